"""GPU parity of the twisted (two-ended) path for small batches (whit_twist.cuh).

The twisted path is a different elimination order of the same SPD system (Eq. (3)): the top half of
the dates is factored forward, the bottom half in reversed time, and the two meet in a d x d block.  So it is
held to the same oracle tolerances as the sequential path (O2 = Algorithm 1 on every series, O1 on a sample),
on the Sentinel-2 mask (90-day trailing gap) and on iid masks, for z, dL/dy and dL/dlambda (per date and
scalar), plus: its fallback -- a group whose half is not safely SPD on its own is handed to the sequential
kernel, whose results it must then equal bit for bit -- and the status rule (every failure case of
test_gpu_status goes through the fallback, so info is the sequential path's exact row).
"""
import numpy as np
import pytest
import torch

import synth
from oracle import banded as O2
from oracle import whittaker as O1
from helpers import check_scalar_lambar, host_inputs, rel_series, ymax_observed

pytestmark = pytest.mark.gpu

TOL = {  # (z, grads) as test_gpu_parity
    (torch.float32, 1): (1e-4, 1e-3), (torch.float32, 2): (1e-4, 1e-3), (torch.float32, 3): (1e-4, 1e-3),
    (torch.float64, 1): (1e-10, 1e-9), (torch.float64, 2): (1e-10, 1e-9), (torch.float64, 3): (1e-8, 1e-5),
}


def run(x, d, dtype, twist, T, B):
    import paper_2604_00048_b200 as P
    per_date = x["lam"].dim() == 2
    ws = P.Workspace(d, T, B, dtype, per_date)
    ws.set_twist(twist)
    y, w, lam, g = (x[k].to(dtype).contiguous() for k in ("y", "w", "lam", "g"))
    z, gy, gl = torch.empty_like(y), torch.empty_like(y), torch.empty_like(lam)
    P.whit_forward(y, w, lam, d, T, B, z, ws)
    P.whit_backward(g, ws, z, gy, gl)
    n, info = P.whit_failures(ws, with_info=True)
    groups = P.whit_twist_groups(ws)
    torch.cuda.synchronize()
    return {"z": z, "ybar": gy, "lambar": gl, "info": info, "nfail": n, "groups": groups}


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("per_date", [True, False])
@pytest.mark.parametrize("d", [1, 2, 3])
@pytest.mark.parametrize("T,mask", [(517, "s2"), (3288, "s2"), (700, "bernoulli")])
def test_twisted_vs_oracle(T, mask, d, per_date, dtype):
    B = 96
    x = synth.make_inputs("hetero", B=B, T=T, d=d, device="cuda", dtype=torch.float64, mask=mask,
                          lam_mode="per_date" if per_date else "scalar", seed=41 + d)
    r = run(x, d, dtype, 1, T, B)
    assert r["groups"] == (B // 32, B // 32), r["groups"]  # healthy data: every group twisted
    assert r["nfail"] == 0
    seq = run(x, d, dtype, 0, T, B)  # the sequential path on the same inputs (d = 3: its own error sets the bar)
    h = host_inputs({k: x[k].to(dtype) for k in ("y", "w", "lam", "g")})
    tz, tg = TOL[(dtype, d)]
    res = {k: r[k].double().cpu().numpy() for k in ("z", "ybar", "lambar")}
    res = {k: (v.T if v.ndim == 2 else v) for k, v in res.items()}
    lam = h["lam"]
    zr, _, info = O2.forward_banded(h["y"], h["w"], lam, d)
    yb, lb = O2.backward_banded(h["g"], h["w"], lam, d, zr)
    if d < 3:  # Algorithm 1 (long double) is the every-series reference where it is fp64-grade
        ez = rel_series(res["z"], zr, ymax_observed(h["y"], h["w"]))
        assert ez.max() <= tz, ez.max()
        assert rel_series(res["ybar"], yb).max() <= tg
        if per_date:
            assert rel_series(res["lambar"], lb).max() <= tg
    zs = seq["z"].double().cpu().numpy().T
    for b in (0, 37, 95):  # O1 (dense + refinement)
        o = O1.forward_backward(h["y"][b], h["w"][b], lam[b], d, h["g"][b])
        ym = ymax_observed(h["y"][b], h["w"][b])
        ez = np.max(np.abs(res["z"][b] - o["z"].astype(float))) / ym
        if d == 3:  # intrinsically ill-conditioned on long gaps: as accurate as the sequential path
            ez_seq = np.max(np.abs(zs[b] - o["z"].astype(float))) / ym
            assert ez <= max(tz, 4 * ez_seq), (b, ez, ez_seq)
        else:
            assert ez <= tz, (b, ez)
        assert rel_series(res["ybar"][b], o["ybar"]).max() <= tg, b
        if per_date:
            assert rel_series(res["lambar"][b], o["lambar"]).max() <= tg, b
        else:
            lam_rep = np.full(T - d, lam[b])
            _, terms = O2.backward_banded(h["g"][b:b + 1], h["w"][b:b + 1], lam_rep[None, :], d, zr[b:b + 1])
            check_scalar_lambar(res["lambar"][b], float(o["lambar"]), np.sum(np.abs(terms.astype(float))), tg,
                                f"twist b={b}")


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("d", [1, 2, 3])
def test_twisted_close_to_sequential(d, dtype):
    """Same system, two elimination orders: at the homo shape's length the two paths agree far inside the
    oracle tolerance (both are fp64 deviation-form eliminations)."""
    T, B = 3288, 64
    x = synth.make_inputs("homo", B=B, T=T, d=d, device="cuda", dtype=torch.float64)
    a = run(x, d, dtype, 1, T, B)
    s = run(x, d, dtype, 0, T, B)
    assert a["groups"][0] == B // 32 and s["groups"][0] == 0
    ym = torch.where(x["w"] > 0, x["y"].abs(), torch.zeros_like(x["y"])).amax(0).to(a["z"].device)
    dz = ((a["z"] - s["z"]).abs().amax(0).double() / ym).max().item()
    # d = 3 on the 90-day trailing gap is conditioned at the 1e-5 level in fp64 (the sweep's
    # accuracy lines): two elimination orders may differ by that much, so it is held to the fp32 tolerance
    lim = 1e-4 if d == 3 else {torch.float32: 1e-6, torch.float64: 1e-10}[dtype]
    assert dz <= lim, dz


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("per_date", [True, False])
def test_twisted_fallback_group_equals_sequential(per_date, dtype):
    """A series whose first half has a single observation (its top block is nearly singular): its group of
    32 goes through the sequential kernel -- bitwise the sequential path's results -- and the other group
    stays twisted."""
    d, T, B = 2, 800, 64
    x = synth.make_inputs("hetero", B=B, T=T, d=d, device="cuda", dtype=torch.float64,
                          lam_mode="per_date" if per_date else "scalar", mask="bernoulli")
    x["w"][: T // 2, 40] = 0.0
    x["w"][5, 40] = 1.0
    a = run(x, d, dtype, 1, T, B)
    s = run(x, d, dtype, 0, T, B)
    assert a["groups"] == (1, 2), a["groups"]
    for k in ("z", "ybar", "lambar"):
        assert torch.equal(a[k][..., 32:], s[k][..., 32:]), k
    tz = TOL[(dtype, d)][0]
    ym = torch.where(x["w"] > 0, x["y"].abs(), torch.zeros_like(x["y"])).amax(0).to(a["z"].device)
    assert ((a["z"][:, :32] - s["z"][:, :32]).abs().amax(0).double() / ym[:32]).max().item() <= tz


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("per_date", [True, False])
@pytest.mark.parametrize("d", [1, 2, 3])
def test_twisted_status_through_fallback(d, per_date, dtype):
    """The failure cases of test_gpu_status (zero row, NaN lambda, negative lambda, subnormal pivot, no
    observation) with the twisted path forced: info, NaN outputs and untouched neighbours as there."""
    import test_gpu_status as S
    import paper_2604_00048_b200 as P

    def run_mode(xh, mode):
        xd = S.dev(xh, dtype)
        ws = P.Workspace(d, S.T_, S.B_, dtype, per_date)
        ws.set_twist(mode)
        z, gy, gl = torch.empty_like(xd["y"]), torch.empty_like(xd["y"]), torch.empty_like(xd["lam"])
        P.whit_forward(xd["y"], xd["w"], xd["lam"], d, S.T_, S.B_, z, ws)
        P.whit_backward(xd["g"], ws, z, gy, gl)
        _, info = P.whit_failures(ws, with_info=True)
        return {"z": z.cpu(), "grad_y": gy.cpu(), "grad_lambda": gl.cpu()}, info

    def run_ok(xh):
        # the failing series sit in group 0, which the bad run hands to the sequential kernel: the healthy
        # reference is the sequential path there and the twisted path in group 1
        seq, info = run_mode(xh, 0)
        tw, _ = run_mode(xh, 1)
        return {k: torch.cat([seq[k][..., :32], tw[k][..., 32:]], dim=-1) for k in seq}, info

    x0 = S.make_x(d, dtype, per_date)
    S.check_family(lambda xh: run_mode(xh, 1), x0, d, dtype, per_date, run_ok=run_ok)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("per_date", [True, False])
def test_hybrid_launch(per_date, dtype):
    """Hybrid launch (B just past one wave): groups [0, g1) (1,504 per date, 1,728 scalar) by the sequential kernel on the workspace
    stream, the rest twisted on a second stream.  The sequential part equals the sequential path bitwise;
    the twisted part agrees with it inside the oracle tolerance (and a failing series there still gets its
    exact status through the fallback); O1 on a sample of both parts."""
    d, T, B = 2, 240, 65536
    x = synth.make_inputs("hetero", B=B, T=T, d=d, device="cuda", dtype=torch.float64, mask="bernoulli",
                          lam_mode="per_date" if per_date else "scalar", seed=77)
    if per_date:
        x["lam"][61, 60000] = float("nan")  # a failing series in the twisted part: info 62
    a = run(x, d, dtype, 2, T, B)
    s = run(x, d, dtype, 0, T, B)
    G1 = (1504 if per_date else 1728) * 32
    assert a["groups"][1] == B // 32 and a["groups"][0] >= (B - G1) // 32 - 1, a["groups"]
    for k in ("z", "ybar", "lambar"):
        assert torch.equal(a[k][..., :G1].nan_to_num(7.0), s[k][..., :G1].nan_to_num(7.0)), k
    assert np.array_equal(a["info"], s["info"])
    if per_date:
        assert a["info"][60000] == 62 and torch.isnan(a["z"][:, 60000]).all()
    ok = torch.isfinite(a["z"]).all(0)
    ym = torch.where(x["w"] > 0, x["y"].abs(), torch.zeros_like(x["y"])).amax(0).to(a["z"].device)
    ez = ((a["z"] - s["z"]).abs().amax(0).double() / ym)[ok].max().item()
    assert ez <= TOL[(dtype, d)][0], ez
    h = host_inputs({k: x[k].to(dtype) for k in ("y", "w", "lam", "g")})
    tz, tg = TOL[(dtype, d)]
    for b in (5, G1 - 1, G1, B - 1):
        o = O1.forward_backward(h["y"][b], h["w"][b], h["lam"][b], d, h["g"][b])
        z = a["z"][:, b].double().cpu().numpy()
        assert np.max(np.abs(z - o["z"].astype(float))) / ymax_observed(h["y"][b], h["w"][b]) <= tz, b
        assert rel_series(a["ybar"][:, b].double().cpu().numpy(), o["ybar"]).max() <= tg, b


def test_posterior_variance_after_twisted_forward_invalidates_backward():
    """whit_posterior_variance rewrites the factor checkpoints in the sequential layout, so after a twisted
    forward the matching backward must be refused (WHIT_ERR_STATE), not run on the wrong layout."""
    import paper_2604_00048_b200 as P
    d, T, B = 2, 300, 64
    x = synth.make_inputs("hetero", B=B, T=T, d=d, device="cuda", mask="bernoulli")
    ws = P.Workspace(d, T, B, torch.float32, True)
    ws.set_twist(1)
    z, gy, gl, var = (torch.empty_like(x["y"]), torch.empty_like(x["y"]), torch.empty_like(x["lam"]),
                      torch.empty_like(x["y"]))
    P.whit_forward(x["y"], x["w"], x["lam"], d, T, B, z, ws)
    P.whit_posterior_variance(x["w"], x["lam"], d, T, B, var, ws)
    with pytest.raises(P.WhitError) as e:
        P.whit_backward(x["g"], ws, z, gy, gl)
    assert e.value.status == 6  # WHIT_ERR_STATE


@pytest.mark.parametrize("d", [1, 2, 3])
def test_twisted_short_series_and_split_offsets(d):
    """Short series down to the smallest T the twisted split accepts, every residue of T - m modulo K (the
    bottom half's chunk boundary relative to the twist block, which may straddle two bottom chunks): twisted
    results against O1 on every series, fp64 I/O."""
    import paper_2604_00048_b200 as P
    K = 16 if d <= 2 else 12
    Tmin = 2 * K + d
    dtype, B = torch.float64, 32
    for T in range(Tmin, Tmin + K + 3):
        x = synth.make_inputs("hetero", B=B, T=T, d=d, device="cuda", dtype=torch.float64, mask="bernoulli",
                              seed=500 + T)
        x["w"][:, :] = torch.where(torch.arange(T, device="cuda")[:, None] % 3 == 1, 0.0, 1.0)  # dense, 2/3
        r = run(x, d, dtype, 1, T, B)
        assert r["groups"] == (1, 1), (T, r["groups"])
        h = host_inputs({k: x[k] for k in ("y", "w", "lam", "g")})
        tz, tg = TOL[(dtype, d)]
        for b in range(0, B, 7):
            o = O1.forward_backward(h["y"][b], h["w"][b], h["lam"][b], d, h["g"][b])
            z = r["z"][:, b].double().cpu().numpy()
            assert np.max(np.abs(z - o["z"].astype(float))) / ymax_observed(h["y"][b], h["w"][b]) <= tz, (T, b)
            assert rel_series(r["ybar"][:, b].double().cpu().numpy(), o["ybar"]).max() <= tg, (T, b)
            assert rel_series(r["lambar"][:, b].double().cpu().numpy(), o["lambar"]).max() <= tg, (T, b)


def test_autograd_default_path_is_twisted_and_correct():
    """The package default (no WHIT_TWIST in the environment): smooth() on a small batch takes the twisted path
    (a subprocess, since the suite pins WHIT_TWIST=0) and its z and gradients match O1."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = r"""
import json, torch, numpy as np, synth, paper_2604_00048_b200 as P
from oracle import whittaker as O1
d, T, B = 2, 400, 96
x = synth.make_inputs("hetero", B=B, T=T, d=d, device="cuda", dtype=torch.float64, mask="bernoulli", seed=3)
y = x["y"].clone().requires_grad_(True); lam = x["lam"].clone().requires_grad_(True)
z = P.smooth(y, x["w"], lam, d)
(z * x["g"]).sum().backward()
out = {"tw": None}
ws = P.Workspace(d, T, B, torch.float64, True); zz = torch.empty_like(y)
P.whit_forward(x["y"], x["w"], x["lam"], d, T, B, zz, ws); out["tw"] = P.whit_twist_groups(ws)
errs = []
for b in (0, 50, 95):
    o = O1.forward_backward(*(t[:, b].cpu().numpy() for t in (x["y"], x["w"], x["lam"])), d, x["g"][:, b].cpu().numpy())
    ym = np.abs(x["y"][:, b].cpu().numpy()[x["w"][:, b].cpu().numpy() > 0]).max()
    errs.append([float(np.abs(z[:, b].detach().cpu().numpy() - o["z"].astype(float)).max() / ym),
                 float(np.abs(y.grad[:, b].cpu().numpy() - o["ybar"].astype(float)).max() / np.abs(o["ybar"].astype(float)).max()),
                 float(np.abs(lam.grad[:, b].cpu().numpy() - o["lambar"].astype(float)).max() / np.abs(o["lambar"].astype(float)).max())])
out["errs"] = errs
print(json.dumps(out))
"""
    env = {k: v for k, v in os.environ.items() if k not in ("WHIT_TWIST", "WHIT_HYBRID")}
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["tw"] == [3, 3], out
    for ez, ey, el in out["errs"]:
        assert ez <= 1e-10 and ey <= 1e-9 and el <= 1e-9, out["errs"]


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("per_date", [True, False])
@pytest.mark.parametrize("d", [2, 3])
def test_twisted_both_register_builds(d, per_date, dtype):
    """The twisted kernel has two builds: 255 registers for launches of <= 592 groups (one wave at 8 warps/SM)
    and 168 for larger ones.  A batch of 600 groups takes the 168-register build; its first 32
    groups, solved alone, take the 255-register one: the same arithmetic, so the results agree bit for bit;
    and the whole batch stays close to the sequential path (as test_twisted_close_to_sequential)."""
    T, G = 300, 600
    B = 32 * G
    x = synth.make_inputs("hetero", B=B, T=T, d=d, device="cuda", dtype=torch.float64, mask="bernoulli",
                          lam_mode="per_date" if per_date else "scalar")
    big = run(x, d, dtype, 1, T, B)
    assert big["groups"][0] == G
    sub = {k: (x[k][..., :32] if x[k].dim() == 2 else x[k][:32]).contiguous() for k in ("y", "w", "lam", "g")}
    small = run(sub, d, dtype, 1, T, 32)
    assert small["groups"][0] == 1
    for k in ("z", "ybar", "lambar"):
        a, b = big[k][..., :32] if big[k].dim() == 2 else big[k][:32], small[k]
        assert torch.equal(a.cpu(), b.cpu()), k
    seq = run(x, d, dtype, 0, T, B)
    ym = torch.where(x["w"] > 0, x["y"].abs(), torch.zeros_like(x["y"])).amax(0).to(big["z"].device)
    dz = ((big["z"] - seq["z"]).abs().amax(0).double() / ym).max().item()
    lim = 1e-4 if d == 3 else {torch.float32: 1e-6, torch.float64: 1e-10}[dtype]
    assert dz <= lim, dz


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_homo_full_size_hybrid_launch_sampled(dtype):
    """BASELINE configs[1] at full size (B = 65,536, T = 3,288, scalar lambda) in the launch configuration
    bench.py times by default -- the hybrid launch (groups [0, 1,728) sequential, the 320-group tail twisted
    with the 255-register build; the suite pins WHIT_TWIST=0, so it is forced here with set_twist(2), which
    picks the same split): sampled series from both parts vs O1 at the BASELINE tolerances."""
    d = 2
    x = synth.make_inputs("homo", device="cuda")
    T, B = x["y"].shape
    r = run(x, d, dtype, 2, T, B)
    assert r["nfail"] == 0
    G1 = 1728  # the scalar-lambda split (hyb_g1_of)
    assert r["groups"][0] == B // 32 - G1  # the twisted tail
    idx = np.unique(np.concatenate([[0, G1 * 32 - 1, G1 * 32, B - 1],
                                    np.linspace(0, B - 1, 6).astype(int),
                                    np.linspace(G1 * 32, B - 1, 4).astype(int)]))
    h = host_inputs({k: (v[:, idx] if v.dim() == 2 else v[idx]) for k, v in x.items() if k in ("y", "w", "lam", "g")})
    tz, tg = TOL[(dtype, d)]
    z = r["z"][:, idx].double().cpu().numpy()
    ybar = r["ybar"][:, idx].double().cpu().numpy()
    lambar = r["lambar"][idx].double().cpu().numpy()
    for i, b in enumerate(idx):
        o = O1.forward_backward(h["y"][i], h["w"][i], h["lam"][i], d, h["g"][i])
        ym = ymax_observed(h["y"][i], h["w"][i])
        assert np.max(np.abs(z[:, i] - o["z"].astype(float))) / ym <= tz, (b, "z")
        assert rel_series(ybar[:, i], o["ybar"]).max() <= tg, (b, "ybar")
        assert abs(lambar[i] - float(o["lambar"])) <= tg * abs(float(o["lambar"])), (b, "lambar")
