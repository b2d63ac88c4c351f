"""GPU: out-of-bounds and race evidence without compute-sanitizer (closed on this pool).

Guard bands: every plane a kernel family reads or writes -- and the workspace -- is placed inside a larger
allocation.  Input margins hold NaN (a read past a plane's end, or before its start, would poison the
results: every output is compared bit for bit with a run on plain, unguarded tensors); output and workspace
margins hold a sentinel byte pattern that must survive the run (a write past a plane would change it).
Determinism: each family runs twice on the same inputs and must reproduce its outputs bit for bit (a
shared-memory race or an mbarrier phase error shows up as run-to-run differences).

Shapes are small but span several chunks, a ragged tail in T and a partial warp / CTA in B, for the
single-series kernels (binary W read as bits, soft W on the float path, caller bits, fused loss),
the irregular-grid kernel, the posterior-variance kernel and the shared-factor kernels (daily and uneven).
"""
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu

PAD = 4096  # elements of margin on each side (16-B aligned offsets for both dtypes)
SENT = 0x5A


class Guarded:
    """Planes carved out of larger tensors with NaN (inputs) or sentinel (outputs) margins."""

    def __init__(self):
        self.outs = []

    def inp(self, t):
        fill = float("nan") if t.dtype.is_floating_point else -1  # (bit planes: all ones)
        flat = torch.full((t.numel() + 2 * PAD,), fill, dtype=t.dtype, device="cuda")
        v = flat[PAD:PAD + t.numel()].view(t.shape)
        v.copy_(t)
        return v

    def out(self, like):
        flat = torch.empty(like.numel() + 2 * PAD, dtype=like.dtype, device="cuda")
        flat.view(torch.uint8).fill_(SENT)
        self.outs.append(flat)
        return flat[PAD:PAD + like.numel()].view(like.shape)

    def ws_buf(self, nbytes):
        flat = torch.full((nbytes + 2 * 256 * 64,), SENT, dtype=torch.uint8, device="cuda")
        self.outs.append(flat)
        self.ws_flat = flat
        return flat[256 * 64:256 * 64 + nbytes]

    def margins_intact(self):
        for flat in self.outs:
            b = flat.view(torch.uint8)
            m = PAD * flat.element_size() if flat.dtype != torch.uint8 else 256 * 64
            if not (bool((b[:m] == SENT).all()) and bool((b[-m:] == SENT).all())):
                return False
        return True


def _family_runs(family, d, dtype, per_date, T, B, C=3):
    """Returns run(guarded: bool) -> dict of output tensors (CPU), plus the margins check."""
    import paper_2604_00048_b200 as P

    bands = family in ("bands", "bands_times")
    times = family in ("times", "bands_times")
    if bands:
        x = synth.make_inputs_bands("hetero", C, B=B, T=T, d=d, device="cuda", dtype=dtype,
                                    lam_mode="per_date" if per_date else "scalar")
    else:
        # (the twisted kernel keeps a group only if each half has >= 2d observed days: the iid mask, so its
        # down sweep -- and its stores -- run under the guards)
        x = synth.make_inputs("hetero", B=B, T=T, d=d, device="cuda", dtype=dtype,
                              lam_mode="per_date" if per_date else "scalar",
                              mask="bernoulli" if family in ("twisted", "hybrid") else None)
    x = {k: x[k].contiguous() for k in ("y", "w", "lam", "g")}
    if family == "soft":
        x["w"] = (x["w"] * 0.75).contiguous()
    tt = synth.make_times(B, T, device="cuda", dtype=dtype) if times else None
    lw = ((torch.arange(T, device="cuda")[:, None] % 3) == 0).to(dtype).expand(T, B).contiguous()

    def run(guarded):
        G = Guarded()
        gi = G.inp if guarded else (lambda t: t)
        go = G.out if guarded else (lambda t: torch.empty_like(t))
        y, w, lam, g = gi(x["y"]), gi(x["w"]), gi(x["lam"]), gi(x["g"])
        kw = {"C": C} if bands else {}
        nbytes = P.Workspace(d, T, B, dtype, per_date, times=times, **kw).nbytes
        ws = P.Workspace(d, T, B, dtype, per_date, times=times, buf=G.ws_buf(nbytes) if guarded else None, **kw)
        if family == "twisted":
            ws.set_twist(1)
        elif family == "hybrid":
            ws.set_twist(2)
        out = {}
        if family == "variance":
            var = go(x["w"])
            P.whit_posterior_variance(w, lam, d, T, B, var, ws)
            out["var"] = var
        else:
            z, gy, gl = go(x["y"]), go(x["y"]), go(x["lam"])
            if family in ("binary", "soft", "twisted", "hybrid"):
                P.whit_forward(y, w, lam, d, T, B, z, ws)
            elif family == "wbits":
                bits = gi(P.whit_pack_mask(x["w"]).contiguous())
                P.whit_forward_wbits(y, bits, lam, d, T, B, z, ws)
            elif family == "mse":
                gz, loss = go(x["y"]), go(torch.empty(B, dtype=dtype, device="cuda"))
                P.whit_forward_mse(y, w, lam, gi(lw), d, T, B, z, gz, loss, ws)
                out.update(grad_z=gz, loss=loss)
                g = gz
            elif family == "times":
                P.whit_forward_times(y, w, lam, gi(tt), d, T, B, z, ws)
            elif family == "bands":
                P.whit_forward_bands(y, w, lam, d, T, B, C, z, ws)
            elif family == "bands_times":
                P.whit_forward_times_bands(y, w, lam, gi(tt), d, T, B, C, z, ws)
            P.whit_backward(g, ws, z, gy, gl)
            out.update(z=z, grad_y=gy, grad_lambda=gl)
            if family in ("binary", "soft"):
                gw = go(x["w"])
                P.whit_grad_w(ws, y, z, gy, gw)
                out["grad_w"] = gw
        torch.cuda.synchronize()
        res = {k: v.cpu().clone() for k, v in out.items()}
        return res, (G.margins_intact() if guarded else True)

    return run


FAMILIES = ["binary", "soft", "wbits", "mse", "times", "variance", "bands", "bands_times", "twisted"]


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("per_date", [True, False])
@pytest.mark.parametrize("d", [1, 2, 3])
@pytest.mark.parametrize("family", FAMILIES)
def test_guard_bands_and_determinism(family, d, per_date, dtype):
    T, B = 203, 100  # ragged chunks in T; a partial warp (and CTA) in B
    run = _family_runs(family, d, dtype, per_date, T, B)
    ref, _ = run(False)
    again, _ = run(False)
    got, intact = run(True)
    assert intact, "a kernel wrote outside its planes or its workspace"
    for k in ref:
        assert torch.equal(ref[k].nan_to_num(nan=7.0), again[k].nan_to_num(nan=7.0)), f"{k}: not deterministic"
        assert torch.equal(ref[k].nan_to_num(nan=7.0), got[k].nan_to_num(nan=7.0)), \
            f"{k}: differs with NaN margins around the inputs (an out-of-bounds read)"
        assert bool(torch.isfinite(ref[k]).all()), f"{k}: non-finite output on a healthy batch"


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("per_date", [True, False])
def test_guard_bands_hybrid_launch(per_date, dtype):
    """The hybrid launch (two streams; 1,792 groups: 1,504 / 1,728 sequential + 288 / 64 twisted, per date /
    scalar) under the same guards."""
    d, T, B = 2, 203, 1792 * 32
    run = _family_runs("hybrid", d, dtype, per_date, T, B)
    ref, _ = run(False)
    again, _ = run(False)
    got, intact = run(True)
    assert intact, "a kernel wrote outside its planes or its workspace"
    for k in ref:
        assert torch.equal(ref[k].nan_to_num(nan=7.0), again[k].nan_to_num(nan=7.0)), f"{k}: not deterministic"
        assert torch.equal(ref[k].nan_to_num(nan=7.0), got[k].nan_to_num(nan=7.0)), k
