"""GPU: the status row on every kernel family -- the pivot-sign backstop, not only the
observed-day count.

P:87 requires Omega SPD; the library reports a series whose factorisation breaks down LAPACK-style
(reading R-8): info = t+1 for the first pivot row t that is not a positive normal double (its
reciprocal must be normal too), T-d+1 when fewer than d days are observed, outputs NaN, the call
still WHIT_OK.  The expected row comes from the oracle: O2's Algorithm 1 on the band of
Omega (``banded_cholesky_alg1``'s info: its first pivot omega <= 0 or non-finite), for the uneven grid
on the band of O1's dense ``omega_dense_times``.  In exact arithmetic the LDL^T pivots D_t of the
kernels are Algorithm 1's omega_t (L_tt^2), so the cases are built where the first failing pivot is
decided exactly, not by rounding:

* zero row:  lambda_{s-d..s} = 0 and w_s = 0 -> row s of Omega vanishes; D_s = 0.0 exactly in both;
* NaN lambda_r -> the first NaN pivot is row r (no earlier row reads lambda_r);
* lambda_r = -1e6 -> D_r ~ -1e6 (data-scale terms cannot flip it);
* scalar lambda: lambda = 0 with w_s = 0 (D_t = w_t exactly), NaN, -1e6 (row 0);
* subnormal pivot (fp64 I/O): lambda_{s-d..s} = 0, w_s = 1e-310 -> D_s = 1e-310 exactly.  Positive,
  so Algorithm 1 passes it (info 0), but 1/D_s is not a normal double: the kernels report s+1
  instead of returning Inf/NaN with info 0 (R-8; the one documented divergence from O2's rule);
* no observations -> T-d+1 (the count rule; O1.is_spd is False).

Every failed series' outputs are NaN; every other series is bitwise identical to a run in which the
failing series were left healthy.
"""
import numpy as np
import pytest
import torch

import synth
from oracle import banded as O2
from oracle import whittaker as O1

pytestmark = pytest.mark.gpu

T_, B_ = 200, 64
S_ZERO, R_NAN, R_NEG, S_SUB = 97, 61, 130, 150
B_ZERO, B_NAN, B_NEG, B_SUB, B_NOOBS = 1, 2, 3, 4, 5


def inject(x, d, per_date, subnormal):
    """Copy of x (host float64 tensors) with the failure cases of the module docstring injected.
    Returns (x_bad, expected_override) where expected_override maps series -> kernel info that is
    fixed by a rule rather than read from O2 (subnormal: s+1; no observations: T-d+1)."""
    xb = {k: v.clone() for k, v in x.items()}
    w, lam = xb["w"], xb["lam"]
    over = {}
    if per_date:
        lam[S_ZERO - d:S_ZERO + 1, B_ZERO] = 0.0
        w[S_ZERO, B_ZERO] = 0.0
        lam[R_NAN, B_NAN] = float("nan")
        lam[R_NEG, B_NEG] = -1e6
    else:
        lam[B_ZERO] = 0.0
        w[S_ZERO, B_ZERO] = 0.0
        w[:S_ZERO, B_ZERO] = torch.where(w[:S_ZERO, B_ZERO] > 0, w[:S_ZERO, B_ZERO], torch.ones_like(w[:S_ZERO, B_ZERO]))
        lam[B_NAN] = float("nan")
        lam[B_NEG] = -1e6
    if subnormal:
        if per_date:
            lam[S_SUB - d:S_SUB + 1, B_SUB] = 0.0
            w[S_SUB, B_SUB] = 1e-310
            over[B_SUB] = S_SUB + 1
        else:
            lam[B_SUB] = 0.0
            w[:, B_SUB] = 1.0
            w[S_SUB, B_SUB] = 1e-310
            over[B_SUB] = S_SUB + 1
    w[:, B_NOOBS] = 0.0
    over[B_NOOBS] = T_ - d + 1
    return xb, over


def band_of_dense(Om, d):
    T = Om.shape[0]
    band = np.zeros((d + 1, T), dtype=Om.dtype)
    for j in range(d + 1):
        band[j, :T - j] = np.diagonal(Om, -j)
    return band


def oracle_info(x, d, times=None):
    """O2's Algorithm 1 info on each series' band (irregular grid: the band of O1's dense Omega)."""
    w = x["w"].double().numpy().T.copy()
    lam = x["lam"].double().numpy()
    lam = lam.T.copy() if lam.ndim == 2 else lam.copy()
    if times is None:
        band = O2.band_from_w_lam(w, lam, d)
    else:
        tt = times.double().numpy().T
        band = np.stack([band_of_dense(O1.omega_dense_times(w[b], lam[b], tt[b], d), d) for b in range(w.shape[0])])
    with np.errstate(invalid="ignore", divide="ignore", over="ignore"):
        _, info = O2.banded_cholesky_alg1(band)
    return info


def check_family(run, x, d, dtype, per_date, times=None, subnormal=None, run_ok=None):
    """run(x) -> (dict of output tensors [..., B] or [B], info array).  Checks info against the
    oracle, NaN in every failed series' outputs, bitwise-unchanged neighbours (against run_ok(x) if given,
    else run(x))."""
    xb, over = inject(x, d, per_date, dtype == torch.float64 if subnormal is None else subnormal)
    out_bad, info = run(xb)
    out_ok, info_ok = (run_ok or run)(x)
    assert np.all(info_ok == 0), info_ok
    ref = oracle_info(xb, d, times)
    bad = sorted(set([B_ZERO, B_NAN, B_NEG, B_NOOBS] + list(over)))
    for b in bad:
        want = over.get(b, ref[b])
        assert want != 0 or b in over, (b, ref[b])
        assert info[b] == want, f"series {b}: kernel info {info[b]} != expected {want} (O2 {ref[b]})"
    if B_SUB in over:
        assert ref[B_SUB] == 0  # the documented divergence: Algorithm 1 accepts the subnormal pivot
    if per_date:
        assert info[B_ZERO] == S_ZERO + 1 and info[B_NAN] == R_NAN + 1 and info[B_NEG] == R_NEG + 1
    else:
        assert info[B_ZERO] == S_ZERO + 1 and info[B_NAN] == 1 and info[B_NEG] == 1
    assert not O1.is_spd(xb["w"][:, B_NOOBS].double().numpy(), xb["lam"][..., B_NOOBS].double().numpy(), d)
    good = [b for b in range(x["w"].shape[1]) if b not in bad]
    assert np.all(info[good] == 0)
    for k, t in out_bad.items():
        tb = t[..., bad].double()
        assert torch.isnan(tb).all(), f"{k}: failed series not NaN"
        assert torch.equal(t[..., good], out_ok[k][..., good]), f"{k}: a healthy series changed"
        assert torch.isfinite(t[..., good]).all(), k


def make_x(d, dtype, per_date, seed=11):
    x = synth.make_inputs("hetero", B=B_, T=T_, d=d, seed=seed, device="cpu", dtype=torch.float64,
                          lam_mode="per_date" if per_date else "scalar")
    return {k: x[k] for k in ("y", "w", "lam", "g")}


def dev(x, dtype):
    return {k: v.to(dtype).cuda().contiguous() for k, v in x.items()}


def run_plain(d, dtype, per_date):
    import paper_2604_00048_b200 as P

    def run(xh):
        x = dev(xh, dtype)
        ws = P.Workspace(d, T_, B_, dtype, per_date)
        z, gy, gl = torch.empty_like(x["y"]), torch.empty_like(x["y"]), torch.empty_like(x["lam"])
        P.whit_forward(x["y"], x["w"], x["lam"], d, T_, B_, z, ws)
        P.whit_backward(x["g"], ws, z, gy, gl)
        _, info = P.whit_failures(ws, with_info=True)
        return {"z": z.cpu(), "grad_y": gy.cpu(), "grad_lambda": gl.cpu()}, info
    return run


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("per_date", [True, False])
@pytest.mark.parametrize("d", [1, 2, 3])
def test_status_plain_kernel(d, per_date, dtype):
    """whit_kernel (whit_forward / whit_backward): the cold exact-row replay from the checkpoint."""
    check_family(run_plain(d, dtype, per_date), make_x(d, dtype, per_date), d, dtype, per_date)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("per_date", [True, False])
def test_status_wbits_kernel(per_date, dtype):
    """Bit-packed W (whit_forward_wbits): binary w only, so the subnormal-w case does not apply."""
    import paper_2604_00048_b200 as P

    d = 2

    def run(xh):
        x = dev(xh, dtype)
        ws = P.Workspace(d, T_, B_, dtype, per_date)
        bits = P.whit_pack_mask(x["w"])
        z, gy, gl = torch.empty_like(x["y"]), torch.empty_like(x["y"]), torch.empty_like(x["lam"])
        P.whit_forward_wbits(x["y"], bits, x["lam"], d, T_, B_, z, ws)
        P.whit_backward(x["g"], ws, z, gy, gl)
        _, info = P.whit_failures(ws, with_info=True)
        return {"z": z.cpu(), "grad_y": gy.cpu(), "grad_lambda": gl.cpu()}, info

    x = make_x(d, dtype, per_date)
    check_family(run, x, d, dtype, per_date, subnormal=False)  # (1e-310 packs as a 1 bit)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_status_fused_loss_kernel(dtype):
    """whit_forward_mse: loss NaN for a failed series (its scored dates see NaN z)."""
    import paper_2604_00048_b200 as P

    d, per_date = 2, True

    def run(xh):
        x = dev(xh, dtype)
        lw = torch.zeros_like(x["w"])
        lw[::7] = 1.0
        ws = P.Workspace(d, T_, B_, dtype, per_date)
        z, gz, gy = torch.empty_like(x["y"]), torch.empty_like(x["y"]), torch.empty_like(x["y"])
        gl, loss = torch.empty_like(x["lam"]), torch.empty(B_, dtype=dtype, device="cuda")
        P.whit_forward_mse(x["y"], x["w"], x["lam"], lw, d, T_, B_, z, gz, loss, ws)
        P.whit_backward(gz, ws, z, gy, gl)
        _, info = P.whit_failures(ws, with_info=True)
        return {"z": z.cpu(), "loss": loss.cpu(), "grad_y": gy.cpu(), "grad_lambda": gl.cpu()}, info

    check_family(run, make_x(d, dtype, per_date), d, dtype, per_date)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("per_date", [True, False])
@pytest.mark.parametrize("d", [1, 2, 3])
def test_status_irregular_kernel(d, per_date, dtype):
    """whit_irr_kernel (whit_forward_times): info = first failing row, not -1."""
    import paper_2604_00048_b200 as P

    tt = synth.make_times(B_, T_, dtype=torch.float64)

    def run(xh):
        x = dev(xh, dtype)
        t = tt.to(dtype).cuda()
        ws = P.Workspace(d, T_, B_, dtype, per_date, times=True)
        z, gy, gl = torch.empty_like(x["y"]), torch.empty_like(x["y"]), torch.empty_like(x["lam"])
        P.whit_forward_times(x["y"], x["w"], x["lam"], t, d, T_, B_, z, ws)
        P.whit_backward(x["g"], ws, z, gy, gl)
        _, info = P.whit_failures(ws, with_info=True)
        return {"z": z.cpu(), "grad_y": gy.cpu(), "grad_lambda": gl.cpu()}, info

    check_family(run, make_x(d, dtype, per_date), d, dtype, per_date, times=tt)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("per_date", [True, False])
@pytest.mark.parametrize("d", [1, 2, 3])
def test_status_variance_kernel(d, per_date, dtype):
    """whit_var_kernel (whit_posterior_variance): info = first failing row, not -1."""
    import paper_2604_00048_b200 as P

    def run(xh):
        x = dev(xh, dtype)
        ws = P.Workspace(d, T_, B_, dtype, per_date)
        var = torch.empty_like(x["w"])
        P.whit_posterior_variance(x["w"], x["lam"], d, T_, B_, var, ws)
        _, info = P.whit_failures(ws, with_info=True)
        return {"var": var.cpu()}, info

    check_family(run, make_x(d, dtype, per_date), d, dtype, per_date)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("per_date", [True, False])
@pytest.mark.parametrize("times", [False, True])
@pytest.mark.parametrize("d", [1, 2, 3])
def test_status_shared_factor_kernel(d, times, per_date, dtype):
    """whit_mb2_kernel (C = 3 bands sharing the factor; daily and uneven grid): the factor warp's
    first failing row, NaN in every band of a failed pixel."""
    import paper_2604_00048_b200 as P

    C = 3
    tt = synth.make_times(B_, T_, dtype=torch.float64)
    xb = synth.make_inputs_bands("hetero", C, B=B_, T=T_, d=d, seed=13, dtype=torch.float64,
                                 lam_mode="per_date" if per_date else "scalar")
    x = {k: xb[k] for k in ("y", "w", "lam", "g")}

    def run(xh):
        xd = dev(xh, dtype)
        ws = P.Workspace(d, T_, B_, dtype, per_date, C=C, times=times)
        z, gy, gl = torch.empty_like(xd["y"]), torch.empty_like(xd["y"]), torch.empty_like(xd["lam"])
        if times:
            P.whit_forward_times_bands(xd["y"], xd["w"], xd["lam"], tt.to(dtype).cuda(), d, T_, B_, C, z, ws)
        else:
            P.whit_forward_bands(xd["y"], xd["w"], xd["lam"], d, T_, B_, C, z, ws)
        P.whit_backward_bands(xd["g"], ws, z, gy, gl)
        _, info = P.whit_failures(ws, with_info=True)
        return {"z": z.cpu(), "grad_y": gy.cpu(), "grad_lambda": gl.cpu()}, info

    check_family(run, x, d, dtype, per_date, times=tt if times else None)
