"""GPU: binary-W detection in the plain forward.

W is binary in the paper.  whit_forward checks every weight; a warp (32 series) whose weights are all
exactly 0 or 1 writes W as a bit plane and reads it back -- in its own back substitution and in the matching
whit_backward -- instead of the float rows.  The bits reconstruct exactly the 1 / 0 the float plane holds,
so the results must be bitwise those of the float path: here every warp of batch B carries one soft weight
in lane 31 (so the whole warp stays on the float path) and lanes 0..30 are compared bit for bit with batch A,
where the detection engaged.  Also: the per-warp flag is exact (-0.0 and soft weights disable it), ragged
T (chunks straddling the 32-date words at d = 3), and the workspace state across forward variants.
"""
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


def _run(x, d, dtype, per_date, T, B, ws=None):
    import paper_2604_00048_b200 as P
    ws = ws or P.Workspace(d, T, B, dtype, per_date)
    z, gy, gl = torch.empty_like(x["y"]), torch.empty_like(x["y"]), torch.empty_like(x["lam"])
    P.whit_forward(x["y"], x["w"], x["lam"], d, T, B, z, ws)
    det = P.whit_wbits_detected(ws)
    P.whit_backward(x["g"], ws, z, gy, gl)
    torch.cuda.synchronize()
    return z, gy, gl, det


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("per_date", [True, False])
@pytest.mark.parametrize("d", [1, 2, 3])
@pytest.mark.parametrize("T", [500, 3288])
def test_binary_w_bits_path_bitwise_equal_float_path(T, d, per_date, dtype):
    B = 128
    x = synth.make_inputs("hetero", B=B, T=T, d=d, device="cuda", dtype=dtype,
                          lam_mode="per_date" if per_date else "scalar")
    x = {k: x[k] for k in ("y", "w", "lam", "g")}
    assert bool(((x["w"] == 0) | (x["w"] == 1)).all())
    za, gya, gla, deta = _run(x, d, dtype, per_date, T, B)
    assert deta == (B // 32, B // 32)  # every warp read W as bits
    xs = dict(x)
    xs["w"] = x["w"].clone()
    xs["w"][T // 3, 31::32] = 0.5  # one soft weight in lane 31 of every warp: the float path
    zb, gyb, glb, detb = _run(xs, d, dtype, per_date, T, B)
    assert detb == (0, B // 32)
    keep = [b for b in range(B) if b % 32 != 31]
    assert torch.equal(za[:, keep], zb[:, keep])
    assert torch.equal(gya[:, keep], gyb[:, keep])
    assert torch.equal(gla[..., keep], glb[..., keep])


def test_binary_w_flag_is_per_warp_and_exact():
    """-0.0 (not the bit pattern of 0) and a soft weight each keep only their own warp on the float path."""
    d, T, B = 2, 300, 128
    x = synth.make_inputs("hetero", B=B, T=T, d=d, device="cuda")
    x = {k: x[k] for k in ("y", "w", "lam", "g")}
    w = x["w"].clone()
    w[10, 33] = -0.0           # warp 1
    w[11, 100] = 1.0 + 2**-20  # warp 3
    x["w"] = w
    _, _, _, det = _run(x, d, torch.float32, True, T, B)
    assert det == (2, 4)


def test_workspace_state_across_forward_variants():
    """One workspace through whit_forward_wbits, then whit_forward_mse, then whit_backward: the backward uses
    the float W of the MSE forward (not the stale caller bits, not stale detection flags) -- bitwise equal
    to the same MSE forward + backward on a fresh workspace.  And whit_grad_w after it is legal."""
    import paper_2604_00048_b200 as P
    d, T, B = 2, 400, 64
    x = synth.make_inputs("hetero", B=B, T=T, d=d, device="cuda")
    y, w, lam = x["y"], x["w"], x["lam"]
    held = (torch.arange(T, device="cuda")[:, None] % 5 == 0) & (w > 0)
    w2 = w.masked_fill(held, 0.0).contiguous()
    lw = held.float().contiguous()

    def mse_bwd(ws):
        z, gz, gy = torch.empty_like(y), torch.empty_like(y), torch.empty_like(y)
        gl, loss = torch.empty_like(lam), torch.empty(B, device="cuda")
        P.whit_forward_mse(y, w2, lam, lw, d, T, B, z, gz, loss, ws)
        P.whit_backward(gz, ws, z, gy, gl)
        gw = torch.empty_like(w2)
        P.whit_grad_w(ws, y, z, gy, gw)
        torch.cuda.synchronize()
        return z, gy, gl, gw

    ws = P.Workspace(d, T, B, torch.float32, True)
    bits = P.whit_pack_mask(w)
    z0 = torch.empty_like(y)
    P.whit_forward_wbits(y, bits, lam, d, T, B, z0, ws)          # leaves caller bits in ws
    z1 = torch.empty_like(y)
    P.whit_forward(y, w, lam, d, T, B, z1, ws)                  # leaves detection flags in ws
    a = mse_bwd(ws)
    b = mse_bwd(P.Workspace(d, T, B, torch.float32, True))
    for name, u, v in zip(("z", "grad_y", "grad_lambda", "grad_w"), a, b):
        if not torch.allclose(u, v, rtol=0.0, atol=0.0, equal_nan=True):  # (held-out dates can leave a
            bad = (u != v) & ~(torch.isnan(u) & torch.isnan(v))                 # series < d observations: NaN)
            idx = bad.nonzero()[:8].tolist()
            raise AssertionError(f"{name}: {int(bad.sum())} differ, first {idx}, "
                                 f"{[(u[tuple(i)].item(), v[tuple(i)].item()) for i in idx]}")
