"""Shared test helpers: run the CUDA path through the C-ABI binding, run the
oracle on the same inputs, and compare with the BASELINE.json metrics.

Error metrics (R-9), per series, then the max over series:
  z:        max_t |z - z_ref| / max_{t: w_t > 0} |y_t|
  grads:    max_t |g - g_ref| / max_t |g_ref|      (normwise relative)
"""
from __future__ import annotations

import numpy as np


def rel_series(a, ref, denom=None):
    """Per-series max-abs error over the last axis / denom (default max|ref| of the series).
    A 1-D input is ONE series; a 0-d input is a scalar per series."""
    a = np.asarray(a, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    if a.ndim == 0:
        a, ref = a[None], ref[None]
    if a.ndim == 1:
        a, ref = a[None, :], ref[None, :]
    err = np.max(np.abs(a - ref), axis=-1)
    den = np.max(np.abs(ref), axis=-1) if denom is None else np.asarray(denom, dtype=np.float64)
    den = np.where(den > 0, den, 1.0)
    return err / den


def ymax_observed(y, w):
    y = np.asarray(y, dtype=np.float64)
    return np.max(np.where(np.asarray(w) > 0, np.abs(y), 0.0), axis=-1)


def run_cuda(x: dict, d: int, dtype, backward: bool = True, twist: int | None = None):
    """Forward (+ backward with x['g']) through the C-ABI; returns host numpy series-major arrays.
    twist: whit_ws_set_twist mode for the workspace (None: the suite's default, WHIT_TWIST=0)."""
    import torch

    import paper_2604_00048_b200 as P

    y, w, lam = (x[k].to(dtype).contiguous() for k in ("y", "w", "lam"))
    T, B = y.shape
    per_date = lam.dim() == 2
    ws = P.Workspace(d, T, B, dtype, per_date, device=y.device)
    if twist is not None:
        ws.set_twist(twist)
    z = torch.empty_like(y)
    P.whit_forward(y, w, lam, d, T, B, z, ws)
    out = {"z": z}
    if backward:
        g = x["g"].to(dtype).contiguous()
        gy = torch.empty_like(g)
        gl = torch.empty_like(lam)
        P.whit_backward(g, ws, z, gy, gl)
        out.update(ybar=gy, lambar=gl)
    nfail, info = P.whit_failures(ws, with_info=True)
    torch.cuda.synchronize()
    res = {k: (v.detach().cpu().double().numpy().T.copy() if v.dim() == 2 else v.detach().cpu().double().numpy())
           for k, v in out.items()}
    res["info"] = info
    res["nfail"] = nfail
    return res


def host_inputs(x: dict, dtype=None):
    """Series-major float64 copies of the exact values the GPU saw."""
    import torch

    out = {}
    for k in ("y", "w", "lam", "g"):
        v = x.get(k)
        if v is None:
            continue
        if dtype is not None:
            v = v.to(dtype)
        a = v.detach().cpu().to(torch.float64).numpy()
        out[k] = a.T.copy() if a.ndim == 2 else a.copy()
    return out


def check_scalar_lambar(got, ref, abs_terms, tol, label="", well_ratio=100.0):
    """Scalar-lambda gradient gate (R-9), two-sided.

    dL/dlambda = sum_r -(Du)_r (Dz)_r is a sum whose rounding scale is sum_r |(Du)_r (Dz)_r|, so the
    primary gate is |got - ref| / sum|terms| <= tol.  That alone is loose where the sum cancels, so
    every series whose cancellation ratio sum|terms| / |ref| is below ``well_ratio`` must ALSO meet
    |got - ref| / |ref| <= tol.  Returns (worst ratio, worst |ref|-relative error on the
    well-conditioned series, number of well-conditioned series)."""
    got = np.atleast_1d(np.asarray(got, dtype=np.float64))
    ref = np.atleast_1d(np.asarray(ref, dtype=np.float64))
    den = np.atleast_1d(np.asarray(abs_terms, dtype=np.float64))
    err = np.abs(got - ref)
    e_sum = err / np.where(den > 0, den, 1.0)
    assert e_sum.max() <= tol, f"{label} lambar err vs sum|terms| {e_sum.max():.3e}"
    ratio = den / np.maximum(np.abs(ref), 1e-300)
    well = ratio < well_ratio
    e_rel = err[well] / np.abs(ref[well]) if well.any() else np.zeros(1)
    assert e_rel.max() <= tol, f"{label} lambar err vs |lambar| {e_rel.max():.3e} (ratio < {well_ratio})"
    print(f"{label} scalar lambar: worst cancellation ratio {ratio.max():.3g}, |lambar|-relative error "
          f"{e_rel.max():.3e} on {int(well.sum())}/{well.size} well-conditioned series")
    return float(ratio.max()), float(e_rel.max()), int(well.sum())
