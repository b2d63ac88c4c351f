"""O2 -- Algorithm 1 of the paper, verbatim, in long double, vectorised over series.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Band storage (Fig. 2; garbled figure read as in R-14):
``band[j, t] = Omega[t+j, t]`` for j = 0..d (row 0 = diagonal, row j = j-th
sub-diagonal, left-aligned, trailing j entries zero).  Here the paper's
``k+1`` is ``d`` (R-1), so the array has ``k+2 = d+1`` rows.

Algorithm 1, numpy index semantics (R-15):

    for t = 0 .. T-1:
        omega = band[0, t];  v = band[1:, t]
        band[0, t] = sqrt(omega);  band[1:, t] = v / sqrt(omega)
        for u = 0 .. min(k+1, T-t-1) - 1:
            band[:k+1-u, t+1+u] -= v[u:u+k+1] * v[u] / omega

(``v[u:u+k+1]`` clips to ``v[u:k+1]``, which has exactly the ``k+1-u`` entries
the left side has.)  A non-positive (or non-finite) ``omega`` at column ``t``
is reported LAPACK-style as ``info = t+1`` (1-based), the series' outputs are
NaN.  Substitutions ``L x = b``, ``L^T z = x`` follow P:93.

Every operation is vectorised across the leading batch axis only; the loops
over t and u are the algorithm's own.
"""
from __future__ import annotations

import numpy as np

from .whittaker import LD, stencil


def _lam_rows(lam, B: int, T: int, d: int) -> np.ndarray:
    lam = np.asarray(lam, dtype=np.float64)
    if lam.ndim == 1 and lam.shape == (B,):
        return np.repeat(lam[:, None], T - d, axis=1)
    if lam.shape != (B, T - d):
        raise ValueError(f"lambda must be (B,) or (B, T-d); got {lam.shape}")
    return lam


def band_from_w_lam(w, lam, d: int, dtype=LD) -> np.ndarray:
    """Lower band storage of ``Omega = W + D^T diag(lam) D`` for a batch.

    ``w``: (B, T); ``lam``: (B,) scalar per series or (B, T-d) per date.
    ``band[:, j, t] = Omega[t+j, t] = w_t [j=0] + sum_r lam_r c_{t+j-r} c_{t-r}``
    over difference rows ``r`` whose stencil (dates r..r+d) covers both
    ``t`` and ``t+j``.
    """
    w = np.asarray(w, dtype=np.float64)
    B, T = w.shape
    lr = _lam_rows(lam, B, T, d).astype(dtype)
    c = stencil(d)
    band = np.zeros((B, d + 1, T), dtype=dtype)
    band[:, 0, :] = w.astype(dtype)
    # Row r contributes lam_r c_a c_b at (r+b, r+a) for 0 <= a <= b <= d.
    for a in range(d + 1):
        for b in range(a, d + 1):
            j = b - a  # sub-diagonal
            # column t = r + a for r = 0..T-d-1
            band[:, j, a : a + T - d] += dtype(c[a] * c[b]) * lr
    return band


def banded_cholesky_alg1(band: np.ndarray):
    """Algorithm 1 on a batch of bands, (B, k+2, T); returns (L, info).

    ``info[b] = 0`` on success, else 1-based column of the first pivot
    ``omega <= 0`` or non-finite (P:87 says Omega is SPD, so this only fires on
    degenerate inputs).
    """
    Om = np.array(band, dtype=LD, copy=True)
    B, kp2, T = Om.shape
    k1 = kp2 - 1  # the paper's k+1 (= d)
    info = np.zeros(B, dtype=np.int64)
    for t in range(T):
        omega = Om[:, 0, t].copy()
        bad = ~(np.isfinite(omega) & (omega > 0))
        newly = bad & (info == 0)
        info[newly] = t + 1
        omega = np.where(bad, LD(np.nan), omega)
        v = Om[:, 1:, t].copy()
        s = np.sqrt(omega)
        Om[:, 0, t] = s
        Om[:, 1:, t] = v / s[:, None]
        for u in range(min(k1, T - t - 1)):
            n = k1 - u  # rows :k+1-u
            Om[:, :n, t + 1 + u] -= v[:, u : u + k1] * (v[:, u] / omega)[:, None]
    return Om, info


def band_solve(L: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Solve ``L L^T x = b`` with the factor from Algorithm 1.

    Forward: ``x_t = (b_t - sum_j L[t, t-j] x_{t-j}) / L[t, t]`` with
    ``L[t, t-j] = band[j, t-j]``; back: ``z_t = (x_t - sum_j L[t+j, t] z_{t+j}) / L[t, t]``.
    """
    B, kp2, T = L.shape
    d = kp2 - 1
    x = np.zeros((B, T), dtype=LD)
    bb = np.asarray(b).astype(LD)
    for t in range(T):
        acc = bb[:, t].copy()
        for j in range(1, d + 1):
            if t - j >= 0:
                acc -= L[:, j, t - j] * x[:, t - j]
        x[:, t] = acc / L[:, 0, t]
    z = np.zeros((B, T), dtype=LD)
    for t in range(T - 1, -1, -1):
        acc = x[:, t].copy()
        for j in range(1, d + 1):
            if t + j < T:
                acc -= L[:, j, t] * z[:, t + j]
        z[:, t] = acc / L[:, 0, t]
    return z


def _apply_D(x: np.ndarray, d: int) -> np.ndarray:
    c = stencil(d)
    T = x.shape[-1]
    out = np.zeros(x.shape[:-1] + (T - d,), dtype=x.dtype)
    for j in range(d + 1):
        out = out + x.dtype.type(c[j]) * x[..., j : j + T - d]
    return out


def forward_banded(y, w, lam, d: int):
    """Batched Eq. (3) via Algorithm 1: returns (z, dz, info), long double."""
    y = np.asarray(y, dtype=np.float64)
    w = np.asarray(w, dtype=np.float64)
    L, info = banded_cholesky_alg1(band_from_w_lam(w, lam, d))
    b = np.where(w != 0, w.astype(LD) * y.astype(LD), LD(0))
    z = band_solve(L, b)
    return z, _apply_D(z, d), info


def backward_banded(g, w, lam, d: int, z):
    """Batched reverse mode (Eq. (4)/(5)) via Algorithm 1.

    Returns (ybar, lambar): lambar is (B, T-d) for per-date lam, (B,) for scalar.
    """
    w = np.asarray(w, dtype=np.float64)
    L, _ = banded_cholesky_alg1(band_from_w_lam(w, lam, d))
    u = band_solve(L, np.asarray(g, dtype=np.float64))
    ybar = w.astype(LD) * u
    lamb = -_apply_D(u, d) * _apply_D(np.asarray(z).astype(LD), d)
    if np.asarray(lam).ndim == 1 and np.asarray(lam).shape == (w.shape[0],):
        lamb = lamb.sum(axis=1)
    return ybar, lamb
