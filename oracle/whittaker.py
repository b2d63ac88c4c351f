"""O1 -- the Whittaker layer as its plain definition (dense, fp64 + long-double refinement).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``): imported by ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / reference legs,
never by the product path.

Notation (PAPER.md line numbers as ``P:n``; readings as DESIGN.md §3 ``R-n``):

* ``y``  -- the observed series, the paper's ``x``, length ``T``.
* ``w``  -- the diagonal of ``W``: 1 observed, 0 cloud/gap/padding.
  Reading R-4: any real ``w >= 0`` is accepted and ``(W y)_t := 0`` where
  ``w_t = 0`` (so values at masked slots never matter).
* ``d``  -- the difference order, the paper's ``k+1`` (R-1).
* ``D``  -- the order-``d`` difference operator, ``(T-d) x T``.  On the
  unit-spaced daily grid the dspline divided difference reduces to the
  binomial stencil ``c_j = (-1)^(d-j) C(d, j)`` with unit scale (R-3); the
  tests pin this against the divided-difference recursion.
* ``lam`` -- the diagonal of ``Lambda``, one weight per difference row:
  ``lam_r`` multiplies ``(D z)_r``, the stencil over dates ``r..r+d`` (R-2).
  A scalar is the homoscedastic case, Eq. (2).
* ``Omega = W + D^T Lambda D``, the matrix of Eq. (3).

Forward:  ``z = Omega^{-1} W y``                       -- Eq. (3)
Backward (reverse mode, upstream cotangent ``g = dL/dz``), ``u = Omega^{-1} g``:
  ``dL/dy = W Omega^{-1} g = w * u``                  -- Eq. (5), P:77 (R-7)
  ``dL/dlam_r = g^T dz/dlam_r = -(D u)_r (D z)_r``    -- Eq. (4), contracted
  scalar ``lam``: ``dL/dlam = sum_r dL/dlam_r``.

The solve is exact up to rounding: Omega is SPD so ``z`` is unique.  To
judge the fp64 tolerance (1e-10, BASELINE.json) the oracle must itself be
accurate well below it; plain dense LAPACK fp64 is only ~1e-10..6e-10 accurate
at T = 3288, so Omega is built entry-exactly in long double and
the fp64 LU solve is followed by iterative refinement with long-double
residuals (reading R-9).  Refinement changes no result, only its rounding.
"""
from __future__ import annotations

import math

import numpy as np
import scipy.linalg as sla

LD = np.longdouble


def stencil(d: int) -> np.ndarray:
    """Row of ``D`` on the unit grid: ``c_j = (-1)^(d-j) C(d, j)``, j = 0..d.

    P:26 (order ``k+1`` difference operator), P:28 (dspline definition, unit
    grid reduction, reading R-3).  E.g. d=1: (-1, 1); d=2: (1, -2, 1).
    """
    if d < 1:
        raise ValueError("order d must be >= 1")
    return np.array([(-1) ** (d - j) * math.comb(d, j) for j in range(d + 1)], dtype=np.int64)


def difference_matrix(T: int, d: int, dtype=np.float64) -> np.ndarray:
    """Dense ``D`` in R^{(T-d) x T} with ``D[r, r+j] = c_j``."""
    if T < d + 1:
        raise ValueError("need T >= d + 1")
    c = stencil(d)
    D = np.zeros((T - d, T), dtype=dtype)
    for r in range(T - d):
        D[r, r : r + d + 1] = c
    return D


def lam_tilde(lam, T: int, d: int) -> np.ndarray:
    """The ``T-d`` penalty weights (diag of Lambda; reading R-2).

    A scalar ``lam`` (Eq. (2)) is broadcast to all ``T-d`` rows.
    """
    lam = np.asarray(lam)
    if lam.ndim == 0:
        return np.full(T - d, lam, dtype=np.float64)
    if lam.shape != (T - d,):
        raise ValueError(f"per-date lambda must have length T-d = {T - d}, got {lam.shape}")
    return lam.astype(np.float64)


def omega_dense(w, lam, d: int, dtype=LD) -> np.ndarray:
    """``Omega = W + D^T diag(lam) D``, dense, built entry-exactly.

    Written as the sum over difference rows ``sum_r lam_r d_r d_r^T`` (the
    expansion of ``D^T Lambda D`` row by row), accumulated in long
    double so every entry is the exact value of the fp32/fp64 inputs up to
    ~1e-19 relative.
    """
    w = np.asarray(w, dtype=np.float64)
    T = w.shape[0]
    lt = lam_tilde(lam, T, d)
    c = stencil(d).astype(dtype)
    Om = np.zeros((T, T), dtype=dtype)
    Om[np.arange(T), np.arange(T)] = w.astype(dtype)
    cc = np.outer(c, c)
    for r in range(T - d):
        Om[r : r + d + 1, r : r + d + 1] += dtype(lt[r]) * cc
    return Om


def _rhs(y, w) -> np.ndarray:
    """``W y`` with the convention ``(W y)_t = 0`` where ``w_t = 0`` (R-4)."""
    y = np.asarray(y, dtype=np.float64)
    w = np.asarray(w, dtype=np.float64)
    return np.where(w != 0, w.astype(LD) * y.astype(LD), LD(0))


class _Factor:
    """fp64 LU of Omega plus the long-double Omega for refinement residuals."""

    def __init__(self, Om_ld: np.ndarray):
        self.Om_ld = Om_ld
        self.lu = sla.lu_factor(Om_ld.astype(np.float64), check_finite=True)

    def solve(self, b_ld: np.ndarray, steps: int = 2) -> np.ndarray:
        x = sla.lu_solve(self.lu, b_ld.astype(np.float64)).astype(LD)
        for _ in range(steps):
            r = b_ld - self.Om_ld @ x
            x = x + sla.lu_solve(self.lu, r.astype(np.float64)).astype(LD)
        return x


def solve_refined(Om_ld: np.ndarray, b, steps: int = 2) -> np.ndarray:
    """``Omega^{-1} b``: fp64 LU solve + ``steps`` long-double refinement steps."""
    return _Factor(Om_ld).solve(np.asarray(b).astype(LD), steps)


def apply_D(x: np.ndarray, d: int) -> np.ndarray:
    """``(D x)_r = sum_j c_j x_{r+j}``, in the dtype of ``x``."""
    c = stencil(d)
    T = x.shape[-1]
    out = np.zeros(x.shape[:-1] + (T - d,), dtype=x.dtype)
    for j in range(d + 1):
        out = out + x.dtype.type(c[j]) * x[..., j : j + T - d]
    return out


def forward(y, w, lam, d: int, steps: int = 2):
    """Eq. (3): ``z = Omega^{-1} W y``; also returns ``D z``.

    Returns long-double arrays ``(z, dz)``.
    """
    Om = omega_dense(w, lam, d)
    z = _Factor(Om).solve(_rhs(y, w), steps)
    return z, apply_D(z, d)


def backward(g, w, lam, d: int, z, steps: int = 2):
    """Reverse mode of the layer for upstream cotangent ``g = dL/dz``.

    ``u = Omega^{-1} g`` (Omega symmetric);
    ``ybar = w * u``              (Eq. (5), as a VJP, reading R-7);
    ``lambar_r = -(D u)_r (D z)_r`` (Eq. (4), contracted with ``g``);
    scalar ``lam``: ``lambar = sum_r lambar_r`` (chain rule, reading R-6).
    """
    Om = omega_dense(w, lam, d)
    u = _Factor(Om).solve(np.asarray(g, dtype=np.float64).astype(LD), steps)
    return _grads(u, w, lam, d, np.asarray(z).astype(LD))


def _grads(u, w, lam, d, z):
    ybar = np.asarray(w, dtype=np.float64).astype(LD) * u
    lamb = -apply_D(u, d) * apply_D(z, d)
    if np.asarray(lam).ndim == 0:
        lamb = lamb.sum()
    return ybar, lamb


def weight_grad(y, w, z, u):
    """``dL/dw_t`` for the layer ``z = Omega^{-1} W y`` (NEXT-3's optional output).

    Differentiating Eq. (3) in ``w_t``: ``Omega dz = e_t (y_t - z_t) dw_t``, so with
    ``u = Omega^{-1} g``: ``dL/dw_t = u_t (y_t - z_t)``.  Reading R-19: at unobserved days
    (``w_t = 0``) ``y_t`` carries no value (R-4) and the gradient is defined as 0.
    """
    y = np.asarray(y, dtype=np.float64)
    w = np.asarray(w, dtype=np.float64)
    ys = np.where(w > 0, y, 0.0).astype(LD)
    return np.where(w > 0, np.asarray(u).astype(LD) * (ys - np.asarray(z).astype(LD)), LD(0))


def forward_backward(y, w, lam, d: int, g, steps: int = 2) -> dict:
    """Forward and backward of one series sharing one factorization of Omega."""
    Om = omega_dense(w, lam, d)
    F = _Factor(Om)
    z = F.solve(_rhs(y, w), steps)
    u = F.solve(np.asarray(g, dtype=np.float64).astype(LD), steps)
    ybar, lamb = _grads(u, w, lam, d, z)
    return {"z": z, "dz": apply_D(z, d), "u": u, "ybar": ybar, "lambar": lamb}


def is_spd(w, lam, d: int) -> bool:
    """Is ``Omega`` symmetric positive definite?

    With every ``lam_r > 0``: ``z^T Omega z = sum w_t z_t^2 + sum lam_r (Dz)_r^2``
    vanishes iff ``D z = 0`` (z a polynomial of degree < d in t) and ``z`` is 0
    on every observed day; a nonzero polynomial of degree < d has at most d-1
    roots, so Omega is SPD iff at least ``d`` days have ``w > 0``.  With some
    ``lam_r = 0`` the count argument does not hold and a dense eigenvalue test
    is used instead.
    """
    w = np.asarray(w, dtype=np.float64)
    lt = lam_tilde(lam, w.shape[0], d)
    if np.all(lt > 0):
        return int(np.count_nonzero(w > 0)) >= d
    ev = np.linalg.eigvalsh(omega_dense(w, lam, d, dtype=np.float64))
    return bool(ev.min() > 0)


def forward_backward_bands(Y, w, lam, d: int, G, steps: int = 2) -> dict:
    """C bands of one pixel sharing ``w`` and ``lam`` (the paper's multivariate batching,
    P:28; C = 10 bands per pixel in its benchmark).

    Omega = W + D^T Lambda D is common to the bands, so for each band c
    ``z_c = Omega^{-1} W y_c`` (Eq. (3)) and ``u_c = Omega^{-1} g_c``; ``dL/dy_c = w * u_c``
    (Eq. (5)); lambda enters every band's solve, so by the chain rule
    ``dL/dlam_r = sum_c -(D u_c)_r (D z_c)_r`` (Eq. (4) contracted with each g_c, summed).
    ``Y``, ``G``: (C, T).  Returns long-double arrays.
    """
    Om = omega_dense(w, lam, d)
    F = _Factor(Om)
    Y = np.atleast_2d(np.asarray(Y, dtype=np.float64))
    G = np.atleast_2d(np.asarray(G, dtype=np.float64))
    zs, us = [], []
    for c in range(Y.shape[0]):
        zs.append(F.solve(_rhs(Y[c], w), steps))
        us.append(F.solve(G[c].astype(LD), steps))
    Z, U = np.array(zs), np.array(us)
    ybar = np.asarray(w, dtype=np.float64).astype(LD)[None, :] * U
    terms = -apply_D(U, d) * apply_D(Z, d)
    lamb = terms.sum(axis=0)
    if np.asarray(lam).ndim == 0:
        lamb = lamb.sum()
    return {"z": Z, "dz": apply_D(Z, d), "u": U, "ybar": ybar, "lambar": lamb, "lambar_terms": terms}


def posterior_variance(w, lam, d: int, rows=None, steps: int = 2) -> np.ndarray:
    """``diag(Omega^{-1})`` (NEXT-4): the pointwise posterior variance of z up to the noise
    variance factor, behind the credibility band of Fig. 4 (its formula, eq. (2.2) of
    the cited Bayesian Whittaker paper, is external -- reading R-15: under the Gaussian model
    y ~ N(z, sigma^2 W^{-1}) with prior precision D^T Lambda D / sigma^2, Cov(z | y) =
    sigma^2 Omega^{-1}).  Plain definition: ``Sigma_tt = e_t^T Omega^{-1} e_t`` by a refined
    dense solve per requested row (all rows by default).  Long double.
    """
    Om = omega_dense(w, lam, d)
    F = _Factor(Om)
    T = Om.shape[0]
    rows = range(T) if rows is None else rows
    out = []
    for t in rows:
        e = np.zeros(T, dtype=LD)
        e[t] = 1
        out.append(F.solve(e, steps)[t])
    return np.array(out, dtype=LD)


def mse_loss_grad(z, y, loss_w):
    """NEXT-3: the training loss of the paper in the form of its MSE metric,
    ``L = T^{-1} sum_t lw_t (z_t - y_t)^2``, and its cotangent ``g = dL/dz = 2 T^{-1} lw (z - y)``.
    ``lw`` selects the scored dates (e.g. the randomly held-out ones, whose W_tt was set to 0 in
    the smoother); terms with ``lw_t = 0`` are exactly 0 (their y may be NaN).  Long double."""
    z = np.asarray(z).astype(LD)
    y = np.asarray(y, dtype=np.float64)
    lw = np.asarray(loss_w, dtype=np.float64)
    T = z.shape[-1]
    e = np.where(lw != 0, z - y.astype(LD), LD(0))
    return (lw.astype(LD) * e * e).sum(axis=-1) / T, 2 * lw.astype(LD) * e / T


# ----------------------------------------------------------------------------- irregular grid (NEXT-2)
def difference_matrix_times(times, d: int, dtype=LD) -> np.ndarray:
    """Order-d difference operator on uneven acquisition times (the dspline divided
    differences it cites, as restated by SPEC S:130): D^(1) = plain forward differences,
    D^(m+1) = Bdiff . diag(m / (t_{i+m} - t_i)) . D^(m).  Row r spans dates r..r+d.
    On unit-spaced times this is exactly the binomial stencil (R-3)."""
    t = np.asarray(times, dtype=np.float64).astype(dtype)
    T = t.shape[0]
    if T < d + 1:
        raise ValueError("need T >= d + 1")
    Dm = np.zeros((T - 1, T), dtype=dtype)
    Dm[np.arange(T - 1), np.arange(T - 1)] = -1
    Dm[np.arange(T - 1), np.arange(1, T)] = 1
    for m in range(1, d):
        n = Dm.shape[0]
        scale = dtype(m) / (t[m:m + n] - t[:n])
        S = Dm * scale[:, None]
        Dm = S[1:] - S[:-1]
    return Dm


def omega_dense_times(w, lam, times, d: int, dtype=LD) -> np.ndarray:
    """Omega = W + D^T diag(lam) D with D from the acquisition times, as sum_r lam_r d_r d_r^T."""
    w = np.asarray(w, dtype=np.float64)
    T = w.shape[0]
    lt = lam_tilde(lam, T, d)
    Dm = difference_matrix_times(times, d, dtype)
    Om = np.zeros((T, T), dtype=dtype)
    Om[np.arange(T), np.arange(T)] = w.astype(dtype)
    for r in range(T - d):
        c = Dm[r, r:r + d + 1]
        Om[r:r + d + 1, r:r + d + 1] += dtype(lt[r]) * np.outer(c, c)
    return Om


def forward_backward_times(y, w, lam, times, d: int, g, steps: int = 2) -> dict:
    """Eq. (3)-(5) on an irregular grid (z, dz = D z, u, ybar, lambar), long double."""
    Om = omega_dense_times(w, lam, times, d)
    F = _Factor(Om)
    z = F.solve(_rhs(y, w), steps)
    u = F.solve(np.asarray(g, dtype=np.float64).astype(LD), steps)
    Dm = difference_matrix_times(times, d)
    dz, du = Dm @ z, Dm @ u
    lamb = -du * dz
    if np.asarray(lam).ndim == 0:
        lamb = lamb.sum()
    return {"z": z, "dz": dz, "u": u, "ybar": np.asarray(w, dtype=np.float64).astype(LD) * u, "lambar": lamb}
