"""Pins of the CPU oracle (O1 dense, O2 Algorithm 1) to facts outside the oracle.

Each test names what fixes the expected value: a worked example in
tests/golden/ (cited), exact rational arithmetic on the objective Eq. (1), a
closed form, a mathematical invariant, or central finite differences.  None
re-types the oracle's formulas.
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
from oracle import banded as O2
from oracle import whittaker as O1

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_worked_examples.json")))
rng = np.random.default_rng(2604_00048)


# ----------------------------------------------------------------- helpers (independent)
def divided_difference_matrix(times, order):
    """dspline recursion restated in SPEC S:130 (cited by P:28): D^(1) plain
    differences; D^(m+1) = Bdiff . diag(m / (t_{i+m} - t_i)) . D^(m)."""
    t = [Fraction(x) for x in times]
    T = len(t)
    D = [[Fraction(0)] * T for _ in range(T - 1)]
    for i in range(T - 1):
        D[i][i], D[i][i + 1] = Fraction(-1), Fraction(1)
    for m in range(1, order):
        n = len(D)
        scaled = [[D[i][j] * Fraction(m) / (t[i + m] - t[i]) for j in range(T)] for i in range(n)]
        D = [[scaled[i + 1][j] - scaled[i][j] for j in range(T)] for i in range(n - 1)]
    return D


def nth_diff(z, d):
    """Repeated first differences (Delta^d), on any element type."""
    for _ in range(d):
        z = [z[i + 1] - z[i] for i in range(len(z) - 1)]
    return z


def objective(z, y, w, lam, d):
    """Eq. (1)/(3) objective: (y-z)^T W (y-z) + sum_r lam_r (D z)_r^2."""
    dz = nth_diff(list(z), d)
    return sum(wi * (yi - zi) ** 2 for wi, yi, zi in zip(w, y, z)) + sum(l * v * v for l, v in zip(lam, dz))


def exact_minimizer(y, w, lam, d):
    """Minimise the quadratic Eq. (1) exactly in rationals: f(z) = f0 + g.z + z^T H z / 2,
    H and g read off f by exact second differences; solve H z = -g by Gauss-Jordan."""
    T = len(y)
    zero = [Fraction(0)] * T
    f0 = objective(zero, y, w, lam, d)

    def e(i, s=1):
        v = list(zero)
        v[i] = Fraction(s)
        return v

    fp = [objective(e(i), y, w, lam, d) for i in range(T)]
    fm = [objective(e(i, -1), y, w, lam, d) for i in range(T)]
    g = [(fp[i] - fm[i]) / 2 for i in range(T)]
    H = [[None] * T for _ in range(T)]
    for i in range(T):
        H[i][i] = fp[i] + fm[i] - 2 * f0
        for j in range(i + 1, T):
            v = list(zero)
            v[i] = v[j] = Fraction(1)
            H[i][j] = H[j][i] = objective(v, y, w, lam, d) - fp[i] - fp[j] + f0
    A = [row[:] + [-g[i]] for i, row in enumerate(H)]
    for c in range(T):
        p = next(r for r in range(c, T) if A[r][c] != 0)
        A[c], A[p] = A[p], A[c]
        piv = A[c][c]
        A[c] = [x / piv for x in A[c]]
        for r in range(T):
            if r != c and A[r][c] != 0:
                f = A[r][c]
                A[r] = [a - f * b for a, b in zip(A[r], A[c])]
    return [A[i][T] for i in range(T)], H


def dyadic(n, lo, hi, bits=8):
    return [Fraction(int(x), 2 ** bits) for x in rng.integers(lo * 2 ** bits, hi * 2 ** bits, size=n)]


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


# ----------------------------------------------------------------- difference operator
@pytest.mark.parametrize("d", [1, 2, 3, 4])
def test_stencil_is_unit_grid_divided_difference(d):
    """P:28 dspline definition on the unit grid (reading R-3) == binomial stencil."""
    T = d + 6
    Dref = divided_difference_matrix(list(range(T)), d)
    D = O1.difference_matrix(T, d)
    assert np.array_equal(D, np.array(Dref, dtype=np.float64))


def test_divided_difference_golden():
    g = GOLD["divided_difference_uneven"]
    assert [float(x) for x in divided_difference_matrix(g["times"], g["order"])[0]] == g["row"]
    g = GOLD["divided_difference_unit_order1"]
    assert O1.difference_matrix(4, 1).tolist() == g["rows"]


@pytest.mark.parametrize("d", [1, 2, 3])
def test_D_null_space(d):
    """Rows annihilate t^0..t^(d-1) and map t^d to the constant d! (finite-difference calculus)."""
    T = 30
    t = np.arange(T, dtype=np.float64)
    for p in range(d):
        assert np.all(O1.apply_D(t ** p, d) == 0)
    assert np.all(O1.apply_D(t ** d, d) == math.factorial(d))


# ----------------------------------------------------------------- Omega
def test_omega_golden():
    for key in ("gram_order1_T3", "omega_order1_T3"):
        g = GOLD[key]
        Om = O1.omega_dense(np.array(g["w"], float), g["lam"], g["d"], dtype=np.float64)
        assert Om.tolist() == g["omega"], key


@pytest.mark.parametrize("d", [1, 2, 3])
def test_omega_symmetric_banded_spd(d):
    """Omega is SPD with bandwidth k+1 (= d)."""
    T = 50
    w = (rng.random(T) < 0.5).astype(float)
    w[:d] = 1
    lam = 10 ** rng.uniform(-1, 4, T - d)
    Om = O1.omega_dense(w, lam, d, dtype=np.float64)
    assert np.array_equal(Om, Om.T)
    i, j = np.nonzero(Om)
    assert np.max(np.abs(i - j)) == d
    assert np.linalg.eigvalsh(Om).min() > 0


def test_band_storage_golden():
    g = GOLD["band_storage_tridiagonal"]
    A = np.array(g["dense"], float)
    T = A.shape[0]
    band = [[A[t + j, t] if t + j < T else 0 for t in range(T)] for j in range(2)]
    assert band == g["band"]
    # O2 builds the same layout for Omega: band[j, t] == Omega[t+j, t]
    for d in (1, 2, 3):
        T = 12
        w = rng.random(T)
        lam = rng.uniform(0.5, 5, T - d)
        Om = O1.omega_dense(w, lam, d, dtype=np.float64)
        bd = O2.band_from_w_lam(w[None], lam[None], d)[0].astype(np.float64)
        for j in range(d + 1):
            for t in range(T):
                assert bd[j, t] == pytest.approx(Om[t + j, t] if t + j < T else 0.0, rel=1e-15, abs=1e-15)


# ----------------------------------------------------------------- Algorithm 1 (O2)
def test_alg1_golden_factor_and_solve():
    g = GOLD["cholesky_spd"]
    A = np.array(g["dense"], float)
    band = np.array([[[A[t + j, t] if t + j < 3 else 0 for t in range(3)] for j in range(2)]])
    L, info = O2.banded_cholesky_alg1(band)
    assert info[0] == 0
    assert L[0, 0].astype(float).tolist() == g["L_diag"]
    assert L[0, 1, :2].astype(float).tolist() == g["L_sub"]
    s = GOLD["solve_first_column"]
    x = O2.band_solve(L, np.array([s["b"]], float))
    assert x[0].astype(float).tolist() == s["x"]


def test_alg1_golden_indefinite():
    g = GOLD["cholesky_indefinite"]
    A = np.array(g["dense"], float)
    band = np.array([[[A[0, 0], A[1, 1]], [A[1, 0], 0]]])
    _, info = O2.banded_cholesky_alg1(band)
    assert info[0] == g["info"]


@pytest.mark.parametrize("d", [1, 2, 3])
def test_alg1_factor_reproduces_omega(d):
    """L L^T == Omega for random SPD bands, entrywise."""
    T, B = 40, 3
    w = (rng.random((B, T)) < 0.6).astype(float)
    lam = 10 ** rng.uniform(-1, 3, (B, T - d))
    band = O2.band_from_w_lam(w, lam, d)
    L, info = O2.banded_cholesky_alg1(band)
    assert np.all(info == 0)
    for b in range(B):
        Ld = np.zeros((T, T))
        for j in range(d + 1):
            for t in range(T - j):
                Ld[t + j, t] = float(L[b, j, t])
        Om = O1.omega_dense(w[b], lam[b], d, dtype=np.float64)
        assert np.max(np.abs(Ld @ Ld.T - Om)) <= 1e-12 * np.max(np.abs(Om))


# ----------------------------------------------------------------- solve: exact & closed forms
@pytest.mark.parametrize("d,T", [(1, 7), (2, 9), (3, 10)])
@pytest.mark.parametrize("per_date", [False, True])
def test_exact_rational_minimizer(d, T, per_date):
    """Eq. (1)/(3) minimised exactly in rationals == O1 and O2 (to fp64/long-double rounding)."""
    y = dyadic(T, -2, 2)
    w = [Fraction(int(b)) for b in (rng.random(T) < 0.6)]
    for i in range(d):
        w[2 * i] = Fraction(1)
    if per_date:
        lam = dyadic(T - d, 1, 40)
    else:
        lam = [dyadic(1, 1, 40)[0]] * (T - d)
    z, H = exact_minimizer(y, w, lam, d)
    # H / 2 is Omega: the Hessian of Eq. (1)
    Om = O1.omega_dense(np.array(w, float), np.array(lam, float) if per_date else float(lam[0]), d, dtype=np.float64)
    assert np.array_equal(np.array([[float(h / 2) for h in r] for r in H]), Om)
    yf, wf = np.array(y, float), np.array(w, float)
    lf = np.array(lam, float) if per_date else float(lam[0])
    z1, _ = O1.forward(yf, wf, lf, d)
    assert rel(z1, [float(v) for v in z]) < 1e-14
    lam2 = np.array(lam, float)[None] if per_date else np.array([float(lam[0])])
    z2, _, info = O2.forward_banded(yf[None], wf[None], lam2, d)
    assert info[0] == 0
    assert rel(z2[0], [float(v) for v in z]) < 1e-14


def test_gap_golden():
    g = GOLD["gap_interpolation"]
    for lam in g["lams"]:
        z, _ = O1.forward(np.array(g["y"]), np.array(g["w"], float), lam, g["d"])
        assert np.max(np.abs(z.astype(float) - g["z"])) < 1e-12


def test_lambda_zero_identity():
    """lambda = 0, w = 1: Omega = I so z = y exactly (north_star invariant)."""
    T = 200
    y = rng.normal(size=T)
    for d in (1, 2, 3):
        z, _ = O1.forward(y, np.ones(T), 0.0, d)
        assert np.array_equal(z.astype(np.float64), y)
        z2, _, _ = O2.forward_banded(y[None], np.ones((1, T)), np.zeros(1), d)
        assert np.array_equal(z2[0].astype(np.float64), y)


@pytest.mark.parametrize("d", [1, 2, 3])
def test_polynomial_passthrough(d):
    """A polynomial of degree < d has D y = 0 and zero objective: z = y everywhere, gaps included."""
    T = 120
    t = np.arange(T) / T
    coef = rng.normal(size=d)
    y = sum(c * t ** k for k, c in enumerate(coef))
    w = (rng.random(T) < 0.2).astype(float)
    w[[3, 50, 90]] = 1
    lam = 10 ** rng.uniform(0, 5, T - d)
    z, dz = O1.forward(y, w, lam, d)
    assert rel(z, y) < 1e-11
    z2, _, _ = O2.forward_banded(y[None], w[None], lam[None], d)
    assert rel(z2[0], y) < 1e-11


@pytest.mark.parametrize("d", [1, 2, 3])
def test_lambda_infinity_is_weighted_polyfit(d):
    """lambda -> inf: z tends to the weighted least-squares polynomial of degree d-1
    (the penalty forces D z = 0); the gap shrinks like 1/lambda."""
    T = 40
    t = np.arange(T, dtype=float)
    y = np.sin(t / 5) + 0.1 * rng.normal(size=T)
    w = (rng.random(T) < 0.7).astype(float)
    w[[0, 20, 39]] = 1
    X = np.vander(t, d, increasing=True)
    beta, *_ = np.linalg.lstsq(X * np.sqrt(w)[:, None], y * np.sqrt(w), rcond=None)
    p = X @ beta
    errs = []
    for lam in ((1e4, 1e6, 1e8) if d < 3 else (1e6, 1e8, 1e10)):
        z, _ = O1.forward(y, w, lam, d)
        errs.append(np.max(np.abs(z.astype(float) - p)))
    assert errs[2] < 1e-3
    assert errs[1] < errs[0] / 30 and errs[2] < errs[1] / 30


def test_mask_zero_independence():
    """Values at w = 0 do not enter Eq. (3) (W y): z is bitwise unchanged."""
    T, d = 300, 2
    y = rng.normal(size=T)
    w = (rng.random(T) < 0.4).astype(float)
    lam = 10 ** rng.uniform(0, 4, T - d)
    z, _ = O1.forward(y, w, lam, d)
    y2 = y.copy()
    y2[w == 0] = rng.normal(size=int((w == 0).sum())) * 1e6
    y2[np.flatnonzero(w == 0)[:3]] = np.nan
    z2, _ = O1.forward(y2, w, lam, d)
    assert np.array_equal(z, z2)


@pytest.mark.parametrize("d", [1, 2, 3])
def test_time_reversal(d):
    """Reversing y, w and lambda reverses z (|c_j| symmetric, penalty squared)."""
    T = 80
    y = rng.normal(size=T)
    w = (rng.random(T) < 0.5).astype(float)
    w[:3] = 1
    lam = 10 ** rng.uniform(0, 4, T - d)
    z, _ = O1.forward(y, w, lam, d)
    zr, _ = O1.forward(y[::-1].copy(), w[::-1].copy(), lam[::-1].copy(), d)
    assert rel(zr[::-1], z) < 1e-13


def test_optimality_and_normal_equations():
    """z minimises Eq. (1): the objective (computed with Delta^d, not D) rises in every
    random direction, and its exact gradient (linear in z) vanishes."""
    T, d = 60, 2
    y = rng.normal(size=T)
    w = (rng.random(T) < 0.5).astype(float)
    w[:3] = 1
    lam = 10 ** rng.uniform(0, 3, T - d)
    z = O1.forward(y, w, lam, d)[0].astype(float)
    f = objective(z, y, w, lam, d)
    for _ in range(10):
        dlt = rng.normal(size=T) * 1e-3
        assert objective(z + dlt, y, w, lam, d) > f
    grad = np.array([(objective(z + h, y, w, lam, d) - objective(z - h, y, w, lam, d)) / 2e-3
                     for h in np.eye(T) * 1e-3])
    assert np.max(np.abs(grad)) < 1e-9 * max(1.0, np.max(np.abs(y)))


# ----------------------------------------------------------------- SPD status
@pytest.mark.parametrize("d", [1, 2, 3])
def test_spd_count_criterion_exact(d):
    """is_spd's count criterion vs exact rational Cholesky (leading pivots) on tiny T."""
    T = 8
    for nobs in range(0, d + 2):
        w = [Fraction(0)] * T
        for i in rng.choice(T, size=nobs, replace=False):
            w[i] = Fraction(1)
        lam = dyadic(T - d, 1, 9)
        _, H = (None, None)
        # exact Omega from the objective's Hessian
        y = [Fraction(0)] * T
        zero = [Fraction(0)] * T

        def f(v):
            return objective(v, y, w, lam, d)

        Om = [[None] * T for _ in range(T)]
        for i in range(T):
            for j in range(T):
                vi = list(zero); vi[i] += 1
                vj = list(zero); vj[j] += 1
                vij = list(zero); vij[i] += 1; vij[j] += 1
                Om[i][j] = (f(vij) - f(vi) - f(vj)) / 2
        # exact LDL^T pivots
        A = [r[:] for r in Om]
        pivots = []
        for k in range(T):
            p = A[k][k]
            pivots.append(p)
            if p == 0:
                break
            for i in range(k + 1, T):
                fct = A[i][k] / p
                for j in range(k, T):
                    A[i][j] -= fct * A[k][j]
        exact_spd = len(pivots) == T and all(p > 0 for p in pivots)
        assert O1.is_spd(np.array(w, float), np.array(lam, float), d) == exact_spd
        assert exact_spd == (nobs >= d)
        if nobs == 0:
            # all-zero mask: first singular leading minor is T-d+1 (1-based)
            assert len(pivots) == T - d + 1 and pivots[-1] == 0


# ----------------------------------------------------------------- gradients
@pytest.mark.parametrize("d", [1, 2, 3])
@pytest.mark.parametrize("per_date", [True, False])
def test_gradients_central_fd(d, per_date):
    """Eq. (4)/(5) contracted == central finite differences of L = g.z."""
    T = 32
    y = rng.normal(size=T)
    w = (rng.random(T) < 0.6).astype(float)
    w[:d + 1] = 1
    lam = 10 ** rng.uniform(0, 2, T - d) if per_date else 10 ** rng.uniform(0, 2)
    g = rng.normal(size=T)
    out = O1.forward_backward(y, w, lam, d, g)

    def L(yv, lv):
        return float(np.dot(g, O1.forward(yv, w, lv, d)[0].astype(float)))

    h = 1e-6
    fd_y = np.array([(L(y + h * e, lam) - L(y - h * e, lam)) / (2 * h) for e in np.eye(T)])
    assert rel(out["ybar"], fd_y) < 1e-7
    if per_date:
        fd_l = np.array([(L(y, lam * np.exp(h * e)) - L(y, lam * np.exp(-h * e))) / (2 * h) for e in np.eye(T - d)]) / lam
    else:
        fd_l = (L(y, lam * np.exp(h)) - L(y, lam * np.exp(-h))) / (2 * h) / lam
    assert rel(out["lambar"], fd_l) < 1e-6


@pytest.mark.parametrize("d", [1, 2, 3])
def test_weight_grad_central_fd(d):
    """dL/dw_t = u_t (y_t - z_t) (NEXT-3 option; Eq. (3) differentiated in w_t) == central finite
    differences of L = g.z in w_t at every observed day, for soft weights; 0 at unobserved days (R-19)."""
    T = 28
    y = rng.normal(size=T)
    w = np.where(rng.random(T) < 0.6, rng.uniform(0.2, 1.0, T), 0.0)
    w[:d + 1] = rng.uniform(0.2, 1.0, d + 1)
    y[w == 0] = np.nan  # unobserved values never enter (R-4)
    lam = 10 ** rng.uniform(0, 2, T - d)
    g = rng.normal(size=T)
    out = O1.forward_backward(y, w, lam, d, g)
    wg = O1.weight_grad(y, w, out["z"], out["u"]).astype(float)
    assert np.all(wg[w == 0] == 0)

    def L(wv):
        return float(np.dot(g, O1.forward(y, wv, lam, d)[0].astype(float)))

    h = 1e-6
    obs = np.flatnonzero(w > 0)
    fd = np.array([(L(w + h * np.eye(T)[t]) - L(w - h * np.eye(T)[t])) / (2 * h) for t in obs])
    assert rel(wg[obs], fd) < 1e-7


def test_eq4_explicit_column_contracts_to_lambar():
    """Eq. (4) as printed, dz/dlam_t = -Omega^{-1} d_t d_t^T z, contracted with g == lambar_t."""
    T, d = 30, 2
    y = rng.normal(size=T)
    w = (rng.random(T) < 0.6).astype(float)
    w[:3] = 1
    lam = 10 ** rng.uniform(0, 2, T - d)
    g = rng.normal(size=T)
    out = O1.forward_backward(y, w, lam, d, g)
    z = out["z"].astype(float)
    Om = O1.omega_dense(w, lam, d, dtype=np.float64)
    D = O1.difference_matrix(T, d)
    cols = np.array([-np.linalg.solve(Om, D[t] * (D[t] @ z)) for t in range(T - d)])
    assert rel(out["lambar"], cols @ g) < 1e-9


def test_scalar_chain_rule_and_zero_cotangent():
    """sum_r lambar_r (per-date, constant lambda) == scalar lambar; g = 0 -> zero grads."""
    T, d = 64, 2
    y = rng.normal(size=T)
    w = (rng.random(T) < 0.5).astype(float)
    w[:3] = 1
    g = rng.normal(size=T)
    a = O1.forward_backward(y, w, 37.5, d, g)
    b = O1.forward_backward(y, w, np.full(T - d, 37.5), d, g)
    assert np.array_equal(a["z"], b["z"])
    assert abs(float(a["lambar"]) - float(b["lambar"].sum())) <= 1e-15 * float(np.abs(b["lambar"]).sum())
    c = O1.forward_backward(y, w, 37.5, d, np.zeros(T))
    assert np.all(c["ybar"] == 0) and c["lambar"] == 0


# ----------------------------------------------------------------- O2 vs O1 at realistic shape
@pytest.mark.parametrize("d", [1, 2, 3])
def test_O2_matches_O1_small(d):
    T, B = 90, 4
    y = rng.normal(size=(B, T))
    w = (rng.random((B, T)) < 0.5).astype(float)
    w[:, :d + 1] = 1
    lam = 10 ** rng.uniform(0, 4, (B, T - d))
    g = rng.normal(size=(B, T))
    z2, dz2, info = O2.forward_banded(y, w, lam, d)
    yb2, lb2 = O2.backward_banded(g, w, lam, d, z2)
    for b in range(B):
        o = O1.forward_backward(y[b], w[b], lam[b], d, g[b])
        assert rel(z2[b], o["z"]) < 1e-13
        assert rel(yb2[b], o["ybar"]) < 1e-12
        assert rel(lb2[b], o["lambar"]) < 1e-12


@pytest.mark.slow
def test_O2_matches_O1_sentinel2_daily():
    """T = 3288 daily grid with the Sentinel-2 gap model (incl. 90-day trailing gap), d = 2."""
    import synth
    x = synth.make_inputs("hetero", B=2)
    y, w, lam, g = (synth.series_major(x[k]) for k in ("y", "w", "lam", "g"))
    z2, _, info = O2.forward_banded(y, w, lam, 2)
    yb2, lb2 = O2.backward_banded(g, w, lam, 2, z2)
    assert np.all(info == 0)
    for b in range(2):
        o = O1.forward_backward(y[b], w[b], lam[b], 2, g[b])
        assert np.max(np.abs(z2[b] - o["z"])) / np.max(np.abs(y[b])) < 1e-11
        assert rel(yb2[b], o["ybar"]) < 1e-10
        assert rel(lb2[b], o["lambar"]) < 1e-10


# ----------------------------------------------------------------- multi-band (NEXT-1)
@pytest.mark.parametrize("per_date", [True, False])
def test_bands_shared_factor_fd_and_per_band(per_date):
    """C bands sharing w, lambda: each band equals the single-band solve, and the summed
    lambda gradient matches central finite differences of L = sum_c g_c . z_c."""
    T, d, C = 30, 2, 3
    Y = rng.normal(size=(C, T))
    G = rng.normal(size=(C, T))
    w = (rng.random(T) < 0.6).astype(float)
    w[:3] = 1
    lam = 10 ** rng.uniform(0, 2, T - d) if per_date else 10 ** rng.uniform(0, 2)
    o = O1.forward_backward_bands(Y, w, lam, d, G)
    for c in range(C):
        s1 = O1.forward_backward(Y[c], w, lam, d, G[c])
        assert rel(o["z"][c], s1["z"]) < 1e-15 and rel(o["ybar"][c], s1["ybar"]) < 1e-15

    def L(lv):
        return sum(float(np.dot(G[c], O1.forward(Y[c], w, lv, d)[0].astype(float))) for c in range(C))

    h = 1e-6
    if per_date:
        fd = np.array([(L(lam * np.exp(h * e)) - L(lam * np.exp(-h * e))) / (2 * h) for e in np.eye(T - d)]) / lam
    else:
        fd = (L(lam * np.exp(h)) - L(lam * np.exp(-h))) / (2 * h) / lam
    assert rel(o["lambar"], fd) < 1e-6


# ----------------------------------------------------------------- posterior variance (NEXT-4)
@pytest.mark.parametrize("d,T", [(1, 7), (2, 8), (3, 9)])
def test_posterior_variance_exact_rational(d, T):
    """diag(Omega^{-1}) == the exact rational inverse of half the Hessian of Eq. (1)."""
    w = [Fraction(int(b)) for b in (rng.random(T) < 0.6)]
    for i in range(d):
        w[2 * i] = Fraction(1)
    lam = dyadic(T - d, 1, 40)
    _, H = exact_minimizer([Fraction(0)] * T, w, lam, d)
    A = [[h / 2 for h in row] + [Fraction(int(i == j)) for j in range(T)] for i, row in enumerate(H)]
    for c in range(T):
        p = next(r for r in range(c, T) if A[r][c] != 0)
        A[c], A[p] = A[p], A[c]
        piv = A[c][c]
        A[c] = [x / piv for x in A[c]]
        for r in range(T):
            if r != c and A[r][c] != 0:
                f = A[r][c]
                A[r] = [a - f * b for a, b in zip(A[r], A[c])]
    exact = [float(A[i][T + i]) for i in range(T)]
    got = O1.posterior_variance(np.array(w, float), np.array(lam, float), d)
    assert rel(got, exact) < 1e-14


def test_posterior_variance_properties():
    """lambda = 0, w = 1 -> Omega = I -> variance 1; an extra observation never increases any
    variance (Omega grows in the Loewner order); time reversal."""
    T, d = 60, 2
    assert np.allclose(O1.posterior_variance(np.ones(T), 0.0, d).astype(float), 1.0, rtol=0, atol=1e-15)
    w = (rng.random(T) < 0.3).astype(float)
    w[[0, 30, 59]] = 1
    lam = 10 ** rng.uniform(0, 3, T - d)
    v0 = O1.posterior_variance(w, lam, d).astype(float)
    w2 = w.copy()
    w2[np.flatnonzero(w == 0)[5]] = 1
    v1 = O1.posterior_variance(w2, lam, d).astype(float)
    assert np.all(v1 <= v0 * (1 + 1e-13))
    vr = O1.posterior_variance(w[::-1].copy(), lam[::-1].copy(), d).astype(float)
    assert rel(vr[::-1], v0) < 1e-13


# ----------------------------------------------------------------- fused masked-MSE (NEXT-3)
def test_mse_chain_rule_fd():
    """The training step: L(y, lam) = T^-1 sum lw (z(y, lam) - y_ref)^2 with z from Eq. (3);
    backward(g = dL/dz) + the explicit dL/dy_ref term equals central finite differences."""
    T, d = 40, 2
    y = rng.normal(size=T)
    w = (rng.random(T) < 0.6).astype(float)
    w[:3] = 1
    lw = ((rng.random(T) < 0.3) & (w == 0)).astype(float)  # score held-out dates
    lw[5] = 1.0
    w[5] = 0.0
    lam = 10 ** rng.uniform(0, 2, T - d)
    z, _ = O1.forward(y, w, lam, d)
    loss, g = O1.mse_loss_grad(z, y, lw)
    ybar, lambar = O1.backward(g.astype(float), w, lam, d, z)

    def Lf(yv, lv):
        zz, _ = O1.forward(yv, w, lv, d)
        return float(O1.mse_loss_grad(zz, yv, lw)[0])

    h = 1e-6
    fd_l = np.array([(Lf(y, lam * np.exp(h * e)) - Lf(y, lam * np.exp(-h * e))) / (2 * h) for e in np.eye(T - d)]) / lam
    assert rel(lambar, fd_l) < 1e-6
    # y enters twice: through z (ybar) and as the reference (-g)
    fd_y = np.array([(Lf(y + h * e, lam) - Lf(y - h * e, lam)) / (2 * h) for e in np.eye(T)])
    assert rel(ybar.astype(float) - g.astype(float), fd_y) < 1e-6
    assert abs(float(loss) - np.sum(lw * (z.astype(float) - y) ** 2) / T) < 1e-15


def test_mse_loss_value_exact_on_polynomial_data():
    """The loss VALUE pinned by the polynomial pass-through, not by restating its formula: observed data on a
    line (degree < d) makes z that line exactly (pinned above); held-out dates carry dyadic offsets e_t, so
    L = T^-1 sum lw_t e_t^2 and g = -2 T^-1 lw e are exact rationals the oracle must reproduce."""
    from fractions import Fraction as F
    T, d = 48, 2
    t = np.arange(T, dtype=float)
    line = 0.5 + 0.25 * t
    w = np.ones(T)
    held = np.array([4, 9, 17, 30, 41])
    e = np.array([0.5, -1.25, 2.0, -0.375, 0.75])
    w[held] = 0.0
    y = line.copy()
    y[held] += e
    lw = np.zeros(T)
    lw[held] = [1.0, 0.5, 1.0, 2.0, 1.0]
    z, _ = O1.forward(y, w, 1e3, d)
    assert np.max(np.abs(z.astype(float) - line)) < 1e-12
    loss, g = O1.mse_loss_grad(line, y, lw)  # the exact z
    exact = sum(F(float(lw[i])) * F(float(v)) ** 2 for i, v in zip(held, e)) / T
    assert float(loss) == float(exact)
    ge = np.zeros(T)
    ge[held] = [-2 * float(lw[i]) * float(v) / T for i, v in zip(held, e)]
    assert np.array_equal(g.astype(float), ge)
    loss_o, _ = O1.mse_loss_grad(z, y, lw)  # through the solve: the same within rounding
    assert abs(float(loss_o) - float(exact)) <= 1e-12 * float(exact)


# ----------------------------------------------------------------- irregular grid (NEXT-2)
def _uneven_times(T, lo=1, hi=12):
    return np.cumsum(rng.integers(lo, hi, size=T)).astype(float)


@pytest.mark.parametrize("d", [1, 2, 3])
def test_times_operator_golden_and_unit_grid(d):
    """SPEC S:134 worked row; unit-spaced times reduce exactly to the daily stencil (R-3)."""
    g = GOLD["divided_difference_uneven"]
    assert O1.difference_matrix_times(g["times"], g["order"]).astype(float)[0].tolist() == g["row"]
    T = 20
    assert np.array_equal(O1.difference_matrix_times(np.arange(T) + 7.0, d).astype(float), O1.difference_matrix(T, d))
    lam = 10 ** rng.uniform(0, 3, T - d)
    w = (rng.random(T) < 0.6).astype(float)
    w[:d] = 1
    y, gg = rng.normal(size=T), rng.normal(size=T)
    a = O1.forward_backward_times(y, w, lam, np.arange(T, dtype=float), d, gg)
    b = O1.forward_backward(y, w, lam, d, gg)
    for k in ("z", "ybar", "lambar"):
        assert rel(a[k], b[k]) < 1e-15


@pytest.mark.parametrize("d", [1, 2, 3])
def test_times_polynomial_annihilation_and_passthrough(d):
    """On ANY increasing grid the rows annihilate t^0..t^(d-1) (divided differences), so a polynomial
    of degree < d in t passes through the smoother unchanged, gaps included."""
    T = 60
    t = _uneven_times(T)
    Dm = O1.difference_matrix_times(t, d).astype(float)
    for p in range(d):
        assert np.max(np.abs(Dm @ (t / t[-1]) ** p)) < 1e-12
    assert np.max(np.abs(Dm @ (t / t[-1]) ** d)) > 1e-9
    coef = rng.normal(size=d)
    y = sum(c * (t / t[-1]) ** k for k, c in enumerate(coef))
    w = (rng.random(T) < 0.3).astype(float)
    w[[1, 20, 40]] = 1
    o = O1.forward_backward_times(y, w, 10 ** rng.uniform(0, 3, T - d), t, d, np.zeros(T))
    assert rel(o["z"], y) < 1e-10


@pytest.mark.parametrize("d", [2, 3])
def test_times_exact_rational(d):
    """Eq. (1) on rational uneven times minimised exactly == oracle."""
    T = 8
    times = [Fraction(int(v)) for v in _uneven_times(T, 1, 5)]
    Drat = divided_difference_matrix(times, d)
    y = dyadic(T, -2, 2)
    w = [Fraction(int(b)) for b in (rng.random(T) < 0.6)]
    for i in range(d):
        w[2 * i] = Fraction(1)
    lam = dyadic(T - d, 1, 20)

    def obj(z):
        dz = [sum(Drat[r][j] * z[j] for j in range(T)) for r in range(T - d)]
        return sum(wi * (yi - zi) ** 2 for wi, yi, zi in zip(w, y, z)) + sum(l * v * v for l, v in zip(lam, dz))

    zero = [Fraction(0)] * T
    f0 = obj(zero)
    fp = [obj([Fraction(int(i == j)) for j in range(T)]) for i in range(T)]
    fm = [obj([Fraction(-int(i == j)) for j in range(T)]) for i in range(T)]
    H = [[None] * T for _ in range(T)]
    for i in range(T):
        H[i][i] = fp[i] + fm[i] - 2 * f0
        for j in range(i + 1, T):
            H[i][j] = H[j][i] = obj([Fraction(int(k in (i, j))) for k in range(T)]) - fp[i] - fp[j] + f0
    A = [row[:] + [-(fp[i] - fm[i]) / 2] for i, row in enumerate(H)]
    for c in range(T):
        p_ = next(r for r in range(c, T) if A[r][c] != 0)
        A[c], A[p_] = A[p_], A[c]
        A[c] = [x / A[c][c] for x in A[c]]
        for r in range(T):
            if r != c and A[r][c] != 0:
                f = A[r][c]
                A[r] = [a - f * b for a, b in zip(A[r], A[c])]
    z_exact = [float(A[i][T]) for i in range(T)]
    o = O1.forward_backward_times(np.array(y, float), np.array(w, float), np.array(lam, float),
                                  np.array(times, float), d, np.zeros(T))
    assert rel(o["z"], z_exact) < 1e-13


def test_times_gradients_fd():
    T, d = 30, 2
    t = _uneven_times(T)
    y, g = rng.normal(size=T), rng.normal(size=T)
    w = (rng.random(T) < 0.6).astype(float)
    w[:3] = 1
    lam = 10 ** rng.uniform(0, 2, T - d)
    o = O1.forward_backward_times(y, w, lam, t, d, g)

    def L(lv):
        return float(np.dot(g, O1.forward_backward_times(y, w, lv, t, d, np.zeros(T))["z"].astype(float)))

    h = 1e-6
    fd = np.array([(L(lam * np.exp(h * e)) - L(lam * np.exp(-h * e))) / (2 * h) for e in np.eye(T - d)]) / lam
    assert rel(o["lambar"], fd) < 1e-6
