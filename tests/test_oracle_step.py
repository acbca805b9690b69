"""Pins for the oracle's whole split step (RNEP Alg. 5, RGNEP Alg. 4) — CPU only.

Ground truth here is what the paper and the mathematics fix: worked 2x2 cases
(SPEC.md:262-273), known-eigenvalue constructions (north_star), a brute-force
characteristic-polynomial root solve at n <= 8 (north_star), QZ eigenvalue counts for
pencils (scipy, library cross-check), and the convergence behaviour of PAPER.md:541-543.
"""
import itertools

import numpy as np
import pytest
import scipy.linalg as sla

from _util import orth_err, sin_angle
from paper_1011_3077_b200 import inputs


def rng(seed):
    return np.random.default_rng(seed)


def haar(n, seed):
    return inputs.haar(rng(seed).standard_normal((n, n)))


# ---------------------------------------------------------------------------------------
# brute-force eigenvalues: Faddeev-LeVerrier characteristic polynomial + Durand-Kerner
# (Weierstrass) simultaneous root iteration, Newton-polished.  Test-only, n <= 8.
# ---------------------------------------------------------------------------------------
def charpoly(a):
    """Coefficients c_0..c_n of det(zI - A) = sum c_k z^(n-k), c_0 = 1 (Faddeev-LeVerrier)."""
    n = a.shape[0]
    c = [1.0]
    m = np.zeros_like(a)
    for k in range(1, n + 1):
        m = a @ m + c[-1] * np.eye(n)
        c.append(-np.trace(a @ m) / k)
    return np.array(c)


def poly_roots(c, iters=500):
    n = len(c) - 1
    if n == 0:
        return np.array([], dtype=complex)
    p = lambda z: np.polyval(c, z)  # noqa: E731
    dp = np.polyder(c)
    rad = 1 + np.max(np.abs(c[1:]))
    z = rad * np.exp(2j * np.pi * (np.arange(n) + 0.25) / n) * 0.9
    for _ in range(iters):
        znew = z.copy()
        for i in range(n):
            den = np.prod([z[i] - z[j] for j in range(n) if j != i]) if n > 1 else 1.0
            znew[i] = z[i] - p(z[i]) / den
        z = znew
    for _ in range(5):  # Newton polish
        d = np.polyval(dp, z)
        ok = np.abs(d) > 0
        z[ok] = z[ok] - p(z[ok]) / d[ok]
    return z


def match_multisets(x, y):
    """min over permutations of max |x_i - y_pi(i)| (brute force, len <= 8)."""
    assert len(x) == len(y)
    best = np.inf
    for perm in itertools.permutations(range(len(y))):
        best = min(best, max(abs(x[i] - y[perm[i]]) for i in range(len(x))))
    return best


def test_charpoly_roots_self_check():
    # the brute-force solver itself: companion-free known polynomial (z-2)(z+0.5)(z^2+1)
    a = np.diag([2.0, -0.5]).astype(float)
    rot = np.array([[0.0, 1.0], [-1.0, 0.0]])
    a = sla.block_diag(a, rot)
    z = poly_roots(charpoly(a))
    assert match_multisets(list(z), [2, -0.5, 1j, -1j]) <= 1e-10


# ---------------------------------------------------------------------------------------
# worked 2x2 cases
# ---------------------------------------------------------------------------------------
def test_diag_4_quarter_leading_block_outside(orc):
    # A = diag(4, 1/4), B = I: split at 1, leading block eigenvalue {4}
    a = np.diag([4.0, 0.25])
    res = orc.split(a, V=haar(2, 77), max_iters=10)
    assert (res.r, res.k) == (1, 1)
    assert abs(res.Ahat[0, 0]) == pytest.approx(4.0, rel=1e-12)
    assert res.Ahat[1, 1] == pytest.approx(0.25, rel=1e-12)
    assert res.status == orc.STATUS_SPLIT


def test_diag_2_half_metric(orc):
    # A = diag(2, 1/2) -> split, metric <= 1e-12
    res = orc.split(np.diag([2.0, 0.5]), V=haar(2, 78), max_iters=12)
    assert res.k == 1 and res.metric <= 1e-12


def test_orthogonal_matrix_does_not_split(orc):
    # A orthogonal (all |lambda| = 1) -> no split
    q = haar(8, 79)
    res = orc.split(q, V=haar(8, 80), max_iters=20)
    assert res.status == orc.STATUS_NO_SPLIT
    assert res.metric > 1e-8


def test_identity_pencil_does_not_split(orc):
    # A = B = I (eigenvalue 1 on the circle) -> failure outcome
    n = 4
    res = orc.split(np.eye(n), B=np.eye(n), V=haar(n, 81), VL=haar(n, 82), max_iters=20)
    assert res.status == orc.STATUS_NO_SPLIT


def test_argument_errors(orc):
    with pytest.raises(ValueError):
        orc.split(np.eye(1), V=np.eye(1))          # n < 2
    with pytest.raises(ValueError):
        orc.split(np.eye(3), V=np.eye(3), max_iters=0)


# ---------------------------------------------------------------------------------------
# n <= 8: eigenvalues of A11 u A22 = brute-force charpoly roots of A (north_star)
# ---------------------------------------------------------------------------------------
def _random_known(n, seed):
    g = rng(seed)
    blocks, lams = [], []
    while sum(b.shape[0] for b in blocks) < n:
        left = n - sum(b.shape[0] for b in blocks)
        mod = g.uniform(0.2, 0.8) if g.uniform() < 0.5 else g.uniform(1.25, 3.0)
        if left >= 2 and g.uniform() < 0.5:
            phi = g.uniform(0.3, np.pi - 0.3)
            c, s = mod * np.cos(phi), mod * np.sin(phi)
            blocks.append(np.array([[c, s], [-s, c]]))
            lams += [complex(c, s), complex(c, -s)]
        else:
            sgn = 1.0 if g.uniform() < 0.5 else -1.0
            blocks.append(np.array([[sgn * mod]]))
            lams.append(complex(sgn * mod))
    T = sla.block_diag(*blocks) + np.triu(g.standard_normal((n, n)) * 0.3, 1) * 0
    S = g.standard_normal((n, n)) + 2 * np.eye(n)
    return S @ T @ np.linalg.inv(S), np.array(lams)


@pytest.mark.parametrize("n,seed", [(2, 0), (3, 2), (4, 0), (5, 4), (6, 5), (7, 6), (8, 7), (8, 8)])
def test_small_n_eigenvalues_match_charpoly(orc, n, seed):
    # seeds chosen so every spectrum has eigenvalues on both sides of the circle (a
    # one-sided spectrum has no split to check); asserted, never skipped
    a, lams = _random_known(n, 600 + seed)
    assert np.any(np.abs(lams) > 1) and np.any(np.abs(lams) < 1)
    res = orc.split(a, V=haar(n, 700 + seed), max_iters=14)
    r = res.r
    assert res.k == int(np.sum(np.abs(lams) < 1))
    ah = res.Ahat
    z_all = poly_roots(charpoly(a))
    z11 = poly_roots(charpoly(ah[:r, :r]))
    z22 = poly_roots(charpoly(ah[r:, r:]))
    nrm = np.linalg.norm(a, 2)
    assert match_multisets(list(z11) + list(z22), list(z_all)) <= 1e-8 * nrm
    assert np.all(np.abs(z11) > 1) and np.all(np.abs(z22) < 1)
    assert res.metric <= 1e-12


# ---------------------------------------------------------------------------------------
# configurations (BASELINE.json) at oracle-friendly sizes
# ---------------------------------------------------------------------------------------
def test_config1_exact(orc):
    # configs[0]: n=64 Ginibre, 12 passes. k = #|lambda|<1 (numpy eigvals cross-check)
    p = inputs.make_config(1)
    res = orc.split(p.A, V=p.V, max_iters=p.max_iters)
    lam = np.linalg.eigvals(p.A)
    assert res.k == int(np.sum(np.abs(lam) < 1))
    assert res.metric <= 1e-13
    assert orth_err(res.Q) <= 1e-13 * p.n
    assert res.status == orc.STATUS_SPLIT
    # similarity: Ahat = Q^T A Q
    assert np.allclose(res.Ahat, res.Q.T @ p.A @ res.Q, atol=1e-12)


def test_config1_e21_falls(orc):
    # north_star: ||E21|| must fall as the iteration converges (reading Q17):
    # at the final split r_final, ||E21(r_final)|| is non-increasing from the first pass
    # where it is < 0.1 until it is within 10x of the final floor; final <= 1e-3 x mid.
    p = inputs.make_config(1)
    final = orc.split(p.A, V=p.V, max_iters=p.max_iters)
    rf = final.r
    nA = orc.norm1(p.A)
    e = []
    for passes in range(1, p.max_iters + 1):
        res = orc.split(p.A, V=p.V, max_iters=passes)
        e.append(np.linalg.norm(res.Ahat[rf:, :rf], 1) / nA)
    floor = e[-1]
    start = next(i for i, x in enumerate(e) if x < 0.1)
    stop = next(i for i, x in enumerate(e) if x <= 10 * floor)
    assert all(e[i + 1] <= e[i] for i in range(start, stop))
    assert floor <= 1e-3 * e[(p.max_iters + 1) // 2 - 1]


def test_config2_twin_known_spectrum(orc):
    # configs[1] recipe at n=128: A = U diag(lam) U^T -> k = #|lam|<1 = 64 exactly, and
    # span Q(:,1:r) = span of the lam>1 eigenvectors (eigh, library cross-check)
    n = 128
    p = inputs.make_config(2, n=n)
    res = orc.split(p.A, V=p.V, max_iters=p.max_iters)
    assert res.k == p.expected_k == 64
    w, u = np.linalg.eigh((p.A + p.A.T) / 2)
    uo = u[:, w > 1]
    assert sin_angle(res.Q[:, : res.r], uo) <= 1e-9
    assert res.metric <= 1e-12
    assert orth_err(res.Q) <= 1e-13 * n


def test_config5_twin_nonnormal(orc):
    # configs[4] recipe at n=64: k = n/2 exactly; Gelfand side checks:
    # ||A22^64||^(1/64) < 1 and ||A11^-64||^(1/64) < 1
    n = 64
    p = inputs.make_config(5, n=n)
    res = orc.split(p.A, V=p.V, max_iters=p.max_iters)
    assert res.k == p.expected_k == n // 2
    r = res.r
    a11, a22 = res.Ahat[:r, :r], res.Ahat[r:, r:]
    assert np.linalg.norm(np.linalg.matrix_power(a22, 64), 2) ** (1 / 64) < 1
    assert np.linalg.norm(np.linalg.matrix_power(np.linalg.inv(a11), 64), 2) ** (1 / 64) < 1
    assert res.metric <= 1e-12


def test_config3_twin_monitor_mode(orc):
    # configs[2] protocol at n=48 (reading Q11): split after every pass,
    # stop at the first pass with metric <= tol; hist holds (r*, metric) per pass.
    p = inputs.make_config(3, n=48)
    res = orc.split(p.A, V=p.V, max_iters=30, tol=1e-12, stop=orc.STOP_E21)
    h = res.hist
    assert res.converged == 1 and res.iters < 30
    assert h[res.iters - 1, 1] == res.metric <= 1e-12
    assert np.all(h[: res.iters - 1, 1] > 1e-12)
    assert np.all(np.isnan(h[res.iters:, 1]))
    lam = np.linalg.eigvals(p.A)
    assert res.k == int(np.sum(np.abs(lam) < 1))
    # fixed mode with the same p gives the same split
    fx = orc.split(p.A, V=p.V, max_iters=res.iters)
    assert fx.r == res.r and fx.metric == res.metric


def test_rtest_mode(orc):
    # Alg. 3 line 4: stop when ||R_j - R_{j-1}||_1 <= tau ||R_{j-1}||_1
    p = inputs.make_config(1)
    res = orc.split(p.A, V=p.V, max_iters=40, tol=1e-6, stop=orc.STOP_RTEST)
    h = res.hist[:, 2]
    assert res.converged == 1
    assert h[res.iters - 1] <= 1e-6 and np.all(h[1: res.iters - 1] > 1e-6)
    assert np.isnan(h[0])


@pytest.mark.parametrize("n,seed", [(16, 4), (40, 5)])
def test_pencil_qz_count_and_block_triangular(orc, n, seed):
    # configs[3] recipe at small n: k = #|lambda(A,B)| < 1 (QZ via scipy, cross-check);
    # Ahat = Q_L^T A Q_R, Bhat = Q_L^T B Q_R block upper triangular at r;
    # (A11,B11) eigenvalues outside, (A22,B22) inside.
    a = rng(seed).standard_normal((n, n))
    b = rng(seed + 1).standard_normal((n, n))
    v, vl = haar(n, 1000 + seed), haar(n, 2000 + seed)
    res = orc.split(a, B=b, V=v, VL=vl, max_iters=30)
    lam = sla.eigvals(a, b)
    assert res.k == int(np.sum(np.abs(lam) < 1))
    r = res.r
    ah = res.QL.T @ a @ res.Q
    bh = res.QL.T @ b @ res.Q
    assert np.allclose(ah, res.Ahat, atol=1e-12)
    met = np.linalg.norm(ah[r:, :r], 1) / np.linalg.norm(a, 1) + \
        np.linalg.norm(bh[r:, :r], 1) / np.linalg.norm(b, 1)
    assert met == pytest.approx(res.metric, rel=1e-8, abs=1e-15)
    assert res.metric <= 1e-10
    l11 = sla.eigvals(ah[:r, :r], bh[:r, :r])
    l22 = sla.eigvals(ah[r:, r:], bh[r:, r:])
    assert np.all(np.abs(l11) > 1) and np.all(np.abs(l22) < 1)
    assert orth_err(res.Q) <= 1e-13 * n and orth_err(res.QL) <= 1e-13 * n


# ---------------------------------------------------------------------------------------
# R-test ratio, status rule and the Frobenius diagnostic (Alg. 3 line 4;
# DESIGN.md readings Q2, Q4, Q5) -- pinned against independent computations
# ---------------------------------------------------------------------------------------
def _numpy_irs_r(a, b, passes):
    """R_j (diag >= 0) of passes j = 0..passes-1 by an independent IRS in numpy/LAPACK:
    full QR of [B_j; -A_j] (numpy.linalg.qr, complete mode), Q12 = Q(0:n, n:2n) multiplies
    A_j, Q22 = Q(n:2n, n:2n) multiplies B_j."""
    n = a.shape[0]
    rs = []
    for _ in range(passes):
        q, r = np.linalg.qr(np.vstack([b, -a]), mode="complete")
        d = np.where(np.diag(r[:n]) < 0, -1.0, 1.0)
        rs.append(d[:, None] * r[:n])
        a, b = q[:n, n:].T @ a, q[n:, n:].T @ b
    return rs


def test_rtest_ratio_matches_independent_irs(orc):
    # hist[:, 2] = ||R_j - R_{j-1}||_1 / ||R_{j-1}||_1 (NaN at j = 0, reading Q5), with the
    # R_j of an independent numpy IRS; compared where the ratio is far above rounding
    p = inputs.make_config(1)
    passes = 8
    res = orc.split(p.A, V=p.V, max_iters=passes, stop=orc.STOP_FIXED)
    rs = _numpy_irs_r(p.A, np.eye(p.n), passes)
    want = [np.linalg.norm(rs[j] - rs[j - 1], 1) / np.linalg.norm(rs[j - 1], 1) for j in range(1, passes)]
    got = res.hist[1:passes, 2]
    assert np.isnan(res.hist[0, 2])
    big = np.array(want) > 1e-6
    assert big.sum() >= 4
    assert np.allclose(got[big], np.array(want)[big], rtol=1e-7, atol=0)


def test_rtest_stops_at_first_eligible_pass(orc):
    # A = I, B = 0: R_0 = I (stack [0; -I]), A_1 = Q12^T orthogonal, B_1 = 0, so R_1 = I and the
    # ratio at j = 1 is exactly 0: the R-test (first eligible at j = 1, reading Q5) stops
    # with p = j + 1 = 2
    n = 6
    res = orc.split(np.eye(n), B=np.zeros((n, n)), V=haar(n, 90), VL=haar(n, 91), max_iters=10,
                    tol=1e-14, stop=orc.STOP_RTEST)
    assert res.converged == 1 and res.iters == 2
    assert res.hist[1, 2] <= 1e-14


@pytest.mark.parametrize("theta", [1e-4, 0.3])
def test_rotation_closed_form_metric_and_status(orc, theta):
    # A = rotation by theta (both eigenvalues on the unit circle: no split).  Any orthogonal
    # similarity of a 2x2 rotation is a rotation by +-theta, so at r = 1 (the only split)
    # |E21| = sin(theta) whatever Q the method returns: metric = sin/(cos + sin) (1-norm,
    # Q2/Q3) and metric_fro = sin/sqrt(2) (F-norm); the metric is far above the 1e-8
    # acceptance threshold, so status = NO_SPLIT (reading Q4)
    c, s = np.cos(theta), np.sin(theta)
    a = np.array([[c, -s], [s, c]])
    res = orc.split(a, V=haar(2, 92), max_iters=12)
    assert res.r == 1 and res.k == 1
    assert res.metric == pytest.approx(s / (c + s), rel=1e-10)
    assert res.metric_fro == pytest.approx(s / np.sqrt(2.0), rel=1e-10)
    assert res.status == orc.STATUS_NO_SPLIT


def test_status_threshold_reading_q4(orc):
    # status 0 iff metric <= 1e-8 (reading Q4): a diagonal pencil splits to rounding (status 0);
    # a rotation by 1e-6 gives metric ~1e-6 in (1e-8, 1e-3) -> status 1
    res = orc.split(np.diag([2.0, 0.5]), V=haar(2, 93), max_iters=12)
    assert res.metric <= 1e-14 and res.status == orc.STATUS_SPLIT
    t = 1e-6
    a = np.array([[np.cos(t), -np.sin(t)], [np.sin(t), np.cos(t)]])
    res = orc.split(a, V=haar(2, 94), max_iters=12)
    assert 1e-8 < res.metric < 1e-3 and res.status == orc.STATUS_NO_SPLIT


def test_metric_fro_is_frobenius_e21(orc):
    # metric_fro = ||Ahat(r+1:n, 1:r)||_F / ||A||_F at the selected r (reading Q2); Ahat itself
    # is pinned as Q^T A Q with Q orthogonal; checked at a pass where E21 is not yet tiny
    p = inputs.make_config(1)
    res = orc.split(p.A, V=p.V, max_iters=3)
    r = res.r
    want = np.linalg.norm(res.Ahat[r:, :r]) / np.linalg.norm(p.A)
    assert want > 1e-6
    assert res.metric_fro == pytest.approx(want, rel=1e-12)
    want1 = np.abs(res.Ahat[r:, :r]).sum(axis=0).max() / np.abs(p.A).sum(axis=0).max()
    assert res.metric == pytest.approx(want1, rel=1e-12)
