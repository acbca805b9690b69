"""Pins for the oracle's IRS pass (Alg. 3), GRURV (Alg. 1/2) and split selection.

Closed forms and identities from the paper (CPU; -m "not gpu").
"""
import numpy as np
import pytest

EPS = np.finfo(np.float64).eps


def rng(seed):
    return np.random.default_rng(seed)


@pytest.mark.parametrize("n", [1, 3, 8])
def test_r_is_cholesky_factor(orc, n):
    # [B;-A] = Q [R;0] with diag(R) >= 0  =>  R^T R = A^T A + B^T B, R = chol (Q6)
    g = rng(100 + n)
    a, b = g.standard_normal((n, n)), g.standard_normal((n, n))
    _, _, r = orc.irs_pass(a, b)
    ref = np.linalg.cholesky(a.T @ a + b.T @ b).T
    assert np.allclose(r, ref, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("n", [2, 4, 8])
def test_squaring_identity(orc, n):
    # A_{j+1}^{-1} B_{j+1} = (A_j^{-1} B_j)^2  (SPEC.md:330 at n <= 8, j <= 3)
    g = rng(200 + n)
    a = g.standard_normal((n, n)) + 2 * np.eye(n)
    b = g.standard_normal((n, n)) * 0.5
    for _ in range(3):
        a1, b1, _ = orc.irs_pass(a, b)
        lhs = np.linalg.solve(a1, b1)
        m = np.linalg.solve(a, b)
        rhs = m @ m
        assert np.linalg.norm(lhs - rhs) <= 1e-8 * np.linalg.norm(rhs)
        # and the Q12^T B = Q22^T A identity behind it: with
        # A_{j+1} = Q12^T A_j, B_{j+1} = Q22^T B_j the pencil stays regular
        a, b = a1, b1


def test_diagonal_pencil_closed_form(orc):
    # Diagonal (a_i, b_i): the stack decouples into 2x2 reflectors; after p passes
    # (A_p+B_p)^{-1} A_p = diag(1/(1+(b_i/a_i)^(2^p))) exactly to rounding, off-diagonal 0.
    av = np.array([2.0, 0.5, 3.0, 1.0 / 3.0, 1.5])
    bv = np.ones_like(av)
    a, b = np.diag(av), np.diag(bv)
    for p in range(1, 6):
        a, b, _ = orc.irs_pass(a, b)
        proj = np.linalg.solve(a + b, a)
        ref = np.diag(1.0 / (1.0 + (bv / av) ** (2 ** p)))
        assert np.allclose(proj, ref, rtol=1e-13, atol=1e-15)
        assert np.count_nonzero(proj - np.diag(np.diag(proj))) == 0


def test_on_circle_shrinks_by_sqrt2(orc):
    # a = b = 1 (eigenvalue on the circle): each pass a' = -a^2/beta, beta = +-sqrt(2)
    a, b = np.eye(3), np.eye(3)
    for p in range(1, 6):
        a, b, _ = orc.irs_pass(a, b)
        assert np.allclose(np.abs(np.diag(a)), 2.0 ** (-p / 2), rtol=1e-14)
        assert np.allclose(np.abs(np.diag(b)), 2.0 ** (-p / 2), rtol=1e-14)


def test_b_zero_stays_zero(orc):
    # B = 0 stays 0
    a = rng(7).standard_normal((4, 4))
    b = np.zeros((4, 4))
    for _ in range(3):
        a, b, _ = orc.irs_pass(a, b)
        assert np.all(b == 0.0)


def test_scalar_lambda_projector_to_identity(orc):
    # A = I, B = lam I, |lam|<1 -> (A_p+B_p)^{-1}A_p -> I, error <= 2 lam^(2^p)
    lam = 0.7
    a, b = np.eye(3), lam * np.eye(3)
    for p in range(1, 7):
        a, b, _ = orc.irs_pass(a, b)
        err = np.linalg.norm(np.linalg.solve(a + b, a) - np.eye(3), 2)
        assert err <= 2 * lam ** (2 ** p) + 1e-15


def test_projector_limit_known_eigenvectors(orc):
    # (A_p+B_p)^{-1}A_p -> P_{R,|z|>1} (projector onto the |lam|>1
    # right eigenvectors along the |lam|<1 ones).  With A = S diag(lam) S^{-1}:
    g = rng(11)
    n = 6
    lam = np.array([4.0, 0.25, 0.5, 3.0, -2.0, 0.1])
    S = g.standard_normal((n, n)) + 3 * np.eye(n)
    a = S @ np.diag(lam) @ np.linalg.inv(S)
    P = S @ np.diag((np.abs(lam) > 1).astype(float)) @ np.linalg.inv(S)
    b = np.eye(n)
    errs = []
    for _ in range(8):
        a, b, _ = orc.irs_pass(a, b)
        errs.append(np.linalg.norm(np.linalg.solve(a + b, a) - P))
    assert errs[-1] <= 1e-10
    # monotone (quadratic) decrease until the rounding floor
    assert all(e2 <= e1 or e2 < 1e-13 for e1, e2 in zip(errs, errs[1:]))
    assert errs[4] <= errs[3] ** 1.5


def _irs(orc, a, b, p):
    for _ in range(p):
        a, b, _ = orc.irs_pass(a, b)
    return a, b


@pytest.mark.parametrize("n", [4, 9, 16])
def test_grurv_lemma(orc, n):
    # PAPER.md:286 lemma with k=2, m=(-1,+1): (A_p+B_p)^{-1} A_p = Q R_1^{-1} R_2 V,
    # i.e. (A_p+B_p)^{-1} A_p V^T = Q R_1^{-1} R_2 (explicit inverse in the test only).
    from paper_1011_3077_b200.inputs import haar
    g = rng(300 + n)
    a = g.standard_normal((n, n)) + 0.5 * np.eye(n)
    ap, bp = _irs(orc, a, np.eye(n), 2)     # not converged: M has full rank
    v = haar(rng(1300 + n).standard_normal((n, n)))
    q, r1, r2 = orc.grurv_right(ap, bp, v)
    lhs = np.linalg.solve(ap + bp, ap) @ v.T
    rhs = q @ np.linalg.solve(r1, r2)
    assert np.linalg.norm(lhs - rhs) <= 1e-10 * np.linalg.norm(lhs)
    assert np.linalg.norm(q.T @ q - np.eye(n)) <= 64 * n * EPS
    assert np.all(np.diag(r1) >= 0) and np.all(np.diag(r2) >= 0)
    assert np.allclose(np.tril(r1, -1), 0) and np.allclose(np.tril(r2, -1), 0)


from _util import sin_angle  # noqa: E402


@pytest.mark.parametrize("n", [6, 12])
def test_grurv_theorem_same_subspace_as_explicit_rurv(orc, n):
    # GRURV gives the same result as RURV on the explicitly formed
    # M = (A_p+B_p)^{-1} A_p: span Q(:,1:r) = span of the leading r columns of QR(M V^T).
    from paper_1011_3077_b200.inputs import haar
    g = rng(400 + n)
    lam = np.concatenate([g.uniform(1.5, 3, n // 2), g.uniform(0.1, 0.6, n - n // 2)])
    S = np.linalg.qr(g.standard_normal((n, n)))[0] + 0.3 * g.standard_normal((n, n))
    a = S @ np.diag(lam) @ np.linalg.inv(S)
    ap, bp = _irs(orc, a, np.eye(n), 8)
    v = haar(rng(1400 + n).standard_normal((n, n)))
    q, _, _ = orc.grurv_right(ap, bp, v)
    M = np.linalg.solve(ap + bp, ap)
    qm = np.linalg.qr(M @ v.T)[0]
    r = n // 2
    assert sin_angle(q[:, :r], qm[:, :r]) <= 1e-12
    # and that subspace is the right invariant subspace of the |lam| > 1 eigenvalues
    qo = np.linalg.qr(S[:, : n // 2])[0]
    assert sin_angle(q[:, :r], qo) <= 1e-12


def test_split_select_hand_cases(orc):
    # SPEC.md:253-255 hand cases.
    ah = np.array([[1.0, 0.0], [1.0, 1.0]])
    r, met, _ = orc.split_select(ah, orc.norm1(ah))
    assert (r, met) == (1, 0.5)
    bt = np.array([[1.0, 2, 3, 4], [5, 6, 7, 8], [0, 0, 9, 1], [0, 0, 2, 3]])
    r, met, _ = orc.split_select(bt, orc.norm1(bt))
    assert (r, met) == (2, 0.0)
    # tie -> smallest r: lower triangle all equal magnitude in a symmetric pattern
    tie = np.array([[1.0, 0, 0], [1, 1, 0], [0, 1, 1]])
    r, met, mv = orc.split_select(tie, 1.0)
    assert mv[0] == mv[1] == 1.0 and r == 1


@pytest.mark.parametrize("n", [2, 3, 7, 20])
def test_split_select_brute_force(orc, n):
    # definition: m(r) = ||Ahat(r+1:n, 1:r)||_1 / ||A||_1, via numpy's matrix 1-norm
    g = rng(500 + n)
    ah = g.standard_normal((n, n)) * np.exp(-np.add.outer(np.arange(n), -np.arange(n)) / 3)
    bh = g.standard_normal((n, n))
    nA, nB = 3.5, 1.25
    r, met, mv = orc.split_select(ah, nA, bh, nB)
    ref = [np.linalg.norm(ah[q:, :q], 1) / nA + np.linalg.norm(bh[q:, :q], 1) / nB
           for q in range(1, n)]
    assert np.allclose(mv, ref, rtol=1e-14, atol=0)
    assert r == 1 + int(np.argmin(ref)) and met == pytest.approx(min(ref), rel=1e-14)
