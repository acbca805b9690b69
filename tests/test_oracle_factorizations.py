"""Pins for the oracle's dense building blocks (CPU; -m "not gpu").

Each test pins an oracle routine to something other than itself: a worked example,
a closed form, an invariant of the mathematics, or an independent library routine
(numpy/scipy LAPACK) used only as a cross-check.
"""
import numpy as np
import pytest
import scipy.linalg as sla

EPS = np.finfo(np.float64).eps


def rng(seed):
    return np.random.default_rng(seed)


def test_qr_worked_example_3_4(orc):
    # SPEC.md:60 worked example: QR([3;4]) gives |R11| = 5.  dlarfg closed form (Q7):
    # beta = -sign(3)*5 = -5, tau = (beta-alpha)/beta = 1.6, v2 = 4/(3-(-5)) = 0.5
    y, tau = orc.geqr2(np.array([[3.0], [4.0]]))
    assert y[0, 0] == -5.0
    assert tau[0] == pytest.approx(1.6, abs=1e-15)
    assert y[1, 0] == pytest.approx(0.5, abs=1e-15)
    q, r = orc.qr_signed(np.array([[3.0], [4.0]]))
    assert r[0, 0] == pytest.approx(5.0, abs=1e-15)
    assert np.allclose(q[:, 0], [0.6, 0.8], atol=1e-15)


def test_householder_zero_tail_is_identity(orc):
    # Q7: ||x|| = 0 -> tau = 0, H = I (beta = alpha, may be negative)
    a = np.array([[-2.0, 1.0], [0.0, 3.0], [0.0, 4.0]])
    y, tau = orc.geqr2(a)
    assert tau[0] == 0.0 and y[0, 0] == -2.0
    q, r = orc.qr_signed(a)
    assert r[0, 0] == 2.0  # sign-normalised
    assert np.allclose(q @ r, a, atol=1e-14)


@pytest.mark.parametrize("m,n", [(2, 1), (7, 5), (16, 8), (40, 20), (65, 33)])
def test_qr_reconstruction_orthogonality(orc, m, n):
    # SPEC.md:127-128 invariants: ||S - QR||_F <= 64 n eps ||S||_F, ||Q^TQ - I|| <= 64 n eps
    s = rng(m * 100 + n).standard_normal((m, n))
    q, r = orc.qr_signed(s)
    assert np.all(np.diag(r) >= 0)
    assert np.allclose(np.tril(r, -1), 0)
    assert np.linalg.norm(s - q @ r) <= 64 * n * EPS * np.linalg.norm(s)
    assert np.linalg.norm(q.T @ q - np.eye(n)) <= 64 * n * EPS
    # independent cross-check: LAPACK's R agrees up to row signs
    r_np = np.linalg.qr(s, mode="r")
    assert np.allclose(np.abs(r_np), np.abs(r), atol=1e-12)


def test_square_explicit_q_matches_lapack(orc):
    s = rng(5).standard_normal((12, 12))
    q, r = orc.qr_signed(s)
    q_np, r_np = np.linalg.qr(s)
    d = np.sign(np.diag(r_np))
    assert np.allclose(q, q_np * d[None, :], atol=1e-13)
    assert np.allclose(r, d[:, None] * r_np, atol=1e-13)


@pytest.mark.parametrize("n", [1, 2, 5, 17])
def test_complement_spans_orthogonal_complement(orc, n):
    # [Q12;Q22] are the last n columns of the 2n x 2n Q of [B;-A];
    # hence C^T C = I, S^T C = 0 and [Q1 | C] is a square orthogonal matrix.
    g = rng(10 + n)
    s = np.vstack([g.standard_normal((n, n)), -g.standard_normal((n, n))])
    y, tau = orc.geqr2(s)
    c = orc.complement(y, tau)
    assert np.linalg.norm(c.T @ c - np.eye(n)) <= 64 * n * EPS
    assert np.linalg.norm(s.T @ c) <= 64 * n * EPS * np.linalg.norm(s)
    q1, _ = orc.qr_signed(s)
    full = np.hstack([q1, c])
    assert np.linalg.norm(full.T @ full - np.eye(2 * n)) <= 64 * n * EPS
    # the complement equals the last n columns of LAPACK's complete Q up to an orthogonal
    # factor: compare projectors
    qf, _ = np.linalg.qr(s, mode="complete")
    p1 = c @ c.T
    p2 = qf[:, n:] @ qf[:, n:].T
    assert np.allclose(p1, p2, atol=1e-13)


@pytest.mark.parametrize("n", [1, 2, 6, 13])
def test_rq_reconstruction(orc, n):
    # PAPER.md:277 (RQ): C = R U' with R upper, diag(R) >= 0, U' orthogonal (Q10)
    c = rng(20 + n).standard_normal((n, n))
    r, q = orc.rq_signed(c)
    assert np.allclose(np.tril(r, -1), 0)
    assert np.all(np.diag(r) >= 0)
    assert np.linalg.norm(q @ q.T - np.eye(n)) <= 64 * n * EPS
    assert np.linalg.norm(r @ q - c) <= 64 * n * EPS * np.linalg.norm(c)
    # independent cross-check: scipy's RQ up to signs
    r2, q2 = sla.rq(c)
    d = np.sign(np.diag(r2))
    assert np.allclose(r, r2 * d[None, :], atol=1e-12)
    assert np.allclose(q, d[:, None] * q2, atol=1e-12)


@pytest.mark.parametrize("n", [1, 3, 9])
def test_ql_reconstruction(orc, n):
    # PAPER.md:252 (QL): X = Q L, L lower with diag >= 0, Q orthogonal
    x = rng(30 + n).standard_normal((n, n))
    q, l = orc.ql_signed(x)
    assert np.allclose(np.triu(l, 1), 0)
    assert np.all(np.diag(l) >= 0)
    assert np.linalg.norm(q.T @ q - np.eye(n)) <= 64 * n * EPS
    assert np.linalg.norm(q @ l - x) <= 64 * n * EPS * np.linalg.norm(x)
    # uniqueness: with a nonsingular X, the QL with positive diag is unique; LAPACK's QR of
    # the column/row-reversed matrix gives the same factors
    J = np.eye(n)[::-1]
    qq, rr = np.linalg.qr(J @ x @ J)
    d = np.sign(np.diag(rr))
    assert np.allclose(q, J @ (qq * d[None, :]) @ J, atol=1e-12)


@pytest.mark.parametrize("ta,tb", [(0, 0), (1, 0), (0, 1), (1, 1)])
def test_gemm_against_numpy(orc, ta, tb):
    g = rng(40 + 2 * ta + tb)
    a = g.standard_normal((7, 5)) if not ta else g.standard_normal((5, 7))
    b = g.standard_normal((5, 9)) if not tb else g.standard_normal((9, 5))
    c = orc.gemm(a, b, bool(ta), bool(tb))
    ref = (a.T if ta else a) @ (b.T if tb else b)
    assert np.allclose(c, ref, atol=1e-13)


def test_norm1(orc):
    a = np.array([[1.0, -7.0], [-2.0, 3.0]])
    assert orc.norm1(a) == 10.0
