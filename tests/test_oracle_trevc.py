"""Pins for the oracle's TREVC (eigenvectors of a triangular matrix, PAPER.md:1018-1027,
SURVEY §8(f) row f4; CPU).

* closed forms: diagonal T -> X = I; 2x2 [[a, b], [0, c]] -> X_01 = b / (c - a);
  3x3 worked by hand;
* TX = XD (D = diag T) to rounding, checked with a plain numpy product;
* library cross-check: every column of X is parallel to numpy's (LAPACK dgeev) eigenvector
  of T for the same eigenvalue;
* back-transform: with Q, X_A = Q X_T and A X_A = X_A D for A = Q T Q^T;
* the near-equal-eigenvalue rule (reading Q19): a repeated diagonal entry gives
  the denominator smin, not a division by zero.
"""
import numpy as np
import pytest

from paper_1011_3077_b200 import inputs


def test_trevc_diagonal(orc):
    T = np.diag([3.0, -1.0, 0.5, 2.0])
    assert np.array_equal(orc.trevc(T), np.eye(4))


def test_trevc_2x2_closed_form(orc):
    a, b, c = 0.7, -1.3, 2.9
    X = orc.trevc(np.array([[a, b], [0.0, c]]))
    assert X[0, 0] == 1.0 and X[1, 1] == 1.0 and X[1, 0] == 0.0
    assert X[0, 1] == pytest.approx(b / (c - a), rel=1e-15)


def test_trevc_3x3_by_hand(orc):
    T = np.array([[1.0, 2.0, 3.0], [0.0, 4.0, 5.0], [0.0, 0.0, 6.0]])
    X = orc.trevc(T)
    # column 1: x0 = 2/(4-1); column 2: x1 = 5/(6-4), x0 = (3 + 2 x1)/(6-1)
    want = np.array([[1.0, 2.0 / 3.0, (3.0 + 2.0 * 2.5) / 5.0], [0.0, 1.0, 2.5], [0.0, 0.0, 1.0]])
    assert np.allclose(X, want, rtol=1e-15, atol=0)


@pytest.mark.parametrize("n", [17, 64, 150])
def test_trevc_residual_and_lapack(orc, n):
    T = inputs.tri_known(n, 70 + n)
    X = orc.trevc(T)
    d = np.diag(T)
    assert np.allclose(np.tril(X, -1), 0.0) and np.all(np.diag(X) == 1.0)
    R = T @ X - X * d[None, :]
    assert np.linalg.norm(R) <= 1e-13 * np.linalg.norm(T) * np.linalg.norm(X)
    w, v = np.linalg.eig(T)
    for j in range(0, n, max(1, n // 10)):
        i = int(np.argmin(np.abs(w - d[j])))
        vj = np.real(v[:, i])
        x = X[:, j] / np.linalg.norm(X[:, j])
        assert min(np.linalg.norm(x - vj), np.linalg.norm(x + vj)) <= 1e-10


def test_trevc_back_transform(orc):
    n = 40
    T = inputs.tri_known(n, 5)
    Q = inputs.haar(np.random.default_rng(6).standard_normal((n, n)))
    A = Q @ T @ Q.T
    XA = orc.trevc(T, Q)
    assert np.allclose(XA, Q @ orc.trevc(T), rtol=0, atol=1e-14)
    R = A @ XA - XA * np.diag(T)[None, :]
    assert np.linalg.norm(R) <= 1e-13 * np.linalg.norm(A) * np.linalg.norm(XA)


def test_trevc_repeated_eigenvalue_guard(orc):
    T = np.array([[2.0, 1.0], [0.0, 2.0]])
    X = orc.trevc(T)
    ulp = 2.0 ** -52
    smin = max(ulp * 2.0, np.finfo(float).tiny * 2 / ulp)
    assert np.isfinite(X).all()
    assert X[0, 1] == -1.0 / smin


def test_trevc_cols_match_full(orc):
    T = inputs.tri_known(90, 11)
    X = orc.trevc(T)
    for j0, j1 in [(0, 1), (37, 41), (89, 90)]:
        assert np.array_equal(orc.trevc_cols(T, j0, j1), X[:, j0:j1])
