"""Pins for the oracle's singular-value split (CPU).

The m x n matrix A is embedded into H = [[0, A], [A^T, 0]], whose eigenvalues are
+-sigma_i(A) and |m - n| zeros with eigenvectors [u_i; +-v_i]/sqrt(2) and [u_perp; 0] /
[0; w_perp]; one RSEP step splits H along |z| = rho.  Pinned against:
* a diagonal A (closed form: sigma = |d_i|, singular vectors = unit vectors, exact);
* A = U diag(s) W^T built with known singular values and vectors (construction), square,
  tall and wide: k = 2 #{s < rho} + |m - n|, the bottom / top rows of the inside block
  span exactly the right / left singular vectors of the small singular values (plus the
  null-space vectors), and the inside block of Ahat has eigenvalues +-s (and zeros);
* Ahat exactly symmetric (Alg. 6 line 3 symmetrisation).
"""
import numpy as np
import pytest

from paper_1011_3077_b200 import inputs
from _util import orth_err, sin_angle


def _orth_basis(x, tol=1e-8):
    """orthonormal basis of the column space of x (rank by relative singular value)."""
    u, sv, _ = np.linalg.svd(x, full_matrices=False)
    return u[:, sv > tol * max(sv[0], 1e-300)]


def test_svd_diagonal_closed_form(orc):
    d = np.array([0.3, -2.0, 0.5, 3.0, -0.1, 1.5, 0.7, -4.0, 0.2, 2.5])
    n = d.size
    A = np.diag(d)
    V = inputs.haar(np.random.default_rng(7).standard_normal((2 * n, 2 * n)))
    res = orc.svd_split(A, 1.0, V, max_iters=20)
    small = np.abs(d) < 1
    assert res.k == 2 * int(small.sum()) == 10
    assert res.status == 0 and res.metric <= 1e-13
    inside = res.Q[:, res.r:]
    e = np.eye(n)[:, small]
    assert sin_angle(_orth_basis(inside[n:, :]), e) <= 1e-12     # right singular vectors
    assert sin_angle(_orth_basis(inside[:n, :]), e) <= 1e-12     # left singular vectors
    assert np.array_equal(res.Ahat, res.Ahat.T)
    assert orth_err(res.Q) <= 1e-13 * 2 * n


@pytest.mark.parametrize("m,n", [(16, 16), (24, 16), (12, 20)])
def test_svd_known_vectors(orc, m, n):
    A, V, U, s, W = inputs.svd_known(m, n, 40 + m, 140 + n)
    p = min(m, n)
    res = orc.svd_split(A, 1.0, V, max_iters=30)
    small = s < 1
    assert res.k == 2 * int(small.sum()) + abs(m - n)
    assert res.status == 0 and res.metric <= 1e-12
    inside = res.Q[:, res.r:]
    # right singular vectors of the small sigma (+ W's null-space columns when n > m)
    right = np.concatenate([W[:, :p][:, small], W[:, p:]], axis=1)
    left = np.concatenate([U[:, :p][:, small], U[:, p:]], axis=1)
    assert sin_angle(_orth_basis(inside[m:, :]), right) <= 1e-10
    assert sin_angle(_orth_basis(inside[:m, :]), left) <= 1e-10
    assert sin_angle(right, _orth_basis(inside[m:, :])) <= 1e-10   # equal dimensions too
    ev = np.sort(np.abs(np.linalg.eigvalsh(res.Ahat[res.r:, res.r:])))
    want = np.sort(np.concatenate([s[small], s[small], np.zeros(abs(m - n))]))
    assert np.allclose(ev, want, atol=1e-12)
    assert np.array_equal(res.Ahat, res.Ahat.T)


def test_svd_all_large_does_not_split(orc):
    # every sigma > rho and m == n: no eigenvalue of H inside -> no valid split index with
    # a small metric (the step reports status 1, not an error)
    n = 8
    A = np.diag(np.linspace(2.0, 5.0, n))
    V = inputs.haar(np.random.default_rng(3).standard_normal((2 * n, 2 * n)))
    res = orc.svd_split(A, 1.0, V, max_iters=12)
    assert res.status == 1
