"""Pins for the cheaper left basis of pencils (FLAG_QL_ORTH; CPU).

Q_L := Q of QR(A Q_R) replaces the left IRS + GRURV of Alg. 4: the
right step is untouched (Q_R bit-identical), the leading r columns of Q_L span the same
left deflating subspace as Alg. 4's Q_L, and Q_L^T A Q_R is the R factor (upper
triangular to rounding), so E21 vanishes for every r and the split is chosen by F21.
"""
import numpy as np

from _util import sin_angle
from paper_1011_3077_b200 import inputs


def test_ql_orth_matches_alg4(orc):
    n = 60
    A, B, V, VL = inputs.pencil(n, 31, 32, 33, 34)
    ref = orc.split(A, B, V, VL, max_iters=30)
    res = orc.split(A, B, V, None, max_iters=30, flags=orc.FLAG_QL_ORTH)
    assert (res.k, res.r, res.status) == (ref.k, ref.r, ref.status) and res.status == 0
    assert np.array_equal(res.Q, ref.Q)                      # right step untouched
    r = res.r
    assert sin_angle(res.QL[:, :r], ref.QL[:, :r]) <= 1e-10
    assert np.linalg.norm(res.QL.T @ res.QL - np.eye(n)) <= 1e-13 * n
    assert res.metric <= 1e-12


def test_ql_orth_triangular_a(orc):
    n = 40
    A, B, V, VL = inputs.pencil(n, 41, 42, 43, 44)
    res = orc.split(A, B, V, None, max_iters=30, flags=orc.FLAG_QL_ORTH)
    Ah = res.Ahat
    assert np.linalg.norm(np.tril(Ah, -1)) <= 1e-13 * np.linalg.norm(A)
    # and Q_L is exactly the orthogonal factor of A Q_R (numpy QR cross-check, signs fixed)
    q, rr = np.linalg.qr(A @ res.Q)
    q = q * np.where(np.diag(rr) < 0, -1.0, 1.0)[None, :]
    assert np.allclose(res.QL, q, atol=1e-12)
