"""Pins for the oracle's other split regions and the RSEP variant (CPU; -m "not gpu").

* half plane Re z < a through the Moebius pencil (A-(a-1)I, A-(a+1)I):
  k = #{Re lambda < a} for a normal matrix with known eigenvalues (construction), and the
  eigenvalues of Ahat11 / Ahat22 lie right / left of the line (library eigvals, test side);
* disk |z| < rho as the unit disk of (A, rho I): k = #{|lambda| < rho};
* RSEP (Alg. 6): Ahat exactly symmetric, k = #{|lambda| < 1}.
"""
import numpy as np
import pytest

from paper_1011_3077_b200 import inputs


def haar(n, seed):
    return inputs.haar(np.random.default_rng(seed).standard_normal((n, n)))


@pytest.mark.parametrize("n,a", [(40, 0.0), (41, -0.5), (30, -0.5)])
def test_halfplane_split(orc, n, a):
    A, V, eig = inputs.normal_random_eigs(n, 500 + n, 1500 + n)
    # (n, a) chosen with every eigenvalue >= 0.06 from the line (converges within 40 passes)
    assert np.min(np.abs(eig.real - a)) >= 0.05
    res = orc.split(A, V=V, max_iters=40, region=orc.REGION_HALFPLANE, param=a)
    assert res.k == int(np.sum(eig.real < a))
    assert res.status == 0 and res.metric <= 1e-12
    r = res.r
    l11 = np.linalg.eigvals(res.Ahat[:r, :r])
    l22 = np.linalg.eigvals(res.Ahat[r:, r:])
    assert np.all(l11.real > a) and np.all(l22.real < a)
    assert np.allclose(res.Ahat, res.Q.T @ A @ res.Q, atol=1e-12)


def test_halfplane_moebius_pencil_identity(orc):
    # the half-plane split IS the unit-disk split of the Moebius pencil: same Q subspace
    n, a = 24, 0.2
    A, V, eig = inputs.normal_random_eigs(n, 7, 8)
    res = orc.split(A, V=V, max_iters=30, region=orc.REGION_HALFPLANE, param=a)
    A1 = A - (a - 1.0) * np.eye(n)
    B1 = A - (a + 1.0) * np.eye(n)
    res2 = orc.split(A1, B=B1, V=V, VL=haar(n, 9), max_iters=30)
    assert res.k == res2.k
    r = res.r
    q1, q2 = res.Q[:, :r], res2.Q[:, :r]
    assert np.linalg.norm(q1 - q2 @ (q2.T @ q1), 2) <= 1e-10


@pytest.mark.parametrize("rho", [0.8, 1.3])
def test_disk_radius_split(orc, rho):
    n = 48
    A, V = inputs.ginibre(n, 77, 1077)
    lam = np.linalg.eigvals(A)
    assert np.min(np.abs(np.abs(lam) - rho)) >= 0.01   # (seed, rho) chosen off the circle
    res = orc.split(A, V=V, max_iters=30, region=orc.REGION_DISK, param=rho)
    assert res.k == int(np.sum(np.abs(lam) < rho))
    r = res.r
    assert np.all(np.abs(np.linalg.eigvals(res.Ahat[:r, :r])) > rho)
    assert np.all(np.abs(np.linalg.eigvals(res.Ahat[r:, r:])) < rho)


def test_rsep_symmetric(orc):
    n = 40
    g = np.random.default_rng(3)
    lam = np.concatenate([g.uniform(-0.8, 0.8, 18), g.uniform(1.2, 2.5, 11), -g.uniform(1.2, 2.5, 11)])
    U = haar(n, 4)
    A = (U * lam) @ U.T
    A = (A + A.T) / 2
    res = orc.split(A, V=haar(n, 5), max_iters=20, flags=orc.FLAG_SYMMETRIC)
    assert np.array_equal(res.Ahat, res.Ahat.T)
    assert res.k == int(np.sum(np.abs(lam) < 1))
    assert res.metric <= 1e-12
    r = res.r
    assert np.allclose(np.sort(np.linalg.eigvalsh(res.Ahat[r:, r:])), np.sort(lam[np.abs(lam) < 1]), atol=1e-10)


def test_region_argument_errors(orc):
    A = np.eye(4) * 2
    with pytest.raises(ValueError):
        orc.split(A, B=np.eye(4), V=np.eye(4), VL=np.eye(4), region=orc.REGION_HALFPLANE, param=0.0)
    with pytest.raises(ValueError):
        orc.split(A, V=np.eye(4), region=orc.REGION_DISK, param=0.0)
