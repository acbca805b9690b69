"""GPU parity (-m gpu) of the recursive divide-and-conquer sdc_schur (SURVEY §8(f) row f2,
DESIGN.md §10) against the oracle's orc_schur.

Both sides take the same discrete decisions (counter-based lines and Haar streams, the
same acceptance rule), so the block lists and split counts are bit-exact; the blocks'
spectra agree to rounding (<= 1e-9) and each block's invariant subspace span Q(:, block)
to a principal angle <= 1e-8; T is exactly zero below its diagonal blocks, Q orthogonal
(<= 1e-13 n) and A = Q T Q^T to the accepted splits' backward error.
"""
import numpy as np
import pytest
import torch

from _util import sin_angle
from paper_1011_3077_b200 import inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def handle():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1011_3077_b200 import api
    return api.Handle(512)


def dev(x):
    return torch.as_tensor(np.asfortranarray(x), dtype=torch.float64).cuda().t().contiguous().t()


def compare(orc, handle, A, leaf, seed):
    n = A.shape[0]
    Qg, Tg, blocks, info = handle.schur(dev(A), leaf=leaf, seed=seed)
    o = orc.schur(A, leaf=leaf, seed=seed)
    assert blocks == o.blocks
    assert (info["splits"], info["failed_attempts"], info["unsplit"]) == (o.splits, o.failed_attempts, o.unsplit)
    Q, T = Qg.cpu().numpy(), Tg.cpu().numpy()
    assert np.linalg.norm(Q.T @ Q - np.eye(n)) <= 1e-13 * n
    mask = np.zeros((n, n), bool)
    for b0, m in blocks:
        mask[b0:b0 + m, b0:b0 + m] = True
    assert np.all(T[np.tril(np.ones((n, n), bool), -1) & ~mask] == 0.0)
    bound = (info["max_metric"] * max(1, info["splits"]) + 1e-13) * np.linalg.norm(A, 1)
    assert np.linalg.norm(Q @ T @ Q.T - A, 1) <= 2 * bound
    for b0, m in blocks:
        eg = np.sort_complex(np.linalg.eigvals(T[b0:b0 + m, b0:b0 + m]))
        eo = np.sort_complex(np.linalg.eigvals(o.T[b0:b0 + m, b0:b0 + m]))
        assert np.max(np.abs(eg - eo)) <= 1e-9
        assert sin_angle(Q[:, b0:b0 + m], o.Q[:, b0:b0 + m]) <= 1e-8
    return blocks, info


def test_schur_complex_pairs_parity(orc, handle):
    A, V, eig = inputs.normal_random_eigs(40, 5, 6)
    blocks, info = compare(orc, handle, A, 1, 3)
    assert all(m <= 2 for _, m in blocks)


def test_schur_real_parity(orc, handle):
    n = 30
    g = np.random.default_rng(8)
    lam = g.uniform(-3, 3, n)
    U = inputs.haar(g.standard_normal((n, n)))
    compare(orc, handle, (U * lam) @ U.T, 1, 9)


# (n, leaf, seed): cases whose oracle decisions are stable under 4e-16 relative input
# perturbations (tests/test_oracle_schur.py::test_gpu_parity_cases_have_decision_margin,
# DESIGN.md reading Q20)
LEAF_CASES = [(60, 8, 4), (150, 16, 4), (201, 64, 5)]


@pytest.mark.parametrize("n,leaf,seed", LEAF_CASES)
def test_schur_leaf_parity(orc, handle, n, leaf, seed):
    A, V, eig = inputs.normal_random_eigs(n, 15 + n, 16 + n)
    blocks, info = compare(orc, handle, A, leaf, seed)
    assert all(m <= leaf for _, m in blocks) and info["unsplit"] == 0


def test_schur_unsplittable(orc, handle):
    A = 2.0 * np.eye(5)
    blocks, info = compare(orc, handle, A, 1, 1)
    assert blocks == [(0, 5)] and info["unsplit"] == 1
