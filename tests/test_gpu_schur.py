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


# ---- batched small blocks (schur_batched.cuh): blocks of order <= 64 run one CTA per block,
# one launch per recursion level ---------------------------------------------------------
# Cases whose oracle decisions are stable under relative input noise up to 2e-14
# (test_oracle_schur.py "batch96" / "batch128" / "batch160"): the batched kernel's contractions
# run in a different order than the large-n path's, so the 4e-16 margin of the cases above
# is not enough -- e.g. (128, 1, seed 1) passes it, and the two sides still accept different
# valid splits of one 8 x 8 block (r = 2 at pass 11 vs r = 4 at pass 9, reading Q20).
BATCH_CASES = [(96, 1, 6), (128, 1, 13), (160, 2, 32)]


@pytest.mark.parametrize("n,leaf,seed", BATCH_CASES)
def test_schur_batched_blocks_parity(orc, handle, n, leaf, seed):
    A, V, eig = inputs.normal_random_eigs(n, 15 + n, 16 + n)
    handle.schedule_counters(reset=True)
    blocks, info = compare(orc, handle, A, leaf, seed)
    c = handle.schedule_counters()
    assert c["schur_batch_launches"] > 0 and c["schur_batch_blocks"] >= len(blocks) // 2
    assert all(m <= 2 for _, m in blocks)


def test_schur_batched_matches_unbatched(orc, monkeypatch):
    # the large-n kernel sequence on every block (SDC_SCHUR_BATCH=0) takes the same decisions
    from paper_1011_3077_b200 import api
    A, V, eig = inputs.normal_random_eigs(128, 15 + 128, 16 + 128)
    seed = 13
    res = []
    for mode in ("1", "0"):
        monkeypatch.setenv("SDC_SCHUR_BATCH", mode)
        h = api.Handle(128)
        Q, T, blocks, info = h.schur(dev(A), leaf=1, seed=seed)
        c = h.schedule_counters()
        assert (c["schur_batch_launches"] > 0) == (mode == "1")
        res.append((blocks, info["splits"], info["failed_attempts"], info["unsplit"], h.launches))
        h.close()
    assert res[0][:4] == res[1][:4]
    assert res[0][4] * 10 <= res[1][4]     # >= 10x fewer kernel launches per decomposition


def test_schur_batched_valid_decomposition(handle):
    # a case whose oracle decisions are NOT margin-stable (block lists may differ between two
    # valid implementations, reading Q20): check what is unique -- A = Q T Q^T, Q
    # orthogonal, T block triangular with blocks <= 2, block spectra = eig(A)
    n = 300
    A, V, eig = inputs.normal_random_eigs(n, 15 + n, 16 + n)
    handle.schedule_counters(reset=True)
    Qg, Tg, blocks, info = handle.schur(dev(A), leaf=1, seed=7)
    assert handle.schedule_counters()["schur_batch_blocks"] > n // 2
    Q, T = Qg.cpu().numpy(), Tg.cpu().numpy()
    assert sum(m for _, m in blocks) == n and all(m <= 2 for _, m in blocks) and info["unsplit"] == 0
    assert np.linalg.norm(Q.T @ Q - np.eye(n)) <= 1e-13 * n
    mask = np.zeros((n, n), bool)
    for b0, m in blocks:
        mask[b0:b0 + m, b0:b0 + m] = True
    assert np.all(T[np.tril(np.ones((n, n), bool), -1) & ~mask] == 0.0)
    bound = (info["max_metric"] * max(1, info["splits"]) + 1e-13) * np.linalg.norm(A, 1)
    assert np.linalg.norm(Q @ T @ Q.T - A, 1) <= 2 * bound
    ev = np.concatenate([np.linalg.eigvals(T[b0:b0 + m, b0:b0 + m]) for b0, m in blocks])
    ref = np.linalg.eigvals(A)
    from scipy.optimize import linear_sum_assignment
    D = np.abs(ev[:, None] - ref[None, :])
    ri, ci = linear_sum_assignment(D)
    assert np.max(D[ri, ci]) <= 1e-8
