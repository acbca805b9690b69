"""Pins for the oracle's recursive divide-and-conquer (PAPER.md:406-410,
472-475, 545; DESIGN.md §10 "recursion"; CPU).

* A = Q T Q^T to rounding, Q orthogonal, T exactly zero below its diagonal blocks;
* the spectra of the diagonal blocks are the construction's eigenvalues (normal matrices
  with known eigenvalues: complex pairs end in 2x2 leaves with complex eigenvalues, real
  spectra in 1x1 leaves);
* every split puts the eigenvalues right of its line first, so with 1x1 leaves and a real
  spectrum diag(T) is non-increasing;
* leaf > 1 bounds the block sizes; an unsplittable block (A = 2I) stays one leaf;
* the counter-based Haar stream is orthogonal and reproducible.
"""
import numpy as np
import pytest

from paper_1011_3077_b200 import inputs


def check_form(A, r):
    n = A.shape[0]
    Q, T = r.Q, r.T
    # backward error: the zeroed E21 blocks (each <= its split's accepted metric) + rounding
    bound = (r.max_metric * max(1, r.splits) + 1e-13) * np.linalg.norm(A, 1)
    assert np.linalg.norm(Q @ T @ Q.T - A, 1) <= 2 * bound
    assert r.max_metric <= 1e-10
    assert np.linalg.norm(Q.T @ Q - np.eye(n)) <= 1e-13 * n
    mask = np.zeros((n, n), bool)
    for o, m in r.blocks:
        mask[o:o + m, o:o + m] = True
    low = np.tril(np.ones((n, n), bool), -1) & ~mask
    assert np.all(T[low] == 0.0)
    assert sorted(r.blocks) == [(o, m) for o, m in sorted(r.blocks)]
    assert sum(m for _, m in r.blocks) == n


def block_eigs(r):
    return np.concatenate([np.linalg.eigvals(r.T[o:o + m, o:o + m]) for o, m in sorted(r.blocks)])


def match_sets(a, b, tol):
    a = sorted(a, key=lambda z: (round(z.real, 6), z.imag))
    b = sorted(b, key=lambda z: (round(z.real, 6), z.imag))
    return max(abs(x - y) for x, y in zip(a, b)) <= tol


def test_schur_complex_pairs(orc):
    A, V, eig = inputs.normal_random_eigs(40, 5, 6)
    r = orc.schur(A, leaf=1, seed=3)
    check_form(A, r)
    assert all(m <= 2 for _, m in r.blocks) and r.unsplit == 0
    for o, m in r.blocks:
        if m == 2:
            ev = np.linalg.eigvals(r.T[o:o + 2, o:o + 2])
            assert abs(ev[0].imag) > 0
    assert match_sets(block_eigs(r), eig, 1e-10)


def test_schur_real_spectrum_sorted(orc):
    n = 30
    g = np.random.default_rng(8)
    lam = g.uniform(-3, 3, n)
    U = inputs.haar(g.standard_normal((n, n)))
    A = (U * lam) @ U.T
    r = orc.schur(A, leaf=1, seed=9)
    check_form(A, r)
    assert [m for _, m in sorted(r.blocks)] == [1] * n
    d = np.diag(r.T)
    assert np.all(np.diff(d) <= 0)
    assert np.allclose(d, np.sort(lam)[::-1], atol=1e-11)


def test_schur_leaf_size(orc):
    A, V, eig = inputs.normal_random_eigs(60, 15, 16)
    r = orc.schur(A, leaf=8, seed=4)
    check_form(A, r)
    assert all(m <= 8 for _, m in r.blocks)
    assert match_sets(block_eigs(r), eig, 1e-10)


def test_schur_unsplittable(orc):
    A = 2.0 * np.eye(5)
    r = orc.schur(A, leaf=1, seed=1)
    assert r.blocks == [(0, 5)] and r.unsplit == 1 and r.splits == 0
    assert np.array_equal(r.T, A) and np.array_equal(r.Q, np.eye(5))


def test_haar_stream(orc):
    V1 = orc.haar_stream(20, 7, 3)
    assert np.linalg.norm(V1.T @ V1 - np.eye(20)) <= 1e-13
    assert np.array_equal(V1, orc.haar_stream(20, 7, 3))
    assert not np.array_equal(V1, orc.haar_stream(20, 7, 5))
    assert np.all(np.diag(np.linalg.qr(V1)[1]) != 0)


def _schur_decisions(r):
    return r.blocks, (r.splits, r.failed_attempts, r.unsplit)


@pytest.mark.parametrize("case", ["cpairs40", "real30", "leaf60", "leaf150", "leaf201", "multirank200",
                                  "batch96", "batch128", "batch160"])
def test_gpu_parity_cases_have_decision_margin(orc, case):
    # The recursion's decisions (accept / reject a line, the split r, interval moves) are
    # discontinuous functions of rounding at their thresholds (reading Q20), so a
    # GPU-vs-oracle block-list comparison is meaningful only where no decision sits on a
    # threshold.  Pin: the cases the GPU parity tests use (test_gpu_schur.py,
    # test_gpu_parallel_schur.py) take identical decisions for inputs perturbed by 4e-16
    # relative noise -- the size of the rounding differences between two implementations.
    if case == "cpairs40":
        A, _, _ = inputs.normal_random_eigs(40, 5, 6); leaf, seed = 1, 3
    elif case == "real30":
        g = np.random.default_rng(8)
        lam = g.uniform(-3, 3, 30)
        U = inputs.haar(g.standard_normal((30, 30)))
        A = (U * lam) @ U.T; leaf, seed = 1, 9
    elif case == "multirank200":
        A, _, _ = inputs.normal_random_eigs(200, 41, 42); leaf, seed = 16, 5
    else:
        n, leaf, seed = {"leaf60": (60, 8, 4), "leaf150": (150, 16, 4), "leaf201": (201, 64, 5),
                         "batch96": (96, 1, 6), "batch128": (128, 1, 13), "batch160": (160, 2, 32)}[case]
        A, _, _ = inputs.normal_random_eigs(n, 15 + n, 16 + n)
    base = _schur_decisions(orc.schur(A, leaf=leaf, seed=seed))
    # the batched small-block kernel orders its contractions differently from the large-n
    # path: its cases must also survive noise of the size of accumulated rounding (2e-14)
    levels = (4e-16, 3e-15, 2e-14) if case.startswith("batch") else (4e-16,)
    for eps in levels:
        for k in range(2):
            noise = np.random.default_rng(100 + k).standard_normal(A.shape)
            assert _schur_decisions(orc.schur(A * (1 + eps * noise), leaf=leaf, seed=seed)) == base
