"""Multi-rank recursive divide-and-conquer (paper_1011_3077_b200/parallel_schur.py; SURVEY
§8(e)/(f) f2; "passes the data associated with the smaller subproblem to an
idle processor") on CPU: world_size 2, 3 and 4 over gloo, with the ORACLE's node and subtree
routines as the backend (test infrastructure; the product backend is GpuBackend on libsdc).

Pinned against the one-rank recursion (orc_schur): identical block list and counters,
bit-identical diagonal blocks of T, exact zeros below them, and A = Q T Q^T with Q orthogonal
to rounding (the off-diagonal blocks are regrouped products, equal to rounding only)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class OracleBackend:
    device = torch.device("cpu")

    def __init__(self, leaf, seed, max_iters, tol):
        from paper_1011_3077_b200.parallel_schur import Stats
        self.kw = dict(leaf=leaf, seed=seed, max_iters=max_iters, tol=tol)
        self.stats = Stats()

    def empty(self, m, n):
        return torch.empty((n, m), dtype=torch.float64).t()

    def node(self, Tb, o):
        import oracle
        a = Tb.numpy()
        assert a.flags.f_contiguous
        r, Qb, st, mm = oracle.schur_node(a, o, **self.kw)
        self.stats.add(st, mm)
        return r, (None if Qb is None else torch.from_numpy(Qb))

    def subtree(self, Tb, o):
        import oracle
        from paper_1011_3077_b200.parallel_schur import Sub
        res = oracle.schur(Tb.numpy(), key_off=o, **self.kw)
        self.stats.add([res.splits, res.failed_attempts, res.unsplit, res.passes], res.max_metric)
        return Sub(torch.from_numpy(res.Q), torch.from_numpy(res.T), [(o + b, m) for b, m in res.blocks])

    def gemm(self, A, B, ta=False, tb=False):
        import oracle
        return torch.from_numpy(oracle.gemm(A.numpy(), B.numpy(), ta, tb))


CASE = dict(n=96, leaf=8, seed=4, max_iters=60, tol=1e-13)


def _problem():
    from paper_1011_3077_b200 import inputs
    A, _, _ = inputs.normal_random_eigs(CASE["n"], 31, 32)
    return A


def _worker(rank, world, port, q):
    sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1011_3077_b200 import parallel_schur as ps
    be = OracleBackend(CASE["leaf"], CASE["seed"], CASE["max_iters"], CASE["tol"])
    A = torch.from_numpy(np.asfortranarray(_problem())) if rank == 0 else None
    out = ps.schur(be, dist, rank, world, A)
    if rank == 0:
        Q, T, blocks, st = out
        q.put((Q.numpy().copy(order="F"), T.numpy().copy(order="F"), blocks, st.counts.tolist(),
               st.max_metric))
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_static_parents():
    from paper_1011_3077_b200 import parallel_schur as ps
    assert ps.delegates(0, 8) == [(4, 4), (2, 2), (1, 1)]
    assert [ps.parent(x, 8)[0] for x in range(1, 8)] == [0, 0, 2, 0, 4, 4, 6]
    assert [ps.parent(x, 3)[0] for x in range(1, 3)] == [0, 0]
    for world in range(1, 9):   # every rank but 0 has exactly one parent; ranges partition
        seen = sorted(d for x in range(world) for d, _ in ps.delegates(x, ps.parent(x, world)[1]))
        assert seen == list(range(1, world))


@pytest.mark.parametrize("world", [2, 3, 4])
def test_multirank_schur_matches_one_rank(orc, world):
    A = _problem()
    ref = orc.schur(A, leaf=CASE["leaf"], seed=CASE["seed"], max_iters=CASE["max_iters"], tol=CASE["tol"])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    Q, T, blocks, counts, mm = q.get(timeout=600)
    for p in procs:
        p.join(600)
        assert p.exitcode == 0
    n = A.shape[0]
    assert sorted(blocks) == sorted(ref.blocks) and blocks == sorted(blocks)
    assert counts[:3] == [ref.splits, ref.failed_attempts, ref.unsplit] and counts[3] == ref.passes
    assert mm == ref.max_metric
    mask = np.zeros((n, n), bool)
    for b0, m in blocks:
        mask[b0:b0 + m, b0:b0 + m] = True
        assert np.array_equal(T[b0:b0 + m, b0:b0 + m], ref.T[b0:b0 + m, b0:b0 + m])
    assert np.all(T[np.tril(np.ones((n, n), bool), -1) & ~mask] == 0.0)
    assert np.linalg.norm(Q.T @ Q - np.eye(n)) <= 1e-13 * n
    assert np.linalg.norm(Q @ T @ Q.T - A) <= 1e-12 * n * np.linalg.norm(A)
    assert np.linalg.norm(T - ref.T) <= 1e-12 * n * np.linalg.norm(A)
