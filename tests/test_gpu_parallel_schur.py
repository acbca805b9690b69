"""GPU (-m gpu): the multi-rank recursion (paper_1011_3077_b200/parallel_schur.py) with the
product backend (libsdc: sdc_schur_node, sdc_schur_keyed, sdc_dgemm).  Only one GPU is
available, so the ranks are threads with their own handles and a queue-based point-to-point
transport (no kernel of one rank ever waits on another rank's kernel: ranks exchange whole
blocks between kernels, as over NCCL).  Pinned against the one-rank sdc_schur (block list,
counters and diagonal blocks bit-identical) and against the oracle's orc_schur."""
import queue
import threading

import numpy as np
import pytest
import torch

from paper_1011_3077_b200 import inputs

pytestmark = pytest.mark.gpu


class ThreadComm:
    """send/recv between threads (rank = thread-local); tensors are copied on send."""

    def __init__(self, world):
        self.q = {(s, d): queue.Queue() for s in range(world) for d in range(world)}
        self.local = threading.local()

    def send(self, t, dst):
        self.q[(self.local.rank, dst)].put(t.clone())

    def recv(self, t, src):
        t.copy_(self.q[(src, self.local.rank)].get(timeout=600))


def run_ranks(world, A, kw):
    from paper_1011_3077_b200 import api, parallel_schur as ps
    comm = ThreadComm(world)
    out, err = {}, []
    n = A.shape[0]

    def body(rank):
        try:
            comm.local.rank = rank
            torch.cuda.set_device(0)
            h = api.Handle(n)
            be = ps.GpuBackend(h, **kw)
            Ad = torch.as_tensor(np.asfortranarray(A)).cuda().t().contiguous().t() if rank == 0 else None
            r = ps.schur(be, comm, rank, world, Ad)
            torch.cuda.synchronize()
            out[rank] = r
        except Exception as e:  # surfaced below
            err.append(e)

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(900)
    assert not err, err
    return out[0]


@pytest.mark.parametrize("world", [2, 3])
def test_gpu_multirank_schur_matches_one_rank(orc, world):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1011_3077_b200 import api
    kw = dict(leaf=16, seed=5, max_iters=60, tol=1e-13)   # decision margin: test_oracle_schur.py
    n = 200
    A, _, _ = inputs.normal_random_eigs(n, 41, 42)
    h = api.Handle(n)
    Q1, T1, blocks1, info1 = h.schur(torch.as_tensor(np.asfortranarray(A)).cuda().t().contiguous().t(), **kw)
    Q, T, blocks, st = run_ranks(world, A, kw)
    assert blocks == blocks1
    assert st.counts.tolist() == [info1["splits"], info1["failed_attempts"], info1["unsplit"], info1["passes"]]
    Qh, Th, T1h = Q.cpu().numpy(), T.cpu().numpy(), T1.cpu().numpy()
    for b0, m in blocks:
        assert np.array_equal(Th[b0:b0 + m, b0:b0 + m], T1h[b0:b0 + m, b0:b0 + m])
    mask = np.zeros((n, n), bool)
    for b0, m in blocks:
        mask[b0:b0 + m, b0:b0 + m] = True
    assert np.all(Th[np.tril(np.ones((n, n), bool), -1) & ~mask] == 0.0)
    assert np.linalg.norm(Qh.T @ Qh - np.eye(n)) <= 1e-13 * n
    assert np.linalg.norm(Qh @ Th @ Qh.T - A) <= 1e-12 * n * np.linalg.norm(A)
    o = orc.schur(A, **kw)
    assert blocks == o.blocks and st.counts[:3].tolist() == [o.splits, o.failed_attempts, o.unsplit]


def test_gpu_thread_ranks_module_helper(orc):
    # parallel_schur.schur_threads: 4 thread-ranks on the one GPU, each with its own handle AND
    # its own stream (the product helper behind `bench.py --config 8 --threads 4`): the same
    # block list, counters and diagonal blocks as one rank
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1011_3077_b200 import api, parallel_schur as ps
    kw = dict(leaf=16, seed=5, max_iters=60, tol=1e-13)
    n = 200
    A, _, _ = inputs.normal_random_eigs(n, 41, 42)
    Ad = torch.as_tensor(np.asfortranarray(A)).cuda().t().contiguous().t()
    h = api.Handle(n)
    Q1, T1, blocks1, info1 = h.schur(Ad, **kw)
    handles = [api.Handle(n) for _ in range(4)]
    Q, T, blocks, st = ps.schur_threads(4, lambda r: ps.GpuBackend(handles[r], **kw), Ad)
    torch.cuda.synchronize()
    assert blocks == blocks1
    assert st.counts.tolist() == [info1["splits"], info1["failed_attempts"], info1["unsplit"], info1["passes"]]
    Qh, Th, T1h = Q.cpu().numpy(), T.cpu().numpy(), T1.cpu().numpy()
    for b0, m in blocks:
        assert np.array_equal(Th[b0:b0 + m, b0:b0 + m], T1h[b0:b0 + m, b0:b0 + m])
    assert np.linalg.norm(Qh.T @ Qh - np.eye(n)) <= 1e-13 * n
    assert np.linalg.norm(Qh @ Th @ Qh.T - A) <= 1e-12 * n * np.linalg.norm(A)
