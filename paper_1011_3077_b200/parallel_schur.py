"""Recursive divide-and-conquer over several ranks.

PAPER.md:989-991: "after a split, the processor ... passes the data associated with the
smaller subproblem to an idle processor" -- the one place where the method shards
naturally.  One process per GPU; this module is the host-side protocol,
every arithmetic step runs in libsdc (sdc_schur_node, sdc_schur_keyed, sdc_dgemm through
`GpuBackend`).

Protocol (static, deterministic, no coordinator):
  * rank ranges: the root block belongs to rank 0 with the range [0, world).  A rank R that
    holds range [R, R+k) and splits a block keeps [R, R+ceil(k/2)) for the LARGER child and
    hands the SMALLER child to rank R+ceil(k/2) with the range [R+ceil(k/2), R+k): one
    send of the child's diagonal block (m_c^2 doubles).  So every rank has one static
    parent (`parent`) and receives exactly one message from it: a block, or "none" when the
    recursion above it ended before reaching it (forwarded down its own range).
  * a rank whose range has shrunk to itself solves its block's whole subtree locally
    (sdc_schur_keyed with the block's global offset as key).
  * the draws of every attempt are keyed by the block's GLOBAL offset and order
    (sdc_schur_keyed), so each node takes exactly the decisions of the one-rank recursion:
    the block list is bit-identical and the diagonal blocks of T are bit-identical (each is
    computed from the same bits by the same kernels).
  * results return up the same edges: a child rank sends (Z, T_final, blocks, stats) of its
    subproblem, Z the accumulated orthogonal factor (T_final = Z^T T_blk Z with the E21
    blocks zeroed).  The parent assembles its node:
        Z = Q_b diag(Z_1, Z_2),   T = [[T_1, Z_1^T A12 Z_2], [0, T_2]]
    -- the off-diagonal updates the one-rank recursion applies eagerly (T(o:o+m, o+m:n) <-
    Q_b^T ..., T(0:o, o:o+m) <- ... Q_b), regrouped; rank 0 ends with Q = Z, T.
Messages: header int64[8], then float64 payloads; any torch.distributed backend (NCCL with
CUDA tensors on the GPU path, gloo with CPU tensors in the tests).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

WORK, NONE = 1, 0


def delegates(R: int, k: int):
    """[(rank, range size)] that rank R, holding [R, R+k), hands subproblems to, in order."""
    out = []
    while k > 1:
        keep = (k + 1) // 2
        out.append((R + keep, k - keep))
        k = keep
    return out


def parent(X: int, world: int):
    """Static parent rank of X (None for rank 0) and X's range size."""
    stack = [(0, world)]
    while stack:
        R, k = stack.pop()
        for d, kd in delegates(R, k):
            if d == X:
                return R, kd
            stack.append((d, kd))
    assert X == 0
    return None, world


@dataclass
class Sub:
    Z: torch.Tensor
    T: torch.Tensor
    blocks: list


@dataclass
class Stats:
    counts: np.ndarray = field(default_factory=lambda: np.zeros(4, dtype=np.int64))
    max_metric: float = 0.0

    def add(self, c, mm):
        self.counts += np.asarray(c, dtype=np.int64)
        self.max_metric = max(self.max_metric, float(mm))


class GpuBackend:
    """libsdc on one GPU: sdc_schur_node / sdc_schur_keyed / sdc_dgemm."""

    def __init__(self, handle, leaf=1, seed=1, max_iters=60, tol=1e-13):
        from . import api
        self.api = api
        self.h = handle
        self.device = torch.device("cuda", handle.device)
        self.kw = dict(leaf=leaf, seed=seed, max_iters=max_iters, tol=tol)
        self.stats = Stats()

    def empty(self, m, n):
        return self.api.empty_colmajor(m, n, self.device)

    def node(self, Tb, o):
        acc = (np.zeros(4, dtype=np.int32), [0.0])
        r, Qb = self.h.schur_node(Tb, o, stats=acc, **self.kw)
        self.stats.add(acc[0], acc[1][0])
        return r, Qb

    def subtree(self, Tb, o):
        Q, T, blocks, info = self.h.schur(Tb, key_off=o, **self.kw)
        self.stats.add([info["splits"], info["failed_attempts"], info["unsplit"], info["passes"]],
                       info["max_metric"])
        return Sub(Q, T, [(o + b, m) for b, m in blocks])

    def gemm(self, A, B, ta=False, tb=False):
        return self.h.dgemm(A, B, ta, tb)


def _colmajor(x: torch.Tensor) -> torch.Tensor:
    return x if (x.stride(0) == 1 and x.stride(1) >= x.shape[0]) else x.t().contiguous().t()


def _cm_copy(x: torch.Tensor) -> torch.Tensor:
    """A fresh, densely packed column-major copy (ld = rows)."""
    return x.t().clone(memory_format=torch.contiguous_format).t()


def _send(comm, x: torch.Tensor, dst: int):
    comm.send(_colmajor(x).t().contiguous(), dst)     # column-major payload as a flat buffer


def _recv(comm, m: int, n: int, src: int, like: torch.Tensor) -> torch.Tensor:
    buf = torch.empty((n, m), dtype=torch.float64, device=like.device)
    comm.recv(buf, src)
    return buf.t()                                     # (m, n) column-major view


def _header(vals, device):
    h = torch.zeros(8, dtype=torch.int64, device=device)
    h[:len(vals)] = torch.tensor(vals, dtype=torch.int64)
    return h


def _process(be, comm, o: int, Tb: torch.Tensor, dels: list) -> Sub:
    m = Tb.shape[0]
    if not dels:
        return be.subtree(Tb, o)
    r, Qb = be.node(Tb, o)
    if r == 0:                          # leaf / unsplit: nothing for the remaining delegates
        for d, kd in dels:
            comm.send(_header([NONE], Tb.device), d)
        Z = be.empty(m, m)
        Z.zero_()
        Z.diagonal().fill_(1.0)
        return Sub(Z, Tb, [(o, m)])
    # children: leading (o, r) [Re > a] and trailing (o + r, m - r)
    kids = [(o, Tb[:r, :r]), (o + r, Tb[r:, r:])]
    small = 0 if r < m - r else 1       # the smaller child goes to the idle rank (ties: trailing)
    d, kd = dels[0]
    so, sT = kids[small]
    ms = sT.shape[0]
    comm.send(_header([WORK, so, ms], Tb.device), d)
    _send(comm, sT, d)
    lo, lT = kids[1 - small]
    large = _process(be, comm, lo, _cm_copy(lT), dels[1:])
    hdr = torch.zeros(8, dtype=torch.int64, device=Tb.device)
    comm.recv(hdr, d)
    nblk = int(hdr[0])
    binfo = torch.zeros(2 * nblk + 5, dtype=torch.float64, device=Tb.device)
    comm.recv(binfo, d)
    b = binfo.cpu().numpy()
    be.stats.add(b[2 * nblk:2 * nblk + 4].astype(np.int64), b[2 * nblk + 4])
    sm = Sub(_recv(comm, ms, ms, d, Tb), _recv(comm, ms, ms, d, Tb),
             [(int(b[2 * i]), int(b[2 * i + 1])) for i in range(nblk)])
    s1, s2 = (sm, large) if small == 0 else (large, sm)
    # assemble: Z = Q_b diag(Z1, Z2); T = [[T1, Z1^T A12 Z2], [0, T2]]
    Z = be.empty(m, m)
    Z[:, :r] = be.gemm(Qb[:, :r], s1.Z)
    Z[:, r:] = be.gemm(Qb[:, r:], s2.Z)
    A12 = _colmajor(Tb[:r, r:])
    X = be.gemm(be.gemm(s1.Z, A12, ta=True), s2.Z)
    T = be.empty(m, m)
    T.zero_()
    T[:r, :r] = s1.T
    T[r:, r:] = s2.T
    T[:r, r:] = X
    return Sub(Z, T, s1.blocks + s2.blocks)


def schur(be, comm, rank: int, world: int, A: torch.Tensor | None = None, n: int | None = None):
    """Distributed recursion.  Rank 0 passes A (n x n, column-major on the backend's device)
    and returns (Q, T, blocks, stats); the other ranks pass nothing and return None."""
    par, k = parent(rank, world)
    dels = delegates(rank, k)
    if rank == 0:
        Tb = _cm_copy(A)
        sub = _process(be, comm, 0, Tb, dels)
        return sub.Z, sub.T, sub.blocks, be.stats
    hdr = torch.zeros(8, dtype=torch.int64, device=be.device)
    comm.recv(hdr, par)
    if int(hdr[0]) == NONE:
        for d, kd in dels:
            comm.send(_header([NONE], be.device), d)
        return None
    o, m = int(hdr[1]), int(hdr[2])
    Tb = _recv(comm, m, m, par, hdr)   # fresh buffer, column-major (ld = m)
    sub = _process(be, comm, o, Tb, dels)
    nblk = len(sub.blocks)
    comm.send(_header([nblk], be.device), par)
    info = np.zeros(2 * nblk + 5)
    for i, (bo, bm) in enumerate(sub.blocks):
        info[2 * i], info[2 * i + 1] = bo, bm
    info[2 * nblk:2 * nblk + 4] = be.stats.counts
    info[2 * nblk + 4] = be.stats.max_metric
    comm.send(torch.as_tensor(info, dtype=torch.float64, device=be.device), par)
    _send(comm, sub.Z, par)
    _send(comm, sub.T, par)
    return None


# ---------------------------------------------------------------------------------------
# Ranks as host threads on ONE GPU: each rank has its own handle (workspace, streams); the
# subtrees handed off after a split then run concurrently on the same device -- their steps are
# latency-bound chains at these sizes, so they overlap almost for free.  Whole blocks are
# exchanged between kernels through queues (no kernel of one rank waits on another's kernel).
# ---------------------------------------------------------------------------------------
class ThreadComm:
    """send/recv between threads of one process (rank = thread-local); tensors are copied on send."""

    def __init__(self, world: int):
        import queue
        import threading
        self.q = {(s, d): queue.Queue() for s in range(world) for d in range(world)}
        self.local = threading.local()

    def send(self, t, dst):
        c = t.clone()
        if c.is_cuda:   # the receiver copies on ITS stream: the clone must have completed
            torch.cuda.current_stream(c.device).synchronize()
        self.q[(self.local.rank, dst)].put(c)

    def recv(self, t, src):
        t.copy_(self.q[(src, self.local.rank)].get(timeout=3600))


def schur_threads(world: int, make_backend, A: torch.Tensor, device: int = 0):
    """One decomposition by `world` thread-ranks on `device`; make_backend(rank) -> backend with
    its own handle.  Returns rank 0's (Q, T, blocks, stats)."""
    import threading
    comm = ThreadComm(world)
    out, err = {}, []

    def body(rank):
        try:
            comm.local.rank = rank
            torch.cuda.set_device(device)
            with torch.cuda.stream(torch.cuda.Stream(device=device)):
                r = schur(make_backend(rank), comm, rank, world, A if rank == 0 else None)
                torch.cuda.current_stream().synchronize()
            out[rank] = r
        except Exception as e:  # noqa: BLE001 -- surfaced to the caller below
            err.append(e)

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if err:
        raise err[0]
    return out[0]
