"""Kernel-level concurrency safety (-m gpu): the C ABI allows one handle per concurrent
stream (include/sdc.h), and the step itself runs two streams (look-ahead QR) or two
factorization contexts (pencil chains, monitor-mode GRURV next to the next IRS pass).
Kernels from different streams then share SMs; every result must stay bit-identical to
the serialized run.  (This caught a missing cross-proxy fence in the TMA GEMM ring: LDS
reads of a slot were not ordered before its TMA refill, and with a second stream loading
the SMs one K slice of a tile was occasionally overwritten under the reads.)
"""
import threading

import numpy as np
import pytest
import torch

from paper_1011_3077_b200 import inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sdc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1011_3077_b200 import api
    return api


def _run_threads(fns):
    out = [None] * len(fns)

    def wrap(i, f):
        out[i] = f()

    ts = [threading.Thread(target=wrap, args=(i, f)) for i, f in enumerate(fns)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    torch.cuda.synchronize()
    return out


def test_two_handles_two_streams_bit_identical(sdc):
    n = 1024
    probs = [inputs.make_config(3, n=n), inputs.make_config(2, n=n)]
    hs = [sdc.Handle(n) for _ in probs]
    ss = [torch.cuda.Stream() for _ in probs]
    dev = [(sdc.colmajor(torch.as_tensor(p.A).cuda()), sdc.colmajor(torch.as_tensor(p.V).cuda()))
           for p in probs]

    def step(i):
        with torch.cuda.stream(ss[i]):
            _, _, Ah, info = hs[i].split(dev[i][0], None, dev[i][1], max_iters=12, want_ahat=True)
        return Ah.clone(), info

    ref = [step(0), step(1)]
    torch.cuda.synchronize()
    for _ in range(4):
        got = _run_threads([lambda: step(0), lambda: step(1)])
        for (a, ia), (b, ib) in zip(got, ref):
            assert torch.equal(a, b)
            assert (ia.k, ia.r, ia.metric) == (ib.k, ib.r, ib.metric)


def test_concurrent_gemms_bit_identical(sdc):
    # every GEMM tile variant (TN: rank-64/256 updates with beta = 1, M = 64 split-K W0,
    # square, small grids with long K, ragged) on two streams at once
    shapes = [(2048, 192, 64, 1.0), (64, 2048, 4096, 0.0), (1024, 1024, 1024, 0.0),
              (4096, 1792, 256, 1.0), (256, 1792, 4096, 0.0), (300, 257, 129, 0.5)]
    hs = [sdc.Handle(256), sdc.Handle(256)]
    ss = [torch.cuda.Stream(), torch.cuda.Stream()]
    data = []
    for side in range(2):
        g = np.random.default_rng(50 + side)
        data.append([(torch.as_tensor(g.standard_normal((K, M))).cuda(),
                      torch.as_tensor(g.standard_normal((K, N))).cuda(),
                      torch.as_tensor(g.standard_normal((M, N))).cuda(), beta)
                     for (M, N, K, beta) in shapes])

    def work(side):
        outs = []
        with torch.cuda.stream(ss[side]):
            for _ in range(2):
                for (a, b, c0, beta) in data[side]:
                    c = sdc.colmajor(c0)
                    hs[side].dgemm(sdc.colmajor(a), sdc.colmajor(b), transa=True, beta=beta, C=c)
                    outs.append(c)
        return outs

    ref = [work(0), work(1)]
    torch.cuda.synchronize()
    for _ in range(3):
        got = _run_threads([lambda: work(0), lambda: work(1)])
        for side in range(2):
            for x, y in zip(got[side], ref[side]):
                assert torch.equal(x, y)
