#!/usr/bin/env python
"""bench.py -- split steps/s and effective FP64 TFLOP/s of one inverse-free split step.

Workload (BASELINE.json metric "at n=16384"): configs[4] -- n = 16384 RNEP, A = U T U^T
(seed 6), 30 IRS passes, Haar V (seed 1006); synthetic inputs resident in HBM.  One "step"
is one full sdc_split (30 IRS passes + GRURV + similarity + split selection).  Inputs (2 GiB
each) exceed the 126 MB L2, so no L2 flush is needed between steps.

Multi-GPU: the step does not shard ("replicas only"): each rank runs its own
independent split; value = N / (max-over-ranks time per step).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--n N]
  python bench.py --impl reference ...   # the CPU oracle arm (bounded sample, extrapolated)
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "split steps/s and effective FP64 TFLOP/s at n=16384 vs FP64 tensor-core peak"
FP64_PEAK_TFLOPS = 37.1   # measured DMMA.8x8x4 peak, profiles/r01_fp64_peak_microbench.txt
MEASURED = os.path.join(ROOT, "MEASURED_PEAKS.json")


def flop_model(n: int, passes: int, pencil: bool = False, monitor: bool = False) -> float:
    """Paper's flop model (PAPER.md:923-945 with Lemma A1):
    per IRS pass 40/3 n^3 (QR 10/3 + complement 6 + 2 GEMMs 4), GRURV + similarity 12 n^3;
    monitor mode (split after every pass) 76/3 n^3 per pass; pencil doubles IRS and GRURV."""
    n3 = float(n) ** 3
    if monitor:
        return passes * (76.0 / 3.0) * n3 * (2 if pencil else 1)
    if pencil:
        return (80.0 * passes / 3.0 + 24.0) * n3
    return (40.0 * passes / 3.0 + 12.0) * n3


def max_over_ranks(x: float, world: int, device=None) -> float:
    """Max of a per-rank time over all ranks (the bench contract's multi-GPU timing)."""
    if world <= 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def replica_throughput(ms_per_step_max: float, world: int) -> float:
    """Whole-job split steps/s of `world` independent replicas ("replicas only")."""
    return world / (ms_per_step_max / 1e3)


def run_config(cfg_name: str, n: int, passes: int, stop: str, world: int) -> dict:
    big = 19 * n * n * 8 >= (256 << 20)
    return {"workload": cfg_name, "n": n, "passes": passes, "stop": stop,
            "parallelism": f"replicas{world}" if world > 1 else "single",
            "l2": (f"working set (~19 n^2 doubles = {19 * n * n * 8 / 2**30:.1f} GiB) exceeds L2; no flush needed" if big
                   else "working set fits in L2: a 256 MB buffer is rewritten between the timed steps "
                        "(each step timed by its own event pair)")}


def hbm_peak():
    try:
        return float(json.load(open(MEASURED))["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.p:
            self.p.terminate()
            try:
                self.p.wait(5)
            except Exception:
                self.p.kill()

    def summary(self):
        self.f.flush()
        try:
            rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines()]
        except Exception:
            rows = []
        rows = [[c.strip() for c in r] for r in rows if len(r) >= 9]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------------------------------
# CPU oracle: a bounded sample, extrapolated by the flop model
# ---------------------------------------------------------------------------------------
def oracle_sample(n_target: int, passes: int, pencil: bool, n_sample: int = 1536, cfg: int = 5,
                  monitor: bool = False, ql_orth: bool = False):
    """Time the plain oracle (as it stands) on a same-recipe sample at n_sample: two IRS
    passes (median) and one full split with a single pass; GRURV + similarity + selection
    = split(1 pass) - IRS pass(es).  A step is passes x IRS (x2 for Alg. 4's left chain) +
    one GRURV/similarity/selection, or one after EVERY pass in monitor mode (config 3,
    PAPER.md:597).  Returns the extrapolated seconds of one full step at n_target (each part
    scaled by n^3, the flop model's order), threads, description, CPU seconds."""
    import oracle
    from paper_1011_3077_b200 import inputs
    oracle.build()
    threads = len(os.sched_getaffinity(0))
    os.environ.setdefault("OMP_NUM_THREADS", str(threads))
    rc = {9: 4, 6: 5, 7: 5, 8: 5, 10: 1}.get(cfg, cfg)
    p = inputs.make_config(rc, n=n_sample)
    if rc == 1 or rc == 3:   # same recipe at n_sample
        p = inputs.make_config(3, n=n_sample)
    b0 = p.B if pencil else np.eye(n_sample)
    oracle.irs_pass(p.A[:64, :64], b0[:64, :64])          # warm the thread pool
    t_spent = time.perf_counter()
    tp = []
    for _ in range(2):
        t0 = time.perf_counter()
        oracle.irs_pass(p.A, b0)
        tp.append(time.perf_counter() - t0)
    chains = 2 if (pencil and not ql_orth) else 1
    per_pass = statistics.median(tp) * chains
    t0 = time.perf_counter()
    oracle.split(p.A, p.B if pencil else None, p.V, None if ql_orth else p.VL, max_iters=1,
                 flags=oracle.FLAG_QL_ORTH if ql_orth else 0)
    t1 = time.perf_counter() - t0
    rest = max(t1 - per_pass, 1e-9)
    scale = (n_target / n_sample) ** 3
    total = (passes * per_pass + (passes if monitor else 1) * rest) * scale
    sample = (f"oracle at n={n_sample} (same recipe): {per_pass:.2f} s per IRS pass"
              f"{' (both chains)' if chains == 2 else ''} (median of 2), {rest:.2f} s "
              f"GRURV+similarity+select{' per pass (monitor mode)' if monitor else ''}; "
              f"extrapolated by n^3 to n={n_target}, {passes} passes")
    return total, threads, sample, time.perf_counter() - t_spent


def run_reference(args, cfg_name, n, passes, pencil, rank, world, cfg=5):
    if rank != 0:
        return 0
    steps = []
    threads = len(os.sched_getaffinity(0))
    sample = ""
    for i in range(args.warmup + args.steps):
        total, threads, sample, _ = oracle_sample(n, passes, pencil, n_sample=args.ref_n, cfg=cfg,
                                                  monitor=(cfg == 3), ql_orth=(cfg == 9))
        if i >= args.warmup:
            steps.append(total)
    t = statistics.median(steps)
    val = 1.0 / t
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "split steps/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": run_config(cfg_name, n, passes, "e21" if cfg == 3 else "fixed", 1),
            "tflops_effective": flop_model(n, passes, pencil and cfg != 9, monitor=(cfg == 3)) / t / 1e12,
            "cpu_baseline": {"value": val, "unit": "split steps/s", "cores": threads,
                             "kind": "oracle", "sample": sample + " (extrapolated)"},
            "e2e": {"value": val, "unit": "split steps/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------------------
# config 7: TREVC -- eigenvectors of an upper triangular T
# ---------------------------------------------------------------------------------------
def run_trevc(args, rank, world, local):
    import torch
    import torch.distributed as dist
    from paper_1011_3077_b200 import api, inputs
    n = args.n or 16384
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    t_in = time.perf_counter()
    T = inputs.tri_known(n, 77, device=dev)
    torch.cuda.synchronize()
    t_in = time.perf_counter() - t_in
    h = api.Handle(n, device=local)
    X = api.empty_colmajor(n, n, dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        h.trevc(T, X=X)
    barrier()
    st = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = h.launches
    h.profile(True)
    with ClockSampler(local) as clk:
        barrier()
        e0.record(st)
        for _ in range(args.steps):
            h.trevc(T, X=X)
        e1.record(st)
        barrier()
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, world, dev)
    launches = (h.launches - launches0) // args.steps
    prof = {c: h.profile_read(c) for c in (0, 7)}
    h.profile(False)
    flops = n ** 3 / 3.0                        # the S GEMMs: sum_i 2 b (n - i b)^2 / 2
    # end to end: pinned host T -> device, trevc, X -> pinned host
    hT = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
    hT.copy_(T.t())
    hX = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
    dT = torch.empty((n, n), dtype=torch.float64, device=dev)

    def e2e_step():
        dT.copy_(hT, non_blocking=True)
        h.trevc(dT.t(), X=X)
        hX.copy_(X.t(), non_blocking=True)
    e2e_step()
    barrier()
    e0.record(st)
    e2e_step()
    e1.record(st)
    barrier()
    ms_e2e = max_over_ranks(e0.elapsed_time(e1), world, dev)
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0
    g_ms, g_n, g_fl = prof[0]
    s_ms, s_n, s_bytes = prof[7]
    achieved = g_fl / (g_ms / 1e3) / 1e12 if g_ms > 0 else None
    hbm, hbm_src = hbm_peak()
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        import oracle
        oracle.build()
        ns = 3072
        Tn = T[:ns, :ns].cpu().numpy()
        t0 = time.perf_counter()
        oracle.trevc(Tn)
        tc = time.perf_counter() - t0
        total = tc * (n / ns) ** 3
        cpu = {"value": 1.0 / total, "unit": "TREVC solves/s", "cores": len(os.sched_getaffinity(0)),
               "kind": "oracle", "sample": f"orc_trevc on the leading {ns}x{ns} block of the same T: "
               f"{tc:.2f} s, extrapolated by n^3 to n={n}"}
    clocks = clk.summary()
    line = {"metric": "TREVC eigenvector solves/s (f4) and effective FP64 TFLOP/s", "value": 1e3 / ms * world,
            "unit": "TREVC solves/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"cfg7: TREVC of T = triu(N(0,1/n^2), 1) + diag(U[-2,2]) (seed 77), n={n}, "
                                   "X_jj = 1", "n": n, "parallelism": f"replicas{world}" if world > 1 else "single",
                       "l2": "T and X (2 GiB each) exceed L2; no flush needed"},
            "tflops_effective": flops / (ms / 1e3) / 1e12, "flop_model": flops,
            "frac_of_fp64_peak": flops / (ms / 1e3) / 1e12 / FP64_PEAK_TFLOPS,
            "clocks": clocks,
            "e2e": {"value": 1e3 / ms_e2e * world, "unit": "TREVC solves/s", "h2d_bytes_per_step": n * n * 8,
                    "d2h_bytes_per_step": n * n * 8, "ms_per_step": ms_e2e, "steps": 1},
            "gpu_launches": int(launches),
            "roofline": {"bound": "tensor", "kernel": "gemm_tn_tma_kernel (S = T[i,:] X, kupper)",
                         "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                         "frac": achieved / FP64_PEAK_TFLOPS if achieved else None, "traffic": None,
                         "share_of_step": (g_ms / args.steps) / ms, "launches_per_step": g_n // args.steps},
            "roofline_solve": {"bound": "latency", "kernel": "k_trevc_block",
                               "achieved": s_bytes / (s_ms / 1e3) / 1e9 if s_ms > 0 else None,
                               "peak": hbm, "unit": "GB/s", "share_of_step": (s_ms / args.steps) / ms,
                               "launches_per_step": s_n // args.steps},
            "cpu_baseline": cpu, "input_gen_s": t_in}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


# ---------------------------------------------------------------------------------------
# config 8: recursive divide-and-conquer to block Schur form
# ---------------------------------------------------------------------------------------
def run_schur(args, rank, world, local):
    import torch
    import torch.distributed as dist
    from paper_1011_3077_b200 import api, inputs
    n = args.n or 4096
    leaf = args.leaf
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    t_in = time.perf_counter()
    A, _, eig = inputs.normal_random_eigs(n, 88, 1088)
    A = torch.as_tensor(np.asfortranarray(A)).to(dev).t().contiguous().t()
    torch.cuda.synchronize()
    t_in = time.perf_counter() - t_in
    h = api.Handle(n, device=local)
    Q = api.empty_colmajor(n, n, dev)
    T = api.empty_colmajor(n, n, dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    kw = dict(leaf=leaf, seed=5, max_iters=60, tol=1e-13)
    if world > 1:
        # one decomposition across the ranks: the smaller subproblem of each split goes to an
        # idle rank (paper_1011_3077_b200/parallel_schur.py), NCCL send/recv
        from paper_1011_3077_b200 import parallel_schur as ps

        def one():
            be = ps.GpuBackend(h, **kw)
            out = ps.schur(be, dist, rank, world, A if rank == 0 else None)
            if out is None:
                return None, None
            Qd, Td, blocks, st_ = out
            c = st_.counts
            return blocks, {"splits": int(c[0]), "failed_attempts": int(c[1]), "unsplit": int(c[2]),
                            "passes": int(c[3]), "max_metric": st_.max_metric}, Qd, Td
    elif args.threads > 1:
        # thread-ranks on this GPU: own handle and stream per rank, queue transport (parallel_schur.py)
        from paper_1011_3077_b200 import parallel_schur as ps
        handles = [h] + [api.Handle(n, device=local) for _ in range(args.threads - 1)]

        def one():
            torch.cuda.synchronize()
            Qd, Td, blocks, st_ = ps.schur_threads(args.threads, lambda r: ps.GpuBackend(handles[r], **kw), A,
                                                    device=local)
            c = st_.counts
            return blocks, {"splits": int(c[0]), "failed_attempts": int(c[1]), "unsplit": int(c[2]),
                            "passes": int(c[3]), "max_metric": st_.max_metric}, Qd, Td
    else:
        def one():
            _, _, blocks, info = h.schur(A, Q=Q, T=T, **kw)
            return blocks, info, Q, T
    for _ in range(args.warmup):
        one()
    barrier()
    st = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = h.launches
    h.profile(True)
    with ClockSampler(local) as clk:
        barrier()
        e0.record(st)
        for _ in range(args.steps):
            res = one()
        e1.record(st)
        barrier()
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, world, dev)
    launches = (h.launches - launches0) // args.steps
    g_ms, g_n, g_fl = h.profile_read(0)
    p_ms, p_n, _ = h.profile_read(1)
    h.profile(False)
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0
    blocks, info, Q, T = res
    # accuracy of this run (test-side torch checks, outside the timed region)
    resid = float(torch.linalg.matrix_norm(Q @ T @ Q.T - A, 1) / torch.linalg.matrix_norm(A, 1))
    achieved = g_fl / (g_ms / 1e3) / 1e12 if g_ms > 0 else None
    clocks = clk.summary()
    line = {"metric": "block Schur decompositions/s by recursive divide-and-conquer (f2)",
            "value": 1e3 / ms, "unit": "decompositions/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"cfg8: sdc_schur of a normal matrix with eigenvalues Re, Im ~ U[-1.5,1.5] "
                                   f"(conjugate pairs, seed 88), n={n}, leaf {leaf}, seed 5, monitor tol 1e-13",
                       "n": n, "leaf": leaf,
                       "parallelism": (f"recursion over {world} ranks (smaller subproblem handed off per split)"
                                       if world > 1 else
                                       f"recursion over {args.threads} thread-ranks on one GPU (own handle each)"
                                       if args.threads > 1 else "single"),
                       "l2": "working set (5 n^2 doubles) exceeds L2; no flush needed"},
            "result": {"blocks": len(blocks), "max_block": max(m for _, m in blocks), **info,
                       "residual_1": resid},
            "clocks": clocks, "gpu_launches": int(launches),
            "roofline": {"bound": "tensor", "kernel": "all DMMA GEMM launches", "achieved": achieved,
                         "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                         "frac": achieved / FP64_PEAK_TFLOPS if achieved else None, "traffic": None,
                         "share_of_step": (g_ms / args.steps) / ms, "launches_per_step": g_n // args.steps},
            "panel_share": (p_ms / args.steps) / ms, "e2e": None, "cpu_baseline": None,
            "input_gen_s": t_in}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


# ---------------------------------------------------------------------------------------
# config 10: batched small-n split steps, config 1's recipe per problem
# ---------------------------------------------------------------------------------------
def run_batched(args, rank, world, local):
    import torch
    import torch.distributed as dist
    from paper_1011_3077_b200 import api, inputs
    n = args.n or 64
    batch = 148 * 16                         # per GPU: the batch shards across ranks (weak)
    passes = args.passes or 12
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    t_in = time.perf_counter()
    g = torch.Generator(device=dev).manual_seed(10 + rank)
    A = (torch.randn((batch, n, n), dtype=torch.float64, device=dev, generator=g) * (2.0 / n) ** 0.5)
    A = A.transpose(1, 2)                    # column-major per problem (any layout: i.i.d.)
    G = torch.randn((batch, n, n), dtype=torch.float64, device=dev, generator=g)
    q, r = torch.linalg.qr(G)                # Haar V per problem (input generation only)
    V = (q * torch.where(torch.diagonal(r, dim1=1, dim2=2) < 0, -1.0, 1.0)[:, None, :])
    V = V.transpose(1, 2).contiguous().transpose(1, 2)
    Q = torch.empty((batch, n, n), dtype=torch.float64, device=dev).transpose(1, 2)
    torch.cuda.synchronize()
    t_in = time.perf_counter() - t_in
    h = api.Handle(n, device=local)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        h.split_batched(A, V, max_iters=passes, Q=Q)
    barrier()
    st = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = h.launches
    with ClockSampler(local) as clk:
        barrier()
        e0.record(st)
        for _ in range(args.steps):
            _, infos = h.split_batched(A, V, max_iters=passes, Q=Q)
        e1.record(st)
        barrier()
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, world, dev)
    launches = (h.launches - launches0) // args.steps
    # end to end: pinned host A, V -> device, batched step, Q -> pinned host
    hA = torch.empty((batch, n, n), dtype=torch.float64, pin_memory=True)
    hV = torch.empty((batch, n, n), dtype=torch.float64, pin_memory=True)
    hQ = torch.empty((batch, n, n), dtype=torch.float64, pin_memory=True)
    hA.copy_(A.transpose(1, 2))
    hV.copy_(V.transpose(1, 2))
    dA = torch.empty_like(hA, device=dev)
    dV = torch.empty_like(hV, device=dev)

    def e2e_step():
        dA.copy_(hA, non_blocking=True)
        dV.copy_(hV, non_blocking=True)
        q2, _ = h.split_batched(dA.transpose(1, 2), dV.transpose(1, 2), max_iters=passes, Q=Q)
        hQ.copy_(q2.transpose(1, 2), non_blocking=True)
    e2e_step()
    barrier()
    e0.record(st)
    e2e_step()
    e1.record(st)
    barrier()
    ms_e2e = max_over_ranks(e0.elapsed_time(e1), world, dev)
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0
    F = batch * flop_model(n, passes)
    tf = F / (ms / 1e3) / 1e12
    ks = [i.k for i in infos]
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        import oracle
        oracle.build()
        ns = 32
        An = A[:ns].transpose(1, 2).cpu().numpy()
        Vn = V[:ns].transpose(1, 2).cpu().numpy()
        t0 = time.perf_counter()
        for b in range(ns):
            oracle.split(np.asfortranarray(An[b].T), V=np.asfortranarray(Vn[b].T), max_iters=passes)
        tc = (time.perf_counter() - t0) / ns
        cpu = {"value": 1.0 / tc, "unit": "split steps/s", "cores": len(os.sched_getaffinity(0)),
               "kind": "oracle", "sample": f"orc_split on {ns} problems of the same batch: {tc * 1e3:.2f} ms each"}
    clocks = clk.summary()
    line = {"metric": "batched split steps/s (f3, n=64, config 1's recipe per problem)",
            "value": batch * world / (ms / 1e3), "unit": "split steps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"cfg10: {batch} independent RNEP steps per GPU, n={n}, A ~ N(0, 2/n), "
                                   f"Haar V, {passes} passes, one CTA per problem (k_split_batched_wy)",
                       "n": n, "batch_per_gpu": batch, "passes": passes,
                       "parallelism": f"batch sharded over {world} GPUs (no collective)" if world > 1 else "single",
                       "l2": "per-problem working set in SMEM; inputs 78 MB read once per step"},
            "tflops_effective": tf, "flop_model": F, "frac_of_fp64_peak": tf / FP64_PEAK_TFLOPS,
            "result": {"k_mean": float(np.mean(ks)), "status0": int(sum(i.status == 0 for i in infos))},
            "clocks": clocks,
            "e2e": {"value": batch * world / (ms_e2e / 1e3), "unit": "split steps/s",
                    "h2d_bytes_per_step": 2 * batch * n * n * 8, "d2h_bytes_per_step": batch * n * n * 8,
                    "ms_per_step": ms_e2e, "steps": 1},
            "gpu_launches": int(launches),
            "roofline": {"bound": "tensor",
                         "kernel": "k_split_batched_wy (DMMA m8n8k4 from SMEM, compact-WY, one CTA per problem)",
                         "achieved": tf, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                         "frac": tf / FP64_PEAK_TFLOPS, "traffic": None,
                         "peak_source": "measured DMMA.8x8x4 microbenchmark (profiles/r01_fp64_peak_microbench.txt)"},
            "cpu_baseline": cpu, "input_gen_s": t_in}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--n", type=int, default=None, help="override n (NOT the headline workload)")
    ap.add_argument("--passes", type=int, default=None)
    ap.add_argument("--impl", default="sdc", choices=["sdc", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-n", type=int, default=1536)
    ap.add_argument("--threads", type=int, default=1,
                    help="config 8: thread-ranks on the one GPU (each with its own handle): the subtree handed "
                         "off after a split runs concurrently on the same device")
    ap.add_argument("--leaf", type=int, default=64,
                    help="config 8: largest diagonal block left unsplit (1 = down to 1x1 / 2x2 blocks; blocks of "
                         "order <= 64 run in the batched kernel)")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # launched without torchrun: spawn one rank per GPU ourselves (same contract)
        port = 29500 + (os.getpid() % 2000)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        return subprocess.call(cmd)
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU",
              file=sys.stderr)
        return 2
    from paper_1011_3077_b200 import inputs
    cfg = args.config
    if cfg == 10:
        if args.impl == "reference":
            print(json.dumps({"impl": "reference", "unavailable": "config 10 reference arm not implemented"}))
            return 0
        return run_batched(args, rank, world, local)
    if cfg == 8:
        if args.impl == "reference":
            print(json.dumps({"impl": "reference", "unavailable": "config 8 reference arm not implemented"}))
            return 0
        return run_schur(args, rank, world, local)
    if cfg == 7:
        if args.impl == "reference":
            print(json.dumps({"impl": "reference", "unavailable": "config 7 reference arm not implemented"}))
            return 0
        return run_trevc(args, rank, world, local)
    n = args.n or inputs.CONFIG_N[cfg]
    pencil = cfg in (4, 9)
    ql_orth = cfg == 9
    cfg_name = f"cfg{cfg}: " + inputs.CONFIG_DOC[cfg] + ("" if args.n is None else f" [n overridden to {n}]")

    if args.impl == "reference":
        passes = args.passes or {1: 12, 2: 20, 3: 30, 4: 30, 5: 30, 6: 30, 9: 30}[cfg]
        return run_reference(args, cfg_name, n, passes, pencil, rank, world, cfg)

    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_1011_3077_b200 import api

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    t_in = time.perf_counter()
    svd = cfg == 6
    if svd:   # singular-value split: the RSEP step on the order-n embedding of an (n/2)^2 A
        A6, V6, _, s6, _ = inputs.svd_known(n // 2, n // 2, 8, 1008, device=dev)
        p = inputs.Problem("cfg6", n, A6, None, V6, None, 30, 0.0, 0,
                           expected_k=2 * int(np.sum(s6 < 1)))
    else:
        p = inputs.make_config(4 if ql_orth else cfg, n=n, device=dev)
        if ql_orth:
            p.VL = None
    passes = args.passes or p.max_iters
    stop = {0: "fixed", 1: "rtest", 2: "e21"}[p.stop]
    torch.cuda.synchronize()
    t_in = time.perf_counter() - t_in
    h = api.Handle(n, pencil=pencil, device=local)
    Q = api.empty_colmajor(n, n, dev)
    QL = api.empty_colmajor(n, n, dev) if pencil else None

    def step():
        if svd:
            q, _, info = h.svd_split(p.A, 1.0, p.V, max_iters=passes, Q=Q)
            return q, None, None, info
        return h.split(p.A, p.B, p.V, p.VL, max_iters=passes, tol=p.tol, stop=stop, Q=Q, QL=QL,
                       ql_orth=ql_orth)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()
    st = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = h.launches
    # per-kernel-class CUDA events: live inside the timed region for large n; for n small
    # enough to run as one CUDA graph (libsdc graph_max_n = 4096) event recording would
    # disable the graph, so the classes are timed on one extra step after the timed region
    live_prof = n > 4096
    if live_prof:
        h.profile(True)
    infos = []
    # timing rule: inputs larger than L2, or an L2 flush between timed iterations.  The working
    # set (~19 n^2 doubles) exceeds twice the 126 MB L2 from n ~ 1300 on; below that a 256 MB
    # buffer is rewritten between the steps, outside their per-step event pairs
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if 19 * n * n * 8 < (256 << 20) else None
    with ClockSampler(local) as clk:
        barrier()
        if flush is None:
            e0.record(st)
            for _ in range(args.steps):
                _, _, _, info = step()
                infos.append(info)
            e1.record(st)
            barrier()
            ms = e0.elapsed_time(e1) / args.steps
        else:
            pairs = []
            for _ in range(args.steps):
                flush.fill_(1)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(st)
                _, _, _, info = step()
                b.record(st)
                infos.append(info)
                pairs.append((a, b))
            barrier()
            ms = sum(a.elapsed_time(b) for a, b in pairs) / args.steps
    launches = (h.launches - launches0) // args.steps
    if not live_prof:
        h.profile(True)
        step()
        barrier()
    prof_steps = args.steps if live_prof else 1
    prof = {c: h.profile_read(c) for c in range(7)}
    h.profile(False)
    ms = max_over_ranks(ms, world, dev)
    info = infos[-1]
    F = flop_model(n, info.iters, pencil, monitor=(stop == "e21"))
    if ql_orth:   # the right IRS + GRURV + similarities, plus A Q_R and QR(A Q_R) with explicit Q
        F = flop_model(n, info.iters) + (2.0 + 8.0 / 3.0 + 4.0) * n ** 3
    value = replica_throughput(ms, world)
    tflops = F / (ms / 1e3) / 1e12

    # ---- end to end: host buffers through the C ABI, copies inside the timed region ----
    e2e = None
    if args.e2e_steps > 0 and svd:
        # public Python API: pinned host A -> device, svd_split, Q -> pinned host, per step
        m6 = n // 2
        hA = torch.empty((m6, m6), dtype=torch.float64, pin_memory=True)
        hA.copy_(p.A.t())
        hQ = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
        dA = torch.empty((m6, m6), dtype=torch.float64, device=dev)

        def e2e_step():
            dA.copy_(hA, non_blocking=True)
            q, _, _ = h.svd_split(dA.t(), 1.0, p.V, max_iters=passes, Q=Q)
            hQ.copy_(q.t(), non_blocking=True)
        e2e_step()
        barrier()
        e0.record(st)
        for _ in range(args.e2e_steps):
            e2e_step()
        e1.record(st)
        barrier()
        ms_e2e = max_over_ranks(e0.elapsed_time(e1) / args.e2e_steps, world, dev)
        e2e = {"value": replica_throughput(ms_e2e, world), "unit": "split steps/s",
               "h2d_bytes_per_step": m6 * m6 * 8, "d2h_bytes_per_step": n * n * 8,
               "ms_per_step": ms_e2e, "steps": args.e2e_steps}
    elif args.e2e_steps > 0 and ql_orth:
        # public Python API with pinned host buffers: A, B, V -> device, split, Q, Q_L -> host
        hs = [torch.empty((n, n), dtype=torch.float64, pin_memory=True) for _ in range(5)]
        for hx, x in zip(hs[:3], (p.A, p.B, p.V)):
            hx.copy_(x.t())
        ds = [torch.empty((n, n), dtype=torch.float64, device=dev) for _ in range(3)]

        def e2e_step():
            for d, hx in zip(ds, hs[:3]):
                d.copy_(hx, non_blocking=True)
            q, ql, _, _ = h.split(ds[0].t(), ds[1].t(), ds[2].t(), None, max_iters=passes, Q=Q, QL=QL,
                                  ql_orth=True)
            hs[3].copy_(q.t(), non_blocking=True)
            hs[4].copy_(ql.t(), non_blocking=True)
        e2e_step()
        barrier()
        e0.record(st)
        for _ in range(args.e2e_steps):
            e2e_step()
        e1.record(st)
        barrier()
        ms_e2e = max_over_ranks(e0.elapsed_time(e1) / args.e2e_steps, world, dev)
        e2e = {"value": replica_throughput(ms_e2e, world), "unit": "split steps/s",
               "h2d_bytes_per_step": 3 * n * n * 8, "d2h_bytes_per_step": 2 * n * n * 8,
               "ms_per_step": ms_e2e, "steps": args.e2e_steps}
    elif args.e2e_steps > 0:
        def pinned(x):
            if x is None:
                return None
            hx = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
            hx.copy_(x.t())                          # row-major (n,n) of x^T == x col-major
            return hx.numpy().T                      # Fortran-ordered view, no copy
        hA, hB, hV, hVL = pinned(p.A), pinned(p.B), pinned(p.V), pinned(p.VL)
        hQ = torch.empty((n, n), dtype=torch.float64, pin_memory=True).numpy().T
        hQL = torch.empty((n, n), dtype=torch.float64, pin_memory=True).numpy().T if pencil else None
        h.split_host(hA, hB, hV, hVL, max_iters=passes, tol=p.tol, stop=stop, Q=hQ, QL=hQL)
        barrier()
        t0 = time.perf_counter()
        e0.record(st)
        for _ in range(args.e2e_steps):
            h.split_host(hA, hB, hV, hVL, max_iters=passes, tol=p.tol, stop=stop, Q=hQ, QL=hQL)
        e1.record(st)
        barrier()
        ms_e2e = max_over_ranks(e0.elapsed_time(e1) / args.e2e_steps, world, dev)
        nin = 2 + (2 if pencil else 0)
        e2e = {"value": replica_throughput(ms_e2e, world), "unit": "split steps/s",
               "h2d_bytes_per_step": nin * n * n * 8, "d2h_bytes_per_step": (2 if pencil else 1) * n * n * 8,
               "ms_per_step": ms_e2e, "steps": args.e2e_steps}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    # ---- roofline of the dominant kernel class (DMMA GEMMs) -----------------------------
    g_ms, g_n, g_flops = prof[0]
    p_ms, p_n, p_bytes = prof[1]
    hbm, hbm_src = hbm_peak()
    achieved = g_flops / (g_ms / 1e3) / 1e12 if g_ms > 0 else None
    traffic = None
    try:   # DRAM bytes per launch of the representative GEMM launches, from the committed ncu capture
        tpath = os.path.join(ROOT, "profiles", "r02_ncu_traffic.json")
        if not os.path.exists(tpath):
            tpath = os.path.join(ROOT, "profiles", "r01_ncu_traffic.json")
        tj = json.load(open(tpath))
        traffic = {k["shape"]: {"dram_bytes": k["dram_read_bytes"] + k["dram_write_bytes"],
                                "algorithmic_bytes": k["algorithmic_bytes"]} for k in tj["kernels"]}
        traffic["source"] = tj["source"]
    except Exception:
        traffic = None
    roof = {"bound": "tensor", "kernel": "gemm_tn_tma_kernel / gemm_tn_tma_persist_kernel (all DMMA GEMM launches)",
            "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
            "frac": (achieved / FP64_PEAK_TFLOPS) if achieved else None, "traffic": traffic,
            "peak_source": "measured DMMA.8x8x4 microbenchmark (profiles/r02_fp64_peak_microbench.txt)",
            "share_of_step": (g_ms / prof_steps) / ms if ms > 0 else None,
            "launches_per_step": g_n // prof_steps, "timed_live": live_prof,
            "flops_per_launch": g_flops / max(1, g_n)}
    panel = {"bound": "hbm", "kernel": "panel factorisations: k_cqs_* chains (tall stack panels) + panel_qr_kernel",
             "achieved":
             (p_bytes / (p_ms / 1e3) / 1e9) if p_ms > 0 else None, "peak": hbm, "unit": "GB/s",
             "peak_source": hbm_src, "share_of_step": (p_ms / prof_steps) / ms if ms > 0 else None,
             "launches_per_step": p_n // prof_steps}
    if panel["achieved"]:
        panel["frac"] = panel["achieved"] / hbm
    others = {name: {"ms_per_step": prof[c][0] / prof_steps, "launches_per_step": prof[c][1] // prof_steps,
                     "tflops": (prof[c][2] / (prof[c][0] / 1e3) / 1e12) if (c >= 4 and prof[c][0] > 0) else None}
              for c, name in ((2, "k_wy_reduce"), (3, "split_select"), (4, "gemm W0=Y^T C (split-K)"),
                              (5, "gemm rank-nb update C-=YW"), (6, "gemm n x n products"))}

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        total, threads, sample, spent = oracle_sample(n, info.iters, pencil, n_sample=args.ref_n, cfg=cfg,
                                                      monitor=(stop == "e21"), ql_orth=ql_orth)
        cpu = {"value": 1.0 / total, "unit": "split steps/s", "cores": threads, "kind": "oracle",
               "sample": sample + " (extrapolated)", "cpu_seconds_spent": spent}

    clocks = clk.summary()
    line = {"metric": METRIC, "value": value, "unit": "split steps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": run_config(cfg_name, n, info.iters, stop, world),
            "tflops_effective": tflops, "fp64_peak_tflops": FP64_PEAK_TFLOPS,
            "frac_of_fp64_peak": tflops / FP64_PEAK_TFLOPS,
            "frac_of_clock_adjusted_peak": (tflops / (FP64_PEAK_TFLOPS * clocks["sm_mhz"] / 1965.0))
            if clocks.get("sm_mhz") else None,
            "flop_model": F,
            "result": {"k": info.k, "r": info.r, "metric": info.metric, "status": info.status,
                       "expected_k": p.expected_k},
            "clocks": clocks, "e2e": e2e, "gpu_launches": int(launches),
            "roofline": roof, "roofline_panel": panel, "other_kernels": others,
            "cpu_baseline": cpu, "input_gen_s": t_in}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
