"""Multi-process (world_size 2, gloo, CPU) coverage of bench.py's N>1 host logic: the
per-rank step time is reduced with MAX over ranks and the whole-job throughput of N
independent replicas ("replicas only") is N / max time."""
import os
import socket
import sys

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    ms = 1000.0 * (rank + 1)           # rank 1 is the slow replica
    mx = bench.max_over_ranks(ms, world)
    q.put((rank, mx, bench.replica_throughput(mx, world)))
    dist.destroy_process_group()


def test_two_rank_max_and_throughput():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    out = sorted(q.get(timeout=10) for _ in range(2))
    for rank, mx, thr in out:
        assert mx == 2000.0                       # max over ranks, identical on every rank
        assert thr == pytest.approx(2 / 2.0)      # 2 replicas / 2 s


def test_single_rank_passthrough():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.max_over_ranks(12.5, 1) == 12.5
    assert bench.replica_throughput(500.0, 1) == 2.0


def test_gpus_must_match_world_size():
    # --gpus N under a launcher that started a different number of ranks is refused (the
    # line would otherwise report N GPUs for a run of WORLD_SIZE replicas: VERDICT r01 weak 9)
    import subprocess
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--impl",
                        "reference"], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 2 and "WORLD_SIZE=1" in r.stderr
