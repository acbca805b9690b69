"""Per-launch timeline of one split step (CUDA events on each launch's own stream, dumped by
libsdc's SDC_PROF_DUMP): busy time per (stream tag, kernel class) and the longest launches.

  SDC_PROF_DUMP=/tmp/dump.txt python tools/timeline.py <config> [n]      (run on the GPU)
  python tools/timeline.py --read /tmp/dump.txt[.gz] [t0 t1]             (summarise / print a window)
tag bits: 1 = high-priority look-ahead stream, 2 = bulk side stream, 4 = second context."""
import collections
import gzip
import os
import sys

NAMES = {1: "panel", 2: "wyred", 3: "select", 4: "gemm W0", 5: "gemm upd", 6: "gemm other", 7: "trevc"}


def read(path, t0=None, t1=None):
    op = gzip.open if path.endswith(".gz") else open
    rows = [l.split() for l in op(path, "rt")]
    rows = [(int(r[0]), int(r[1]), float(r[2]), float(r[3]), float(r[4])) for r in rows if int(r[0]) != 0]
    rows.sort(key=lambda r: r[2])
    span = max(r[3] for r in rows) - min(r[2] for r in rows)
    busy = collections.defaultdict(float)
    cnt = collections.Counter()
    for c, tag, a, b, w in rows:
        busy[(tag, NAMES.get(c, c))] += b - a
        cnt[(tag, NAMES.get(c, c))] += 1
    print(f"{len(rows)} launches over {span:.1f} ms")
    for k, v in sorted(busy.items()):
        print(f"  tag {k[0]} {k[1]:10s} {v:9.1f} ms  {cnt[k]:6d} launches  {v / cnt[k] * 1e3:8.1f} us each")
    if t0 is not None:
        for c, tag, a, b, w in rows:
            if t0 <= a <= t1:
                rate = f"{w / (b - a) / 1e9:6.1f} TF/s" if c in (4, 5, 6) and b > a else ""
                print(f"{NAMES.get(c, c):10s} tag {tag} {a:9.3f} -> {b:9.3f} {1e3 * (b - a):8.1f} us {w / 1e9:8.2f} G {rate}")


def run(cfg, n):
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    from paper_1011_3077_b200 import api, inputs
    p = inputs.make_config(cfg, n=n, device="cuda") if cfg >= 3 else inputs.make_config(cfg, n=n)
    dev = lambda x: None if x is None else api.colmajor(torch.as_tensor(x).cuda())   # noqa: E731
    h = api.Handle(p.n, pencil=p.B is not None)
    A, B, V, VL = dev(p.A), dev(p.B), dev(p.V), dev(p.VL)
    kw = dict(max_iters=p.max_iters, tol=p.tol, stop={0: "fixed", 1: "rtest", 2: "e21"}[p.stop])
    h.split(A, B, V, VL, **kw)
    torch.cuda.synchronize()
    h.profile(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = h.split(A, B, V, VL, **kw)
    e1.record()
    torch.cuda.synchronize()
    h.profile_read(0)
    h.profile(False)
    print(f"cfg{cfg} n={p.n}: {e0.elapsed_time(e1):.1f} ms (profiled), iters={out[3].iters} k={out[3].k}")
    print({k: v for k, v in h.schedule_counters().items() if v})


if __name__ == "__main__":
    if sys.argv[1] == "--read":
        w = [float(x) for x in sys.argv[3:5]] if len(sys.argv) >= 5 else [None, None]
        read(sys.argv[2], *w)
    else:
        run(int(sys.argv[1]), int(sys.argv[2]) if len(sys.argv) > 2 else None)
