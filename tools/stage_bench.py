"""Stage timing of one IRS pass at order n (default 16384): the blocked QR of the 2n x n
stack alone, and the whole pass (QR + complement + the two products), each by CUDA events
and by the paper's flop model (QR 10/3 n^3, complement 6 n^3, products 4 n^3).

  python tools/stage_bench.py [n] [KNOB=VALUE,KNOB=VALUE ...]   (one line per knob set)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1011_3077_b200 import api  # noqa: E402
from paper_1011_3077_b200.api import _ptr_ld, _stream, check  # noqa: E402

NAMES = ["gemm(all)", "panel", "wy_reduce", "select", "gemm W0", "gemm update", "gemm other"]


def timed(fn, reps=2):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def run(n, knobs):
    saved = {}
    for kv in knobs:
        k, v = kv.split("=")
        saved[k] = os.environ.get(k)
        os.environ[k] = v
    h = api.Handle(n)
    dev = torch.device("cuda")
    g = torch.Generator(device="cuda").manual_seed(0)
    A = api.colmajor(torch.randn((n, n), dtype=torch.float64, device=dev, generator=g) * (2.0 / n) ** 0.5)
    B = api.colmajor(torch.eye(n, dtype=torch.float64, device=dev) +
                     0.1 * torch.randn((n, n), dtype=torch.float64, device=dev, generator=g) * (1.0 / n) ** 0.5)
    S = api.empty_colmajor(2 * n, n, dev)
    S0 = api.empty_colmajor(2 * n, n, dev)
    S0[:n].copy_(B)
    S0[n:].copy_(-A)
    Ao, Bo = (api.empty_colmajor(n, n, dev) for _ in range(2))
    ps, ls = _ptr_ld(S)

    def qr():
        S.copy_(S0)
        check(h.lib.sdc_qr(h._h, _stream(dev), 2 * n, n, ps, ls, None, 0), "sdc_qr")

    def cp():
        S.copy_(S0)

    args = []
    for x in (A, B, Ao, Bo, None):
        args += list(_ptr_ld(x))

    def irs():
        check(h.lib.sdc_irs_pass(h._h, _stream(dev), n, *args), "sdc_irs_pass")

    t_cp = timed(cp)
    t_qr = timed(qr) - t_cp
    noprof = bool(os.environ.get("STAGE_NOPROF"))   # per-class events off (they disable some schedules)
    if not noprof:
        h.profile(True)
    t_irs = timed(irs, reps=1)
    prof = [h.profile_read(c) for c in range(7)] if not noprof else []
    h.profile(False)
    n3 = float(n) ** 3
    tf = lambda c, ms: c * n3 / (ms * 1e-3) / 1e12   # noqa: E731
    rest = t_irs - t_qr
    print(f"n={n} {' '.join(knobs) or '(defaults)'}: QR {t_qr:.1f} ms = {tf(10 / 3, t_qr):.2f} TF/s | "
          f"pass {t_irs:.1f} ms = {tf(40 / 3, t_irs):.2f} TF/s | complement+products {rest:.1f} ms = "
          f"{tf(10, rest):.2f} TF/s", flush=True)
    for c, (ms, cnt, w) in enumerate(prof):
        if cnt:
            extra = f" {w / (ms / 1e3) / 1e12:6.2f} TF/s" if c in (0, 4, 5, 6) and ms > 0 else ""
            print(f"   {NAMES[c]:12s} {ms:9.2f} ms  {cnt:6d} launches{extra}")
    print("   sched:", {k: v for k, v in h.schedule_counters().items() if v})
    h.close()
    del h
    torch.cuda.empty_cache()
    for k, v in saved.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 16384
    sets = [a for a in sys.argv[1:] if "=" in a or a == "-"]
    if not sets:
        sets = ["-"]
    for s in sets:
        run(n, [] if s == "-" else s.split(","))
