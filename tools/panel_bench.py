"""Panel-kernel phase timing: one blocked QR of a 2n x n stack with SDC_DEBUG_COUNTERS=1.
Reports, per timed CTA, the clock64 cycles spent in the four phases of a column step."""
import ctypes
import os
import sys

os.environ.setdefault("SDC_DEBUG_COUNTERS", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1011_3077_b200 import api  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
h = api.Handle(n)
S = api.colmajor(torch.randn((2 * n, n), dtype=torch.float64, device="cuda"))
h.qr(S, want_q=False)
buf = (ctypes.c_ulonglong * 32)()
h.lib.sdc_debug_counters(h._h, buf, 32, 1)
h.profile(True)
h.qr(S, want_q=False)
ms, cnt, _ = h.profile_read(1)
h.profile(False)
h.lib.sdc_debug_counters(h._h, buf, 32, 1)
cols = n
names = ["partials", "grid barrier", "sum partials", "update+T"]
print(f"n={n} panel_rows={os.environ.get('SDC_PANEL_ROWS', '128')}: panels {ms:.2f} ms total, "
      f"{ms / cnt * 1e3:.1f} us/panel, {ms / cols * 1e3:.2f} us/column")
for who, o in (("CTA 0", 0), ("last CTA", 4)):
    tot = sum(buf[o + q] for q in range(4))
    print(f"  {who}: " + ", ".join(f"{names[q]} {buf[o + q] / cols / 1.965e3:.2f} us" for q in range(4))
          + f"  (sum {tot / cols / 1.965e3:.2f} us/col)")
ncall = max(1, buf[8] // 2)
for who, o in (("CTA 0", 9), ("last CTA", 12)):
    print(f"  {who}: per panel: prologue {buf[o] / ncall / 1.965e3:.1f} us, loop gaps "
          f"{buf[o + 1] / ncall / 1.965e3:.1f} us, tail {buf[16 + (o > 9)] / ncall / 1.965e3:.1f} us, "
          f"write-back {buf[o + 2] / ncall / 1.965e3:.1f} us")
spn = ["fma", "sync+sum", "push", "Tcol", "wait", "leaders", "sum(b)", "reflector", "update", "stage+sync"]
print("  CTA 0 sub-phases (us/col): " + ", ".join(f"{spn[q]} {buf[20 + q] / cols / 1.965e3:.2f}" for q in range(10)))
