"""CholeskyQR2 panel phase timing (SDC_DEBUG_COUNTERS): one blocked QR of an m x n matrix,
per-panel time with SDC_CQR on/off and the CQR phases of CTA 0 / the last CTA."""
import ctypes
import os
import sys

os.environ.setdefault("SDC_DEBUG_COUNTERS", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1011_3077_b200 import api  # noqa: E402

m, n = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (2048, 1024)
h = api.Handle(max(n, (m + 1) // 2))
S0 = api.colmajor(torch.randn((m, n), dtype=torch.float64, device="cuda"))
h.qr(S0.clone(), want_q=False)
buf = (ctypes.c_ulonglong * 64)()
h.lib.sdc_debug_counters(h._h, buf, 64, 1)
h.profile(True)
h.qr(S0.clone(), want_q=False)
ms, cnt, _ = h.profile_read(1)
h.profile(False)
h.lib.sdc_debug_counters(h._h, buf, 64, 1)
c = h.schedule_counters()
names = ["gram1", "reduce1", "gather1", "chol1", "trinv1", "Q1", "keepR1", "gram2+xchg", "chol2", "Qtop",
         "LU", "R/W/M", "T|waitM", "Y"]
npan = max(1, c["panel_cqr_done"] // 2)   # warm-up + timed QR
print(f"m={m} n={n} SDC_CQR={os.environ.get('SDC_CQR', 'default')}: {cnt} panels, {ms / cnt * 1e3:.1f} us/panel, "
      f"cqr done {c['panel_cqr_done']} fallback {c['panel_cqr_fallback']} | {c}")
for who, o in (("CTA 0", 32), ("last CTA", 48)):
    print(f"  {who}: " + ", ".join(f"{names[q]} {buf[o + q] / npan / 1.965e3:.2f}" for q in range(14)) + " (us/panel)")
