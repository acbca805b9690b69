"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel class.

usage: python tools/summarize_launches.py launches.csv [title]
Per-launch times under ncu are cold-cache and serialised: compare SHARES of the step, not
absolute times.  Kernels not from libsdc (torch input preparation) are listed but excluded
from the shares.
"""
import csv
import sys
from collections import defaultdict


def kernel_class(name: str) -> str:
    if "gemm_tn_tma_persist_kernel" in name:
        return "gemm_tn_tma_persist_kernel (DMMA, TMA, rank-nb updates)"
    if "gemm_tn_tma_kernel" in name:
        return "gemm_tn_tma_kernel (DMMA, TMA)"
    if "gemm_dmma_kernel" in name:
        return "gemm_dmma_kernel (DMMA, cp.async)"
    if "panel_qr" in name:
        return "panel_qr_kernel"
    if "k_cqs_" in name:
        return "k_cqs_* (split CholeskyQR2 panel chain: 6 kernels per panel)"
    if "sdc::" in name or name.startswith("k_") or "k_split_batched" in name or "trevc" in name:
        return name.split("(")[0].replace("void ", "")
    return "torch (input prep, outside the timed region)"


def main():
    path = sys.argv[1]
    title = sys.argv[2] if len(sys.argv) > 2 else path
    t = defaultdict(float)
    c = defaultdict(int)
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for row in csv.DictReader(lines):
        if row.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = kernel_class(row["Kernel Name"])
        v = float(row["Metric Value"].replace(",", ""))
        unit = row.get("Metric Unit", "ns")
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(unit, 1e-6)
        t[k] += v * scale
        c[k] += 1
    own = sum(v for k, v in t.items() if not k.startswith("torch"))
    print(title)
    print("(ncu per-launch times: cold-cache, serialised -> compare shares)\n")
    for k in sorted(t, key=lambda x: -t[x]):
        share = t[k] / own if not k.startswith("torch") else float("nan")
        print(f"{k:58s} launches {c[k]:7d}  time {t[k]:11.3f} ms  share {share:6.3f}")
    print(f"\nlibsdc kernels: {sum(v for k, v in c.items() if not k.startswith('torch'))} launches, {own:.3f} ms")


if __name__ == "__main__":
    main()
