"""Time libsdc GEMM shapes of the split step in isolation (CUDA events via sdc_profile)."""
import sys
import os
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1011_3077_b200 import api  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    h = api.Handle(n)
    g = torch.Generator(device="cuda").manual_seed(0)
    dev = torch.device("cuda")
    shapes = [("TN square", True, False, n, n, n), ("NN square (cp.async)", False, False, n, n, n),
              ("TN rank-64 update", True, False, 2 * n, n, 64),
              ("TN rank-128 update", True, False, 2 * n, n, 128),
              ("TN rank-256 update", True, False, 2 * n, n, 256),
              ("TN rank-256 update b=0", True, False, 2 * n, n, -256),
              ("TN rank-512 update", True, False, 2 * n, n, 512),
              ("TN W0 (no split-K)", True, False, 64, n, 2 * n)]
    for name, ta, tb, M, N, K in shapes:
        beta = 1.0
        if K < 0:
            K, beta = -K, 0.0
        A = torch.randn((K, M) if ta else (M, K), dtype=torch.float64, device=dev, generator=g)
        B = torch.randn((N, K) if tb else (K, N), dtype=torch.float64, device=dev, generator=g)
        A, B = api.colmajor(A), api.colmajor(B)
        C = api.empty_colmajor(M, N, dev)
        C.zero_()
        for _ in range(2):
            h.dgemm(A, B, ta, tb, alpha=-1.0, beta=beta, C=C)
        torch.cuda.synchronize()
        h.profile(True)
        reps = 5
        for _ in range(reps):
            h.dgemm(A, B, ta, tb, alpha=-1.0, beta=beta, C=C)
        ms, cnt, fl = h.profile_read(0)
        h.profile(False)
        print(f"{name:24s} M={M} N={N} K={K}: {ms / cnt:8.3f} ms  {fl / (ms / 1e3) / 1e12:6.2f} TFLOP/s")
    # one blocked QR of a 2n x n stack with the breakdown
    S = api.colmajor(torch.randn((2 * n, n), dtype=torch.float64, device=dev, generator=g))
    h.qr(S, want_q=False)
    torch.cuda.synchronize()
    h.profile(True)
    t0 = time.perf_counter()
    h.qr(S, want_q=False)
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    names = ["gemm(all)", "panel", "wy_reduce", "select", "gemm W0", "gemm update", "gemm other"]
    print(f"blocked QR {2*n}x{n}: {t*1e3:.1f} ms wall, model {(2*(2*n)*n*n - 2*n**3/3)/t/1e12:.2f} TF/s")
    for c in range(7):
        ms, cnt, w = h.profile_read(c)
        extra = f" {w / (ms / 1e3) / 1e12:6.2f} TF/s" if c in (0, 4, 5, 6) and ms > 0 else ""
        print(f"   {names[c]:12s} {ms:9.2f} ms  {cnt:6d} launches{extra}")
    h.profile(False)


if __name__ == "__main__":
    main()
