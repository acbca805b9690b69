// latency of the 16 x 16 warp-level routines of csrc/cqr.cuh (one warp, cycles per call)
#include <cstdio>
#include "../../paper_1011_3077_b200/csrc/cqr.cuh"
using namespace sdc;
__global__ void k(double* out) {
  __shared__ double A[64 * CQ_LD], g[64], d[64], ri[16];
  const int lane = threadIdx.x;
  for (int e = lane; e < 64 * CQ_LD; e += 32) A[e] = 0.01 * ((e * 37) % 17) + (e % (CQ_LD + 1) == 0 ? 20.0 : 0.0);
  for (int e = lane; e < 64; e += 32) { g[e] = 1.0; }
  if (lane < 16) ri[lane] = 0.05;
  __syncwarp();
  double a[16];
  long long t[8];
  for (int rep = 0; rep < 3; ++rep) {
    t[0] = clock64();
    cq_blk_load(A, CQ_LD, 0, 0, a);
    t[1] = clock64();
    cq_chol16(a, g);
    t[2] = clock64();
    cq_lu16(a, d);
    t[3] = clock64();
    cq_blk_store(A, CQ_LD, 16, 16, a, 0, false);
    __syncwarp();
    t[4] = clock64();
    double x[16];
    cq_trinv16([=](int i, int j) { return i <= j ? CQX(A, CQ_LD, i, j) : 0.0; }, false, x);
    t[5] = clock64();
    cq_solve_rows_upper([=](int kk, int j) { return CQX(A, CQ_LD, kk, j); }, ri,
                        [=](int i, int j) -> double& { return CQX(A, CQ_LD, 32 + i, j); });
    __syncwarp();
    t[6] = clock64();
    if (lane < 16) out[lane] = a[lane] + x[lane];
  }
  if (lane == 0) for (int i = 0; i < 6; ++i) out[16 + i] = (double)(t[i + 1] - t[i]);
}
int main() {
  double* d; cudaMalloc(&d, 64 * 8);
  k<<<1, 32>>>(d);
  double h[64]; cudaMemcpy(h, d, 64 * 8, cudaMemcpyDeviceToHost);
  const char* nm[6] = {"blk_load", "chol16", "lu16", "blk_store", "trinv16", "solve_rows_upper"};
  for (int i = 0; i < 6; ++i) printf("%-18s %6.0f cycles\n", nm[i], h[16 + i]);
}
