// Microbenchmark of the 64 x 64 CholeskyQR2 building blocks (csrc/cqr.cuh) in one CTA of 512
// threads: clock64 cycles per call (median of the repetitions), plus residual checks.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <algorithm>
#include "../../paper_1011_3077_b200/csrc/cqr.cuh"
using namespace sdc;

__global__ void __launch_bounds__(512) bench(const double* G, double* out, unsigned long long* cyc, int reps) {
  extern __shared__ double smem[];
  double *A = smem, *B = A + 64 * CQ_LD, *gd = B + 64 * CQ_LD, *dsg = gd + 64, *sc = dsg + 64;
  __shared__ int flag;
  const int tid = threadIdx.x;
  for (int r = 0; r < reps; ++r) {
    for (int e = tid; e < 4096; e += 512) A[(e & 63) + (e >> 6) * CQ_LD] = G[e];
    __syncthreads();
    unsigned long long t0 = clock64();
    bool ok = cq_chol64(A, gd, sc, &flag);
    __syncthreads();
    unsigned long long t1 = clock64();
    cq_trinv64([=](int i, int j) { return CQX(A, CQ_LD, i, j); }, false, B, CQ_LD);
    unsigned long long t2 = clock64();
    cq_gemm64([=](int i, int k) { return CQX(A, CQ_LD, i, k); }, [=](int k, int j) { return CQX(B, CQ_LD, k, j); },
              [](int ti, int tj) { return ti; }, [](int ti, int tj) { return tj + 1; }, 1.0,
              [=](int i, int j, double v) { CQX(B, CQ_LD, i, j) = v; });
    unsigned long long t3 = clock64();
    for (int e = tid; e < 4096; e += 512) A[(e & 63) + (e >> 6) * CQ_LD] = G[4096 + e];
    __syncthreads();
    unsigned long long t4 = clock64();
    cq_lu64(A, CQ_LD, dsg, sc);
    unsigned long long t5 = clock64();
    if (tid == 0) {
      cyc[4 * r + 0] = t1 - t0; cyc[4 * r + 1] = t2 - t1; cyc[4 * r + 2] = t3 - t2; cyc[4 * r + 3] = t5 - t4;
    }
    if (r == reps - 1) {
      for (int e = tid; e < 4096; e += 512) { out[e] = B[(e & 63) + (e >> 6) * CQ_LD]; out[4096 + e] = A[(e & 63) + (e >> 6) * CQ_LD]; }
      if (tid < 64) out[8192 + tid] = dsg[tid];
      if (tid == 0) out[8192 + 64] = ok;
    }
    __syncthreads();
  }
}

int main() {
  const int reps = 20;
  std::vector<double> G(8192);
  srand(1);
  // SPD Gram of a random 256 x 64 matrix; and an orthonormal-ish matrix for the LU
  std::vector<double> X(256 * 64);
  for (auto& x : X) x = (rand() / (double)RAND_MAX) * 2 - 1;
  for (int i = 0; i < 64; ++i)
    for (int j = 0; j < 64; ++j) {
      double s = 0; for (int k = 0; k < 256; ++k) s += X[k * 64 + i] * X[k * 64 + j];
      G[i + 64 * j] = s;
    }
  for (int e = 0; e < 4096; ++e) G[4096 + e] = ((rand() / (double)RAND_MAX) * 2 - 1) * 0.2;
  double *dG, *dO; unsigned long long* dc;
  cudaMalloc(&dG, 8192 * 8); cudaMalloc(&dO, 8300 * 8); cudaMalloc(&dc, reps * 4 * 8);
  cudaMemcpy(dG, G.data(), 8192 * 8, cudaMemcpyHostToDevice);
  const int smem = (2 * 64 * CQ_LD + 128 + 512) * 8;
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  bench<<<1, 512, smem>>>(dG, dO, dc, reps);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  std::vector<unsigned long long> c(reps * 4);
  std::vector<double> o(8300);
  cudaMemcpy(c.data(), dc, reps * 4 * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(o.data(), dO, 8300 * 8, cudaMemcpyDeviceToHost);
  const char* nm[4] = {"chol64", "trinv64", "gemm64(upper x upper)", "lu64"};
  for (int q = 0; q < 4; ++q) {
    std::vector<unsigned long long> v;
    for (int r = 1; r < reps; ++r) v.push_back(c[4 * r + q]);
    std::sort(v.begin(), v.end());
    printf("%-24s %8llu cycles = %.2f us\n", nm[q], v[v.size() / 2], v[v.size() / 2] / 1965.0);
  }
  // checks: B = R R^{-1} = I (gemm of R and its inverse); LU: (L U)_ij = A_ij - D_i delta_ij
  double err = 0;
  for (int i = 0; i < 64; ++i) for (int j = 0; j < 64; ++j) err = fmax(err, fabs(o[i + 64 * j] - (i == j)));
  printf("chol ok=%g  |R R^-1 - I|max = %.2e\n", o[8192 + 64], err);
  double lerr = 0;
  for (int i = 0; i < 64; ++i) for (int j = 0; j < 64; ++j) {
    double s = 0;
    for (int k = 0; k <= std::min(i, j); ++k) {
      double l = (k == i) ? 1.0 : o[4096 + i + 64 * k];
      double u = o[4096 + k + 64 * j];
      s += l * u;
    }
    double want = G[4096 + i + 64 * j] - (i == j ? o[8192 + i] : 0.0);
    lerr = fmax(lerr, fabs(s - want));
  }
  printf("|L U - (A - D)|max = %.2e\n", lerr);
  return 0;
}
