// Microbenchmark: FP64 tensor (DMMA m8n8k4) vs DFMA throughput on sm_100a.
// Used once to pin the FP64 roofline figure.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void dmma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[CHAINS][2];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}

template <int CHAINS>
__global__ void dfma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) c[i] = fma(a, c[i], b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i];
  if (s == 12345.0) out[0] = s;
}

// half the warps DMMA, half DFMA (same flops per iteration per warp: 8 DMMA = 4096 flop;
// DFMA 64 chains * 32 lanes * 2 = 4096 flop)
__global__ void mixed_loop(double* out, int iters) {
  int w = threadIdx.x / 32;
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double s = 0;
  if (w & 1) {
    double c[8][2] = {};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  } else {
    double c[64];
    for (int i = 0; i < 64; ++i) c[i] = i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 64; ++i) c[i] = fma(a, c[i], b);
    }
    for (int i = 0; i < 64; ++i) s += c[i];
  }
  if (s == 12345.0) out[0] = s;
}

int main(int argc, char** argv) {
  double* d; cudaMalloc(&d, 8);
  int dev; cudaGetDevice(&dev); cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  printf("%s SMs=%d clock(kHz)=%d\n", p.name, p.multiProcessorCount, p.clockRate);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = argc > 1 ? atoi(argv[1]) : 20000;   // run_fp64_peak.sh: long enough to sample clocks
  for (int warps : {4, 8, 16}) {
    for (int bps : {1, 2}) {
      int blocks = p.multiProcessorCount * bps;
      dmma_loop<8><<<blocks, warps * 32>>>(d, 100);
      cudaEventRecord(e0);
      dmma_loop<8><<<blocks, warps * 32>>>(d, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = double(blocks) * warps * iters * 8 * 512.0;
      printf("DMMA m8n8k4 warps=%2d blocks/SM=%d: %.2f TFLOP/s\n", warps, bps, flops / ms / 1e9);
    }
  }
  for (int warps : {4, 8, 16, 32}) {
    int blocks = p.multiProcessorCount;
    dfma_loop<16><<<blocks, warps * 32>>>(d, 100);
    cudaEventRecord(e0);
    dfma_loop<16><<<blocks, warps * 32>>>(d, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = double(blocks) * warps * 32 * iters * 16 * 2.0;
    printf("DFMA warps=%2d: %.2f TFLOP/s\n", warps, flops / ms / 1e9);
  }
  for (int warps : {8, 16}) {
    int blocks = p.multiProcessorCount;
    mixed_loop<<<blocks, warps * 32>>>(d, 100);
    cudaEventRecord(e0);
    mixed_loop<<<blocks, warps * 32>>>(d, iters / 4);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    const cudaError_t e = cudaGetLastError();   // 16 warps x 64 DFMA chains: too many registers
    if (e != cudaSuccess) { printf("MIXED warps=%2d: not launchable (%s)\n", warps, cudaGetErrorString(e)); continue; }
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = double(blocks) * warps * (iters / 4) * 4096.0;
    printf("MIXED warps=%2d: %.2f TFLOP/s\n", warps, flops / ms / 1e9);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
