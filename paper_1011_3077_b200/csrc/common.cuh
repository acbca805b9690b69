// common.cuh -- shared device helpers for the sm_100a split-step kernels.
//
// FP64 tensor-core math on sm_100a: tcgen05.mma has no f64 kind, so the FP64 tensor
// path is the warp-level mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4); measured peak on B200:
// 37.1 TFLOP/s (profiles/r01_fp64_peak_microbench.txt), 128 flop/clk/SM.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define SDC_DEV __device__ __forceinline__

namespace sdc {

// ---- DMMA: D(8x8) += A(8x4) * B(4x8), fp64 -----------------------------------------
// Fragments (PTX ISA, mma.m8n8k4 .f64): lane t holds A[t/4][t%4], B[t%4][t/4],
// C/D[t/4][2*(t%4) + {0,1}].
SDC_DEV void dmma_8x8x4(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// ---- cp.async (LDGSTS) with zero-fill ----------------------------------------------
SDC_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
template <int BYTES>
SDC_DEV void cp_async_zfill(void* smem, const void* gmem, int src_bytes) {
  static_assert(BYTES == 8 || BYTES == 16, "cp.async size");
  if constexpr (BYTES == 16) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)),
                 "l"(gmem), "r"(src_bytes));
  } else {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(smem)),
                 "l"(gmem), "r"(src_bytes));
  }
}
SDC_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
SDC_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// ---- grid barrier for cooperative launches ------------------------------------------
// Monotonic counter; the caller passes the absolute target (epoch scheme: the host tracks
// how many barriers were already completed on this counter).  All CTAs of the grid must
// be co-resident (cudaLaunchCooperativeKernel guarantees it or fails).
SDC_DEV unsigned int ld_acquire_gpu(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
SDC_DEV void red_release_gpu_add(unsigned int* p, unsigned int v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
// Bounded spin: a barrier that has not completed after ~2^26 polls (seconds) records an
// error in ctr[1] and releases the CTA instead of hanging the GPU; the host reports it.
SDC_DEV void grid_barrier(unsigned int* ctr, unsigned int target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    red_release_gpu_add(ctr, 1u);
    unsigned int polls = 0;
    while (ld_acquire_gpu(ctr) < target) {
      if (++polls > (1u << 26)) {
        atomicExch(ctr + 1, 1u);
        break;
      }
      if (polls > 64) __nanosleep(32);
    }
  }
  __syncthreads();
}

// Barrier where only `arrive` CTAs (cluster leaders) add to the counter but every CTA waits
// for the target; bounded spin as grid_barrier.
SDC_DEV void leaders_barrier(unsigned int* ctr, unsigned int target, bool arrive) {
  __syncthreads();
  if (threadIdx.x == 0) {
    if (arrive) red_release_gpu_add(ctr, 1u);
    unsigned int polls = 0;
    while (ld_acquire_gpu(ctr) < target) {
      if (++polls > (1u << 26)) {
        atomicExch(ctr + 1, 1u);
        break;
      }
      if (polls > 64) __nanosleep(32);
    }
  }
  __syncthreads();
}

SDC_DEV double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
SDC_DEV double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

}  // namespace sdc
