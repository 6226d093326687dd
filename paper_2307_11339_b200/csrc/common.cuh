// Shared device helpers: gate nonlinearities, the grid-wide step barrier,
// L2-only loads for data produced by other CTAs within the same launch.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace hs {

// kernels launched by the current forward call on this host thread
// (hs_rnn_last_launch_count; reset at the start of every forward entry point)
inline thread_local int g_launch_count = 0;

// Full-precision activations: the f32 mode is held to max-abs 1e-4 against
// the float64 oracle, so no __expf / tanh.approx here.
__device__ __forceinline__ float sigmoidf_(float v) { return 1.0f / (1.0f + expf(-v)); }
__device__ __forceinline__ float tanhf_(float v) { return tanhf(v); }

// Short-latency forms for the tensor-core epilogue (on the per-step critical
// path): ex2.approx has ~2 ulp relative error, so sigmoid/tanh built on it
// stay within ~1e-7 absolute — far below the 1e-4 budget.
__device__ __forceinline__ float sigmoid_fast(float v) { return __fdividef(1.0f, 1.0f + __expf(-v)); }
__device__ __forceinline__ float tanh_fast(float v) { return 1.0f - __fdividef(2.0f, __expf(2.0f * v) + 1.0f); }

// Grid barrier for persistent kernels.  `ctr` is zeroed by the host before
// the launch; round r (0-based) completes when every CTA has arrived r+1
// times.  All CTAs must be co-resident (cooperative launch enforces it).
// Release: bar.sync then a gpu-scope fence by the arriving thread (cumulative
// over the CTA's writes).  Acquire: ld.acquire spin, fence, bar.sync.
__device__ __forceinline__ void grid_barrier(unsigned int* ctr, unsigned int target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
    unsigned int seen;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(ctr) : "memory");
    } while (seen < target);
    __threadfence();
  }
  __syncthreads();
}

// Loads of values written by other CTAs earlier in the same launch must not
// hit a stale L1 line: cache-global (L2 only).
__device__ __forceinline__ float ld_l2(const float* p) { return __ldcg(p); }
__device__ __forceinline__ float4 ld_l2_v4(const float* p) {
  return __ldcg(reinterpret_cast<const float4*>(p));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

}  // namespace hs
