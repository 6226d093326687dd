// Shared device helpers: gate nonlinearities, the grid-wide step barrier,
// L2-only loads for data produced by other CTAs within the same launch.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace hs {

// kernels launched by the current forward call on this host thread
// (hs_rnn_last_launch_count; reset at the start of every forward entry point)
inline thread_local int g_launch_count = 0;

// Per-device one-time setup (cudaFuncSetAttribute and lazy module loading act
// on the current device only): flags are indexed by the current device.
constexpr int kMaxDev = 16;
inline int cur_device() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= kMaxDev) d = 0;
  return d;
}

// ------------------------------------------------------------------ watchdog
// Every spin on a value another CTA or another kernel publishes (per-chunk h
// counters, XP readiness, the dynamic K1's progress poll, the SIMT grid
// barrier) is bounded: if the awaited condition has not held for
// g_watchdog_ns (HS_WATCHDOG_MS, default 10 s; 0 = off) the spinning thread
// records where it was in a host-mapped word and traps.  A lost co-residency
// (another process / MPS client holding the SMs a persistent launch counted
// on) then surfaces as a CUDA error with a message (hs_last_error) instead of
// a silent hang.  Sites:
enum WatchSite : unsigned int {
  kWatchRecurChunk = 1,   // recurrence producer: h_{t-1} chunk counter
  kWatchRecurXready = 2,  // recurrence: K1 tiles of the next timestep (XP streaming)
  kWatchGemmProgress = 3, // dynamic K1: recurrence progress for the tile's rows
  kWatchGridBarrier = 4,  // SIMT recurrence grid barrier
  kWatchPeerFlag = 5,     // pipeline hand-off: previous stage's step flag
};
__device__ unsigned long long g_watchdog_ns = 0;
__device__ unsigned int* g_watch_word = nullptr;  // host-mapped; 0 = no event

__device__ __noinline__ void watchdog_fire(unsigned int site) {
  unsigned int* w = g_watch_word;
  if (w) {
    atomicCAS_system(w, 0u, 0x80000000u | ((blockIdx.x & 0xffffu) << 8) | (site & 0xffu));
    __threadfence_system();
  }
  __trap();
}

struct Spin {
  unsigned long long t0 = 0;
  unsigned int n = 0;
  // call once per unsuccessful poll
  __device__ __forceinline__ void tick(unsigned int site) {
    if ((++n & 63u) != 0u) return;
    const unsigned long long lim = g_watchdog_ns;
    if (lim == 0ull) return;
    unsigned long long now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    if (t0 == 0ull) t0 = now;
    else if (now - t0 > lim) watchdog_fire(site);
  }
};

// spin until *p >= target (acquire, gpu scope), bounded by the watchdog
__device__ __forceinline__ unsigned int wait_geq(const unsigned int* p, unsigned int target, unsigned int site) {
  unsigned int v;
  Spin sp;
  for (;;) {
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    if (v >= target) return v;
    sp.tick(site);
  }
}

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
    wait_geq(ctr, target, kWatchGridBarrier);
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
