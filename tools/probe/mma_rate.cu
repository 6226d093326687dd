// tcgen05.mma issue rate at the recurrence's shapes (M=128, small N, K=16,
// kind::f16): cycles per MMA for a back-to-back stream issued by one thread,
// A from shared memory (SS) or tensor memory (TS), 1/2/4 accumulators.
// Built and run by tools/mma_rate.py.
#include "../../paper_2307_11339_b200/csrc/tc_common.cuh"

using namespace hs;

__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__global__ void __launch_bounds__(288) mma_rate_kernel(int ts, int N, int R, int nacc, int spin, unsigned long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __nv_bfloat16* A = reinterpret_cast<__nv_bfloat16*>(smem);              // 128 x 64
  __nv_bfloat16* B = reinterpret_cast<__nv_bfloat16*>(smem + 16384);      // 256 x 64
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 16384 + 32768);
  uint64_t* ready = bar + 1;  // two barriers whose phase 0 has completed (waits return at once)
  uint64_t* spare = bar + 3;  // commit target of the per-chunk "slot free" commits
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 4);
  for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    ptx::mbar_init(bar, 1);
    ptx::mbar_init(ready, 1);
    ptx::mbar_init(ready + 1, 1);
    ptx::mbar_init(spare, 1 << 20);
    ptx::fence_mbar_init();
    ptx::mbar_arrive(ready);
    ptx::mbar_arrive(ready + 1);
  }
  ptx::fence_proxy_async_smem();
  if (threadIdx.x < 32) ptx::tmem_alloc_dyn(slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, *slot, 0);  // warp-uniform: MMA operands stay in uniform registers
  if (threadIdx.x < 32 && ptx::elect_one()) {
    const uint32_t idesc = idesc_f16(128, N);
    const unsigned long long t0 = clock64();
    for (int i = 0; i < (ts >= 4 ? 0 : R); ++i) {
      const int kk = i & 3;
      // chunk mode (ts >= 2): every 8 MMAs = one chunk of the recurrence's loop:
      // wait on the h barrier (+ the W slot barrier for SS), fence, and (SS) commit the slot
      if (ts >= 2 && (i & 7) == 0) {
        if (ts == 3 && i) ptx::mma_commit(spare);
        if (ts == 3) ptx::mbar_wait(ready + 1, 0);
        ptx::mbar_wait(ready, 0);
        ptx::tc_fence_after();
      }
      const uint32_t acc = tmem + (uint32_t)((i & (nacc - 1)) * N);
      const uint64_t bd = ptx::sdesc_k_sw128(B + kk * 16);
      if (ts == 1 || ts == 2)
        ptx::mma_bf16_ts(acc, tmem + 256u + (uint32_t)(kk * 8), bd, idesc, i >= nacc);
      else
        ptx::mma_bf16_ss(acc, ptx::sdesc_k_sw128(A + kk * 16), bd, idesc, i >= nacc);
    }
    if (ts >= 4) {  // unrolled chunks of 8 (4 K-steps x 2 planes), descriptors hoisted; ts 5/7: + per-chunk waits
      const bool tsm = ts < 6;
      const bool waits = ts == 5 || ts == 7;
      uint64_t bd[4], ad[4];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        bd[kk] = ptx::sdesc_k_sw128(B + kk * 16);
        ad[kk] = ptx::sdesc_k_sw128(A + kk * 16);
      }
      for (int c = 0; c < R / 8; ++c) {
        if (waits) {
          if (!tsm) ptx::mbar_wait(ready + 1, 0);
          ptx::mbar_wait(ready, 0);
          ptx::tc_fence_after();
        }
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          if (tsm) {
            ptx::mma_bf16_ts(tmem, tmem + 256u + (uint32_t)(kk * 8), bd[kk], idesc, c | kk);
            ptx::mma_bf16_ts(tmem, tmem + 288u + (uint32_t)(kk * 8), bd[kk], idesc, 1);
          } else {
            ptx::mma_bf16_ss(tmem, ad[kk], bd[kk], idesc, c | kk);
            ptx::mma_bf16_ss(tmem, ad[kk] + 2, bd[kk], idesc, 1);
          }
        }
        if (waits && !tsm) ptx::mma_commit(spare);
      }
    }
    const unsigned long long t1 = clock64();
    ptx::mma_commit(bar);
    ptx::mbar_wait(bar, 0);
    const unsigned long long t2 = clock64();
    out[2 * blockIdx.x] = t1 - t0;
    out[2 * blockIdx.x + 1] = t2 - t0;
  } else if (spin && threadIdx.x >= 32) {
    ptx::mbar_wait(bar, 0);  // like the recurrence's epilogue warps waiting on the accumulator
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

extern "C" int mma_rate(int ts, int N, int R, int nacc, int grid, int threads, double* issue_cyc, double* done_cyc) {
  unsigned long long* d;
  if (cudaMalloc(&d, 2 * sizeof(unsigned long long) * grid) != cudaSuccess) return 1;
  const int smem = 16384 + 32768 + 64 + 1024;
  cudaFuncSetAttribute(mma_rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
  // > half of shared memory: one CTA per SM (each allocates all 512 TMEM columns)
  for (int rep = 0; rep < 2; ++rep) mma_rate_kernel<<<grid, threads, 120 * 1024>>>(ts, N, R, nacc, threads > 128, d);
  (void)smem;
  if (cudaDeviceSynchronize() != cudaSuccess) return 2;
  unsigned long long h[2 * 1024];
  cudaMemcpy(h, d, 2 * sizeof(unsigned long long) * grid, cudaMemcpyDeviceToHost);
  double a = 0, b = 0;
  for (int i = 0; i < grid; ++i) {
    a += h[2 * i];
    b += h[2 * i + 1];
  }
  *issue_cyc = a / grid / R;
  *done_cyc = b / grid / R;
  cudaFree(d);
  return 0;
}
