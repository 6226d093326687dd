// K2/K3 — persistent recurrent wavefront on the tensor cores.
//
// Per timestep t of layer l (both directions concurrently):
//   gatesᵀ[G·H, B] = W_hh[G·H, H] · h_{t-1}ᵀ[H, B]  (+ XP[t] from K1, + b_hh for GRU)
// fused with the gate nonlinearities and the c/h update.
//
// Decomposition (B200-first, W_hh never leaves the SM):
//   * row block rb = 32 hidden units x G gates = 128 MMA rows (GRU pads 96->128)
//   * the row block's K = H contraction is split over a cluster of S CTAs
//     (rank q owns k in [q·H/S, (q+1)·H/S)); each CTA keeps its W_hh slice
//     (split-bf16 hi/lo planes) resident in shared memory for all T steps
//   * per step each CTA TMA-loads only its K-slice of h_{t-1} (bf16 planes,
//     written by the previous step's epilogues), runs M=128, N=Bpad, K=16
//     tcgen05 MMAs into TMEM (3 passes hi·hi + hi·lo + lo·hi in f32 mode),
//     reduce-scatters the f32 partial gates to the unit owners through DSMEM
//     (st.shared::cluster), and each owner finishes 32/S units: +XP, σ/tanh,
//     c/h update (c and h stay in registers for all T), writes h_t planes
//   * steps are ordered by per-K-slice arrival counters in global memory
//     (release/acquire), not a full grid barrier: a CTA starts step t as soon
//     as the H/32 row-block owners of *its* K-slice have published h_{t-1};
//     h_t is triple-buffered so no CTA can overwrite a slice still being read.
#pragma once
#include "common.cuh"
#include "tc_common.cuh"

namespace hs {
namespace tc {

constexpr int RMAXCH = 16;   // max 64-wide K chunks per CTA (K-slice <= 1024)
constexpr int RMAXCELLS = 32;

struct TcRecurArgs {
  int H, B, Npad, T, D, S;
  int RB;                       // row blocks per direction = H / 32
  const float* xproj[2];        // per dir [T][B][G*H] f32 (includes b_ih (+ b_hh for LSTM))
  const float* bias_h[2];       // per dir [G*H] (GRU b_hh) or nullptr
  const float* h0[2];           // per dir [B][H]
  const float* c0[2];
  float* hn[2];                 // per dir [B][H]
  float* cn[2];
  float* y;                     // [T][B][D*H] f32, or nullptr
  __nv_bfloat16* ypl;           // [2][T*B][D*H] bf16 planes for the next layer's K1, or nullptr
  __nv_bfloat16* hbuf;          // [3][D][NPL][Npad][H] bf16
  unsigned int* counters;       // [D][S]
};

struct RecurLayout {
  int nch;        // K chunks per CTA
  size_t w_off, h_off, red_off, bar_off, total;
};

__host__ __device__ inline RecurLayout recur_layout(int G, int H, int Npad, int S, int NPL) {
  RecurLayout L;
  const int KS = H / S;
  L.nch = KS / 64;
  size_t off = 0;
  L.w_off = off;   off += (size_t)NPL * L.nch * 128 * 128;
  L.h_off = off;   off += (size_t)NPL * L.nch * Npad * 128;
  L.red_off = off; off += (size_t)G * 32 * (Npad + 4) * 4;
  off = (off + 15) / 16 * 16;
  L.bar_off = off; off += 8 * (2 + RMAXCH) + 16;
  L.total = off;  // dynamic smem starts 1024-aligned (checked in-kernel)
  return L;
}

__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int G, int NPL>
__global__ void __launch_bounds__(256, 1)
    recur_tc_kernel(const __grid_constant__ CUtensorMap tmW0, const __grid_constant__ CUtensorMap tmW1,
                    const __grid_constant__ CUtensorMap tmH, const TcRecurArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if (ptx::smem_u32(smem_raw) & 1023) __trap();  // SW128 atoms need 1024-B alignment
  const int H = a.H, B = a.B, Npad = a.Npad, T = a.T, D = a.D, S = a.S, RB = a.RB;
  const RecurLayout L = recur_layout(G, H, Npad, S, NPL);
  const int nch = L.nch;
  const int KS = H / S;
  const int UO = 32 / S;  // units finished by each rank
  __nv_bfloat16* sW = reinterpret_cast<__nv_bfloat16*>(smem + L.w_off);
  __nv_bfloat16* sH = reinterpret_cast<__nv_bfloat16*>(smem + L.h_off);
  float* red = reinterpret_cast<float*>(smem + L.red_off);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bar_off);
  uint64_t* w_full = bars;
  uint64_t* acc_full = bars + 1;
  uint64_t* h_full = bars + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 + RMAXCH);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = (int)ptx::cluster_rank();
  const int cl = blockIdx.x / S;          // cluster index
  const int d = cl / RB;
  const int rb = cl % RB;
  const CUtensorMap* tmW = d == 0 ? &tmW0 : &tmW1;
  const int GH = G * H;
  const int rstride = Npad + 4;
  const uint32_t tcols = Npad <= 32 ? 32 : Npad <= 64 ? 64 : Npad <= 128 ? 128 : 256;
  const int own_slice = (rb * 32) / KS;
  unsigned int* my_counter = a.counters + d * S + own_slice;
  const unsigned int* in_counter = a.counters + d * S + q;
  const size_t plane_stride = (size_t)Npad * H;  // elements per (buf, d, plane) slab of hbuf

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch(tmW);
    ptx::tma_prefetch(&tmH);
    ptx::mbar_init(w_full, 1);
    ptx::mbar_init(acc_full, 1);
    for (int c = 0; c < nch; ++c) ptx::mbar_init(&h_full[c], 1);
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc_dyn(tmem_slot, tcols);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // resident W_hh slice: NPL planes x nch chunks of [128 rows x 64 k]
  if (warp == 0 && ptx::elect_one()) {
    ptx::mbar_arrive_expect_tx(w_full, (uint32_t)(NPL * nch * 128 * 128));
    for (int p = 0; p < NPL; ++p)
      for (int c = 0; c < nch; ++c)
        ptx::tma_load_3d(sW + ((size_t)p * nch + c) * 128 * 64, tmW, w_full, q * KS + c * 64, rb * 128, p);
  }

  // owner cells: unit u_loc in [0, UO), batch rows b = b0 + k*bstep
  const int e = threadIdx.x - 128;
  const int u_loc = e >= 0 ? e % UO : 0;
  const int b0 = e >= 0 ? e / UO : 0;
  const int bstep = 128 / UO;
  const int ncell = Npad / bstep;
  const int unit = rb * 32 + q * UO + u_loc;
  float c_reg[RMAXCELLS], h_reg[RMAXCELLS];
  if (warp >= 4) {
#pragma unroll
    for (int k = 0; k < RMAXCELLS; ++k) {
      c_reg[k] = 0.f;
      h_reg[k] = 0.f;
      const int b = b0 + k * bstep;
      if (k < ncell && b < B) {
        h_reg[k] = a.h0[d][(size_t)b * H + unit];
        if (G == 4) c_reg[k] = a.c0[d][(size_t)b * H + unit];
        __nv_bfloat16 hi, lo;
        ptx::split_bf16(h_reg[k], hi, lo);
        __nv_bfloat16* hb = a.hbuf + ((size_t)(0 * D + d) * NPL) * plane_stride + (size_t)b * H + unit;
        hb[0] = NPL == 2 ? hi : __float2bfloat16_rn(h_reg[k]);
        if (NPL == 2) hb[plane_stride] = lo;
      }
    }
    ptx::fence_proxy_async_global();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(my_counter) : "memory");
  }
  cluster_arrive();

  const uint32_t idesc = ptx::idesc_bf16_f32(128, Npad);
  for (int s = 0; s < T; ++s) {
    const int t = d == 0 ? s : T - 1 - s;
    const int buf_in = s % 3, buf_out = (s + 1) % 3;
    if (warp == 0) {
      if (ptx::elect_one()) {
        const unsigned int target = (unsigned int)RB * (unsigned int)(s + 1);
        unsigned int seen;
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(in_counter) : "memory");
        } while (seen < target);
        ptx::fence_proxy_async_global();
        for (int c = 0; c < nch; ++c) {
          ptx::mbar_arrive_expect_tx(&h_full[c], (uint32_t)(NPL * Npad * 128));
          for (int p = 0; p < NPL; ++p)
            ptx::tma_load_3d(sH + ((size_t)p * nch + c) * Npad * 64, &tmH, &h_full[c], q * KS + c * 64, 0,
                             (buf_in * D + d) * NPL + p);
        }
      }
      __syncwarp();
    } else if (warp == 1) {
      if (ptx::elect_one()) {
        if (s == 0) ptx::mbar_wait(w_full, 0);
        for (int c = 0; c < nch; ++c) {
          ptx::mbar_wait(&h_full[c], s & 1);
          ptx::tc_fence_after();
          const __nv_bfloat16* wh = sW + (size_t)c * 128 * 64;
          const __nv_bfloat16* hh = sH + (size_t)c * Npad * 64;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            ptx::mma_bf16_ss(tmem, ptx::sdesc_k_sw128(wh + kk * 16), ptx::sdesc_k_sw128(hh + kk * 16), idesc,
                             (c | kk) != 0);
            if (NPL == 2) {
              const __nv_bfloat16* wl = wh + (size_t)nch * 128 * 64;
              const __nv_bfloat16* hl = hh + (size_t)nch * Npad * 64;
              ptx::mma_bf16_ss(tmem, ptx::sdesc_k_sw128(wh + kk * 16), ptx::sdesc_k_sw128(hl + kk * 16), idesc, 1);
              ptx::mma_bf16_ss(tmem, ptx::sdesc_k_sw128(wl + kk * 16), ptx::sdesc_k_sw128(hh + kk * 16), idesc, 1);
            }
          }
        }
        ptx::mma_commit(acc_full);
      }
      __syncwarp();
    }
    cluster_wait();  // peers finished reading last step's partials
    if (warp >= 4) {
      const int sub = warp & 3;
      ptx::mbar_wait(acc_full, s & 1);
      ptx::tc_fence_after();
      if (sub < G) {
        const int o = lane / UO, ul = lane % UO;
        const uint32_t local = ptx::smem_u32(red + ((size_t)(q * G + sub) * UO + ul) * rstride);
        const uint32_t remote = ptx::mapa(local, (uint32_t)o);
        for (int c16 = 0; c16 < Npad / 16; ++c16) {
          float v[16];
          ptx::tmem_ld_32x32b_x16(tmem + ((uint32_t)(sub * 32) << 16) + c16 * 16, v);
#pragma unroll
          for (int j = 0; j < 16; j += 4)
            ptx::st_cluster_v4(remote + (uint32_t)(c16 * 16 + j) * 4u, v[j], v[j + 1], v[j + 2], v[j + 3]);
        }
      }
      ptx::tc_fence_before();
    }
    cluster_arrive();
    cluster_wait();  // all partials for my units are in my shared memory
    if (warp >= 4) {
      const bool last = s == T - 1;
      const float* xp = a.xproj[d] + (size_t)t * B * GH + unit;
      const float* bh = a.bias_h[d];
#pragma unroll
      for (int k = 0; k < RMAXCELLS; ++k) {
        const int b = b0 + k * bstep;
        if (k >= ncell) break;
        float pre[4];
#pragma unroll
        for (int g = 0; g < G; ++g) {
          float acc = 0.f;
          for (int sr = 0; sr < S; ++sr) acc += red[((size_t)(sr * G + g) * UO + u_loc) * rstride + b];
          pre[g] = acc;
        }
        if (b >= B) continue;
        const float* xr = xp + (size_t)b * GH;
        float h;
        if (G == 4) {
          const float ig = sigmoidf_(pre[0] + xr[0]), fg = sigmoidf_(pre[1] + xr[H]);
          const float gg = tanhf_(pre[2] + xr[2 * H]), og = sigmoidf_(pre[3] + xr[3 * H]);
          const float cnew = fg * c_reg[k] + ig * gg;
          c_reg[k] = cnew;
          h = og * tanhf_(cnew);
        } else {
          const float r = sigmoidf_(xr[0] + pre[0] + (bh ? bh[unit] : 0.f));
          const float z = sigmoidf_(xr[H] + pre[1] + (bh ? bh[H + unit] : 0.f));
          const float n = tanhf_(xr[2 * H] + r * (pre[2] + (bh ? bh[2 * H + unit] : 0.f)));
          h = (1.f - z) * n + z * h_reg[k];
        }
        h_reg[k] = h;
        __nv_bfloat16 hi, lo;
        ptx::split_bf16(h, hi, lo);
        if (!last) {
          __nv_bfloat16* hb = a.hbuf + ((size_t)(buf_out * D + d) * NPL) * plane_stride + (size_t)b * H + unit;
          hb[0] = NPL == 2 ? hi : __float2bfloat16_rn(h);
          if (NPL == 2) hb[plane_stride] = lo;
        }
        const size_t yrow = (size_t)t * B + b;
        if (a.y) a.y[yrow * D * H + (size_t)d * H + unit] = h;
        if (a.ypl) {
          const size_t plane = (size_t)T * B * D * H;
          a.ypl[yrow * D * H + (size_t)d * H + unit] = hi;
          a.ypl[plane + yrow * D * H + (size_t)d * H + unit] = lo;
        }
        if (last) {
          a.hn[d][(size_t)b * H + unit] = h;
          if (G == 4) a.cn[d][(size_t)b * H + unit] = c_reg[k];
        }
      }
      ptx::fence_proxy_async_global();
    }
    __syncthreads();
    if (threadIdx.x == 0 && s + 1 < T) {
      __threadfence();
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(my_counter) : "memory");
    }
    cluster_arrive();
  }
  cluster_wait();
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, tcols);
  }
}

}  // namespace tc
}  // namespace hs
