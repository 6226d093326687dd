// K1 — input projection on the 5th-gen tensor cores.
//
//   XP[M, N] = X[M, K] · W_ih[N, K]ᵀ + bias[N]      M = T·B, N = G·H, K = I_l
//
// Pass schemes (npass): 3 = f32 mode for layer 0 (the raw input): bf16
// hi/lo X and W, X_hi·W_hi + X_hi·W_lo + X_lo·W_hi accumulated in f32 in TMEM
// (≈16-bit operands); 2 = f32 mode for the hidden layers: X = h rounded to
// fp16 once times fp16 hi/lo of the row-scaled W_ih (X·W_hi + X·W_lo, the
// recurrence's own h·W_hh scheme; the epilogue applies the row scales);
// 1 = bf16 mode, one product.  The f32-mode kernels issue the products of a
// 64-wide K-block from one load of its tiles (a slot pair of the ring) in the
// same order everywhere (load_kblock_fused / mma_kblock_fused); bf16 mode and
// HS_K1_FUSED3=0 run the passes as a longer K loop over (plane_a, plane_b)
// pairs.  ncu at c2 (scheme 3): 158.6 -> 153.2 us per layer fused, L2
// throughput 56% -> 43%.  The pipeline is a plain warp-specialised GEMM:
//   warp 0   TMA producer (one elected lane), 4-stage smem ring, 128B swizzle
//   warp 1   MMA issuer: tcgen05.mma.cta_group::1.kind::f16, M=128, N=BN, K=16
//   warp 2   TMEM allocator (BN f32 columns)
//   warps 4-7 epilogue: tcgen05.ld 32x32b -> +bias -> st.global f32
#pragma once
#include "common.cuh"
#include "tc_common.cuh"

namespace hs {
namespace tc {

constexpr int GBM = 128;
constexpr int GBK = 64;

// K1 fused K-blocks (f32 mode, pass schemes 2 and 3); HS_K1_FUSED3=0 selects
// the pass-major loop (A/B).  Set per device by the host before the first K1.
__constant__ int c_k1_fused3 = 1;
__device__ __forceinline__ bool k1_fused3() { return c_k1_fused3 != 0; }

// Pass schemes (npass): 3 = f32 mode, bf16 hi/lo X and W, three products
// (layer 0: the raw input); 2 = f32 mode for hidden-state inputs, X rounded
// to fp16 once (plane 0) times fp16 hi/lo W of the row-scaled weights —
// exactly the recurrence's own h·W_hh operand scheme — with the row scales
// applied in the epilogue; 1 = bf16 mode, one bf16 product.
__device__ __forceinline__ uint32_t k1_idesc(int npass, int BN) {
  return npass == 2 ? ptx::idesc_f16_f32(GBM, BN) : ptx::idesc_bf16_f32(GBM, BN);
}
// accumulator columns of W_ih rows scaled by 2^e -> times 2^-e
__device__ __forceinline__ void apply_scale(float (&v)[32], const float* __restrict__ sc) {
#pragma unroll
  for (int j = 0; j < 32; j += 4) {
    const float4 f = *reinterpret_cast<const float4*>(sc + j);
    v[j] *= f.x;
    v[j + 1] *= f.y;
    v[j + 2] *= f.z;
    v[j + 3] *= f.w;
  }
}

// Fused K-block (pass schemes 2 and 3): every product of one 64-wide K-block
// from ONE load of its tiles, staged in a slot pair (s0, s1) of the ring:
//   a[s0] = X plane 0, b[s0] = W hi, b[s1] = W lo, a[s1] = X lo (scheme 3)
// products per K=16 step: X0·W_hi, X0·W_lo (+ X_lo·W_hi for scheme 3).
// Every kernel issues them in this order, so a layer's K1 is bit-identical
// whichever kernel (persistent, one tile per CTA, dynamic, wave) runs it.
template <int BN>
__device__ __forceinline__ void load_kblock_fused(int np, __nv_bfloat16* a0, __nv_bfloat16* a1, __nv_bfloat16* b0,
                                                  __nv_bfloat16* b1, const CUtensorMap* ta, const CUtensorMap* tb,
                                                  uint64_t* bar, int kk, int m0, int n0) {
  ptx::mbar_arrive_expect_tx(bar, (uint32_t)((np == 3 ? 2 * (GBM + BN) : GBM + 2 * BN) * GBK * 2));
  ptx::tma_load_3d(a0, ta, bar, kk * GBK, m0, 0);
  ptx::tma_load_3d(b0, tb, bar, kk * GBK, n0, 0);
  ptx::tma_load_3d(b1, tb, bar, kk * GBK, n0, 1);
  if (np == 3) ptx::tma_load_3d(a1, ta, bar, kk * GBK, m0, 1);
}
__device__ __forceinline__ void mma_kblock_fused(int np, uint32_t acc, const __nv_bfloat16* a0, const __nv_bfloat16* a1,
                                                 const __nv_bfloat16* b0, const __nv_bfloat16* b1, uint32_t idesc,
                                                 bool first) {
#pragma unroll
  for (int k = 0; k < GBK / 16; ++k) {
    const uint64_t ad0 = ptx::sdesc_k_sw128(a0 + k * 16), bd0 = ptx::sdesc_k_sw128(b0 + k * 16);
    const uint64_t bd1 = ptx::sdesc_k_sw128(b1 + k * 16);
    ptx::mma_bf16_ss(acc, ad0, bd0, idesc, !(first && k == 0));
    ptx::mma_bf16_ss(acc, ad0, bd1, idesc, 1);
    if (np == 3) ptx::mma_bf16_ss(acc, ptx::sdesc_k_sw128(a1 + k * 16), bd0, idesc, 1);
  }
}

// BN = 256: 4-stage ring, one CTA per SM.  BN = 128: 3-stage ring and two
// CTAs per SM, so one CTA's epilogue overlaps the other's MMAs.
template <int BN>
constexpr int gemm_stages() { return BN == 256 ? 4 : 3; }

template <int BN>
struct GemmSmem {
  static constexpr int GSTAGES = gemm_stages<BN>();
  __nv_bfloat16 a[GSTAGES][GBM * GBK];
  __nv_bfloat16 b[GSTAGES][BN * GBK];
  uint64_t full[GSTAGES];
  uint64_t empty[GSTAGES];
  uint64_t acc_full;
  uint32_t tmem_base;
};

template <int BN>
constexpr size_t gemm_smem_bytes() {
  return sizeof(GemmSmem<BN>) + 1024;
}

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

// tmA: 3D {K, M, 2 planes} bf16, box {64, 128, 1}; tmB: 3D {K, N, 2}, box {64, BN, 1}.
template <int BN>
__global__ void __launch_bounds__(256, BN == 256 ? 1 : 2)
    gemm_xproj_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      const float* __restrict__ bias, const float* __restrict__ scale, float* __restrict__ C, int M,
                      int N, int K, int npass) {
  extern __shared__ uint8_t smem_raw[];
  GemmSmem<BN>& sm = *reinterpret_cast<GemmSmem<BN>*>(align1024(smem_raw));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.y * GBM, n0 = blockIdx.x * BN;
  const int nk = K / GBK;
  const int nkb = npass * nk;
  constexpr int GSTAGES = gemm_stages<BN>();
  const bool fz = npass >= 2 && k1_fused3();  // fused K-blocks in slot pairs (GSTAGES / 2 of them)

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch(&tmA);
    ptx::tma_prefetch(&tmB);
    for (int s = 0; s < GSTAGES; ++s) {
      ptx::mbar_init(&sm.full[s], 1);
      ptx::mbar_init(&sm.empty[s], 1);
    }
    ptx::mbar_init(&sm.acc_full, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc<BN>(&sm.tmem_base);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp == 0) {
    if (ptx::elect_one()) {
      for (int kk = 0; fz && kk < nk; ++kk) {
        const int s0 = 2 * (kk % (GSTAGES / 2)), s1 = s0 + 1;
        if (kk >= GSTAGES / 2) ptx::mbar_wait(&sm.empty[s0], ((kk / (GSTAGES / 2)) - 1) & 1);
        load_kblock_fused<BN>(npass, sm.a[s0], sm.a[s1], sm.b[s0], sm.b[s1], &tmA, &tmB, &sm.full[s0], kk, m0, n0);
      }
      for (int kb = 0; !fz && kb < nkb; ++kb) {
        const int st = kb % GSTAGES;
        if (kb >= GSTAGES) ptx::mbar_wait(&sm.empty[st], ((kb / GSTAGES) - 1) & 1);
        const int pass = kb / nk, kk = kb % nk;
        const int pa = pass == 2 ? 1 : 0, pb = pass == 1 ? 1 : 0;
        ptx::mbar_arrive_expect_tx(&sm.full[st], (GBM + BN) * GBK * 2);
        ptx::tma_load_3d(sm.a[st], &tmA, &sm.full[st], kk * GBK, m0, pa);
        ptx::tma_load_3d(sm.b[st], &tmB, &sm.full[st], kk * GBK, n0, pb);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (ptx::elect_one()) {
      const uint32_t idesc = k1_idesc(npass, BN);
      for (int kk = 0; fz && kk < nk; ++kk) {
        const int s0 = 2 * (kk % (GSTAGES / 2)), s1 = s0 + 1;
        ptx::mbar_wait(&sm.full[s0], (kk / (GSTAGES / 2)) & 1);
        ptx::tc_fence_after();
        mma_kblock_fused(npass, tmem, sm.a[s0], sm.a[s1], sm.b[s0], sm.b[s1], idesc, kk == 0);
        ptx::mma_commit(&sm.empty[s0]);
      }
      for (int kb = 0; !fz && kb < nkb; ++kb) {
        const int st = kb % GSTAGES;
        ptx::mbar_wait(&sm.full[st], (kb / GSTAGES) & 1);
        ptx::tc_fence_after();
#pragma unroll
        for (int k = 0; k < GBK / 16; ++k) {
          const uint64_t ad = ptx::sdesc_k_sw128(sm.a[st] + k * 16);
          const uint64_t bd = ptx::sdesc_k_sw128(sm.b[st] + k * 16);
          ptx::mma_bf16_ss(tmem, ad, bd, idesc, (kb | k) != 0);
        }
        ptx::mma_commit(&sm.empty[st]);
      }
      ptx::mma_commit(&sm.acc_full);
    }
    __syncwarp();
  } else if (warp >= 4) {
    const int sub = warp & 3;
    ptx::mbar_wait(&sm.acc_full, 0);
    ptx::tc_fence_after();
    const int row = m0 + sub * 32 + lane;
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
      float v[32];
      ptx::tmem_ld_32x32b_x32(tmem + ((uint32_t)(sub * 32) << 16) + c * 32, v);
      if (row < M) {
        const int n = n0 + c * 32;
        float* dst = C + (size_t)row * N + n;
        if (scale) apply_scale(v, scale + n);
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          const float4 bb = *reinterpret_cast<const float4*>(bias + n + j);
          *reinterpret_cast<float4*>(dst + j) = make_float4(v[j] + bb.x, v[j + 1] + bb.y, v[j + 2] + bb.z, v[j + 3] + bb.w);
        }
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, BN);
  }
}

// Persistent form of K1: one CTA per SM walks the (M/128) x (N/256) output
// tiles (tile = blockIdx.x + k * gridDim.x).  The TMA ring runs across tile
// boundaries and the accumulator is double-buffered in TMEM (2 x 256 of the
// 512 columns), so the epilogue of tile j (TMEM -> +bias -> global) overlaps
// the MMAs of tile j+1 — the non-persistent kernel leaves the tensor pipe idle
// during every epilogue.
struct GemmPSmem {
  static constexpr int ST = 4;
  __nv_bfloat16 a[ST][GBM * GBK];
  __nv_bfloat16 b[ST][256 * GBK];
  uint64_t full[ST];
  uint64_t empty[ST];
  uint64_t tmem_full[2];
  uint64_t tmem_empty[2];
  uint32_t tmem_base;
};

constexpr size_t gemm_p_smem_bytes() { return sizeof(GemmPSmem) + 1024; }

__global__ void __launch_bounds__(256, 1)
    gemm_xproj_persistent(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                          const float* __restrict__ bias, const float* __restrict__ scale, float* __restrict__ C,
                          int M, int N, int K, int npass) {
  constexpr int BN = 256, ST = GemmPSmem::ST;
  extern __shared__ uint8_t smem_raw[];
  GemmPSmem& sm = *reinterpret_cast<GemmPSmem*>(align1024(smem_raw));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nk = K / GBK, nkb = npass * nk;
  // f32 mode: the three products of a K-block from one load of its four tiles
  // (X_hi, X_lo, W_hi, W_lo) instead of three passes re-loading X_hi and W_hi
  const bool f3 = npass >= 2 && k1_fused3();
  const int tiles_n = N / BN, tiles = ((M + GBM - 1) / GBM) * tiles_n;
  const int my_tiles = blockIdx.x < tiles ? (tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch(&tmA);
    ptx::tma_prefetch(&tmB);
    for (int s = 0; s < ST; ++s) {
      ptx::mbar_init(&sm.full[s], 1);
      ptx::mbar_init(&sm.empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&sm.tmem_full[b], 1);
      ptx::mbar_init(&sm.tmem_empty[b], 4);  // one arrive per epilogue warp
    }
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc<512>(&sm.tmem_base);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp == 0) {
    if (ptx::elect_one()) {
      for (int j = 0; j < my_tiles; ++j) {
        const int t = blockIdx.x + j * gridDim.x;
        const int m0 = (t / tiles_n) * GBM, n0 = (t % tiles_n) * BN;
        if (f3) {  // one super-stage (slot pair) per K-block: hi planes in slot 2p, lo planes in 2p+1
          for (int kk = 0; kk < nk; ++kk) {
            const int g = j * nk + kk, sp = g % (ST / 2), s0 = 2 * sp, s1 = s0 + 1;
            if (g >= ST / 2) ptx::mbar_wait(&sm.empty[s0], ((g / (ST / 2)) - 1) & 1);
            load_kblock_fused<BN>(npass, sm.a[s0], sm.a[s1], sm.b[s0], sm.b[s1], &tmA, &tmB, &sm.full[s0], kk, m0, n0);
          }
          continue;
        }
        for (int kb = 0; kb < nkb; ++kb) {
          const int g = j * nkb + kb, st = g % ST;
          if (g >= ST) ptx::mbar_wait(&sm.empty[st], ((g / ST) - 1) & 1);
          const int pass = kb / nk, kk = kb % nk;
          const int pa = pass == 2 ? 1 : 0, pb = pass == 1 ? 1 : 0;
          ptx::mbar_arrive_expect_tx(&sm.full[st], (GBM + BN) * GBK * 2);
          ptx::tma_load_3d(sm.a[st], &tmA, &sm.full[st], kk * GBK, m0, pa);
          ptx::tma_load_3d(sm.b[st], &tmB, &sm.full[st], kk * GBK, n0, pb);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (ptx::elect_one()) {
      const uint32_t idesc = k1_idesc(npass, BN);
      for (int j = 0; j < my_tiles; ++j) {
        const int buf = j & 1;
        if (j >= 2) ptx::mbar_wait(&sm.tmem_empty[buf], ((j >> 1) - 1) & 1);  // epilogue drained it
        ptx::tc_fence_after();
        const uint32_t acc = tmem + (uint32_t)(buf * BN);
        if (f3) {
          for (int kk = 0; kk < nk; ++kk) {
            const int g = j * nk + kk, sp = g % (ST / 2), s0 = 2 * sp, s1 = s0 + 1;
            ptx::mbar_wait(&sm.full[s0], (g / (ST / 2)) & 1);
            ptx::tc_fence_after();
            mma_kblock_fused(npass, acc, sm.a[s0], sm.a[s1], sm.b[s0], sm.b[s1], idesc, kk == 0);
            ptx::mma_commit(&sm.empty[s0]);
          }
          ptx::mma_commit(&sm.tmem_full[buf]);
          continue;
        }
        for (int kb = 0; kb < nkb; ++kb) {
          const int g = j * nkb + kb, st = g % ST;
          ptx::mbar_wait(&sm.full[st], (g / ST) & 1);
          ptx::tc_fence_after();
#pragma unroll
          for (int k = 0; k < GBK / 16; ++k) {
            const uint64_t ad = ptx::sdesc_k_sw128(sm.a[st] + k * 16);
            const uint64_t bd = ptx::sdesc_k_sw128(sm.b[st] + k * 16);
            ptx::mma_bf16_ss(acc, ad, bd, idesc, (kb | k) != 0);
          }
          ptx::mma_commit(&sm.empty[st]);
        }
        ptx::mma_commit(&sm.tmem_full[buf]);
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    const int sub = warp & 3;
    for (int j = 0; j < my_tiles; ++j) {
      const int t = blockIdx.x + j * gridDim.x;
      const int m0 = (t / tiles_n) * GBM, n0 = (t % tiles_n) * BN;
      const int buf = j & 1;
      ptx::mbar_wait(&sm.tmem_full[buf], (j >> 1) & 1);
      ptx::tc_fence_after();
      const int row = m0 + sub * 32 + lane;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        float v[32];
        ptx::tmem_ld_32x32b_x32(tmem + ((uint32_t)(sub * 32) << 16) + (uint32_t)(buf * BN + c * 32), v);
        if (row < M) {
          const int n = n0 + c * 32;
          float* dst = C + (size_t)row * N + n;
          if (scale) apply_scale(v, scale + n);
#pragma unroll
          for (int q = 0; q < 32; q += 4) {
            const float4 bb = *reinterpret_cast<const float4*>(bias + n + q);
            *reinterpret_cast<float4*>(dst + q) =
                make_float4(v[q] + bb.x, v[q + 1] + bb.y, v[q + 2] + bb.z, v[q + 3] + bb.w);
          }
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&sm.tmem_empty[buf]);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

// ---------------------------------------------------------------------------
// Dynamic-schedule K1 for the layer overlap: layer l+1's input projection
// while layer l's recurrence is still running.  Tiles are claimed in time
// order from one global counter (atomicAdd), unit t -> (M-tile m, direction
// d, N-tile n), and the producer polls the recurrence's per-step progress
// counter for the M-tile's last timestep before loading its rows.  Launched
// with one CTA per SM once the recurrence is resident: the CTAs that find a
// free SM (those the persistent recurrence leaves idle) start right away and
// wait for rows as they are published; the rest start when the recurrence
// exits and take the remaining tiles at full width.  Same pipeline as
// gemm_xproj_persistent (TMA ring across tiles, double-buffered TMEM
// accumulators), plus a 16-slot tile-id queue in shared memory (tq_full
// mbarriers) from the producer to the MMA and epilogue warps.
constexpr int kMaxSeg = 8;  // segments of a dynamic K1 launch (directions, or the layers of a wave)
struct GemmDynArgs {
  const float* bias[kMaxSeg];      // per segment [N]
  float* C[kMaxSeg];               // per segment [M, N]
  const float* scale[kMaxSeg];     // per segment [N] W_ih row inverse scales (pass scheme 2), else nullptr
  int M, N, K, npass, D, T, B;     // npass: pass scheme (see k1_idesc); wave mode: per segment in wnpass
  unsigned int* claim;             // zeroed before launch
  const unsigned int* progress;    // [T] CTAs of the recurrence that finished step s
  unsigned int ncta;               // progress[s] value meaning "step s complete everywhere"
  int tile_begin, tile_end;        // claimable tile range (tile_end <= 0: all)
  unsigned int* xready;            // optional [M-tiles]: +1 per stored tile (XP streaming into a running recurrence)
  // Wave mode (nseg > 0, D == 1): segment j is layer j+1 of a layer wavefront
  // (recur_tc_wave_kernel).  It has its own A map (layer j's output planes),
  // B map (layer j+1's W_ih), progress counters (layer j's steps) and xready
  // (layer j+1's M-tiles).  Tiles are claimed along skewed diagonals: claim
  // index u -> (k = u / per_m, segment j, N-tile n), M-tile m = k - j*lag, so
  // a tile is claimed about when its rows are produced, and every tile a
  // claimed tile depends on (m' <= m of segment j-1) was claimed before it.
  int nseg, lag;
  int wK[kMaxSeg];                 // wave mode: contraction length of each segment (layer input width)
  int wnpass[kMaxSeg];             // wave mode: pass scheme of each segment
  const unsigned int* wprogress[kMaxSeg];
  unsigned int wncta[kMaxSeg];
  unsigned int* wxready[kMaxSeg];
};

struct DynMaps {
  CUtensorMap a[kMaxSeg];  // A planes: [0] only, except in wave mode
  CUtensorMap b[kMaxSeg];  // W_ih planes per segment
};

// ST: TMA ring stages; NACC: TMEM accumulators (2 = double-buffered, 512
// columns; 1 = 256 columns, for two CTAs per SM in the 2-CTA/SM layer wave)
template <int ST_ = 4>
struct GemmDSmem {
  static constexpr int ST = ST_, NQ = 16;
  __nv_bfloat16 a[ST][GBM * GBK];
  __nv_bfloat16 b[ST][256 * GBK];
  uint64_t full[ST];
  uint64_t empty[ST];
  uint64_t tmem_full[2];
  uint64_t tmem_empty[2];
  uint64_t tq_full[NQ];
  int tq[NQ];
  uint32_t tmem_base;
};

template <int ST = 4>
constexpr size_t gemm_d_smem_bytes() { return sizeof(GemmDSmem<ST>) + 1024; }

// The body: also run by the K1 CTAs of the fused layer-wave kernel (tc_wave.cuh).
template <int ST = 4, int NACC = 2>
__device__ __forceinline__ void gemm_dyn_body(const DynMaps& mp, const GemmDynArgs& g, uint8_t* smem_raw) {
  constexpr int BN = 256, NQ = GemmDSmem<ST>::NQ;
  constexpr uint32_t TCOLS = NACC * BN;
  GemmDSmem<ST>& sm = *reinterpret_cast<GemmDSmem<ST>*>(align1024(smem_raw));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool wave = g.nseg > 0;
  // k-blocks of a tile of segment sg (passes x K/64); the ring position is a
  // running count because wave segments may differ in K
  auto np_of = [&](int sg) -> int { return wave ? g.wnpass[sg] : g.npass; };  // pass scheme of segment sg
  auto nkb_of = [&](int sg) -> int { return np_of(sg) * ((wave ? g.wK[sg] : g.K) / GBK); };
  const int nseg = wave ? g.nseg : g.D;
  // f32-mode schemes (2, 3): fused K-blocks, one slot pair each (ST / 2
  // pairs; one, unpipelined, for ST = 2), in the same product order as the
  // other K1 kernels.  bf16 mode (1) runs pass-major.
  bool f3 = k1_fused3();
  for (int j = 0; j < nseg; ++j) f3 = f3 && np_of(j) >= 2;
  const int tiles_n = g.N / BN, per_m = nseg * tiles_n;
  const int tiles_m = (g.M + GBM - 1) / GBM;
  const int tiles_all = tiles_m * per_m;
  const int tiles = g.tile_end > 0 && g.tile_end < tiles_all ? g.tile_end : tiles_all;
  const int claims = wave ? (tiles_m + (nseg - 1) * g.lag) * per_m : tiles;

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch(&mp.a[0]);
    for (int j = 0; j < nseg; ++j) {
      ptx::tma_prefetch(&mp.b[j]);
      if (wave && j) ptx::tma_prefetch(&mp.a[j]);
    }
    for (int s = 0; s < ST; ++s) {
      ptx::mbar_init(&sm.full[s], 1);
      ptx::mbar_init(&sm.empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&sm.tmem_full[b], 1);
      ptx::mbar_init(&sm.tmem_empty[b], 4);
    }
    for (int q = 0; q < NQ; ++q) ptx::mbar_init(&sm.tq_full[q], 1);
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc<TCOLS>(&sm.tmem_base);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = sm.tmem_base;
  // the queue slot of tile j is rewritten at j + NQ; the producer runs at most
  // ST stages + 2 TMEM buffers (< NQ tiles) ahead of the epilogue
  auto next_tile = [&](int j) -> int {
    ptx::mbar_wait(&sm.tq_full[j % NQ], (uint32_t)((j / NQ) & 1));
    return sm.tq[j % NQ];
  };

  if (warp == 0) {
    if (ptx::elect_one()) {
      int gi = 0;  // ring position
      for (int j = 0;; ++j) {
        int t = -1;
        for (;;) {  // next claim (wave mode skips a diagonal's out-of-range M-tiles)
          const int u = g.tile_begin + (int)atomicAdd(g.claim, 1u);
          if (u >= claims) break;
          if (!wave) {
            t = u;
            break;
          }
          const int r = u % per_m, m = u / per_m - (r / tiles_n) * g.lag;
          if (m >= 0 && m < tiles_m) {
            t = m * per_m + r;
            break;
          }
        }
        sm.tq[j % NQ] = t;
        ptx::mbar_arrive(&sm.tq_full[j % NQ]);
        if (t < 0) break;
        const int mt = t / per_m, sg = (t % per_m) / tiles_n, n0 = (t % tiles_n) * BN;
        const int m0 = mt * GBM;
        // rows [m0, m0+128) hold timesteps [t0, t1); they are final once the
        // recurrence finished step s_need (a backward direction runs T-1 .. 0)
        const int t0 = m0 / g.B, t1 = min(g.T, (m0 + GBM + g.B - 1) / g.B);
        const int s_need = g.D == 1 ? t1 - 1 : max(t1 - 1, g.T - 1 - t0);
        const unsigned int* prog = wave ? g.wprogress[sg] : g.progress;
        if (prog) {  // nullptr: every row is already in memory
          wait_geq(prog + s_need, wave ? g.wncta[sg] : g.ncta, kWatchGemmProgress);
          ptx::fence_proxy_async_global();  // generic-proxy y stores -> TMA reads
        }
        const CUtensorMap* ta = &mp.a[wave ? sg : 0];
        const CUtensorMap* tb = &mp.b[sg];
        const int nkb = nkb_of(sg), nk = nkb / np_of(sg);
        if (f3) {
          for (int kk = 0; kk < nk; ++kk, ++gi) {
            const int sp = gi % (ST / 2), s0 = 2 * sp, s1 = s0 + 1;
            if (gi >= ST / 2) ptx::mbar_wait(&sm.empty[s0], ((gi / (ST / 2)) - 1) & 1);
            load_kblock_fused<BN>(np_of(sg), sm.a[s0], sm.a[s1], sm.b[s0], sm.b[s1], ta, tb, &sm.full[s0], kk, m0, n0);
          }
          continue;
        }
        for (int kb = 0; kb < nkb; ++kb, ++gi) {
          const int st = gi % ST;
          if (gi >= ST) ptx::mbar_wait(&sm.empty[st], ((gi / ST) - 1) & 1);
          const int pass = kb / nk, kk = kb % nk;
          const int pa = pass == 2 ? 1 : 0, pb = pass == 1 ? 1 : 0;
          ptx::mbar_arrive_expect_tx(&sm.full[st], (GBM + BN) * GBK * 2);
          ptx::tma_load_3d(sm.a[st], ta, &sm.full[st], kk * GBK, m0, pa);
          ptx::tma_load_3d(sm.b[st], tb, &sm.full[st], kk * GBK, n0, pb);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (ptx::elect_one()) {
      int gi = 0;  // ring position
      for (int j = 0;; ++j) {
        const int t = next_tile(j);
        if (t < 0) break;
        const int buf = j % NACC;
        if (j >= NACC) ptx::mbar_wait(&sm.tmem_empty[buf], ((j / NACC) - 1) & 1);
        ptx::tc_fence_after();
        const uint32_t acc = tmem + (uint32_t)(buf * BN);
        const int nkb = nkb_of((t % per_m) / tiles_n);
        const uint32_t idesc = k1_idesc(np_of((t % per_m) / tiles_n), BN);
        if (f3) {
          const int np = np_of((t % per_m) / tiles_n);
          for (int kk = 0; kk < nkb / np; ++kk, ++gi) {
            const int sp = gi % (ST / 2), s0 = 2 * sp, s1 = s0 + 1;
            ptx::mbar_wait(&sm.full[s0], (gi / (ST / 2)) & 1);
            ptx::tc_fence_after();
            mma_kblock_fused(np, acc, sm.a[s0], sm.a[s1], sm.b[s0], sm.b[s1], idesc, kk == 0);
            ptx::mma_commit(&sm.empty[s0]);
          }
          ptx::mma_commit(&sm.tmem_full[buf]);
          continue;
        }
        for (int kb = 0; kb < nkb; ++kb, ++gi) {
          const int st = gi % ST;
          ptx::mbar_wait(&sm.full[st], (gi / ST) & 1);
          ptx::tc_fence_after();
#pragma unroll
          for (int k = 0; k < GBK / 16; ++k) {
            const uint64_t ad = ptx::sdesc_k_sw128(sm.a[st] + k * 16);
            const uint64_t bd = ptx::sdesc_k_sw128(sm.b[st] + k * 16);
            ptx::mma_bf16_ss(acc, ad, bd, idesc, (kb | k) != 0);
          }
          ptx::mma_commit(&sm.empty[st]);
        }
        ptx::mma_commit(&sm.tmem_full[buf]);
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    const int sub = warp & 3;
    for (int j = 0;; ++j) {
      const int t = next_tile(j);
      if (t < 0) break;
      const int mt = t / per_m, sg = (t % per_m) / tiles_n, n0 = (t % tiles_n) * BN;
      const int m0 = mt * GBM;
      const float* __restrict__ bias = g.bias[sg];
      const float* __restrict__ scale = g.scale[sg];
      float* __restrict__ C = g.C[sg];
      unsigned int* xr = wave ? g.wxready[sg] : g.xready;
      const int buf = j % NACC;
      ptx::mbar_wait(&sm.tmem_full[buf], (j / NACC) & 1);
      ptx::tc_fence_after();
      const int row = m0 + sub * 32 + lane;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        float v[32];
        ptx::tmem_ld_32x32b_x32(tmem + ((uint32_t)(sub * 32) << 16) + (uint32_t)(buf * BN + c * 32), v);
        if (row < g.M) {
          const int n = n0 + c * 32;
          float* dst = C + (size_t)row * g.N + n;
          if (scale) apply_scale(v, scale + n);
#pragma unroll
          for (int q = 0; q < 32; q += 4) {
            const float4 bb = *reinterpret_cast<const float4*>(bias + n + q);
            *reinterpret_cast<float4*>(dst + q) =
                make_float4(v[q] + bb.x, v[q + 1] + bb.y, v[q + 2] + bb.z, v[q + 3] + bb.w);
          }
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&sm.tmem_empty[buf]);
      if (xr) {  // the 4 epilogue warps' stores of this tile -> one release
        ptx::named_bar(1, 128);
        if (warp == 4 && lane == 0)
          asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(xr + mt) : "memory");
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, TCOLS);
  }
}

__global__ void __launch_bounds__(256, 1) gemm_xproj_dyn(const __grid_constant__ DynMaps mp, const GemmDynArgs g) {
  extern __shared__ uint8_t smem_raw[];
  gemm_dyn_body(mp, g, smem_raw);
}

// fp32 [rows, cols] (row stride ld) -> the K1 A operand planes [2][rows][cols]:
// f16 = 1 (pass scheme 2, hidden-state inputs): fp16(x) in plane 0 only;
// else bf16 hi/lo, the lo plane `pstride` elements after the hi plane
// (pstride = 0: rows*cols)
__global__ void split_planes_kernel(const float* __restrict__ x, __nv_bfloat16* __restrict__ out, size_t rows, int cols,
                                    int ld, size_t pstride, int f16) {
  const size_t total = rows * (size_t)cols;
  for (size_t i = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) * 4; i < total; i += (size_t)gridDim.x * blockDim.x * 4) {
    const size_t r = i / cols;
    const int c = (int)(i % cols);
    const float4 v = *reinterpret_cast<const float4*>(x + r * ld + c);
    if (f16) {
      __align__(8) __half h4[4] = {__float2half_rn(v.x), __float2half_rn(v.y), __float2half_rn(v.z), __float2half_rn(v.w)};
      *reinterpret_cast<uint2*>(out + i) = *reinterpret_cast<uint2*>(h4);
      continue;
    }
    const float f[4] = {v.x, v.y, v.z, v.w};
    __align__(8) __nv_bfloat16 hi[4], lo[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) ptx::split_bf16(f[j], hi[j], lo[j]);
    *reinterpret_cast<uint2*>(out + i) = *reinterpret_cast<uint2*>(hi);
    *reinterpret_cast<uint2*>(out + (pstride ? pstride : total) + i) = *reinterpret_cast<uint2*>(lo);
  }
}

}  // namespace tc
}  // namespace hs
