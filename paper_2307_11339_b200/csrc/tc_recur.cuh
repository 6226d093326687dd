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
//     (fp16 hi/lo planes) resident in shared memory for all T steps
//   * per step each CTA TMA-loads only its K-slice of h_{t-1} (one fp16
//     plane, written by the previous step's epilogues), runs M=128, N=Bpad,
//     K=16 tcgen05 MMAs into TMEM (2 passes W_hi·h + W_lo·h in f32 mode),
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
constexpr int RMAXCELLS = 32;  // owner cells per epilogue thread (template CELLS <= this)

struct TcRecurArgs {
  int H, B, Npad, T, D, S;
  int Bst;                      // batch stride of xproj / y / ypl rows (>= B when the batch is sliced)
  int RB;                       // row blocks per direction = H / 32
  const float* xproj[2];        // per dir [T][B][G*H] f32 (includes b_ih (+ b_hh for LSTM))
  const float* bias_h[2];       // per dir [G*H] (GRU b_hh) or nullptr
  const float* whh_scale[2];    // per dir [H/32*128] 2^-e of each packed W_hh row (see whh_row_scale_kernel)
  const float* h0[2];           // per dir [B][H]
  const float* c0[2];
  float* hn[2];                 // per dir [B][H]
  float* cn[2];
  float* y;                     // [T][B][D*H] f32, or nullptr
  __nv_bfloat16* ypl;           // [2][T*B][D*H] planes for the next layer's K1, or nullptr
  int ypl_f16;                  // 1: fp16(h) in plane 0 only (next K1 on pass scheme 2), 0: bf16 hi/lo
  uint16_t* hbuf;               // [3][D][Npad][H] h_{t-1} operand: fp16 (f32 mode) / bf16 (bf16 mode)
  unsigned int* counters;       // [D][S]
  unsigned long long* trace;    // optional [grid][kTraceSteps][16] %globaltimer stamps (debug)
  unsigned int* progress;       // optional [T]: progress[s] counts CTAs whose outputs of step s are in memory
  unsigned int group_offset_ns; // two-group kernel: initial phase offset of group 1 (0 = none)
  // XP streaming (K1 of this layer still running): xready[m] counts the K1
  // tiles of M-tile m (rows [128m, 128m+128) of xproj) already stored;
  // timestep t may be read once its M-tiles reach xready_target.  nullptr = all present.
  const unsigned int* xready;
  unsigned int xready_target;
  unsigned int* started;        // optional: +1 per CTA once resident (gates the side-stream K1)
  // L2 eviction policies (kL2Hint*): the streamed W_hh ring evict_last, the
  // read-once xproj rows and the y stores evict_first, so the W_hh bytes the
  // streaming variant re-reads every step stay in L2 (c4: 64 MiB of 126 MB)
  int l2_hints;
  // A segment of a layer-direction (hs_rnn_run_cells): the launch runs T
  // steps starting at processing step s_base of a T_full-step sequence; rev
  // = 1 walks it backwards (the reverse direction launched alone, D = 1);
  // ycols = floats per y row (0 = D*H).  All zero = the whole layer.
  int s_base, T_full, rev, ycols;
  // optional per-step %globaltimer stamps of cluster 0 rank 0 of each
  // direction: stamps[d*(T+1)] at the first step's start, stamps[d*(T+1)+s+1]
  // when step s's h is released (hs_rnn_profile_cells)
  unsigned long long* stamps;
  // W_hh resident in TENSOR memory instead of shared memory (A operand of
  // tcgen05.mma read from TMEM): in SS mode every M=128, K=16 MMA re-reads
  // 4 KiB of W from shared memory, which paced the MMA phase of a step at
  // ~75 cycles per instruction (c2 trace: 32 MMAs = 1.2 of 5.4 us)
  const uint16_t* whh_g[2];     // per dir: packed planes [NPL][RB*128][H] (global)
  int w_tmem;                   // 1 = load the CTA's slice into TMEM and run TS-mode MMAs
  int w_tmem_chunks;            // W-streaming variant: chunks [0, n) of the slice stay in TMEM, the rest stream
};

// TMEM columns of the CTA's W_hh slice (16-bit elements, two per column)
__host__ __device__ inline int w_tmem_cols(int H, int S, int NPL) { return NPL * (H / S) / 2; }
// The CTA's W_hh slice -> TMEM columns [wcol, wcol + w_tmem_cols): lane r =
// MMA row r (warp w writes lanes 32*(w%4)..), the K elements of plane p at
// columns p*KS/2 .. in order, the lower K index in the low 16 bits.  Warps
// w and w+4 split the planes (NPL = 2) or the K halves (NPL = 1).
__device__ __forceinline__ void load_w_tmem(const uint16_t* __restrict__ wg, size_t plane_elems, int H, int row0,
                                            int k0, int KS, int NPL, uint32_t tmem_w) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp >= 8) return;
  const int quarter = warp & 3, half = warp >> 2;
  const int row = row0 + quarter * 32 + lane;
  const int per = NPL * KS / 2;                   // elements this thread writes
  const int p = NPL == 2 ? half : 0;
  const int kb = NPL == 2 ? 0 : half * (KS / 2);  // first K element of this thread's part
  const uint16_t* src = wg + (size_t)p * plane_elems + (size_t)row * H + k0 + kb;
  const uint32_t col0 = (uint32_t)((p * KS + kb) / 2);
  for (int e = 0; e < per; e += 32) {             // 32 elements = 16 columns per store
    uint32_t r[16];
    const uint4* v = reinterpret_cast<const uint4*>(src + e);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint4 u = __ldg(v + j);
      r[4 * j] = u.x; r[4 * j + 1] = u.y; r[4 * j + 2] = u.z; r[4 * j + 3] = u.w;
    }
    ptx::tmem_st_32x32b_x16(tmem_w + ((uint32_t)(quarter * 32) << 16) + col0 + (uint32_t)(e / 2), r);
  }
  ptx::tmem_wait_st();
}
// timestep (row of xproj / y) of processing step `step` of direction d
__device__ __forceinline__ int seg_time(const TcRecurArgs& a, int d, int step) {
  const int Tf = a.T_full ? a.T_full : a.T;
  return ((d == 0) != (a.rev != 0)) ? a.s_base + step : Tf - 1 - a.s_base - step;
}
constexpr int kL2HintW = 1, kL2HintStream = 2;

// Block until the K1 tiles holding timestep tt's rows of xproj are stored.
// In the time loop ONE lane of an epilogue-only warp does this for step s+1
// while step s waits for its partial sums; the group / CTA barrier before the
// h release then orders every thread's XP prefetch after that acquire, so
// neither the producer nor the MMA warp ever waits on it.
__device__ __forceinline__ void wait_xready(const TcRecurArgs& a, int tt) {
  if (!a.xready) return;
  const int lo = (tt * a.Bst) / 128, hi = (tt * a.Bst + a.Bst - 1) / 128;
  for (int mt = lo; mt <= hi; ++mt) wait_geq(a.xready + mt, a.xready_target, kWatchRecurXready);
}
constexpr int kCtrStrideWords = 32;  // chunk readiness counters: one 128-B line each

// The h_{t-1} all-gather of one step: lane c of the producer warp polls the
// readiness counter of chunk c of this CTA's K-slice and, once it is
// published, issues that chunk's TMA load itself (`issue(c)`).  All chunks are
// polled in one round trip — polling them one after another from one lane
// cost a serial L2 round trip per chunk (c3 at S=2, 4 chunks: 1.5 us of the
// 5.1 us step; c2's 4 chunks: 1.2 us).  The MMA warp still consumes the
// chunks in order, so the accumulation order is unchanged.  Whole warp.
template <typename Issue>
__device__ __forceinline__ void poll_chunks(const unsigned int* in_counter, int nch, unsigned int target, Issue&& issue) {
  const int lane = threadIdx.x & 31;
  const unsigned int all = nch >= 32 ? 0xffffffffu : (1u << nch) - 1u;
  unsigned int done = 0u;
  Spin sp;
  while (done != all) {
    bool ok = false;
    if (lane < nch && !((done >> lane) & 1u)) {
      unsigned int v;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(in_counter + lane * kCtrStrideWords) : "memory");
      if (v >= target) {
        ok = true;
        issue(lane);
      }
    }
    const unsigned int ready = __ballot_sync(0xffffffffu, ok);
    if (!ready) sp.tick(kWatchRecurChunk);
    done |= ready;
  }
}

__device__ __forceinline__ void signal_started(const TcRecurArgs& a) {
  if (a.started && threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(a.started) : "memory");
}

constexpr int kTraceSteps = 64;
constexpr int kTraceCtas = 320;  // CTAs with a trace slot (the 2-CTA/SM wave runs up to 296)

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define HS_TRACE_AT(phase)                                                                       \
  do {                                                                                           \
    if (a.trace && s < kTraceSteps && blockIdx.x < kTraceCtas)                                   \
      a.trace[((size_t)blockIdx.x * kTraceSteps + s) * 16 + (phase)] = globaltimer();             \
  } while (0)
// HS_TRACE_CHUNKS (diagnostic variant build, tools/trace_chunks.py): the MMA
// issuer first waits for every h chunk of the step in order, recording when
// each landed (slots 0..13), then times the W-streaming variant's TMEM-chunk
// MMAs alone into a scratch accumulator (slot 14); no phase stamps
#ifdef HS_TRACE_CHUNKS
#define HS_TRACE(phase) do { } while (0)
#else
#define HS_TRACE(phase) HS_TRACE_AT(phase)
#endif

constexpr int kMaxSW = 8;  // W-streaming ring depth limit

struct RecurLayout {
  int nch;        // K chunks per CTA
  size_t w_off, h_off, red_off, stage_off, bar_off, total;
};

// nsw = 0: the CTA's W_hh slice is resident in shared memory (NPL planes x
// nch chunks); nsw = kTmemW: resident in tensor memory, no shared-memory copy;
// nsw > 0: W_hh does not fit on chip and streams through an nsw-stage ring of
// [NPL planes x 128 rows x 64 k] chunks, re-read from L2 every step.
constexpr int kTmemW = -1;
__host__ __device__ inline RecurLayout recur_layout(int G, int H, int Npad, int S, int NPL, int nsw = 0) {
  RecurLayout L;
  const int KS = H / S;
  L.nch = KS / 64;
  size_t off = 0;
  L.w_off = off;   off += nsw < 0 ? 0 : (size_t)NPL * (nsw ? nsw : L.nch) * 128 * 128;
  L.h_off = off;   off += (size_t)L.nch * Npad * 128;  // one h plane
  L.red_off = off; off += (size_t)G * 32 * (Npad + 4) * 4;
  // outgoing partials for the S-1 peers, laid out like their destination regions
  L.stage_off = off; off += (size_t)(S - 1) * G * (32 / S) * (Npad + 4) * 4;
  off = (off + 15) / 16 * 16;
  L.bar_off = off; off += 8 * (5 + RMAXCH + 1 + 2 * kMaxSW) + 16;
  L.total = off;  // dynamic smem starts 1024-aligned (checked in-kernel)
  return L;
}

__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
// arrive without release: used once this CTA's reads of the partial-sum
// buffer have completed (their values are already consumed in registers)
__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// One CTA = 8 warps.  Roles inside a timestep:
//   warp 0 lane 0  producer: polls the per-chunk readiness counters of its
//                  K-slice in order and TMA-loads each h chunk once published
//   warp 1 lane 0  MMA issuer: tcgen05.mma per landed chunk, commit -> acc_full
//   warp 2         TMEM allocator
//   all 8 warps    drain TMEM (warp w reads lane quarter w%4; warps w, w+4
//                  split the columns), reduce-scatter partial gates to the unit
//                  owners over DSMEM, cluster barrier, then finish the gates of
//                  the CTA's own units (c, h in registers), publish h_t planes
//                  and release the chunk counter.
constexpr int kRecurThreads = 256;  // + one W-producer warp in the streaming variant
constexpr int kEpiThreads = 256;

using ptx::idesc_f16_f32;  // tcgen05 instruction descriptor, kind::f16 with fp16 A/B and f32 D

// The streamed h_{t-1} MMA operand.  f32 mode (NPL = 2 W_hh planes): fp16,
// 11 significant bits, exact range for |h| < 1; W_hh is carried as fp16
// hi + lo (~22 bits), so gates = W_hi·h + W_lo·h in two passes with fp32
// accumulation (max-abs vs the float64 oracle <= 1.5e-5 on the BASELINE
// configs, budget 1e-4).  bf16 mode: bf16.
template <int NPL>
__device__ __forceinline__ uint16_t h_operand(float h) {
  if (NPL == 2) return __half_as_ushort(__float2half_rn(h));
  return __bfloat16_as_ushort(__float2bfloat16_rn(h));
}

// The kernel body: one row-block cluster `cl` of one recurrence (a layer,
// both directions).  recur_tc_kernel runs one layer per launch;
// recur_tc_wave_kernel runs several unidirectional layers side by side.
template <int G, int NPL, int CELLS, int NSW>
__device__ __forceinline__ void recur_tc_body(const CUtensorMap& tmW0, const CUtensorMap& tmW1, const CUtensorMap& tmH,
                                              const TcRecurArgs& a, const int cl, uint8_t* smem_raw) {
  uint8_t* smem = smem_raw;
  if (ptx::smem_u32(smem_raw) & 1023) __trap();  // SW128 atoms need 1024-B alignment
  signal_started(a);
  const int H = a.H, B = a.B, Npad = a.Npad, T = a.T, D = a.D, S = a.S, RB = a.RB;
  const RecurLayout L = recur_layout(G, H, Npad, S, NPL, NSW == 0 && a.w_tmem ? kTmemW : NSW);
  const int nch = L.nch;
  const int KS = H / S;
  const int UO = 32 / S;  // units finished by each rank
  __nv_bfloat16* sW = reinterpret_cast<__nv_bfloat16*>(smem + L.w_off);
  __nv_bfloat16* sH = reinterpret_cast<__nv_bfloat16*>(smem + L.h_off);
  float* red = reinterpret_cast<float*>(smem + L.red_off);
  float* stage = reinterpret_cast<float*>(smem + L.stage_off);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bar_off);
  uint64_t* w_full = bars;
  uint64_t* acc_full = bars + 1;
  uint64_t* red_full = bars + 2;   // 8 local warps + the owner's expect_tx for the peers' bulk copies
  uint64_t* red_free = bars + 3;   // S ranks x 8 owner warps finished reading the partials
  uint64_t* tmem_free = bars + 4;  // 8 warps drained the accumulator
  uint64_t* h_full = bars + 5;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 5 + RMAXCH);
  uint64_t* wfull = bars + 5 + RMAXCH + 1;   // streaming ring (NSW > 0)
  uint64_t* wempty = wfull + kMaxSW;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = (int)ptx::cluster_rank();
  const int d = cl / RB;
  const int rb = cl % RB;
  const CUtensorMap* tmW = d == 0 ? &tmW0 : &tmW1;
  const int GH = G * H;
  const int rstride = Npad + 4;
  const uint32_t tcols_acc = Npad <= 32 ? 32 : Npad <= 64 ? 64 : Npad <= 128 ? 128 : 256;
  // W_hh in TMEM (a.w_tmem, resident variant only): columns [256, 256 + NPL*KS/2)
  const bool wt = NSW == 0 && a.w_tmem;
  const uint32_t wcol = 256u;
  // W-streaming variant: the first `nres` chunks (both planes) stay in TMEM
  // after the accumulator, only the rest cross the ring each step
  const int nres = NSW ? a.w_tmem_chunks : 0;
  const uint32_t tcols = (wt || nres) ? 512u : tcols_acc;
  // readiness counters, one per 64-unit chunk of h (= 2 row blocks = 2S producer
  // CTAs), each on its own 128-B line
  constexpr int kCtrStride = kCtrStrideWords;
  const int nchunk_all = H / 64;
  unsigned int* my_counter = a.counters + (d * nchunk_all + (rb * 32) / 64) * kCtrStride;
  const unsigned int* in_counter = a.counters + (d * nchunk_all + (q * KS) / 64) * kCtrStride;
  const unsigned int per_round = 2u * (unsigned int)S;
  const size_t plane_stride = (size_t)Npad * H;  // elements per (buf, d) slab of hbuf

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch(tmW);
    ptx::tma_prefetch(&tmH);
    ptx::mbar_init(w_full, 1);
    ptx::mbar_init(acc_full, 1);
    for (int c = 0; c < nch; ++c) ptx::mbar_init(&h_full[c], 1);
    for (int i = 0; i < NSW; ++i) {
      ptx::mbar_init(&wfull[i], 1);
      ptx::mbar_init(&wempty[i], 1);
    }
#ifdef HS_TRACE_CHUNKS
    if (NSW < kMaxSW) ptx::mbar_init(&wfull[kMaxSW - 1], 1);
#endif
    ptx::mbar_init(red_full, 9);
    ptx::mbar_init(red_free, (uint32_t)(S * 8));
    ptx::mbar_init(tmem_free, 8);
    ptx::fence_mbar_init();
    ptx::mbar_arrive_expect_tx(red_full, (uint32_t)((S - 1) * G * UO * (Npad + 4) * 4));  // phase 0
  }
  if (warp == 2) ptx::tmem_alloc_dyn(tmem_slot, tcols);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // resident W_hh slice: NPL planes x nch chunks of [128 rows x 64 k]
  if (wt) {
    load_w_tmem(a.whh_g[d], (size_t)RB * 128 * H, H, rb * 128, q * KS, KS, NPL, tmem + wcol);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
  } else if (NSW == 0 && warp == 0 && ptx::elect_one()) {
    ptx::mbar_arrive_expect_tx(w_full, (uint32_t)(NPL * nch * 128 * 128));
    for (int p = 0; p < NPL; ++p)
      for (int c = 0; c < nch; ++c)
        ptx::tma_load_3d(sW + ((size_t)p * nch + c) * 128 * 64, tmW, w_full, q * KS + c * 64, rb * 128, p);
  }
  __syncwarp();

  if (nres) {  // resident part of the streamed slice: chunk c plane p at column tcols_acc + (c*NPL + p)*32
    const int quarter = warp & 3, half = warp >> 2, row = rb * 128 + quarter * 32 + lane;
    if (warp < 8) {
      for (int i = half; i < nres * NPL; i += 2) {
        const int c = i / NPL, p = i % NPL;
        const uint16_t* src = a.whh_g[d] + (size_t)p * RB * 128 * H + (size_t)row * H + q * KS + c * 64;
        for (int e = 0; e < 64; e += 32) {
          uint32_t r[16];
          const uint4* v = reinterpret_cast<const uint4*>(src + e);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint4 u = __ldg(v + j);
            r[4 * j] = u.x; r[4 * j + 1] = u.y; r[4 * j + 2] = u.z; r[4 * j + 3] = u.w;
          }
          ptx::tmem_st_32x32b_x16(tmem + ((uint32_t)(quarter * 32) << 16) + tcols_acc + (uint32_t)(i * 32 + e / 2), r);
        }
      }
      ptx::tmem_wait_st();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
  }
  // streaming variant: warp 8 keeps the W ring NSW chunks ahead of the MMAs.
  // Ring item gi = s*nstream + (c - nres) holds streamed chunk c (the same
  // weights every step).
  const int nstream = nch - nres;
  const int total_items = T * nstream;
  int w_next = 0;  // next ring item to load (warp 8 lane 0)
  const uint64_t pol_w = ptx::policy_evict_last();
  const uint64_t pol_s = ptx::policy_evict_first();
  const bool hint_s = (a.l2_hints & kL2HintStream) != 0;
  auto w_produce_until = [&](int last_item) {
    for (; w_next <= last_item && w_next < total_items; ++w_next) {
      const int slot = w_next % NSW, c = nres + w_next % nstream;
      if (w_next >= NSW) ptx::mbar_wait(&wempty[slot], ((w_next / NSW) - 1) & 1);
      ptx::mbar_arrive_expect_tx(&wfull[slot], (uint32_t)(NPL * 128 * 128));
      for (int p = 0; p < NPL; ++p) {
        if (a.l2_hints & kL2HintW)
          ptx::tma_load_3d_hint(sW + ((size_t)slot * NPL + p) * 128 * 64, tmW, &wfull[slot], q * KS + c * 64, rb * 128,
                                p, pol_w);
        else
          ptx::tma_load_3d(sW + ((size_t)slot * NPL + p) * 128 * 64, tmW, &wfull[slot], q * KS + c * 64, rb * 128, p);
      }
    }
  };

  // owner cells: unit u_loc in [0, UO), batch rows b = b0 + k*bstep, k < CELLS
  // (threads of the W-producer warp own no cells)
  const int e = threadIdx.x;
  const bool owner = e < kEpiThreads;
  const int u_loc = e % UO;
  const int b0 = owner ? e / UO : (1 << 20);  // non-owners: every row index out of range
  const int bstep = kEpiThreads / UO;
  const int unit = rb * 32 + q * UO + u_loc;
  float c_reg[CELLS], h_reg[CELLS], xq[CELLS][G];
  float wsc[G];  // undo the per-row power-of-two W_hh scaling (exact)
#pragma unroll
  for (int g = 0; g < G; ++g) wsc[g] = a.whh_scale[d][rb * 128 + g * 32 + q * UO + u_loc];
  float bias_r = 0.f, bias_z = 0.f, bias_n = 0.f;
  if (G == 3 && a.bias_h[d]) {
    bias_r = a.bias_h[d][unit];
    bias_z = a.bias_h[d][H + unit];
    bias_n = a.bias_h[d][2 * H + unit];
  }
  auto load_xproj = [&](int step, bool poll) {
    const int tt = seg_time(a, d, step);
    if (poll) wait_xready(a, tt);
    const float* __restrict__ xp = a.xproj[d] + (size_t)tt * a.Bst * GH + unit;
#pragma unroll
    for (int k = 0; k < CELLS; ++k) {
      const int b = b0 + k * bstep;
#pragma unroll
      for (int g = 0; g < G; ++g) xq[k][g] = b < B ? (hint_s ? ptx::ldcg_hint(xp + (size_t)b * GH + g * H, pol_s)
                                                                 : __ldcg(xp + (size_t)b * GH + g * H))
                                   : 0.f;  // may be written by a running K1
    }
  };
#pragma unroll
  for (int k = 0; k < CELLS; ++k) {
    c_reg[k] = 0.f;
    h_reg[k] = 0.f;
    const int b = b0 + k * bstep;
    if (b < B) {
      h_reg[k] = a.h0[d][(size_t)b * H + unit];
      if (G == 4) c_reg[k] = a.c0[d][(size_t)b * H + unit];
      a.hbuf[(size_t)(0 * D + d) * plane_stride + (size_t)b * H + unit] = h_operand<NPL>(h_reg[k]);
    }
  }
  ptx::fence_proxy_async_global();
  load_xproj(0, true);
  __syncthreads();
  if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(my_counter) : "memory");
  cluster_arrive();  // every CTA's barriers initialised before any remote op
  cluster_wait();
  const bool stamper = a.stamps && rb == 0 && q == 0 && threadIdx.x == 0;
  if (stamper) a.stamps[(size_t)d * (T + 1)] = globaltimer();

  // f32 mode: fp16 W hi/lo x fp16 h; bf16 mode: bf16 x bf16
  const uint32_t idesc = NPL == 2 ? idesc_f16_f32(128, Npad) : ptx::idesc_bf16_f32(128, Npad);
  const int sub = warp & 3;  // TMEM lane quarter
  const bool split = (Npad % 32) == 0;
  const int ncol = split ? Npad / 2 : Npad;
  const int col0 = split ? (warp >> 2) * ncol : 0;
  const bool active = warp < 8 && sub < G && (split || warp >= 4);
  const uint32_t region_floats = (uint32_t)(G * UO * rstride);  // one sender's rows in an owner's buffer
  const int dst_rank = lane / UO;
  // this lane's partial row: in my own buffer (dst == me) or in peer dst's staging slot
  float* part_row = dst_rank == q ? red + ((size_t)(q * G + sub) * UO + lane % UO) * rstride
                                  : stage + (size_t)(dst_rank < q ? dst_rank : dst_rank - 1) * region_floats +
                                        ((size_t)sub * UO + lane % UO) * rstride;

  for (int s = 0; s < T; ++s) {
    const int t = seg_time(a, d, s);
    const int buf_in = s % 3, buf_out = (s + 1) % 3;
    const bool last = s == T - 1;
    if (warp == 0) {
      if (lane == 0) HS_TRACE(0);
      poll_chunks(in_counter, nch, per_round * (unsigned int)(s + 1), [&](int c) {
        if (c == 0) HS_TRACE(1);
        if (c == nch - 1) HS_TRACE(12);
        ptx::fence_proxy_async_global();
        ptx::mbar_arrive_expect_tx(&h_full[c], (uint32_t)(Npad * 128));
        ptx::tma_load_3d(sH + (size_t)c * Npad * 64, &tmH, &h_full[c], q * KS + c * 64, 0, buf_in * D + d);
        if (c == nch - 1) HS_TRACE(13);
      });
      __syncwarp();
    } else if (NSW && warp == 8) {
      // keep the W ring NSW items ahead: this step's chunks, then the next step's first NSW
      if (lane == 0) w_produce_until((s + 1) * nstream + NSW - 1);
      __syncwarp();
    } else if (warp == 1) {
      if (ptx::elect_one()) {
        if (NSW == 0 && s == 0 && !wt) ptx::mbar_wait(w_full, 0);
        if (s > 0) ptx::mbar_wait(tmem_free, (s - 1) & 1);  // every warp drained step s-1
#ifdef HS_TRACE_CHUNKS
        for (int c = 0; c < nch; ++c) {
          ptx::mbar_wait(&h_full[c], s & 1);
          if (c < 14) HS_TRACE_AT(c);
        }
        if (nres && tcols_acc + (uint32_t)(nres * NPL * 32) + 32u <= 512u) {
          // the TMEM chunks' MMAs once more into a scratch accumulator (the
          // free columns after the resident W), back to back
          const uint32_t scratch = tmem + tcols_acc + (uint32_t)(nres * NPL * 32);
          ptx::tc_fence_after();
          for (int c = 0; c < nres; ++c) {
            const __nv_bfloat16* hh = sH + (size_t)c * Npad * 64;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint64_t bd = ptx::sdesc_k_sw128(hh + kk * 16);
              const uint32_t wc = tmem + tcols_acc + (uint32_t)(c * NPL * 32 + kk * 8);
              ptx::mma_bf16_ts(scratch, wc, bd, idesc, (c | kk) != 0);
              if (NPL == 2) ptx::mma_bf16_ts(scratch, wc + 32u, bd, idesc, 1);
            }
          }
          ptx::mma_commit(&wfull[kMaxSW - 1]);
          ptx::mbar_wait(&wfull[kMaxSW - 1], s & 1);
          HS_TRACE_AT(14);
        }
#endif
        for (int c = 0; c < nch; ++c) {
          const bool in_tmem = c < nres;  // W-streaming variant: resident chunk, no ring slot
          const int gi = s * nstream + (c - nres), wslot = NSW && !in_tmem ? gi % NSW : 0;
          if (NSW && !in_tmem) ptx::mbar_wait(&wfull[wslot], (gi / NSW) & 1);
          ptx::mbar_wait(&h_full[c], s & 1);
          ptx::tc_fence_after();
          if (c == 0) HS_TRACE(15);
          if (c == nch - 1) HS_TRACE(14);
          const __nv_bfloat16* wh = NSW ? sW + (size_t)wslot * NPL * 128 * 64 : sW + (size_t)c * 128 * 64;
          const __nv_bfloat16* hh = sH + (size_t)c * Npad * 64;
          if (wt) {  // A = W columns of (plane, chunk, kk) in TMEM: 8 columns per K=16
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint64_t bd = ptx::sdesc_k_sw128(hh + kk * 16);
              ptx::mma_bf16_ts(tmem, tmem + wcol + (uint32_t)(c * 32 + kk * 8), bd, idesc, (c | kk) != 0);
              if (NPL == 2) ptx::mma_bf16_ts(tmem, tmem + wcol + (uint32_t)(KS / 2 + c * 32 + kk * 8), bd, idesc, 1);
            }
          } else if (in_tmem) {  // resident chunk of the streamed slice
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint64_t bd = ptx::sdesc_k_sw128(hh + kk * 16);
              const uint32_t wc = tmem + tcols_acc + (uint32_t)(c * NPL * 32 + kk * 8);
              ptx::mma_bf16_ts(tmem, wc, bd, idesc, (c | kk) != 0);
              if (NPL == 2) ptx::mma_bf16_ts(tmem, wc + 32u, bd, idesc, 1);
            }
          } else {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              ptx::mma_bf16_ss(tmem, ptx::sdesc_k_sw128(wh + kk * 16), ptx::sdesc_k_sw128(hh + kk * 16), idesc,
                               (c | kk) != 0);
              if (NPL == 2) {  // + W_lo · h
                const __nv_bfloat16* wl = wh + (size_t)(NSW ? 1 : nch) * 128 * 64;
                ptx::mma_bf16_ss(tmem, ptx::sdesc_k_sw128(wl + kk * 16), ptx::sdesc_k_sw128(hh + kk * 16), idesc, 1);
              }
            }
          }
          if (NSW && !in_tmem) ptx::mma_commit(&wempty[wslot]);  // ring slot free once these MMAs have read it
        }
        ptx::mma_commit(acc_full);
        HS_TRACE(2);
      }
      __syncwarp();
    }
    // 1. drain TMEM into LOCAL shared memory (own rows -> my buffer, peers'
    //    rows -> staging); one thread then moves each peer's slice with a bulk
    //    copy whose complete_tx lands on the peer's red_full
    ptx::mbar_wait(acc_full, s & 1);
    ptx::tc_fence_after();
    if (e == 128) HS_TRACE(3);
    if (active) {
      for (int c16 = 0; c16 < ncol / 16; ++c16) {
        float v[16];
        const int col = col0 + c16 * 16;
        ptx::tmem_ld_32x32b_x16(tmem + ((uint32_t)(sub * 32) << 16) + col, v);
#pragma unroll
        for (int j = 0; j < 16; j += 4)
          *reinterpret_cast<float4*>(part_row + col + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      }
    }
    ptx::tc_fence_before();
    if (warp < 8) {
      ptx::fence_proxy_async_smem();  // staging writes -> the bulk copy (async proxy)
      __syncwarp();
      if (lane == 0) {
        ptx::mbar_arrive(tmem_free);
        ptx::mbar_arrive(red_full);  // my own rows are in place
      }
      ptx::named_bar(1, 256);  // staging complete
      if (e == 0) {
        if (s > 0) ptx::mbar_wait_cluster(red_free, (s - 1) & 1);  // peers read step s-1's partials
        for (int r = 0; r < S; ++r) {
          if (r == q) continue;
          const float* src = stage + (size_t)(r < q ? r : r - 1) * region_floats;
          const uint32_t dst = ptx::mapa(ptx::smem_u32(red + (size_t)q * region_floats), (uint32_t)r);
          ptx::bulk_s2cluster(dst, src, region_floats * 4u, ptx::mapa(ptx::smem_u32(red_full), (uint32_t)r));
        }
        ptx::bulk_commit();
        ptx::bulk_wait_read0();  // staging reusable
      }
    }
    if (e == 128) HS_TRACE(4);
    if (e == kEpiThreads - 32 && !last) {  // next step's XP (see wait_xready)
      HS_TRACE(7);
      wait_xready(a, seg_time(a, d, s + 1));
      HS_TRACE(9);
    }
    ptx::mbar_wait_cluster(red_full, s & 1);  // all partials for my units are in my shared memory
    if (e == 0 && !last)  // next phase: the peers' bulk copies of step s+1
      ptx::mbar_arrive_expect_tx(red_full, (uint32_t)((S - 1) * region_floats * 4));
    if (e == 128) HS_TRACE(5);
    // 2. owner: gates -> h_t planes (critical path)
#pragma unroll
    for (int k = 0; k < CELLS; ++k) {
      const int b = b0 + k * bstep;
      if (b >= Npad) break;
      float pre[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const float* rp = red + ((size_t)g * UO + u_loc) * rstride + b;
        float acc = rp[0];
#pragma unroll
        for (int sr = 1; sr < 8; ++sr)
          if (sr < S) acc += rp[(size_t)sr * G * UO * rstride];
        pre[g] = acc * wsc[g];
      }
      float h;
      if (G == 4) {
        const float ig = sigmoid_fast(pre[0] + xq[k][0]), fg = sigmoid_fast(pre[1] + xq[k][1]);
        const float gg = tanh_fast(pre[2] + xq[k][2]), og = sigmoid_fast(pre[3] + xq[k][3]);
        const float cnew = fg * c_reg[k] + ig * gg;
        c_reg[k] = cnew;
        h = og * tanh_fast(cnew);
      } else {
        const float r = sigmoid_fast(xq[k][0] + pre[0] + bias_r);
        const float z = sigmoid_fast(xq[k][1] + pre[1] + bias_z);
        const float n = tanh_fast(xq[k][2] + r * (pre[2] + bias_n));
        h = (1.f - z) * n + z * h_reg[k];
      }
      h_reg[k] = h;
      if (!last && b < B) {
        a.hbuf[(size_t)(buf_out * D + d) * plane_stride + (size_t)b * H + unit] = h_operand<NPL>(h);
      }
    }
    if (e == 128) HS_TRACE(6);
    if (warp < 8) {  // partials read (values consumed above): peers may refill the buffer
      __syncwarp();
      if (lane < S) ptx::mbar_arrive_remote_relaxed(ptx::mapa(ptx::smem_u32(red_free), (uint32_t)lane));
    }
    ptx::fence_proxy_async_global();
    __syncthreads();  // all h_t stores of this CTA issued
    if (e == 128) HS_TRACE(8);
    if (e == 0 && !last) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(my_counter) : "memory");
    if (stamper) a.stamps[(size_t)d * (T + 1) + s + 1] = globaltimer();
    // the barrier above also ordered every thread's y stores of step s-1:
    // publish them for the overlapped device->host copy (off the critical path)
    if (a.progress && e == kEpiThreads - 32 && s > 0)
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(a.progress + s - 1) : "memory");
    if (e == 0) HS_TRACE(10);
    // 3. off the critical path: layer outputs, final state, next step's XP
#pragma unroll
    for (int k = 0; k < CELLS; ++k) {
      const int b = b0 + k * bstep;
      if (b >= B) continue;
      const float hv = h_reg[k];
      const size_t yidx = ((size_t)t * a.Bst + b) * (a.ycols ? a.ycols : D * H) + (size_t)d * H + unit;
      if (a.y) {
        if (hint_s) ptx::st_hint(a.y + yidx, hv, pol_s);
        else a.y[yidx] = hv;
      }
      if (a.ypl) {
        if (a.ypl_f16) {  // a hidden layer's K1 input: fp16(h), the recurrence's own h operand
          reinterpret_cast<uint16_t*>(a.ypl)[yidx] = __half_as_ushort(__float2half_rn(hv));
        } else {
          __nv_bfloat16 hi, lo;
          ptx::split_bf16(hv, hi, lo);
          a.ypl[yidx] = hi;
          a.ypl[(size_t)T * a.Bst * D * H + yidx] = lo;
        }
      }
      if (last) {
        a.hn[d][(size_t)b * H + unit] = hv;
        if (G == 4) a.cn[d][(size_t)b * H + unit] = c_reg[k];
      }
    }
    if (!last) load_xproj(s + 1, false);  // ordered after warp 7's wait_xready by the barrier above
    if (e == 0) HS_TRACE(11);
  }
  cluster_arrive();  // no CTA leaves while peers may still copy into it / arrive on its barriers
  cluster_wait();
  ptx::tc_fence_before();
  __syncthreads();
  if (a.progress && e == kEpiThreads - 32)
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(a.progress + T - 1) : "memory");
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, tcols);
  }
}

template <int G, int NPL, int CELLS, int NSW>
__global__ void __launch_bounds__(kRecurThreads + 32, 1)
    recur_tc_kernel(const __grid_constant__ CUtensorMap tmW0, const __grid_constant__ CUtensorMap tmW1,
                    const __grid_constant__ CUtensorMap tmH, const TcRecurArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  recur_tc_body<G, NPL, CELLS, NSW>(tmW0, tmW1, tmH, a, (int)(blockIdx.x / a.S), smem_raw);
}

// Per-layer arguments of the single-GPU layer wavefront (tc_wave.cuh).
constexpr int kMaxWave = 8;
struct WaveMaps {
  CUtensorMap w[kMaxWave];  // per layer: W_hh planes
  CUtensorMap h[kMaxWave];  // per layer: h exchange planes
};
struct TcWaveArgs {
  TcRecurArgs layer[kMaxWave];  // D = 1 each
  int L;
  int RB;  // row-block clusters per layer
};

}  // namespace tc
}  // namespace hs
