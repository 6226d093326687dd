// Single-GPU layer wavefront: every layer's recurrence AND every layer's input
// projection in ONE cooperative launch.
//
// north_star (b): "layer l step t overlaps layer l+1 step t-1".  The cell
// DAG's edges are (l-1,t)->(l,t) and (l,t-1)->(l,t) (reference
// graph.py:207-228) and the reference executor starts a node as soon as its
// inputs have arrived (engine.py:359-372).  Layer-by-layer launches serialise
// the L recurrences (L·T dependent steps); here they run side by side, so the
// critical path is about T + (L-1)·lag steps.
//
//   CTAs [0, L·RB·S)          recurrences: layer l on row-block clusters
//                             [l·RB, (l+1)·RB), its W_hh slices resident in
//                             shared memory (recur_tc_body, tc_recur.cuh), its
//                             own h exchange planes, chunk counters and
//                             per-step progress counters
//   CTAs [L·RB·S, grid)       input projections (gemm_dyn_body, tc_gemm.cuh,
//                             wave mode): segment l = layer l's
//                             XP_l = W_ih^l · in_l + b.  in_0 = the x planes;
//                             in_l = layer l-1's output planes, a tile of which
//                             waits for layer l-1's progress counters.  Each
//                             stored tile bumps layer l's per-M-tile xready,
//                             which layer l's recurrence polls before step t.
//
// Forward progress: every CTA is resident at once (cooperative launch), every
// wait is on work with a smaller claim index or an earlier step (see
// GemmDynArgs), and every spin is watchdog-bounded (common.cuh).  Being one
// kernel, the schedule needs no concurrent-kernel probe and profiles under
// Nsight Compute and compute-sanitizer like any other launch.
//
// Shared memory: max(recurrence layout, K1 ring); one CTA per SM.
// Unidirectional layers only: a bidirectional layer's output at t depends on
// all of t..T-1, so the next layer cannot start early.
#pragma once
#include <mutex>
#include <set>
#include <utility>

#include "tc_gemm.cuh"
#include "tc_recur.cuh"

namespace hs {
namespace tc {

struct WaveArgs {
  TcWaveArgs rec;  // per-layer recurrence args (D = 1), L, RB
  int nrec;        // recurrence CTAs (L·RB·S); the rest of the grid runs K1
  int nk1;         // K1 CTAs that work (HS_WAVE_K1_CTAS experiments; the rest exit)
};

// PER_SM = CTAs per SM.  1: the recurrences at the K-split S whose slices fit
// one CTA per SM, the K1 on a 4-stage ring with double-buffered accumulators.
// 2 (twice the K-split, two CTAs per SM, the K1 on a 2-stage ring with one
// 256-column accumulator so any two CTAs share an SM's shared memory and
// TMEM) was measured and is not instantiated: c3 22.56k seqs/s at S=4 / two
// per SM vs 22.57k at S=2 / one per SM — the step is bound by the h
// exchange's round trips, not by the per-CTA slice.
template <int PER_SM>
struct WaveK1 {
  static constexpr int ST = PER_SM == 2 ? 2 : 4, NACC = PER_SM == 2 ? 1 : 2;
};

template <int G, int NPL, int CELLS, int PER_SM>
__global__ void __launch_bounds__(kRecurThreads, PER_SM)
    wave_fused_kernel(const __grid_constant__ WaveMaps rmaps, const __grid_constant__ WaveArgs wa,
                      const __grid_constant__ DynMaps gmaps, const __grid_constant__ GemmDynArgs ga) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if ((int)blockIdx.x < wa.nrec) {
    const int cl = (int)(blockIdx.x / wa.rec.layer[0].S);
    const int l = cl / wa.rec.RB;
    recur_tc_body<G, NPL, CELLS, 0>(rmaps.w[l], rmaps.w[l], rmaps.h[l], wa.rec.layer[l], cl - l * wa.rec.RB, smem_raw);
  } else if ((int)blockIdx.x < wa.nrec + wa.nk1) {
    gemm_dyn_body<WaveK1<PER_SM>::ST, WaveK1<PER_SM>::NACC>(gmaps, ga, smem_raw);
  }
}

// SMs' worth of CTAs the wave leaves to its K1 (at least).
constexpr int kWaveMinK1 = 16;
constexpr size_t kSmemPerSm = 233472;  // 228 KB per SM, 1 KB of it reserved per resident CTA

struct WavePlan {
  int S = 0;       // recurrence K-split (cluster size); 0 = no wave
  int per_sm = 1;  // CTAs per SM
};

inline size_t wave_k1_smem(int per_sm) { return per_sm == 2 ? gemm_d_smem_bytes<2>() : gemm_d_smem_bytes<4>(); }

inline size_t wave_smem(int G, int H, int B, int S, int NPL, int per_sm) {
  const size_t r = recur_layout(G, H, pad16(B), S, NPL, 0).total;
  const size_t k = wave_k1_smem(per_sm);
  return r > k ? r : k;
}

// Wave plan for this shape: every layer's W_hh slices resident at once,
// L·RB·S recurrence CTAs co-resident with >= kWaveMinK1 K1 CTAs.  `lim(S,
// per_sm)` = co-resident CTAs.  Prefers the larger K-split (shorter steps);
// on a tie, one CTA per SM.
template <typename Limit>
inline WavePlan choose_wave(int G, int H, int B, int L, int NPL, int GH, Limit lim) {
  WavePlan best;
  if (L < 2 || L > kMaxWave || GH % 256) return best;
  const int Npad = pad16(B);
  if (H % 64 || Npad > 256) return best;
  const int RB = H / 32;
  for (int per_sm = 1; per_sm <= 1; ++per_sm) {
    const size_t cap = kSmemPerSm / per_sm - 1024;
    for (int S = 1; S <= 8; S *= 2) {
      if (H % (64 * S)) continue;
      const RecurLayout Lo = recur_layout(G, H, Npad, S, NPL, 0);
      if (Lo.nch > RMAXCH || wave_smem(G, H, B, S, NPL, per_sm) > cap) continue;
      const int cells = (Npad + 8 * S - 1) / (8 * S);
      if (cells > (per_sm == 2 ? 2 : 4)) continue;  // instantiated owner cells per thread
      if (L * RB * S + kWaveMinK1 > lim(S, per_sm)) continue;
      if (S > best.S) best = WavePlan{S, per_sm};
    }
  }
  return best;
}
// Static co-residency estimate (the launch re-checks with the occupancy
// query): at two CTAs per SM a cluster of S packs onto S/2 SMs.
inline int static_wave_limit(int S, int per_sm) { return per_sm == 2 ? 2 * static_cta_limit(S > 1 ? S / 2 : 1) : static_cta_limit(S); }

// Co-resident CTAs of the fused kernel (occupancy query).
template <int G, int NPL, int PER_SM>
inline int wave_coresident_t(int S, size_t smem) {
  static bool init_d[kMaxDev] = {};
  bool& init = init_d[cur_device()];
  std::string err;
  if (!init) {
    if (set_smem(wave_fused_kernel<G, NPL, 1, PER_SM>, kSmemMax, err)) return 0;
    init = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(S * 16);
  cfg.blockDim = dim3(kRecurThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = S;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (occ_clusters(&n, wave_fused_kernel<G, NPL, 1, PER_SM>, cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n * S;
}
inline int wave_coresident(int G, int NPL, const WavePlan& p, size_t smem) {
  (void)p;
  if (G == 4) return NPL == 2 ? wave_coresident_t<4, 2, 1>(p.S, smem) : wave_coresident_t<4, 1, 1>(p.S, smem);
  return NPL == 2 ? wave_coresident_t<3, 2, 1>(p.S, smem) : wave_coresident_t<3, 1, 1>(p.S, smem);
}

// Launch the fused wave.  wa.rec.layer[l] carries each layer's recurrence
// args (D = 1, S and RB filled in here); whh[l] its W_hh planes; ga the wave-
// mode K1 args with apl[j] / a_pstride[j] / wih[j] segment j's operand planes
// (segment j = layer L - nseg + j; layers before it have their XP already).
// The grid is every co-resident CTA: L·RB·S recurrence CTAs, the rest K1.
inline int launch_wave(int G, int NPL, const WavePlan& p, const __nv_bfloat16* const* whh, WaveArgs& wa,
                       const __nv_bfloat16* const* apl, const size_t* a_pstride, const __nv_bfloat16* const* wih,
                       GemmDynArgs& ga, cudaStream_t s, std::string& err) {
  const int S = p.S;
  const int L = wa.rec.L;
  const TcRecurArgs& a0 = wa.rec.layer[0];
  const int H = a0.H, Npad = a0.Npad;
  const int RB = H / 32;
  wa.rec.RB = RB;
  wa.nrec = L * RB * S;
  WaveMaps rm;
  DynMaps gm;
  int rc = k1_mode_init(err);
  for (int l = 0; l < L && !rc; ++l) {
    TcRecurArgs& a = wa.rec.layer[l];
    a.S = S;
    a.RB = RB;
    set_w_tmem(a, &whh[l], S, NPL, 0);
    rc = make_map3(&rm.w[l], whh[l], H, (uint64_t)RB * 128, 2, 128, err);
    if (!rc) rc = make_map3(&rm.h[l], a.hbuf, H, Npad, 3, Npad, err);
  }
  for (int j = 0; j < ga.nseg && !rc; ++j) {  // K1 segments (apl / a_pstride / wih indexed by segment)
    rc = make_map3(&gm.a[j], apl[j], ga.wK[j], ga.M, 2, GBM, err, a_pstride[j]);
    if (!rc) rc = make_map3(&gm.b[j], wih[j], ga.wK[j], ga.N, 2, 256, err);
    ga.scale[j] = ga.wnpass[j] == 2 ? wih_scales(wih[j], ga.N, ga.wK[j]) : nullptr;  // pass scheme 2: row-scaled W_ih
  }
  if (rc) return rc;
  const size_t smem = wave_smem(G, H, a0.B, S, NPL, p.per_sm);
  const int cores = wave_coresident(G, NPL, p, smem);
  const int grid = cores / S * S;
  if (grid < wa.nrec + kWaveMinK1) {
    err = "layer wave needs " + std::to_string(wa.nrec + kWaveMinK1) + " co-resident CTAs, device fits " +
          std::to_string(cores);
    return 3;
  }
  static const char* cap_env = getenv("HS_WAVE_K1_CTAS");
  wa.nk1 = grid - wa.nrec;
  if (cap_env && atoi(cap_env) > 0 && atoi(cap_env) < wa.nk1) wa.nk1 = atoi(cap_env);
  int cells = 1;
  while (cells * (kEpiThreads / (32 / S)) < Npad) cells *= 2;
  auto launch = [&](auto kernel) -> int {
    // every instantiation shares this lambda (same function-pointer type), so
    // the one-time smem opt-in is keyed by the kernel itself and the device
    static std::mutex mu;
    static std::set<std::pair<const void*, int>> done;
    {
      std::lock_guard<std::mutex> lk(mu);
      const auto key = std::make_pair(reinterpret_cast<const void*>(kernel), cur_device());
      if (!done.count(key)) {
        const int rc2 = set_smem(kernel, kSmemMax, err);
        if (rc2) return rc2;
        done.insert(key);
      }
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kRecurThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = S;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeCooperative;  // the whole grid resident: waits between CTAs never starve
    attr[1].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = coop_launch() ? 2 : 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, rm, wa, gm, ga);
    if (e != cudaSuccess) {
      err = std::string("wave_fused_kernel launch: ") + cudaGetErrorString(e);
      return 2;
    }
    ++g_launch_count;
    return 0;
  };
  return dispatch_cells(G, NPL, cells, [&](auto g_, auto npl_, auto c_) -> int {
    constexpr int Gv = decltype(g_)::value, NPLv = decltype(npl_)::value, Cv = decltype(c_)::value;
    if constexpr (Cv > 4) {
      err = "layer wave supports at most 4 cells per thread";
      return 3;
    } else {
      return launch(wave_fused_kernel<Gv, NPLv, Cv, 1>);
    }
  }, err);
}

}  // namespace tc
}  // namespace hs
