// Host glue of the tensor-core path: feasibility, packed-weight layout,
// tensor maps, launches of K1 (tc_gemm.cuh) and K2/K3 (tc_recur.cuh).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <type_traits>

#include "simt_kernels.cuh"
#include "tc_gemm.cuh"
#include "tc_recur.cuh"
#include "tc_recur2.cuh"

namespace hs {
namespace tc {

constexpr size_t kSmemMax = 232448;  // 227 KB opt-in per block on sm_100

inline int pad16(int b) { return (b + 15) / 16 * 16; }

// Pick the K-split (cluster size) for the recurrence: the largest grid that
// still fits one CTA per SM, with the W_hh slice + h staging + partial-sum
// buffer inside 227 KB of shared memory.
// Co-resident CTA limits per cluster size when the device cannot be queried
// (cluster placement strands SMs: measured 15 clusters of 8 on a B200).
inline int static_cta_limit(int S) { return S <= 2 ? 148 : S == 4 ? 132 : 120; }

// W-streaming ring depth, used when the W_hh slices cannot stay resident
// (e.g. c4, H = 2048: 64 MiB of fp16 hi/lo planes per layer-direction).
constexpr int kSW = 4;

template <typename Limit>
inline int choose_split(int G, int H, int B, int D, int NPL, Limit max_ctas, int nsw = 0) {
  const int Npad = pad16(B);
  if (H % 64 || Npad > 256) return 0;
  const int RB = H / 32;
  int best = 0;
  for (int S = 1; S <= 8; S *= 2) {
    if (H % (64 * S)) continue;
    const RecurLayout L = recur_layout(G, H, Npad, S, NPL, nsw);
    if (L.nch > RMAXCH || L.total > kSmemMax) continue;
    // W_hh in TMEM: its NPL*KS/2 columns at column 256 beside an accumulator of <= 256
    if (nsw == kTmemW && (w_tmem_cols(H, S, NPL) > 256 || Npad > 256)) continue;
    if ((Npad + 8 * S - 1) / (8 * S) > RMAXCELLS) continue;
    // streaming and TMEM-resident variants: <= 4 cells per thread (8 spill: c5 at 96 rows ran 16.7 vs 7.5 us/step)
    if (nsw != 0 && (Npad + 8 * S - 1) / (8 * S) > 4) continue;
    if (D * RB * S > max_ctas(S)) continue;
    best = S;  // increasing S -> larger grid; keep the largest that fits
  }
  return best;
}

// Resident W_hh when possible — in shared memory, else in tensor memory (the
// shared-memory layout then holds no W, which fits c5's batch-64 bf16 slices
// and lets larger slices in) — else the W-streaming variant.
// *nsw = 0 (smem-resident), kTmemW (TMEM-resident) or the ring depth.
template <typename Limit>
inline int plan_split(int G, int H, int B, int D, int NPL, Limit max_ctas, int* nsw) {
  int S = choose_split(G, H, B, D, NPL, max_ctas, 0);
  *nsw = 0;
  if (!S) {
    S = choose_split(G, H, B, D, NPL, max_ctas, kTmemW);
    *nsw = S ? kTmemW : 0;
  }
  if (!S) {
    S = choose_split(G, H, B, D, NPL, max_ctas, kSW);
    *nsw = S ? kSW : 0;
  }
  return S;
}

// Batch slice of the recurrence: the largest equal split of B whose slice
// has a feasible K-split (slices run one after another; 0 = infeasible).
inline int batch_slice(int G, int H, int B, int D, int NPL) {
  for (int n = 1; n <= B; ++n) {
    const int Bs = (B + n - 1) / n;
    int nsw;
    if (Bs <= 256 && plan_split(G, H, Bs, D, NPL, static_cta_limit, &nsw) > 0) return Bs;
    if (Bs <= 16) break;
  }
  return 0;
}

inline bool supports(int G, int H, int B, int I0, int DH, int D = 1, int NPL = 2) {
  if (I0 % 64 || DH % 64 || (G * H) % 128 || H % 64) return false;
  return batch_slice(G, H, B, D, NPL) > 0;
}

inline bool profitable(int G, int H, int B, int T) { return H >= 256 && B >= 4 && (long)T * B >= 128; }

inline int gemm_bn(int N) {
  static const char* env = getenv("HS_GEMM_BN");  // experiments: force the N tile
  if (env) return atoi(env) == 128 || N % 256 ? 128 : 256;
  return N % 256 == 0 ? 256 : 128;
}

// packed planes per layer-direction:
//   W_ih [2][G*H][I] 16-bit hi/lo planes — bf16 for pass scheme 3 / 1 (layer
//        0, bf16 mode), fp16 of the row-scaled weights for scheme 2 (hidden
//        layers in f32 mode) — then their per-row inverse scales [G*H] f32
//        (ones for bf16 planes), padded to 256 B;
//   W_hh row-block packed [2][H/32*128][H] 16-bit planes, then their per-row
//        inverse scales [H/32*128] f32.
inline size_t wih_plane_elems(int G, int H, int I) { return (size_t)G * H * I; }
inline size_t whh_plane_elems(int H) { return (size_t)(H / 32) * 128 * H; }
inline size_t wih_scale_bytes(int N) { return ((size_t)N * 4 + 255) / 256 * 256; }
inline size_t packed_bytes(int G, int H, int I) {
  if (H % 32) return 0;
  return 2 * 2 * (wih_plane_elems(G, H, I) + whh_plane_elems(H)) + wih_scale_bytes(G * H) + 4 * (size_t)(H / 32) * 128;
}
// per-row inverse scales of the W_ih planes starting at `wih` ([2][N][K])
inline const float* wih_scales(const void* wih, int N, int K) {
  return reinterpret_cast<const float*>(static_cast<const unsigned char*>(wih) + 2 * 2 * (size_t)N * K);
}
// the W_hh planes of the layer whose W_ih planes start at `wih`
inline const __nv_bfloat16* whh_of(const __nv_bfloat16* wih, int G, int H, int I) {
  return reinterpret_cast<const __nv_bfloat16*>(reinterpret_cast<const unsigned char*>(wih) +
                                                2 * 2 * wih_plane_elems(G, H, I) + wih_scale_bytes(G * H));
}
inline float* whh_scales(void* packed_layer, int G, int H, int I) {
  return reinterpret_cast<float*>(static_cast<unsigned char*>(packed_layer) +
                                  2 * 2 * (wih_plane_elems(G, H, I) + whh_plane_elems(H)) + wih_scale_bytes(G * H));
}

__global__ void fill_ones_kernel(float* p, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = 1.f;
}

struct TcWs {
  size_t xpl, hbuf, counters, trace, progress, claim, xready, total;
};
inline TcWs tc_ws_layout(int G, int H, int B, int T, int D, int I0) {
  (void)G;
  TcWs w{};
  size_t off = 0;
  const size_t cols = (size_t)(I0 > D * H ? I0 : D * H);
  w.xpl = off;      off += ((2 * (size_t)T * B * cols * 2) + 255) / 256 * 256;
  w.hbuf = off;     off += ((3 * (size_t)D * 2 * pad16(B) * H * 2) + 255) / 256 * 256;
  w.counters = off; off += 128 * 128;  // <= 128 chunk counters, one 128-B line each
  w.trace = off;    off += (size_t)kTraceCtas * kTraceSteps * 16 * 8;
  w.progress = off; off += ((size_t)T * 4 + 255) / 256 * 256;  // per-step output counters (host-buffer forward)
  w.claim = off;    off += 512;  // tile claim counters of the dynamic K1 launches ([0], [32], [64]) + started ([96])
  w.xready = off;   off += (((size_t)T * B + 127) / 128 * 4 + 255) / 256 * 256;  // per-M-tile XP readiness
  w.total = off;
  return w;
}
inline size_t workspace_bytes(int G, int H, int B, int T, int D, int I0) {
  if (H % 64) return 0;
  return tc_ws_layout(G, H, B, T, D, I0).total;
}

// Per packed W_hh row: the power-of-two exponent e that brings the row's
// max |w| to ~2^14 before the fp16 split, so W_lo = fp16(w*2^e - W_hi) stays
// a normal fp16 (the tensor cores flush fp16 subnormals: unscaled, W_lo of
// |w| ~ 1/32 weights would vanish).  Stores 2^-e, which the recurrent
// epilogue applies to the gate pre-activation.  One warp per row.
__global__ void whh_row_scale_kernel(const float* __restrict__ w_hh, float* __restrict__ inv_scale, int G, int H) {
  const int rows = (H / 32) * 128;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  for (int r = warp; r < rows; r += (gridDim.x * blockDim.x) >> 5) {
    const int rb = r / 128, g = (r % 128) / 32, u = r % 32;
    float m = 0.f;
    if (g < G)
      for (int k = lane; k < H; k += 32) m = fmaxf(m, fabsf(w_hh[((size_t)g * H + rb * 32 + u) * H + k]));
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) {
      int e = 0;
      if (m > 0.f) {
        int ex;
        frexpf(m, &ex);  // m in [2^(ex-1), 2^ex)
        e = 14 - ex;
        e = e > 60 ? 60 : e < -60 ? -60 : e;
      }
      inv_scale[r] = ldexpf(1.f, -e);
    }
  }
}

// Per W_ih row (pass scheme 2): the same power-of-two scaling as W_hh's, so
// the fp16 lo plane stays normal.  One warp per row.
__global__ void wih_row_scale_kernel(const float* __restrict__ w_ih, float* __restrict__ inv_scale, int N, int K) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  for (int r = warp; r < N; r += (gridDim.x * blockDim.x) >> 5) {
    float m = 0.f;
    for (int k = lane; k < K; k += 32) m = fmaxf(m, fabsf(w_ih[(size_t)r * K + k]));
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) {
      int e = 0;
      if (m > 0.f) {
        int ex;
        frexpf(m, &ex);
        e = 14 - ex;
        e = e > 60 ? 60 : e < -60 ? -60 : e;
      }
      inv_scale[r] = ldexpf(1.f, -e);
    }
  }
}

// W_ih: bf16 hi/lo planes, or (wih_f16, pass scheme 2) fp16 hi/lo planes of
// the row-scaled weights.  W_hh: fp16 hi/lo planes of the row-scaled weights
// (f32 mode, whh_f16) or bf16 (bf16 mode uses plane 0 only), row-block packed.
__global__ void pack_tc_kernel(const float* __restrict__ w_ih, const float* __restrict__ w_hh,
                               __nv_bfloat16* __restrict__ wih_pl, __nv_bfloat16* __restrict__ whh_pl, int G, int H,
                               int I, int whh_f16, const float* __restrict__ inv_scale, int wih_f16,
                               const float* __restrict__ wih_inv_scale) {
  const size_t n_ih = (size_t)G * H * I;
  const size_t n_hh = (size_t)(H / 32) * 128 * H;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n_ih; i += stride) {
    if (wih_f16) {
      const float vs = w_ih[i] / wih_inv_scale[i / I];  // exact: power of two
      const __half hi = __float2half_rn(vs);
      const __half lo = __float2half_rn(vs - __half2float(hi));
      reinterpret_cast<uint16_t*>(wih_pl)[i] = __half_as_ushort(hi);
      reinterpret_cast<uint16_t*>(wih_pl)[n_ih + i] = __half_as_ushort(lo);
    } else {
      __nv_bfloat16 hi, lo;
      ptx::split_bf16(w_ih[i], hi, lo);
      wih_pl[i] = hi;
      wih_pl[n_ih + i] = lo;
    }
  }
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n_hh; i += stride) {
    const int k = (int)(i % H);
    const size_t r = i / H;
    const int rb = (int)(r / 128), g = (int)((r % 128) / 32), u = (int)(r % 32);
    const float v = g < G ? w_hh[((size_t)g * H + rb * 32 + u) * H + k] : 0.f;
    if (whh_f16) {
      const float vs = v / inv_scale[r];  // exact: power of two
      const __half hi = __float2half_rn(vs);
      const __half lo = __float2half_rn(vs - __half2float(hi));
      reinterpret_cast<uint16_t*>(whh_pl)[i] = __half_as_ushort(hi);
      reinterpret_cast<uint16_t*>(whh_pl)[n_hh + i] = __half_as_ushort(lo);
    } else {
      __nv_bfloat16 hi, lo;
      ptx::split_bf16(v, hi, lo);
      whh_pl[i] = hi;
      whh_pl[n_hh + i] = lo;
    }
  }
}

// wih_f16: pack W_ih for pass scheme 2 (a hidden layer's K1 in f32 mode)
inline int pack_layer(int G, int H, int I, const float* w_ih, const float* w_hh, unsigned char* dst, bool whh_f16,
                      bool wih_f16, cudaStream_t s, std::string& err) {
  __nv_bfloat16* wih = reinterpret_cast<__nv_bfloat16*>(dst);
  __nv_bfloat16* whh = const_cast<__nv_bfloat16*>(whh_of(wih, G, H, I));
  float* inv_scale = whh_scales(dst, G, H, I);
  float* wih_inv = const_cast<float*>(wih_scales(wih, G * H, I));
  whh_row_scale_kernel<<<148, 256, 0, s>>>(w_hh, inv_scale, G, H);
  if (!whh_f16) {  // bf16 mode: unscaled
    fill_ones_kernel<<<16, 256, 0, s>>>(inv_scale, (H / 32) * 128);
  }
  if (wih_f16) wih_row_scale_kernel<<<148, 256, 0, s>>>(w_ih, wih_inv, G * H, I);
  else fill_ones_kernel<<<16, 256, 0, s>>>(wih_inv, G * H);
  pack_tc_kernel<<<592, 256, 0, s>>>(w_ih, w_hh, wih, whh, G, H, I, whh_f16 ? 1 : 0, inv_scale, wih_f16 ? 1 : 0,
                                     wih_inv);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    err = std::string("pack_tc_kernel: ") + cudaGetErrorString(e);
    return 2;
  }
  return 0;
}

// ------------------------------------------------------------ tensor maps
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 3D bf16 map {inner, rows, planes}, 128B swizzle, box {64, box_rows, 1};
// planes are `pstride` elements apart (0: inner*rows, i.e. dense).
inline int make_map3(CUtensorMap* map, const void* base, uint64_t inner, uint64_t rows, uint64_t planes, uint32_t box_rows,
                     std::string& err, uint64_t pstride = 0) {
  // memoised: a forward encodes ~10 maps over the same few buffers every call
  // (~1-3 us of host time each, on the enqueue path of every layer)
  struct Entry {
    const void* base;
    uint64_t inner, rows, planes, pstride;
    uint32_t box_rows;
    CUtensorMap map;
  };
  static thread_local Entry cache[32];
  static thread_local int next = 0;
  for (const Entry& e : cache)
    if (e.base == base && e.inner == inner && e.rows == rows && e.planes == planes && e.pstride == pstride &&
        e.box_rows == box_rows && base) {
      *map = e.map;
      return 0;
    }
  EncodeTiledFn fn = encode_fn();
  if (!fn) {
    err = "cuTensorMapEncodeTiled unavailable";
    return 2;
  }
  cuuint64_t dims[3] = {inner, rows, planes};
  cuuint64_t strides[2] = {inner * 2, (pstride ? pstride : inner * rows) * 2};
  cuuint32_t box[3] = {64, box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    err = "cuTensorMapEncodeTiled failed with CUresult " + std::to_string((int)r);
    return 2;
  }
  Entry& e = cache[next];
  next = (next + 1) % 32;
  e = Entry{base, inner, rows, planes, pstride, box_rows, *map};
  return 0;
}

template <typename K>
inline int set_smem(K kernel, size_t bytes, std::string& err) {
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) {
    err = std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e);
    return 2;
  }
  return 0;
}

// HS_K1_FUSED3=0 (A/B): the f32-mode K1 runs its three products pass-major
// (three sweeps over K re-loading X_hi / W_hi) instead of fused per K-block.
// The flag lives in each device's module constant; set once per device.
inline int k1_mode_init(std::string& err) {
  static const char* env = getenv("HS_K1_FUSED3");
  if (!env || atoi(env) != 0) return 0;
  static bool done_d[kMaxDev] = {};
  bool& done = done_d[cur_device()];
  if (!done) {
    const int zero = 0;
    cudaError_t e = cudaMemcpyToSymbol(c_k1_fused3, &zero, sizeof zero);
    if (e != cudaSuccess) {
      err = std::string("k1_mode_init: ") + cudaGetErrorString(e);
      return 2;
    }
    done = true;
  }
  return 0;
}

// K1 on planes: A planes [2][M][K], W_ih planes [2][N][K]
// (a_pstride: element distance between the A hi and lo planes; 0 = M*K)
// persistent = false: one CTA per tile.  Required when the launch shares the
// GPU with a running persistent recurrence: a persistent GEMM's tile lists are
// fixed per CTA, so its CTAs queued behind the recurrence would hold back their
// tiles until the recurrence ends; one-tile CTAs trickle onto the free SMs.
inline int gemm_planes(const __nv_bfloat16* apl, const __nv_bfloat16* wpl, const float* bias, float* C, int M, int N, int K,
                       int npass, cudaStream_t s, std::string& err, size_t a_pstride = 0, bool persistent = true) {
  CUtensorMap ta, tb;
  const int BN = gemm_bn(N);
  int rc = k1_mode_init(err);
  if (!rc) rc = make_map3(&ta, apl, K, M, 2, GBM, err, a_pstride);
  if (!rc) rc = make_map3(&tb, wpl, K, N, 2, BN, err);
  if (rc) return rc;
  dim3 grid(N / BN, (M + GBM - 1) / GBM);
  const float* scale = npass == 2 ? wih_scales(wpl, N, K) : nullptr;  // pass scheme 2: row-scaled W_ih
  cudaError_t e;
  static const char* np_env = getenv("HS_GEMM_NONPERSISTENT");  // A/B runs
  if (BN == 256 && persistent && !np_env) {
    static bool initp_d[kMaxDev] = {};
    static int sms_d[kMaxDev] = {};
    const int dev = cur_device();
    if (!initp_d[dev]) {
      if ((rc = set_smem(gemm_xproj_persistent, gemm_p_smem_bytes(), err))) return rc;
      cudaDeviceGetAttribute(&sms_d[dev], cudaDevAttrMultiProcessorCount, dev);
      initp_d[dev] = true;
    }
    const int sms = sms_d[dev];
    const int tiles = (int)(grid.x * grid.y);
    gemm_xproj_persistent<<<tiles < sms ? tiles : sms, 256, gemm_p_smem_bytes(), s>>>(ta, tb, bias, scale, C, M, N, K, npass);
  } else if (BN == 256) {
    static bool init_d[kMaxDev] = {};
  bool& init = init_d[cur_device()];
    if (!init) { if ((rc = set_smem(gemm_xproj_kernel<256>, gemm_smem_bytes<256>(), err))) return rc; init = true; }
    gemm_xproj_kernel<256><<<grid, 256, gemm_smem_bytes<256>(), s>>>(ta, tb, bias, scale, C, M, N, K, npass);
  } else {
    static bool init_d[kMaxDev] = {};
  bool& init = init_d[cur_device()];
    if (!init) { if ((rc = set_smem(gemm_xproj_kernel<128>, gemm_smem_bytes<128>(), err))) return rc; init = true; }
    gemm_xproj_kernel<128><<<grid, 256, gemm_smem_bytes<128>(), s>>>(ta, tb, bias, scale, C, M, N, K, npass);
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) {
    err = std::string("gemm_xproj_kernel launch: ") + cudaGetErrorString(e);
    return 2;
  }
  ++g_launch_count;
  return 0;
}

// Overlapped K1 of the next layer (gemm_xproj_dyn): one CTA per SM on stream
// s, launched once the recurrence is resident; *claim must be zeroed before.
inline int gemm_dyn_preload(std::string& err) {  // loads the module (lazy loading) + smem opt-in, once
  static bool init_d[kMaxDev] = {};
  bool& init = init_d[cur_device()];
  if (!init) {
    int rc = set_smem(gemm_xproj_dyn, gemm_d_smem_bytes(), err);
    if (rc) return rc;
    init = true;
  }
  return 0;
}

inline int gemm_planes_dyn(const __nv_bfloat16* apl, size_t a_pstride, const __nv_bfloat16* const* wpl,
                           const GemmDynArgs& ga, int grid, cudaStream_t s, std::string& err) {
  DynMaps mp;
  int rc = k1_mode_init(err);
  if (!rc) rc = make_map3(&mp.a[0], apl, ga.K, ga.M, 2, GBM, err, a_pstride);
  for (int d = 0; d < ga.D && !rc; ++d) rc = make_map3(&mp.b[d], wpl[d], ga.K, ga.N, 2, 256, err);
  if (rc) return rc;
  if ((rc = gemm_dyn_preload(err))) return rc;
  GemmDynArgs g = ga;
  for (int d = 0; d < ga.D; ++d) g.scale[d] = ga.npass == 2 ? wih_scales(wpl[d], ga.N, ga.K) : nullptr;
  gemm_xproj_dyn<<<grid, 256, gemm_d_smem_bytes(), s>>>(mp, g);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    err = std::string("gemm_xproj_dyn launch: ") + cudaGetErrorString(e);
    return 2;
  }
  ++g_launch_count;
  return 0;
}

// Wave-mode K1 (GemmDynArgs::nseg > 0): segment j projects layer j's output
// planes apl[j] ([2][M][K], hi/lo `a_pstride` apart) with layer j+1's W_ih
// planes wpl[j].  ga.bias/C/wprogress/wncta/wxready are filled per segment.
inline int gemm_planes_wave(const __nv_bfloat16* const* apl, size_t a_pstride, const __nv_bfloat16* const* wpl,
                            const GemmDynArgs& ga, int grid, cudaStream_t s, std::string& err) {
  DynMaps mp;
  int rc = k1_mode_init(err);
  for (int j = 0; j < ga.nseg && !rc; ++j) {
    rc = make_map3(&mp.a[j], apl[j], ga.K, ga.M, 2, GBM, err, a_pstride);
    if (!rc) rc = make_map3(&mp.b[j], wpl[j], ga.K, ga.N, 2, 256, err);
  }
  if (rc) return rc;
  if ((rc = gemm_dyn_preload(err))) return rc;
  GemmDynArgs g = ga;
  for (int j = 0; j < ga.nseg; ++j) g.scale[j] = g.wnpass[j] == 2 ? wih_scales(wpl[j], ga.N, ga.K) : nullptr;
  gemm_xproj_dyn<<<grid, 256, gemm_d_smem_bytes(), s>>>(mp, g);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    err = std::string("gemm_xproj_dyn (wave) launch: ") + cudaGetErrorString(e);
    return 2;
  }
  ++g_launch_count;
  return 0;
}

// f16: pass scheme 2's single fp16 plane (hidden-state inputs); else bf16 hi/lo
inline int split_planes(const float* x, __nv_bfloat16* out, size_t rows, int cols, bool f16, cudaStream_t s,
                        std::string& err, size_t pstride = 0) {
  const size_t total = rows * cols;
  int blocks = (int)((total / 4 + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  split_planes_kernel<<<blocks, 256, 0, s>>>(x, out, rows, cols, cols, pstride, f16 ? 1 : 0);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    err = std::string("split_planes_kernel: ") + cudaGetErrorString(e);
    return 2;
  }
  ++g_launch_count;
  return 0;
}

// cudaOccupancyMaxActiveClusters, memoised per (kernel, device, smem, block,
// cluster): the query costs ~10 us of host time and sits on the launch path of
// every layer (the first layer's K1 head waited ~36 us for the host at c2)
template <typename K>
inline cudaError_t occ_clusters(int* n, K kernel, const cudaLaunchConfig_t& cfg) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, size_t, unsigned, unsigned>, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(reinterpret_cast<const void*>(kernel), dev, cfg.dynamicSmemBytes, cfg.blockDim.x,
                                   cfg.attrs[0].val.clusterDim.x);
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      *n = it->second;
      return cudaSuccess;
    }
  }
  const cudaError_t e = cudaOccupancyMaxActiveClusters(n, kernel, &cfg);
  if (e == cudaSuccess) {
    std::lock_guard<std::mutex> lk(mu);
    cache[key] = *n;
  }
  return e;
}

template <int G, int NPL>
inline int max_coresident_ctas_t(int S, size_t smem) {
  static bool init_d[kMaxDev] = {};
  bool& init = init_d[cur_device()];
  std::string err;
  if (!init) {
    if (set_smem(recur_tc_kernel<G, NPL, 1, 0>, kSmemMax, err)) return 0;
    init = true;
  }
  if (smem > kSmemMax) return 0;
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
  if (occ_clusters(&n, recur_tc_kernel<G, NPL, 1, 0>, cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n * S;
}

inline int max_coresident_ctas(int G, int NPL, int S, size_t smem) {
  if (G == 4) return NPL == 2 ? max_coresident_ctas_t<4, 2>(S, smem) : max_coresident_ctas_t<4, 1>(S, smem);
  return NPL == 2 ? max_coresident_ctas_t<3, 2>(S, smem) : max_coresident_ctas_t<3, 1>(S, smem);
}

// A CTA holding W_hh in TMEM allocates all 512 columns: two such CTAs on one
// SM would block each other's allocation inside a persistent, co-dependent
// grid.  Dynamic shared memory is padded past half an SM so the hardware
// places one per SM; 0 = the grid would not fit that way (keep W in smem).
inline size_t one_cta_per_sm(size_t smem, int ctas, int sms) {
  constexpr size_t kHalf = 116 * 1024;  // > (228 KB per SM - 2 KB reserved) / 2
  if (smem > kHalf) return smem;
  return ctas <= sms ? kHalf + 1024 : 0;
}

inline const char* wt_env0() {
  static const char* env = getenv("HS_W_TMEM");
  return env;
}

// W_hh in TMEM for the resident single-group recurrence (tc_recur.cuh
// load_w_tmem): the slice's NPL*KS/2 columns at column 256, the accumulator
// (<= 256 columns) below.  HS_W_TMEM=0 keeps W_hh in shared memory (A/B).
inline void set_w_tmem(TcRecurArgs& a, const __nv_bfloat16* const* whh, int S, int NPL, int nsw) {
  static const char* env = getenv("HS_W_TMEM");
  a.whh_g[0] = reinterpret_cast<const uint16_t*>(whh[0]);
  a.whh_g[1] = reinterpret_cast<const uint16_t*>(whh[a.D > 1 ? 1 : 0]);
  a.w_tmem = !(env && atoi(env) == 0) && nsw == 0 && w_tmem_cols(a.H, S, NPL) <= 256 && pad16(a.B) <= 256 &&
             (a.H / S) % 64 == 0;
}

// persistent recurrences launch cooperatively (HS_COOP=0: plain cluster launch,
// A/B only).  Nsight Compute fails cooperative cluster launches with
// LaunchFailed; it replays one kernel at a time, so the occupancy check
// before every launch already guarantees the whole grid is resident there.
inline bool coop_launch() {
  static const char* env = getenv("HS_COOP");
  static const bool ncu = getenv("NV_NSIGHT_INJECTION_TRANSPORT_TYPE") || getenv("NV_COMPUTE_PROFILER_PERFWORKS_DIR");
  return !(env && atoi(env) == 0) && !ncu;
}

template <int G, int NPL, int CELLS, int NSW>
inline int launch_recur(const CUtensorMap& w0, const CUtensorMap& w1, const CUtensorMap& hm, const TcRecurArgs& a,
                        int S, size_t smem, cudaStream_t s, std::string& err) {
  static bool init_d[kMaxDev] = {};
  bool& init = init_d[cur_device()];
  int rc;
  if (!init) {
    if ((rc = set_smem(recur_tc_kernel<G, NPL, CELLS, NSW>, kSmemMax, err))) return rc;
    init = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.D * a.RB * S);
  cfg.blockDim = dim3(kRecurThreads + (NSW ? 32 : 0));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = S;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int nclusters = 0;
  cudaError_t e = occ_clusters(&nclusters, recur_tc_kernel<G, NPL, CELLS, NSW>, cfg);
  if (e != cudaSuccess) {
    err = std::string("cudaOccupancyMaxActiveClusters: ") + cudaGetErrorString(e);
    return 2;
  }
  if (nclusters * S < (int)cfg.gridDim.x) {
    err = "recurrent kernel needs " + std::to_string(cfg.gridDim.x / S) + " co-resident clusters of " +
          std::to_string(S) + ", device fits " + std::to_string(nclusters);
    return 3;
  }
  // cooperative: every CTA of the persistent grid is resident at once or the
  // launch waits / fails — never a partial grid spinning on absent peers
  attr[1].id = cudaLaunchAttributeCooperative;
  attr[1].val.cooperative = 1;
  cfg.numAttrs = coop_launch() ? 2 : 1;
  e = cudaLaunchKernelEx(&cfg, recur_tc_kernel<G, NPL, CELLS, NSW>, w0, w1, hm, a);
  if (e != cudaSuccess) {
    err = std::string("recur_tc_kernel launch: ") + cudaGetErrorString(e);
    return 2;
  }
  ++g_launch_count;
  return 0;
}

template <int V>
using IC = std::integral_constant<int, V>;

// Map runtime (G, NPL, cells per owner thread) to a kernel instantiation.
template <typename F>
inline int dispatch_cells(int G, int NPL, int cells, F&& f, std::string& err) {
  auto by_cells = [&](auto g_, auto npl_) -> int {
    switch (cells) {
      case 1: return f(g_, npl_, IC<1>{});
      case 2: return f(g_, npl_, IC<2>{});
      case 4: return f(g_, npl_, IC<4>{});
      case 8: return f(g_, npl_, IC<8>{});
      case 16: return f(g_, npl_, IC<16>{});
      case 32: return f(g_, npl_, IC<32>{});
      default: err = "unsupported cells-per-thread " + std::to_string(cells); return 3;
    }
  };
  if (G == 4) return NPL == 2 ? by_cells(IC<4>{}, IC<2>{}) : by_cells(IC<4>{}, IC<1>{});
  return NPL == 2 ? by_cells(IC<3>{}, IC<2>{}) : by_cells(IC<3>{}, IC<1>{});
}

// One layer of recurrence (both directions).  W_hh planes for dir d at whh[d].
inline int recurrence_layer(int G, int NPL, const __nv_bfloat16* const* whh, TcRecurArgs& a, int sms,
                            cudaStream_t s, std::string& err) {
  int nsw_try = 0;  // ring depth the limit is evaluated for
  auto limit = [&](int S_) -> int {
    size_t sm_ = recur_layout(G, a.H, pad16(a.B), S_, NPL, nsw_try).total;
    if (nsw_try == kTmemW && sm_ < 117 * 1024) sm_ = 117 * 1024;  // padded to one CTA per SM (see one_cta_per_sm)
    return max_coresident_ctas(G, NPL, S_, sm_);
  };
  int nsw = 0;
  static const char* force_sw = getenv("HS_FORCE_STREAM");  // experiments: stream W even if it fits
  int S = force_sw ? 0 : choose_split(G, a.H, a.B, a.D, NPL, limit, 0);
  static const char* force_s0 = getenv("HS_FORCE_S");  // experiments: cap the K-split
  if (S && force_s0 && atoi(force_s0) > 0 && atoi(force_s0) < S) S = atoi(force_s0);
  bool tmem_only = false;  // W_hh fits on chip only in TMEM (no shared-memory copy)
  if (!S && !force_sw) {
    nsw_try = kTmemW;
    S = choose_split(G, a.H, a.B, a.D, NPL, limit, kTmemW);
    tmem_only = S > 0;
  }
  if (!S) {
    nsw_try = kSW;
    S = choose_split(G, a.H, a.B, a.D, NPL, limit, kSW);
    static const char* force_s = getenv("HS_FORCE_S");
    if (force_s && S) S = atoi(force_s) < S ? atoi(force_s) : S;
    nsw = S ? kSW : 0;
  }
  if (!S) {
    err = "no feasible tensor-core split for this shape";
    return 3;
  }
  a.S = S;
  a.RB = a.H / 32;
  set_w_tmem(a, whh, S, NPL, nsw);
  if (tmem_only) a.w_tmem = 1;  // the layout has no shared-memory W (HS_W_TMEM=0 cannot apply)
  CUtensorMap w0, w1, hm;
  int rc = make_map3(&w0, whh[0], a.H, (uint64_t)a.RB * 128, 2, 128, err);
  if (!rc) rc = make_map3(&w1, whh[a.D > 1 ? 1 : 0], a.H, (uint64_t)a.RB * 128, 2, 128, err);
  if (!rc) rc = make_map3(&hm, a.hbuf, a.H, a.Npad, (uint64_t)3 * a.D, a.Npad, err);
  if (rc) return rc;
  size_t smem = recur_layout(G, a.H, a.Npad, S, NPL, nsw).total;  // with W in smem: >= the kernel's TMEM layout
  if (tmem_only) smem = recur_layout(G, a.H, a.Npad, S, NPL, kTmemW).total;
  if (a.w_tmem && one_cta_per_sm(smem, a.D * a.RB * S, sms) == 0) {
    if (tmem_only) {
      err = "TMEM-resident recurrence needs one CTA per SM";
      return 3;
    }
    a.w_tmem = 0;
  }
  if (a.w_tmem) smem = one_cta_per_sm(smem, a.D * a.RB * S, sms);
  // W-streaming: keep as many chunks of the slice in TMEM as fit after the
  // accumulator (c4: 7 of 16 per step never cross the ring); HS_W_TMEM=0: none
  a.w_tmem_chunks = 0;
  if (nsw > 0 && !(wt_env0() && atoi(wt_env0()) == 0)) {
    const int acc = a.Npad <= 32 ? 32 : a.Npad <= 64 ? 64 : a.Npad <= 128 ? 128 : 256;
    const int nch = (a.H / S) / 64;
    int n = (512 - acc) / (NPL * 32);
    if (n >= nch) n = nch - 1;
    if (n > 0 && one_cta_per_sm(smem, a.D * a.RB * S, sms) == smem) a.w_tmem_chunks = n;
  }
  int cells = 1;
  while (cells * (kEpiThreads / (32 / S)) < a.Npad) cells *= 2;
  if (nsw) {  // streaming variant: instantiated for <= 4 cells per thread
    return dispatch_cells(G, NPL, cells, [&](auto g_, auto npl_, auto c_) -> int {
      if constexpr (decltype(c_)::value <= 4) {
        return launch_recur<decltype(g_)::value, decltype(npl_)::value, decltype(c_)::value, kSW>(w0, w1, hm, a, S, smem,
                                                                                                  s, err);
      } else {
        err = "W-streaming recurrence supports at most 4 cells per thread";
        return 3;
      }
    }, err);
  }
  return dispatch_cells(G, NPL, cells, [&](auto g_, auto npl_, auto c_) {
    return launch_recur<decltype(g_)::value, decltype(npl_)::value, decltype(c_)::value, 0>(w0, w1, hm, a, S, smem, s, err);
  }, err);
}


// ------------------------------------------- two-group recurrence (tc_recur2.cuh)
// K-split for two batch halves per CTA; 0 = infeasible.
// With wtmem the layout holds no W_hh (it lives in TMEM): bidirectional
// batch-64 slices (c5) fit at S=2, which the shared-memory layout does not.
inline int choose_split2(int G, int H, int B, int D, int NPL, bool wtmem) {
  if (B < 2 || H % 64) return 0;
  const int Np = pad16((B + 1) / 2);
  if (Np > 64) return 0;
  const int RB = H / 32;
  int best = 0;
  for (int S = 1; S <= 8; S *= 2) {
    if (H % (64 * S)) continue;
    const Recur2Layout L = recur2_layout(G, H, Np, S, NPL, wtmem);
    if (L.nch > RMAXCH || L.total > kSmemMax) continue;
    if (wtmem && w_tmem_cols(H, S, NPL) > 256) continue;
    if ((Np + (128 / (32 / S)) - 1) / (128 / (32 / S)) > 4) continue;  // <= 4 cells per thread
    if (D * RB * S > static_cta_limit(S)) continue;
    best = S;
  }
  return best;
}
// K-split of the two-group recurrence, W_hh in shared memory when that fits
// (*tmem_only = false), else in tensor memory; 0 = infeasible.
inline int choose_split2(int G, int H, int B, int D, int NPL, bool* tmem_only = nullptr) {
  int S = choose_split2(G, H, B, D, NPL, false);
  bool t = false;
  if (!S) {
    S = choose_split2(G, H, B, D, NPL, true);
    t = S > 0;
  }
  if (tmem_only) *tmem_only = t;
  return S;
}

template <int G, int NPL, int CELLS>
inline int launch_recur2(const CUtensorMap& w0, const CUtensorMap& w1, const CUtensorMap& hm, const TcRecurArgs& a,
                         int S, size_t smem, cudaStream_t s, std::string& err) {
  static bool init_d[kMaxDev] = {};
  bool& init = init_d[cur_device()];
  int rc;
  if (!init) {
    if ((rc = set_smem(recur_tc2_kernel<G, NPL, CELLS>, kSmemMax, err))) return rc;
    init = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.D * a.RB * S);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = S;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int nclusters = 0;
  cudaError_t e = occ_clusters(&nclusters, recur_tc2_kernel<G, NPL, CELLS>, cfg);
  if (e != cudaSuccess || nclusters * S < (int)cfg.gridDim.x) {
    err = "two-group recurrent kernel cannot be co-resident";
    return 3;
  }
  attr[1].id = cudaLaunchAttributeCooperative;  // whole grid resident (see launch_recur)
  attr[1].val.cooperative = 1;
  cfg.numAttrs = coop_launch() ? 2 : 1;
  e = cudaLaunchKernelEx(&cfg, recur_tc2_kernel<G, NPL, CELLS>, w0, w1, hm, a);
  if (e != cudaSuccess) {
    err = std::string("recur_tc2_kernel launch: ") + cudaGetErrorString(e);
    return 2;
  }
  ++g_launch_count;
  return 0;
}

// a.B = full batch; a.Npad is set to the per-group padding; a.S / a.RB filled in.
inline int recurrence_layer2(int G, int NPL, const __nv_bfloat16* const* whh, TcRecurArgs& a, cudaStream_t s,
                             std::string& err) {
  bool tmem_only = false;
  const int S = choose_split2(G, a.H, a.B, a.D, NPL, &tmem_only);
  if (!S) {
    err = "no feasible two-group split";
    return 3;
  }
  a.S = S;
  a.RB = a.H / 32;
  a.Npad = pad16((a.B + 1) / 2);
  // W_hh slice in TMEM (TS-mode MMAs) when it fits beside the two accumulators
  static const char* wt_env = getenv("HS_W_TMEM");  // HS_W_TMEM=0: W_hh in shared memory (A/B)
  a.whh_g[0] = reinterpret_cast<const uint16_t*>(whh[0]);
  a.whh_g[1] = reinterpret_cast<const uint16_t*>(whh[a.D > 1 ? 1 : 0]);
  a.w_tmem = (tmem_only || !(wt_env && atoi(wt_env) == 0)) && w_tmem_cols(a.H, S, NPL) <= 256 &&
             a.Npad <= 64 && (a.H / S) % 64 == 0;
  CUtensorMap w0, w1, hm;
  int rc = make_map3(&w0, whh[0], a.H, (uint64_t)a.RB * 128, 2, 128, err);
  if (!rc) rc = make_map3(&w1, whh[a.D > 1 ? 1 : 0], a.H, (uint64_t)a.RB * 128, 2, 128, err);
  if (!rc) rc = make_map3(&hm, a.hbuf, a.H, a.Npad, (uint64_t)3 * a.D * kNG, a.Npad, err);
  if (rc) return rc;
  size_t smem = recur2_layout(G, a.H, a.Npad, S, NPL, tmem_only).total;
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cur_device()) != cudaSuccess) sms = 0;
  if (a.w_tmem && one_cta_per_sm(smem, a.D * a.RB * S, sms) == 0) {
    if (tmem_only) {
      err = "TMEM-resident two-group recurrence needs one CTA per SM";
      return 3;
    }
    a.w_tmem = 0;
  }
  if (a.w_tmem) smem = one_cta_per_sm(smem, a.D * a.RB * S, sms);
  int cells = 1;
  while (cells * (128 / (32 / S)) < a.Npad) cells *= 2;
  return dispatch_cells(G, NPL, cells, [&](auto g_, auto npl_, auto c_) -> int {
    if constexpr (decltype(c_)::value <= 4) {
      return launch_recur2<decltype(g_)::value, decltype(npl_)::value, decltype(c_)::value>(w0, w1, hm, a, S, smem, s,
                                                                                             err);
    } else {
      err = "two-group recurrence supports at most 4 cells per thread";
      return 3;
    }
  }, err);
}

// CTAs the recurrence launch for this layer will use (same split choice as
// recurrence_layer / recurrence_layer2), without launching; 0 = infeasible.
inline int recurrence_ctas(int G, int NPL, const TcRecurArgs& a, bool two) {
  if (two) {
    const int S = choose_split2(G, a.H, a.B, a.D, NPL);
    return S ? a.D * (a.H / 32) * S : 0;
  }
  int nsw_try = 0;
  auto limit = [&](int S_) -> int {
    size_t sm_ = recur_layout(G, a.H, pad16(a.B), S_, NPL, nsw_try).total;
    if (nsw_try == kTmemW && sm_ < 117 * 1024) sm_ = 117 * 1024;
    return max_coresident_ctas(G, NPL, S_, sm_);
  };
  int S = choose_split(G, a.H, a.B, a.D, NPL, limit, 0);
  if (!S) {
    nsw_try = kTmemW;
    S = choose_split(G, a.H, a.B, a.D, NPL, limit, kTmemW);
  }
  if (!S) {
    nsw_try = kSW;
    S = choose_split(G, a.H, a.B, a.D, NPL, limit, kSW);
  }
  return S ? a.D * (a.H / 32) * S : 0;
}

}  // namespace tc
}  // namespace hs
