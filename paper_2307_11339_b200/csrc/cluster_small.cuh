// K2/K3, small-shape form: one thread-block cluster per direction runs a whole
// layer (input projection + recurrence) in FP32 FFMA, W resident in SMEM.
//
// For the latency regime of the paper's own models (hidden 32-256, batch 1-16,
// e.g. BASELINE c1: 1x128, T16, B1) the tensor-core path and the grid-barrier
// SIMT path are dominated by synchronisation: a grid barrier costs a few us per
// step.  Here a cluster of C CTAs (16, 8 or 4; one GPC) owns the layer:
//   * CTA q owns U = H/C units and all G of their gate rows: W_ih and W_hh
//     slices (G*U rows, fp32) live in its shared memory for all T steps;
//   * every CTA holds the full h_{t-1} [B][H] in shared memory; each step a
//     CTA computes its units' h_t and broadcasts them to all C CTAs with
//     st.shared::cluster (DSMEM), then one cluster barrier (~0.2 us) orders the
//     step — no global-memory round trip on the recurrence critical path;
//   * the input term W_ih x_{t+1} does not depend on h, so it is computed
//     between barrier arrive and wait, hiding the barrier latency.
// FP32 FFMA arithmetic, ex2-based gate functions (max-abs ~1e-7 vs the float64 oracle).
#pragma once
#include "common.cuh"
#include "tc_common.cuh"

namespace hs {

constexpr int kSmallThreads = 256;

struct SmallArgs {
  int H, I, B, T, D, C;          // C = cluster size (CTAs per direction); D = directions launched
  // directions dir0 .. dir0+D-1 of a Dy-direction layer, steps s_base .. s_base+T-1
  // of T_full (one plan segment, hs_rnn_run_cells); the fused forward runs
  // dir0 = 0, Dy = D, s_base = 0, T_full = T
  int dir0, Dy, s_base, T_full;
  const float* x;                // layer input [T][B][I]
  const float* w_ih[2];          // per dir [G*H][I] fp32 (PyTorch layout)
  const float* w_hh[2];          // per dir [G*H][H] fp32
  const float* bias_x[2];        // per dir [G*H] (b_ih (+ b_hh for LSTM))
  const float* bias_h[2];        // per dir [G*H] (GRU b_hh) or nullptr
  const float* h0[2];            // per dir [B][H], nullptr = zeros
  const float* c0[2];            // nullptr = zeros
  float* y;                      // [T_full][B][Dy*H]
  float* hn[2];                  // per dir [B][H]
  float* cn[2];
};

__host__ __device__ inline size_t small_smem_bytes(int G, int H, int I, int B, int C) {
  const int rows = G * (H / C);
  return sizeof(float) * ((size_t)rows * (I + H)       // W_ih, W_hh slices
                          + 2 * (size_t)B * H           // h double buffer
                          + 2 * (size_t)rows * B        // x-part double buffer
                          + (size_t)rows * B            // h-part
                          + (size_t)(H / C) * B         // c state of owned cells
                          + 2 * (size_t)rows            // x- and h-side biases of the slice
                          + (size_t)(H / C) * B);       // h_t of owned cells, staged for the y store
}

// dot products of `rows` weight rows (row stride K, in smem) with `nb`
// vectors (stride vstride) -> out[r*B + b]; `tpi` threads cooperate per (r, b).
// K % 4 == 0 and 16-B aligned rows: float4 loads, 4 independent FMA chains.
__device__ __forceinline__ void small_matvec(const float* __restrict__ w, const float* __restrict__ v, int rows, int nb,
                                             int K, int vstride, float* __restrict__ out, int B, int tpi,
                                             const float* __restrict__ bias) {
  const int items = rows * nb;
  const int groups = kSmallThreads / tpi;
  const int g = threadIdx.x / tpi, l = threadIdx.x % tpi;
  const int K4 = K / 4;
  for (int it = g; it < (items + groups - 1) / groups * groups; it += groups) {
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    const bool valid = it < items;
    const int r = valid ? it / nb : 0, b = valid ? it % nb : 0;
    if (valid) {
      const float4* wr = reinterpret_cast<const float4*>(w + (size_t)r * K);
      const float4* vb = reinterpret_cast<const float4*>(v + (size_t)b * vstride);
#pragma unroll 4
      for (int k = l; k < K4; k += tpi) {
        const float4 ww = wr[k], vv = vb[k];
        a0 = fmaf(ww.x, vv.x, a0);
        a1 = fmaf(ww.y, vv.y, a1);
        a2 = fmaf(ww.z, vv.z, a2);
        a3 = fmaf(ww.w, vv.w, a3);
      }
    }
    float acc = (a0 + a1) + (a2 + a3);
    for (int o = tpi / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o, tpi);
    if (valid && l == 0) out[r * B + b] = acc + (bias ? bias[r] : 0.f);
  }
}

template <int G>
__global__ void __launch_bounds__(kSmallThreads, 1) recur_cluster_small(const SmallArgs a) {
  extern __shared__ __align__(16) float sm[];
  const int H = a.H, I = a.I, B = a.B, T = a.T, C = a.C;
  const int U = H / C, rows = G * U;
  const int q = (int)ptx::cluster_rank();
  const int d = a.dir0 + (int)blockIdx.x / C;
  const int Tf = a.T_full, sb = a.s_base, Dy = a.Dy;
  float* w_ih = sm;                                  // [rows][I]
  float* w_hh = w_ih + (size_t)rows * I;             // [rows][H]
  float* hbuf = w_hh + (size_t)rows * H;             // [2][B][H]
  float* xpart = hbuf + 2 * (size_t)B * H;           // [2][rows][B]
  float* hpart = xpart + 2 * (size_t)rows * B;       // [rows][B]
  float* cst = hpart + (size_t)rows * B;             // [U][B]
  float* bx = cst + (size_t)U * B;                   // [rows] x-side bias (b_ih (+ b_hh for LSTM))
  float* bhh = bx + rows;                            // [rows] h-side bias (GRU b_hh), else 0
  float* ystage = bhh + rows;                        // [U][B]
  const int tid = threadIdx.x;

  // resident slices: local row r = g*U + u  <->  global row g*H + q*U + u
  {
    const int I4 = I / 4, H4 = H / 4;
#pragma unroll 4
    for (int i = tid; i < rows * I4; i += kSmallThreads) {
      const int r = i / I4, k = i % I4;
      reinterpret_cast<float4*>(w_ih)[i] =
          __ldg(reinterpret_cast<const float4*>(a.w_ih[d] + ((size_t)(r / U) * H + q * U + r % U) * I) + k);
    }
#pragma unroll 4
    for (int i = tid; i < rows * H4; i += kSmallThreads) {
      const int r = i / H4, k = i % H4;
      reinterpret_cast<float4*>(w_hh)[i] =
          __ldg(reinterpret_cast<const float4*>(a.w_hh[d] + ((size_t)(r / U) * H + q * U + r % U) * H) + k);
    }
#pragma unroll 4
    for (int i = tid; i < B * H4; i += kSmallThreads)
      reinterpret_cast<float4*>(hbuf)[i] =
          a.h0[d] ? __ldg(reinterpret_cast<const float4*>(a.h0[d]) + i) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  for (int i = tid; i < U * B; i += kSmallThreads) {
    const int u = i / B, b = i % B;
    cst[i] = (G == 4 && a.c0[d]) ? a.c0[d][(size_t)b * H + q * U + u] : 0.f;
  }
  for (int r = tid; r < rows; r += kSmallThreads) {
    const int grow = (r / U) * H + q * U + r % U;
    bx[r] = a.bias_x[d][grow];
    bhh[r] = a.bias_h[d] ? a.bias_h[d][grow] : 0.f;
  }
  // threads per dot product: enough to keep all 256 threads busy, <= 32
  int tpi_x = 1, tpi_h = 1;
  while (tpi_x < 32 && rows * B * tpi_x * 2 <= kSmallThreads && tpi_x * 2 <= I / 4) tpi_x *= 2;
  while (tpi_h < 32 && rows * B * tpi_h * 2 <= kSmallThreads && tpi_h * 2 <= H / 4) tpi_h *= 2;
  __syncthreads();
  auto x_term = [&](int step, float* out) {
    const int tt = d == 0 ? sb + step : Tf - 1 - sb - step;
    small_matvec(w_ih, a.x + (size_t)tt * B * I, rows, B, I, I, out, B, tpi_x, bx);
  };
  x_term(0, xpart);
  // peers' shared memory is initialised before anyone writes into it
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");

  for (int s = 0; s < T; ++s) {
    const int t = d == 0 ? sb + s : Tf - 1 - sb - s;
    const float* hcur = hbuf + (size_t)(s & 1) * B * H;
    float* hnext_local = hbuf + (size_t)((s + 1) & 1) * B * H;
    const float* xp = xpart + (size_t)(s & 1) * rows * B;
    small_matvec(w_hh, hcur, rows, B, H, H, hpart, B, tpi_h, bhh);
    __syncthreads();
    // cells (u, b): gates, state update, broadcast h_t to every CTA of the cluster
    for (int i = tid; i < U * B; i += kSmallThreads) {
      const int u = i / B, b = i % B;
      const int unit = q * U + u;
      float hval;
      if (G == 4) {
        float pre[4];
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          const int r = g * U + u;
          pre[g] = xp[r * B + b] + hpart[r * B + b];
        }
        const float ig = sigmoid_fast(pre[0]), fg = sigmoid_fast(pre[1]), gg = tanh_fast(pre[2]), og = sigmoid_fast(pre[3]);
        const float cnew = fg * cst[i] + ig * gg;
        cst[i] = cnew;
        hval = og * tanh_fast(cnew);
      } else {
        const int r0 = u, r1 = U + u, r2 = 2 * U + u;
        const float px0 = xp[r0 * B + b], ph0 = hpart[r0 * B + b];
        const float px1 = xp[r1 * B + b], ph1 = hpart[r1 * B + b];
        const float px2 = xp[r2 * B + b], ph2 = hpart[r2 * B + b];
        const float r = sigmoid_fast(px0 + ph0), z = sigmoid_fast(px1 + ph1);
        const float n = tanh_fast(px2 + r * ph2);
        hval = (1.f - z) * n + z * hcur[(size_t)b * H + unit];
      }
      const uint32_t loc = ptx::smem_u32(hnext_local + (size_t)b * H + unit);
      for (int p = 0; p < C; ++p) {
        const uint32_t rem = ptx::mapa(loc, (uint32_t)p);
        asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(rem), "f"(hval) : "memory");
      }
      ystage[i] = hval;
    }
    // the release covers only the DSMEM h stores above; the global y / h_n
    // stores below stay off the step's critical path
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    for (int i = tid; i < U * B; i += kSmallThreads) {
      const int u = i / B, b = i % B;
      const int unit = q * U + u;
      a.y[((size_t)t * B + b) * Dy * H + (size_t)d * H + unit] = ystage[i];
      if (s == T - 1) {
        a.hn[d][(size_t)b * H + unit] = ystage[i];
        if (G == 4) a.cn[d][(size_t)b * H + unit] = cst[i];
      }
    }
    if (s + 1 < T) x_term(s + 1, xpart + (size_t)((s + 1) & 1) * rows * B);  // hides the barrier latency
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
}

}  // namespace hs
