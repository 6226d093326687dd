// SIMT (FP32 FFMA) kernels: the any-shape path and the numerics reference for
// the tensor-core path.
//
//   sgemm_tn_bias      K1 input projection  XP = X · W_ihᵀ + bias   (all T at once)
//   recur_simt<G>      K2/K3 persistent recurrent wavefront over timesteps:
//                      gates = XP[t] + h_{t-1} · W_hhᵀ (+ b_hh for GRU), fused
//                      gate nonlinearities and c/h update, one grid barrier
//                      per timestep.
#pragma once
#include "common.cuh"

namespace hs {

// ---------------------------------------------------------------- K1 (SIMT)
// C[M,N] = A[M,K] · B[N,K]ᵀ + bias[N]; A, B row-major (K contiguous), K % 4 == 0.
// 128x128x8 block tile, 256 threads, 8x8 register tile per thread.
__global__ void __launch_bounds__(256) sgemm_tn_bias(const float* __restrict__ A,
                                                      const float* __restrict__ Bm,
                                                      const float* __restrict__ bias,
                                                      float* __restrict__ C, int M, int N, int K) {
  __shared__ __align__(16) float As[8][128];
  __shared__ __align__(16) float Bs[8][128];
  const int tid = threadIdx.x;
  const int m0 = blockIdx.y * 128, n0 = blockIdx.x * 128;
  const int lr = tid >> 1, lk = (tid & 1) * 4;
  const int ty = tid >> 4, tx = tid & 15;
  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

  for (int k0 = 0; k0 < K; k0 += 8) {
    float4 av = make_float4(0.f, 0.f, 0.f, 0.f), bv = av;
    const int kk = k0 + lk;
    if (m0 + lr < M && kk < K) av = *reinterpret_cast<const float4*>(A + (size_t)(m0 + lr) * K + kk);
    if (n0 + lr < N && kk < K) bv = *reinterpret_cast<const float4*>(Bm + (size_t)(n0 + lr) * K + kk);
    As[lk + 0][lr] = av.x; As[lk + 1][lr] = av.y; As[lk + 2][lr] = av.z; As[lk + 3][lr] = av.w;
    Bs[lk + 0][lr] = bv.x; Bs[lk + 1][lr] = bv.y; Bs[lk + 2][lr] = bv.z; Bs[lk + 3][lr] = bv.w;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      float a[8], b[8];
      *reinterpret_cast<float4*>(a) = *reinterpret_cast<const float4*>(&As[k][ty * 4]);
      *reinterpret_cast<float4*>(a + 4) = *reinterpret_cast<const float4*>(&As[k][64 + ty * 4]);
      *reinterpret_cast<float4*>(b) = *reinterpret_cast<const float4*>(&Bs[k][tx * 4]);
      *reinterpret_cast<float4*>(b + 4) = *reinterpret_cast<const float4*>(&Bs[k][64 + tx * 4]);
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int m = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int n = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + (j - 4));
      if (n < N) C[(size_t)m * N + n] = acc[i][j] + (bias ? bias[n] : 0.f);
    }
  }
}

// ---------------------------------------------------------- K2/K3 (SIMT)
constexpr int RU = 16;   // hidden units per tile
constexpr int RB = 32;   // batch rows per tile
constexpr int RKC = 64;  // K chunk staged in shared memory
constexpr int RTHREADS = 128;

struct RecurArgs {
  int H, B, T, D;     // hidden, batch, seq, directions of the layer output
  int dir_lo, ndir;   // directions handled by this launch
  int s0, s1;         // processing-step range [s0, s1)
  int tiles_u, tiles_b;
  const float* whh[2];     // per dir: unit-block packed [ceil(H/16)][H][G][16]
  const float* bias_h[2];  // per dir: [G*H] hidden-side bias (GRU) or nullptr
  const float* xproj[2];   // per dir: [T][B][G*H]
  float* out;              // [T][B][D*H]
  const float* hprev[2];   // per dir: [B][H] state entering step s0
  const float* cprev[2];
  float* hlast[2];         // per dir: [B][H] state after step s1-1
  float* clast[2];
  float* cst;              // [D][B][H] cell-state scratch
  unsigned int* barrier;
};

template <int G>
struct RecurSmem {
  union {
    struct {
      float w[RKC][G * RU];
      float h[RKC][RB];
    } stage;
    float red[4][G * RU][RB];
  };
};

template <int G>
__global__ void __launch_bounds__(RTHREADS) recur_simt(RecurArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  RecurSmem<G>& sm = *reinterpret_cast<RecurSmem<G>*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ug = lane & 3, bg = lane >> 2;
  const int H = a.H, B = a.B, T = a.T, D = a.D;
  const int tiles_per_dir = a.tiles_u * a.tiles_b;
  const int ntiles = a.ndir * tiles_per_dir;
  unsigned int round = 0;

  for (int s = a.s0; s < a.s1; ++s) {
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const int d = a.dir_lo + tile / tiles_per_dir;
      const int rem = tile % tiles_per_dir;
      const int ub = rem % a.tiles_u, bb = rem / a.tiles_u;
      const int t = (d == 0) ? s : T - 1 - s;
      const bool first = (s == a.s0);
      const int tprev = (d == 0) ? t - 1 : t + 1;
      const float* hsrc = first ? a.hprev[d] : a.out + (size_t)tprev * B * D * H + (size_t)d * H;
      const size_t hstride = first ? (size_t)H : (size_t)D * H;
      const float* wblk = a.whh[d] + (size_t)ub * H * G * RU;

      float acc[G][4][4];
#pragma unroll
      for (int g = 0; g < G; ++g)
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[g][i][j] = 0.f;

      for (int k0 = 0; k0 < H; k0 += RKC) {
        // W chunk: contiguous [RKC][G][16] slab of the unit block
        constexpr int WV4 = RKC * G * RU / 4;
        for (int v = tid; v < WV4; v += RTHREADS) {
          const int kk = (v * 4) / (G * RU);
          float4 w4 = make_float4(0.f, 0.f, 0.f, 0.f);
          if (k0 + kk < H) w4 = *reinterpret_cast<const float4*>(wblk + (size_t)k0 * G * RU + v * 4);
          *reinterpret_cast<float4*>(&sm.stage.w[0][0] + v * 4) = w4;
        }
        // h chunk, transposed to [k][b]
        {
          const int b = tid & 31, kq = tid >> 5;
          const int gb = bb * RB + b;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int kl = (kq + 4 * i) * 4;
            float4 hv = make_float4(0.f, 0.f, 0.f, 0.f);
            if (gb < B && k0 + kl < H) hv = ld_l2_v4(hsrc + (size_t)gb * hstride + k0 + kl);
            sm.stage.h[kl + 0][b] = hv.x;
            sm.stage.h[kl + 1][b] = hv.y;
            sm.stage.h[kl + 2][b] = hv.z;
            sm.stage.h[kl + 3][b] = hv.w;
          }
        }
        __syncthreads();
#pragma unroll 4
        for (int kk = warp * 16; kk < warp * 16 + 16; ++kk) {
          const float4 hv = *reinterpret_cast<const float4*>(&sm.stage.h[kk][bg * 4]);
          const float hb[4] = {hv.x, hv.y, hv.z, hv.w};
#pragma unroll
          for (int g = 0; g < G; ++g) {
            const float4 wv = *reinterpret_cast<const float4*>(&sm.stage.w[kk][g * RU + ug * 4]);
            const float wu[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
              for (int j = 0; j < 4; ++j) acc[g][i][j] = fmaf(wu[i], hb[j], acc[g][i][j]);
          }
        }
        __syncthreads();
      }
      // cross-warp K reduction through shared memory
#pragma unroll
      for (int g = 0; g < G; ++g)
#pragma unroll
        for (int i = 0; i < 4; ++i)
          *reinterpret_cast<float4*>(&sm.red[warp][g * RU + ug * 4 + i][bg * 4]) =
              make_float4(acc[g][i][0], acc[g][i][1], acc[g][i][2], acc[g][i][3]);
      __syncthreads();
      const bool last = (s == a.s1 - 1);
      for (int c = tid; c < RU * RB; c += RTHREADS) {
        const int u = c % RU, b = c / RU;
        const int unit = ub * RU + u, gb = bb * RB + b;
        if (unit >= H || gb >= B) continue;
        float pre[G];
#pragma unroll
        for (int g = 0; g < G; ++g)
          pre[g] = sm.red[0][g * RU + u][b] + sm.red[1][g * RU + u][b] + sm.red[2][g * RU + u][b] +
                   sm.red[3][g * RU + u][b];
        const float* xp = a.xproj[d] + ((size_t)t * B + gb) * G * H + unit;
        float h;
        if (G == 4) {
          const float gi = pre[0] + xp[0], gf = pre[1] + xp[H], gg = pre[2] + xp[2 * H],
                      go = pre[3] + xp[3 * H];
          const float cp = first ? a.cprev[d][(size_t)gb * H + unit]
                                 : a.cst[((size_t)d * B + gb) * H + unit];
          const float cn = sigmoidf_(gf) * cp + sigmoidf_(gi) * tanhf_(gg);
          h = sigmoidf_(go) * tanhf_(cn);
          a.cst[((size_t)d * B + gb) * H + unit] = cn;
          if (last) a.clast[d][(size_t)gb * H + unit] = cn;
        } else {
          const float* bh = a.bias_h[d];
          const float hr = pre[0] + (bh ? bh[unit] : 0.f), hz = pre[1] + (bh ? bh[H + unit] : 0.f),
                      hn = pre[2] + (bh ? bh[2 * H + unit] : 0.f);
          const float r = sigmoidf_(xp[0] + hr), z = sigmoidf_(xp[H] + hz);
          const float n = tanhf_(xp[2 * H] + r * hn);
          const float hp = ld_l2(hsrc + (size_t)gb * hstride + unit);
          h = (1.f - z) * n + z * hp;
        }
        a.out[((size_t)t * B + gb) * D * H + (size_t)d * H + unit] = h;
        if (last) a.hlast[d][(size_t)gb * H + unit] = h;
      }
      __syncthreads();
    }
    if (s + 1 < a.s1) {
      ++round;
      grid_barrier(a.barrier, round * gridDim.x);
    }
  }
}

// Pack W_hh [G*H, H] (PyTorch) into unit blocks [ceil(H/16)][H][G][16].
__global__ void pack_whh_simt(const float* __restrict__ w, float* __restrict__ out, int G, int H) {
  const int nub = (H + RU - 1) / RU;
  const size_t total = (size_t)nub * H * G * RU;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int u = i % RU;
    const int g = (i / RU) % G;
    const int k = (i / ((size_t)RU * G)) % H;
    const int ub = i / ((size_t)RU * G * H);
    const int unit = ub * RU + u;
    out[i] = unit < H ? w[((size_t)g * H + unit) * H + k] : 0.f;
  }
}

}  // namespace hs
