// K2/K3, two-group form of the cluster K-split recurrence (tc_recur.cuh).
//
// The batch rows of a sequence batch are independent recurrences, so each CTA
// runs TWO of them — batch halves ("groups") — side by side on the same
// resident W_hh slice: warps 0-3 serve group 0, warps 4-7 group 1, each with
// its own producer lane, MMA lane, TMEM accumulator, h_{t-1} staging, partial
// buffer, readiness counters and barriers.  A step of the recurrence is a
// latency chain (h all-gather through L2, MMA, DSMEM reduce-scatter, gates,
// release); with two independent chains in flight, one group's waits overlap
// the other group's work.  The cluster-wide reduce-scatter is therefore
// synchronised per group with mbarriers instead of barrier.cluster:
//   red_full[g]   owner side: the 4 local warps arrive after writing their own
//                 rows; the S-1 peers' slices arrive as bulk copies
//                 (cp.async.bulk shared::cta -> shared::cluster) whose
//                 complete_tx settles the expected byte count
//   red_free[g]   sender side: S ranks x 4 owner warps arrive (relaxed) after
//                 reading the previous step's partials
//   tmem_free[g]  the group's 4 warps drained the accumulator
// Numerics are identical to tc_recur.cuh (fp16 W hi/lo x fp16 h, f32 TMEM).
#pragma once
#include "common.cuh"
#include "tc_common.cuh"
#include "tc_recur.cuh"

namespace hs {
namespace tc {

constexpr int kNG = 2;  // groups per CTA

struct Recur2Layout {
  int nch;
  size_t w_off, h_off, red_off, stage_off, bar_off, total;
  size_t h_group, red_group, stage_group;  // bytes per group
};

// Np = padded rows of ONE group; wtmem: W_hh in tensor memory (no smem copy)
__host__ __device__ inline Recur2Layout recur2_layout(int G, int H, int Np, int S, int NPL, bool wtmem = false) {
  Recur2Layout L;
  const int KS = H / S;
  L.nch = KS / 64;
  size_t off = 0;
  L.w_off = off;   off += wtmem ? 0 : (size_t)NPL * L.nch * 128 * 128;
  L.h_group = (size_t)L.nch * Np * 128;
  L.h_off = off;   off += kNG * L.h_group;
  L.red_group = (size_t)G * 32 * (Np + 4) * 4;
  L.red_off = off; off += kNG * L.red_group;
  // outgoing partials for the S-1 peers, laid out like their destination regions
  L.stage_group = (size_t)(S - 1) * G * (32 / S) * (Np + 4) * 4;
  L.stage_off = off; off += kNG * L.stage_group;
  off = (off + 15) / 16 * 16;
  // per group: acc_full, red_full, red_free, tmem_free, h_full[RMAXCH]; + w_full, tmem slot
  L.bar_off = off; off += 8 * (2 + kNG * (4 + RMAXCH)) + 16;
  L.total = off;
  return L;
}

template <int G, int NPL, int CELLS>
__global__ void __launch_bounds__(256, 1)
    recur_tc2_kernel(const __grid_constant__ CUtensorMap tmW0, const __grid_constant__ CUtensorMap tmW1,
                     const __grid_constant__ CUtensorMap tmH, const TcRecurArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if (ptx::smem_u32(smem_raw) & 1023) __trap();
  signal_started(a);
  // a.B = total batch, a.Npad = padded rows of one group (Bh = ceil(B/2) rows each)
  const int H = a.H, B = a.B, Np = a.Npad, T = a.T, D = a.D, S = a.S, RB = a.RB;
  const int Bh = (B + 1) / 2;
  const Recur2Layout L = recur2_layout(G, H, Np, S, NPL, a.w_tmem != 0);
  const int nch = L.nch;
  const int KS = H / S;
  const int UO = 32 / S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = warp >> 2;           // group of this warp
  const int sub = warp & 3;            // TMEM lane quarter
  const int eg = threadIdx.x & 127;    // thread index within the group
  const int Bg = grp == 0 ? Bh : B - Bh;  // real rows of this group
  const int brow0 = grp * Bh;              // first global batch row of the group

  __nv_bfloat16* sW = reinterpret_cast<__nv_bfloat16*>(smem + L.w_off);
  __nv_bfloat16* sH = reinterpret_cast<__nv_bfloat16*>(smem + L.h_off + grp * L.h_group);
  float* red = reinterpret_cast<float*>(smem + L.red_off + grp * L.red_group);
  float* stage = reinterpret_cast<float*>(smem + L.stage_off + grp * L.stage_group);
  const uint32_t region_floats = (uint32_t)(G * UO * (Np + 4));  // one sender's rows in an owner's buffer
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bar_off);
  uint64_t* w_full = bars;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 1);
  uint64_t* gb = bars + 2 + grp * (4 + RMAXCH);  // this group's barriers
  uint64_t* acc_full = gb;
  uint64_t* red_full = gb + 1;
  uint64_t* red_free = gb + 2;
  uint64_t* tmem_free = gb + 3;
  uint64_t* h_full = gb + 4;

  const int q = (int)ptx::cluster_rank();
  const int cl = blockIdx.x / S;
  const int d = cl / RB;
  const int rb = cl % RB;
  const CUtensorMap* tmW = d == 0 ? &tmW0 : &tmW1;
  const int GH = G * H;
  const int rstride = Np + 4;
  const uint32_t tcols_g = Np <= 32 ? 32 : Np <= 64 ? 64 : 128;
  // accumulators in columns [0, 2*tcols_g); W_hh (a.w_tmem) from column 256
  const uint32_t wcol = 256u;
  const uint32_t tcols = a.w_tmem ? 512u : 2 * tcols_g;
  constexpr int kCtrStride = kCtrStrideWords;
  const int nchunk_all = H / 64;
  unsigned int* ctr_g = a.counters + (size_t)grp * D * nchunk_all * kCtrStride;
  unsigned int* my_counter = ctr_g + (d * nchunk_all + (rb * 32) / 64) * kCtrStride;
  const unsigned int* in_counter = ctr_g + (d * nchunk_all + (q * KS) / 64) * kCtrStride;
  const unsigned int per_round = 2u * (unsigned int)S;
  const size_t slab = (size_t)Np * H;  // hbuf elements per (buf, d, group)

  if (threadIdx.x == 0) {
    ptx::tma_prefetch(tmW);
    ptx::tma_prefetch(&tmH);
    ptx::mbar_init(w_full, 1);
    for (int g2 = 0; g2 < kNG; ++g2) {
      uint64_t* b2 = bars + 2 + g2 * (4 + RMAXCH);
      ptx::mbar_init(b2 + 0, 1);                       // acc_full
      ptx::mbar_init(b2 + 1, 5);                       // red_full: 4 local warps + the owner's expect_tx
      ptx::mbar_init(b2 + 2, (uint32_t)(S * 4));       // red_free
      ptx::mbar_init(b2 + 3, 4);                       // tmem_free
      for (int c = 0; c < nch; ++c) ptx::mbar_init(b2 + 4 + c, 1);
    }
    ptx::fence_mbar_init();
    for (int g2 = 0; g2 < kNG; ++g2)  // phase 0: the S-1 peers' bulk copies
      ptx::mbar_arrive_expect_tx(bars + 2 + g2 * (4 + RMAXCH) + 1, (uint32_t)((S - 1) * G * UO * (Np + 4) * 4));
  }
  if (warp == 2) ptx::tmem_alloc_dyn(tmem_slot, tcols);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot + (uint32_t)(grp * tcols_g);

  if (a.w_tmem) {  // the CTA's W_hh slice into TMEM (all 8 warps), visible to the MMA issuer below
    load_w_tmem(a.whh_g[d], (size_t)RB * 128 * H, H, rb * 128, q * KS, KS, NPL, *tmem_slot + wcol);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
  } else if (warp == 0 && ptx::elect_one()) {
    ptx::mbar_arrive_expect_tx(w_full, (uint32_t)(NPL * nch * 128 * 128));
    for (int p = 0; p < NPL; ++p)
      for (int c = 0; c < nch; ++c)
        ptx::tma_load_3d(sW + ((size_t)p * nch + c) * 128 * 64, tmW, w_full, q * KS + c * 64, rb * 128, p);
  }
  __syncwarp();
  const uint32_t tmem_w = *tmem_slot + wcol;

  // owner cells of this group: unit u_loc, group rows b = b0 + k*bstep
  const int u_loc = eg % UO;
  const int b0 = eg / UO;
  const int bstep = 128 / UO;
  const int unit = rb * 32 + q * UO + u_loc;
  float c_reg[CELLS], h_reg[CELLS], xq[CELLS][G];
  float wsc[G];
#pragma unroll
  for (int g = 0; g < G; ++g) wsc[g] = a.whh_scale[d][rb * 128 + g * 32 + q * UO + u_loc];
  float bias_r = 0.f, bias_z = 0.f, bias_n = 0.f;
  if (G == 3 && a.bias_h[d]) {
    bias_r = a.bias_h[d][unit];
    bias_z = a.bias_h[d][H + unit];
    bias_n = a.bias_h[d][2 * H + unit];
  }
  auto load_xproj = [&](int step, bool poll) {
    const int tt = d == 0 ? step : T - 1 - step;
    if (poll) wait_xready(a, tt);
    const float* __restrict__ xp = a.xproj[d] + (size_t)tt * a.Bst * GH + unit;
#pragma unroll
    for (int k = 0; k < CELLS; ++k) {
      const int b = b0 + k * bstep;
#pragma unroll
      for (int g = 0; g < G; ++g) xq[k][g] = b < Bg ? __ldcg(xp + (size_t)(brow0 + b) * GH + g * H) : 0.f;
    }
  };
  auto group_release = [&](unsigned int* ctr) {  // the group's 4 warps, then one release
    ptx::named_bar(1 + grp, 128);
    if (eg == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
  };
#pragma unroll
  for (int k = 0; k < CELLS; ++k) {
    c_reg[k] = 0.f;
    h_reg[k] = 0.f;
    const int b = b0 + k * bstep;
    if (b < Bg) {
      h_reg[k] = a.h0[d][(size_t)(brow0 + b) * H + unit];
      if (G == 4) c_reg[k] = a.c0[d][(size_t)(brow0 + b) * H + unit];
      a.hbuf[((size_t)(0 * D + d) * kNG + grp) * slab + (size_t)b * H + unit] = h_operand<NPL>(h_reg[k]);
    }
  }
  ptx::fence_proxy_async_global();
  load_xproj(0, true);
  group_release(my_counter);
  cluster_arrive();  // every CTA's barriers initialised before any remote op
  cluster_wait();
  const bool stamper = a.stamps && rb == 0 && q == 0 && threadIdx.x == 0;  // group 0's chain
  if (stamper) a.stamps[(size_t)d * (T + 1)] = globaltimer();

  const uint32_t idesc = NPL == 2 ? idesc_f16_f32(128, Np) : ptx::idesc_bf16_f32(128, Np);
  const bool active = sub < G;
  const int dst_rank = lane / UO;
  // this lane's row: in my own buffer (dst == me) or in the staging slot of peer dst
  float* part_row = dst_rank == q ? red + ((size_t)(q * G + sub) * UO + lane % UO) * rstride
                                  : stage + (size_t)(dst_rank < q ? dst_rank : dst_rank - 1) * region_floats +
                                        ((size_t)sub * UO + lane % UO) * rstride;

  for (int s = 0; s < T; ++s) {
    const int t = d == 0 ? s : T - 1 - s;
    const int buf_in = s % 3, buf_out = (s + 1) % 3;
    const bool last = s == T - 1;
    if (sub == 0) {  // producer of this group (whole warp: lane-parallel chunk polls)
      if (lane == 0) {
        if (grp == 0) HS_TRACE(0);
        if (s == 0 && grp == 1 && a.group_offset_ns) {  // start group 1 out of phase
          const unsigned long long t0 = globaltimer();
          while (globaltimer() - t0 < a.group_offset_ns) {
          }
        }
      }
      __syncwarp();
      poll_chunks(in_counter, nch, per_round * (unsigned int)(s + 1), [&](int c) {
        if (grp == 0 && c == 0) HS_TRACE(1);
        if (grp == 0 && c == nch - 1) HS_TRACE(12);
        ptx::fence_proxy_async_global();
        ptx::mbar_arrive_expect_tx(&h_full[c], (uint32_t)(Np * 128));
        ptx::tma_load_3d(sH + (size_t)c * Np * 64, &tmH, &h_full[c], q * KS + c * 64, 0, (buf_in * D + d) * kNG + grp);
      });
      __syncwarp();
    } else if (sub == 1) {  // MMA issuer of this group
      if (ptx::elect_one()) {
        if (s == 0) {
          if (!a.w_tmem) ptx::mbar_wait(w_full, 0);
        } else {
          ptx::mbar_wait(tmem_free, (s - 1) & 1);
        }
        for (int c = 0; c < nch; ++c) {
          ptx::mbar_wait(&h_full[c], s & 1);
          ptx::tc_fence_after();
          if (grp == 0 && c == 0) HS_TRACE(14);
          if (grp == 0 && c == nch - 1) HS_TRACE(15);
          const __nv_bfloat16* wh = sW + (size_t)c * 128 * 64;
          const __nv_bfloat16* hh = sH + (size_t)c * Np * 64;
          if (a.w_tmem) {  // A = W columns of (plane, chunk, kk): 8 columns per K=16
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint64_t bd = ptx::sdesc_k_sw128(hh + kk * 16);
              ptx::mma_bf16_ts(tmem, tmem_w + (uint32_t)(c * 32 + kk * 8), bd, idesc, (c | kk) != 0);
              if (NPL == 2) ptx::mma_bf16_ts(tmem, tmem_w + (uint32_t)(KS / 2 + c * 32 + kk * 8), bd, idesc, 1);
            }
          } else {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              ptx::mma_bf16_ss(tmem, ptx::sdesc_k_sw128(wh + kk * 16), ptx::sdesc_k_sw128(hh + kk * 16), idesc,
                               (c | kk) != 0);
              if (NPL == 2) {
                const __nv_bfloat16* wl = wh + (size_t)nch * 128 * 64;
                ptx::mma_bf16_ss(tmem, ptx::sdesc_k_sw128(wl + kk * 16), ptx::sdesc_k_sw128(hh + kk * 16), idesc, 1);
              }
            }
          }
        }
        ptx::mma_commit(acc_full);
        if (grp == 0) HS_TRACE(2);
      }
      __syncwarp();
    }
    // 1. drain TMEM, reduce-scatter the group's partial gates to the unit owners
    ptx::mbar_wait(acc_full, s & 1);
    ptx::tc_fence_after();
    if (threadIdx.x == 64) HS_TRACE(3);
    // partials go to LOCAL shared memory (own rows -> my buffer, peers' rows ->
    // staging), then one thread moves each peer's slice with a bulk copy whose
    // complete_tx lands on the peer's red_full: no per-thread DSMEM stores and
    // no release fence on the sender side
    if (active) {
      if (threadIdx.x == 64) HS_TRACE(7);
      for (int c16 = 0; c16 < Np / 16; ++c16) {
        float v[16];
        ptx::tmem_ld_32x32b_x16(tmem + ((uint32_t)(sub * 32) << 16) + c16 * 16, v);
#pragma unroll
        for (int j = 0; j < 16; j += 4)
          *reinterpret_cast<float4*>(part_row + c16 * 16 + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      }
    }
    if (threadIdx.x == 64) HS_TRACE(8);
    ptx::tc_fence_before();
    ptx::fence_proxy_async_smem();  // staging writes -> the bulk copy (async proxy)
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(tmem_free);
    if (lane == 0) ptx::mbar_arrive(red_full);  // my own rows are in place
    ptx::named_bar(1 + grp, 128);               // the group's staging is complete
    if (eg == 0) {
      if (s > 0) ptx::mbar_wait_cluster(red_free, (s - 1) & 1);  // peers read step s-1's partials
      for (int r = 0; r < S; ++r) {
        if (r == q) continue;
        const float* src = stage + (size_t)(r < q ? r : r - 1) * region_floats;
        const uint32_t dst = ptx::mapa(ptx::smem_u32(red + (size_t)q * region_floats), (uint32_t)r);
        ptx::bulk_s2cluster(dst, src, region_floats * 4u, ptx::mapa(ptx::smem_u32(red_full), (uint32_t)r));
      }
      ptx::bulk_commit();
      ptx::bulk_wait_read0();  // staging reusable (next step's drain comes long after)
    }
    if (threadIdx.x == 64) HS_TRACE(4);
    if (eg == 96 && !last) wait_xready(a, d == 0 ? s + 1 : T - 2 - s);  // next step's XP (see wait_xready)
    ptx::mbar_wait_cluster(red_full, s & 1);  // all partials for my units landed
    if (threadIdx.x == 64) HS_TRACE(5);
    if (eg == 0 && !last)  // next phase: the peers' bulk copies of step s+1
      ptx::mbar_arrive_expect_tx(red_full, (uint32_t)((S - 1) * region_floats * 4));
    // 2. owner: gates -> h_t (critical path)
#pragma unroll
    for (int k = 0; k < CELLS; ++k) {
      const int b = b0 + k * bstep;
      if (b >= Np) break;
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
      if (!last && b < Bg)
        a.hbuf[((size_t)(buf_out * D + d) * kNG + grp) * slab + (size_t)b * H + unit] = h_operand<NPL>(h);
    }
    if (threadIdx.x == 64) HS_TRACE(6);
    // partials read (values consumed above): senders may refill the buffer
    __syncwarp();
    if (lane < S) ptx::mbar_arrive_remote_relaxed(ptx::mapa(ptx::smem_u32(red_free), (uint32_t)lane));
    if (!last) {
      ptx::fence_proxy_async_global();
      group_release(my_counter);
      if (stamper) a.stamps[(size_t)d * (T + 1) + s + 1] = globaltimer();
      // the group barrier inside group_release also ordered the group's y stores
      // of step s-1: publish them for the overlapped K1 / device->host copy from
      // a thread off the critical path (warp 3 of the group: neither the
      // producer nor the MMA warp), without a barrier or fence of its own
      if (a.progress && s > 0 && eg == 96)
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(a.progress + s - 1) : "memory");
    }
    if (stamper && last) a.stamps[(size_t)d * (T + 1) + T] = globaltimer();
    if (threadIdx.x == 0) HS_TRACE(10);
    // 3. off the critical path: outputs, final state, next step's XP
#pragma unroll
    for (int k = 0; k < CELLS; ++k) {
      const int b = b0 + k * bstep;
      if (b >= Bg) continue;
      const float hv = h_reg[k];
      const size_t yidx = ((size_t)t * a.Bst + brow0 + b) * D * H + (size_t)d * H + unit;
      if (a.y) a.y[yidx] = hv;
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
        a.hn[d][(size_t)(brow0 + b) * H + unit] = hv;
        if (G == 4) a.cn[d][(size_t)(brow0 + b) * H + unit] = c_reg[k];
      }
    }
    if (a.progress && last) {  // y of the last two steps in memory: one increment each per group per CTA
      ptx::named_bar(1 + grp, 128);
      if (eg == 96) {
        if (s > 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(a.progress + s - 1) : "memory");
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(a.progress + s) : "memory");
      }
    }
    if (!last) load_xproj(s + 1, false);  // ordered after warp 3's wait_xready by group_release's barrier
  }
  cluster_arrive();  // no CTA leaves while peers may still write its partials / barriers
  cluster_wait();
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(*tmem_slot, tcols);
  }
}

}  // namespace tc
}  // namespace hs
