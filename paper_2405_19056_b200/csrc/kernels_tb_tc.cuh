// kernels_tb_tc.cuh -- the fused T + B + psi kernel on tcgen05.
//
// PAPER.md Eq. eq:SymmetricNN: tau = sum_i h(b_i), h shared; B;
// the psi projection is reading R15.  One CTA = one 128-pixel tile at a time,
// thread r owns pixel r (= TMEM lane r = MMA row r).  Per tile:
//   1. each thread loads its pixel's K records into registers and gives every valid
//      record its rank in the canonical order (reading R5: lexicographic on the storage
//      bits, slot index as the last tie-break, which only orders identical records); the
//      record's A1 row [record | 1 1 1 | 0 0] is stored at that rank, masked slots get
//      zero rows.  No data moves between registers: ranks are computed, rows scattered.
//   2. software-pipelined slot rounds t = 0 .. Kt (Kt = the tile's largest valid count):
//        epilogue 2 of slot t-1:  A3 = ReLU(acc2) (/n in mean mode) -> f16
//        epilogue 1 of slot t:    A2 = [ReLU(acc1) -> bf16 | 1 1 1 0..] (1s only if valid)
//        then one MMA batch:      accB += A3 W_B,tau^T   (slot t-1)
//                                 acc2  = A2 W2ext^T      (slot t)
//                                 acc1  = A1[t+1] W1ext^T (slot t+1)
//      so each slot costs one MMA round trip.  accB starts as e0 W_B,e0^T; the pool
//      g = sum is the tensor core's accumulation (W_B sum_s a2_s = sum_s W_B a2_s).
//      Masked slots are all-zero rows (bias columns included) and contribute exactly 0;
//      per-fragment activations never leave the SM.
//   3. phi = ReLU(accB + b_B + w_Bn n);  psi = W_O,d0 phi + W_O,L L_d + b_O  -> HBM (fp32).
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <type_traits>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace gn {

#ifdef GN_PROFILE_TB
// clock64 breakdown of chain 0 of CTA 0 (diagnostic build only)
__device__ unsigned long long gn_tb_prof[16];
#define TBP_NOW(v) const long long v = clock64()
#define TBP_ADD(i, a, b) \
  if (threadIdx.x == 0 && blockIdx.x == 0) gn_tb_prof[i] += (unsigned long long)((b) - (a))
#else
#define TBP_NOW(v)
#define TBP_ADD(i, a, b)
#endif

template <int K, int H, int C0>
struct TbLayout {
  static constexpr int KA2 = H + 16;
  static constexpr int W1_B = H * 16 * 2;
  static constexpr int W2_B = H * KA2 * 2;
  static constexpr int WBT_B = C0 * H * 2;
  static constexpr int WBE_B = C0 * C0 * 2;
  static constexpr int WIMG_B = W1_B + W2_B + WBT_B + WBE_B;
  static constexpr int NPAR = C0 + C0 + 3 * (C0 + 3) + 3;
  static constexpr int OFF_W1 = 0, OFF_W2 = OFF_W1 + W1_B, OFF_WBT = OFF_W2 + W2_B, OFF_WBE = OFF_WBT + WBT_B;
  static constexpr int PL = 128 * 16;                 // one 8-column K-plane of a 128-row operand
  // one chain (= one warpgroup working on its own tile stream):
  static constexpr int CH_A1 = 0;                     // K slots x 2 planes
  static constexpr int CH_A2 = CH_A1 + K * 2 * PL;    // KA2/8 planes
  static constexpr int CH_A3 = CH_A2 + (KA2 / 8) * PL;  // H/8 planes; the e0 operand aliases it
  static constexpr int SBT = 4;                       // tiles per superblock (pixels sorted by count)
  // superblock sort scratch (perm: SBT*128 u16, wsum: 4 warps x (K+2) ints) lives in the
  // A2 region, which is free while a superblock is sorted
  static constexpr int CH_PERM = CH_A2;
  static constexpr int CH_SCAN = CH_PERM + SBT * 128 * 2;
  static_assert(SBT * 128 * 2 + 4 * (K + 2) * 4 <= (KA2 / 8) * PL, "sort scratch must fit A2");
  static constexpr int CH_B = CH_A3 + (H / 8) * PL;
  static constexpr int OFF_PAR = WIMG_B;
  static constexpr int OFF_BAR = (OFF_PAR + NPAR * 4 + 15) / 16 * 16;   // 4 mbarriers + tmem ptr
  static constexpr int OFF_RED = OFF_BAR + 48;        // 4 chains x 8 ints: per-warp max count, superblock ids
  static constexpr int OFF_CH = (OFF_RED + 128 + 127) / 128 * 128;
  static constexpr int TCOLS = (2 * H + C0 + 31) / 32 * 32;   // TMEM columns per chain
  static constexpr int NCH_T = 512 / TCOLS;
  static constexpr int NCH_S = (232448 - 1024 - OFF_CH) / CH_B;
  static constexpr int NCH = NCH_T < NCH_S ? (NCH_T < 4 ? NCH_T : 4) : (NCH_S < 4 ? NCH_S : 4);
  static constexpr int SMEM = OFF_CH + NCH * CH_B;
  static constexpr int TMEM_COLS = 512;
  static constexpr int REC_B = K * 22;                // bytes of one pixel's records
  static constexpr int VW = REC_B % 16 == 0 ? 16 : REC_B % 8 == 0 ? 8 : REC_B % 4 == 0 ? 4 : 2;
  static constexpr int NV = REC_B / VW;
  static constexpr bool PREFETCH = K <= 8;            // register budget of the next tile's records
};

template <int K, int H, int C0, int POOL>
__global__ void __launch_bounds__(128 * TbLayout<K, H, C0>::NCH, 1)
k_tb_tc(const uint16_t* __restrict__ tbuf, const uint8_t* __restrict__ tcount, const uint16_t* __restrict__ e0,
        const uint16_t* __restrict__ direct, const uint8_t* __restrict__ wimg, const float* __restrict__ params,
        float* __restrict__ psi, long P, int r_takes_ld, int* __restrict__ sched) {
  using S = TbLayout<K, H, C0>;
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int NCH = S::NCH;
  const int g = threadIdx.x >> 7;                    // chain (warpgroup) index
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + S::OFF_BAR) + g;
  uint32_t* tptr = reinterpret_cast<uint32_t*>(smem + S::OFF_BAR + 32);
  int* red = reinterpret_cast<int*>(smem + S::OFF_RED) + 8 * g;
  const int tid = threadIdx.x & 127, warp = tid >> 5, lane = tid & 31;
  const int bar_id = 1 + g;                          // named barrier of this warpgroup

  for (int i = threadIdx.x; i < S::WIMG_B / 16; i += blockDim.x)
    reinterpret_cast<int4*>(smem)[i] = reinterpret_cast<const int4*>(wimg)[i];
  float* par = reinterpret_cast<float*>(smem + S::OFF_PAR);
  for (int i = threadIdx.x; i < S::NPAR; i += blockDim.x) par[i] = params[i];
  if (threadIdx.x == 0) {
    for (int c = 0; c < NCH; ++c) tc::mbar_init(reinterpret_cast<uint64_t*>(smem + S::OFF_BAR) + c, 1);
    tc::fence_mbar_init();
  }
  if (threadIdx.x < 32) tc::tmem_alloc<S::TMEM_COLS>(tptr);
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tptr + g * S::TCOLS;
  const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
  const uint32_t t_acc1 = tmem, t_acc2 = tmem + H, t_accB = tmem + 2 * H;
  uint8_t* chs = smem + S::OFF_CH + g * S::CH_B;
  const float* bB = par;
  const float* wBn = par + C0;
  constexpr int NO = C0 + 3;
  const float* WO = par + 2 * C0;
  const float* bO = WO + 3 * NO;

  constexpr uint32_t PL = S::PL;
  const uint32_t sA1 = tc::smem_u32(chs + S::CH_A1), sA2 = tc::smem_u32(chs + S::CH_A2);
  const uint32_t sA3 = tc::smem_u32(chs + S::CH_A3);
  const uint32_t sW1 = tc::smem_u32(smem + S::OFF_W1), sW2 = tc::smem_u32(smem + S::OFF_W2);
  const uint32_t sWBT = tc::smem_u32(smem + S::OFF_WBT), sWBE = tc::smem_u32(smem + S::OFF_WBE);
  constexpr uint32_t ID_T = tc::idesc_f16(128, H, 1, 1);
  constexpr uint32_t ID_BE = tc::idesc_f16(128, C0, 1, 1);
  constexpr uint32_t ID_BT = tc::idesc_f16(128, C0, 0, 0);
  uint32_t phase = 0;
  const int r = tid;
  constexpr int SBT = S::SBT, SBP = SBT * 128;
  uint16_t* perm = reinterpret_cast<uint16_t*>(chs + S::CH_PERM);
  int* wsum = reinterpret_cast<int*>(chs + S::CH_SCAN);     // [warp][bin]
  const long nsb = (P + SBP - 1) / SBP;
  using V = typename std::conditional<S::VW == 16, uint4,
            typename std::conditional<S::VW == 8, uint2,
            typename std::conditional<S::VW == 4, uint32_t, uint16_t>::type>::type>::type;
  auto load_records = [&](V* dst, long pp, bool ok) {   // the pixel's K*22 contiguous bytes
    if (ok) {
      const V* src = reinterpret_cast<const V*>(tbuf + pp * (K * 11));
#pragma unroll
      for (int i = 0; i < S::NV; ++i) dst[i] = __ldg(src + i);
    } else {
#pragma unroll
      for (int i = 0; i < S::NV; ++i) memset(&dst[i], 0, sizeof(V));
    }
  };

  // Superblocks of SBT tiles: the superblock's pixels are stably sorted by their valid
  // count (bins 0..K, absent pixels last) so that each 128-row tile runs only as many slot
  // rounds as its own largest count.  Per-pixel results do not depend on the row a pixel
  // lands in (each MMA row is an independent dot product), so this is a pure schedule.
  // Superblocks are handed out dynamically (global counter, zeroed before the launch); the
  // next one is claimed one ahead so its inputs can be staged into L2 meanwhile.
  volatile int* sbn = red + 4;
  if (tid == 0) sbn[0] = atomicAdd(sched, 1);
  tc::bar_sync(bar_id, 128);
  long sb = sbn[0];
  for (int it = 0; sb < nsb; ++it) {
    const long q0 = sb * SBP;
    TBP_NOW(tp_sb0);
    if (tid == 0) {   // claim the next superblock and stage its inputs into L2
      const int nx = atomicAdd(sched, 1);
      sbn[(it + 1) & 1] = nx;
      const long q1 = (long)nx * SBP;
      if (q1 < P) {
        const long np = min((long)SBP, P - q1);
        const uint32_t rb = (uint32_t)(np * K * 22) & ~15u, eb = (uint32_t)(np * C0 * 2) & ~15u;
        if (rb) tc::bulk_prefetch_l2(tbuf + q1 * K * 11, rb);
        if (eb) tc::bulk_prefetch_l2(e0 + q1 * C0, eb);
        const uint32_t db = (uint32_t)(np * 6) & ~15u, cb = (uint32_t)np & ~15u;
        if (db && ((q1 * 6) & 15) == 0) tc::bulk_prefetch_l2(direct + q1 * 3, db);
        if (cb) tc::bulk_prefetch_l2(tcount + q1, cb);
      }
    }
    int mj[SBT];
#pragma unroll
    for (int j = 0; j < SBT; ++j) {
      const long q = q0 + j * 128 + r;
      mj[j] = q < P ? min((int)__ldg(tcount + q), K) : K + 1;
    }
    int cnt[K + 2], incl[K + 2];
#pragma unroll
    for (int b = 0; b < K + 2; ++b) {
      int c = 0;
#pragma unroll
      for (int j = 0; j < SBT; ++j) c += mj[j] == b ? 1 : 0;
      cnt[b] = c;
      int x = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xFFFFFFFFu, x, o);
        if (lane >= o) x += y;
      }
      incl[b] = x;
      if (lane == 31) wsum[warp * (K + 2) + b] = x;
    }
    tc::bar_sync(bar_id, 128);
    {
      int base = 0;
#pragma unroll
      for (int b = 0; b < K + 2; ++b) {
        int woff = 0, tot = 0;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const int v = wsum[w * (K + 2) + b];
          woff += w < warp ? v : 0;
          tot += v;
        }
        int pos = base + woff + incl[b] - cnt[b];
#pragma unroll
        for (int j = 0; j < SBT; ++j)
          if (mj[j] == b) perm[pos++] = (uint16_t)((j * 128 + r) | (b << 11));   // row | count
        base += tot;
      }
    }
    tc::bar_sync(bar_id, 128);
    int pe_all[SBT];   // this thread's row of every tile of the superblock (row | count << 11)
#pragma unroll
    for (int v = 0; v < SBT; ++v) pe_all[v] = perm[v * 128 + r];
    TBP_NOW(tp_sb1);
    TBP_ADD(0, tp_sb0, tp_sb1);
  V nraw[S::NV];   // the next tile's records, loaded while this tile's MMAs run
  for (int v = 0; v < SBT; ++v) {
    TBP_NOW(tp_t0);
    int pe = pe_all[0];
#pragma unroll
    for (int u = 1; u < SBT; ++u) pe = v == u ? pe_all[u] : pe;
    const long p = q0 + (pe & 2047);
    const bool pv = p < P;
    const int m = pv ? (pe >> 11) : 0;   // min(tcount, K), read once by the superblock sort
    // ---- 1. records -> registers -> canonical rank -> A1 rows ----
    {
      V raw[S::NV];
      if (v == 0 || !S::PREFETCH) load_records(raw, p, pv);   // else prefetched during the rounds
      else {
#pragma unroll
        for (int i = 0; i < S::NV; ++i) raw[i] = nraw[i];
      }
      // the pixel's K*11 halfwords as 32-bit words; record k starts at halfword 11k
      constexpr int NW = (K * 11 + 1) / 2 + 1;
      uint32_t rw[NW];
#pragma unroll
      for (int i = 0; i < NW; ++i) rw[i] = 0;
      memcpy(rw, raw, K * 22);
#ifdef GN_PROFILE_TB
      {  // force the loads to complete for the phase timer
        uint32_t acc = 0;
#pragma unroll
        for (int i = 0; i < NW; ++i) acc ^= rw[i];
        if (acc == 0x12345u) gn_tb_prof[15] += 1;
      }
#endif
      TBP_NOW(tp_l1);
      TBP_ADD(12, tp_t0, tp_l1);
      // A1 words of each record (ch0|ch1, .., ch8|ch9, ch10|1.0) and its 64-bit sort key
      // (depth, ch0, ch1, ch2): one PRMT per word for records at odd halfword offsets.
      uint32_t w[K][6];
      uint64_t key[K];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int s0 = 11 * k, wi = s0 >> 1;
        if ((s0 & 1) == 0) {
#pragma unroll
          for (int j = 0; j < 5; ++j) w[k][j] = rw[wi + j];
          w[k][5] = (rw[wi + 5] & 0xFFFFu) | 0x3F800000u;
        } else {
#pragma unroll
          for (int j = 0; j < 5; ++j) w[k][j] = __byte_perm(rw[wi + j], rw[wi + j + 1], 0x5432);
          w[k][5] = (rw[wi + 5] >> 16) | 0x3F800000u;
        }
        const uint32_t khi = __byte_perm(w[k][0], w[k][3], 0x7610);   // depth<<16 | ch0
        const uint32_t klo = __byte_perm(w[k][1], w[k][0], 0x7610);   // ch1<<16 | ch2
        key[k] = ((uint64_t)khi << 32) | klo;
      }
      TBP_NOW(tp_l2);
      TBP_ADD(13, tp_l1, tp_l2);
      int rank[K];
#pragma unroll
      for (int k = 0; k < K; ++k) rank[k] = 0;
#pragma unroll
      for (int i = 1; i < K; ++i) {
#pragma unroll
        for (int j = 0; j < i; ++j) {
          // is record j before record i?  (key, then remaining words, then slot index)
          bool jf = key[j] < key[i];
          if (key[j] == key[i]) {   // rare: full-record tie-break
            jf = true;
#pragma unroll
            for (int c = 1; c < 6; ++c)
              if (w[j][c] != w[i][c]) { jf = w[j][c] < w[i][c]; break; }
          }
          const bool both = i < m;  // both valid (j < i < m); masked slots are never read
          rank[i] += (both && jf) ? 1 : 0;
          rank[j] += (both && !jf) ? 1 : 0;
        }
      }
#pragma unroll
      for (int k = 0; k < K; ++k) {
        if (k < m) {
          const uint32_t dst = sA1 + rank[k] * 2 * PL + r * 16;
          tc::sts128(dst, w[k][0], w[k][1], w[k][2], w[k][3]);
          tc::sts128(dst + PL, w[k][4], w[k][5], 0x3F803F80u, 0);
        } else {
          const uint32_t dst = sA1 + k * 2 * PL + r * 16;
          tc::sts128(dst, 0, 0, 0, 0);
          tc::sts128(dst + PL, 0, 0, 0, 0);
        }
      }
      TBP_NOW(tp_l3);
      TBP_ADD(14, tp_l2, tp_l3);
    }
    // the tile's largest count: slots no pixel uses are skipped (they would add 0)
    {
      const int wm = __reduce_max_sync(0xFFFFFFFFu, (unsigned)m);
      if (lane == 0) red[warp] = wm;
    }
    float ld0 = 0.f, ld1 = 0.f, ld2 = 0.f;
    if (pv) {
      ld0 = __uint_as_float((uint32_t)__ldg(direct + p * 3 + 0) << 16);
      ld1 = __uint_as_float((uint32_t)__ldg(direct + p * 3 + 1) << 16);
      ld2 = __uint_as_float((uint32_t)__ldg(direct + p * 3 + 2) << 16);
    }
    const float inv_m = (POOL == 1 && m > 0) ? 1.f / (float)m : 1.f;
    // e0 operand in the A3 region (A3 is first written after the round-0 commit).
    if (pv) {
      const uint4* e = reinterpret_cast<const uint4*>(e0 + p * C0);
#pragma unroll
      for (int j = 0; j < C0 / 8; ++j) {
        uint4 v = __ldg(e + j);
        tc::sts128(sA3 + j * PL + r * 16, v.x, v.y, v.z, v.w);
      }
    } else {
#pragma unroll
      for (int j = 0; j < C0 / 8; ++j) tc::sts128(sA3 + j * PL + r * 16, 0, 0, 0, 0);
    }
    tc::fence_proxy_async();
    TBP_NOW(tp_t1);
    TBP_ADD(1, tp_t0, tp_t1);
    tc::bar_sync(bar_id, 128);
    TBP_NOW(tp_t2);
    TBP_ADD(2, tp_t1, tp_t2);
    const int Kt = max(max(red[0], red[1]), max(red[2], red[3]));
    TBP_ADD(10, 0, Kt + 1);
    TBP_ADD(11, 0, 1);
    if (tid == 0) {
      tc::fence_after_sync();
#pragma unroll
      for (int q = 0; q < C0 / 16; ++q)
        tc::mma_f16_ss(t_accB, tc::smem_desc(sA3 + 2 * q * PL, PL, 128),
                       tc::smem_desc(sWBE + 2 * q * C0 * 16, C0 * 16, 128), ID_BE, q > 0);
      if (Kt > 0)
        tc::mma_f16_ss(t_acc1, tc::smem_desc(sA1, PL, 128), tc::smem_desc(sW1, H * 16, 128), ID_T, 0);
      tc::mma_commit(mbar);
    }
    if (S::PREFETCH && v + 1 < SBT) {   // prefetch the next tile's records (latency hidden by the rounds)
      int pe2 = pe_all[0];
#pragma unroll
      for (int u = 1; u < SBT; ++u) pe2 = v + 1 == u ? pe_all[u] : pe2;
      const long p2 = q0 + (pe2 & 2047);
      load_records(nraw, p2, p2 < P);
    }
#pragma unroll 1
    for (int t = 0; t <= Kt; ++t) {
      TBP_NOW(tp_r0);
      tc::mbar_wait(mbar, phase);
      TBP_NOW(tp_r1);
      TBP_ADD(3, tp_r0, tp_r1);
      phase ^= 1;
      tc::fence_after_sync();
      if (t >= 1) {  // epilogue 2 of slot t-1 -> A3 (MMA3(t-2) and the e0 MMA are done)
#pragma unroll
        for (int c = 0; c < H / 32; ++c) {
          uint32_t v[32];
          tc::tmem_ld32(t_acc2 + lane_off + c * 32, v);
          tc::tmem_ld_wait();
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            uint32_t o[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              float lo = __uint_as_float(v[8 * g + 2 * i]), hi = __uint_as_float(v[8 * g + 2 * i + 1]);
              if (POOL == 1) { lo *= inv_m; hi *= inv_m; }
              o[i] = tc::cvt_relu_f16x2(lo, hi);
            }
            tc::sts128(sA3 + (4 * c + g) * PL + r * 16, o[0], o[1], o[2], o[3]);
          }
        }
      }
      if (t < Kt) {  // epilogue 1 of slot t -> A2 (MMA2(t-1) is done)
#pragma unroll
        for (int c = 0; c < H / 32; ++c) {
          uint32_t v[32];
          tc::tmem_ld32(t_acc1 + lane_off + c * 32, v);
          tc::tmem_ld_wait();
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            uint32_t o[4];
#pragma unroll
            for (int i = 0; i < 4; ++i)
              o[i] = tc::cvt_relu_bf16x2(__uint_as_float(v[8 * g + 2 * i]), __uint_as_float(v[8 * g + 2 * i + 1]));
            tc::sts128(sA2 + (4 * c + g) * PL + r * 16, o[0], o[1], o[2], o[3]);
          }
        }
        const uint32_t one = t < m ? 0x3F80u : 0u;
        tc::sts128(sA2 + (H / 8) * PL + r * 16, one | (one << 16), one, 0, 0);
        tc::sts128(sA2 + (H / 8 + 1) * PL + r * 16, 0, 0, 0, 0);
      }
      TBP_NOW(tp_r2);
      TBP_ADD(4, tp_r1, tp_r2);
      tc::fence_before_sync();
      tc::fence_proxy_async();
      tc::bar_sync(bar_id, 128);
      TBP_NOW(tp_r3);
      TBP_ADD(5, tp_r2, tp_r3);
      if (tid == 0) {
        tc::fence_after_sync();
        if (t >= 1) {
#pragma unroll
          for (int q = 0; q < H / 16; ++q)
            tc::mma_f16_ss(t_accB, tc::smem_desc(sA3 + 2 * q * PL, PL, 128),
                           tc::smem_desc(sWBT + 2 * q * C0 * 16, C0 * 16, 128), ID_BT, 1);
        }
        if (t < Kt) {
#pragma unroll
          for (int q = 0; q < S::KA2 / 16; ++q)
            tc::mma_f16_ss(t_acc2, tc::smem_desc(sA2 + 2 * q * PL, PL, 128),
                           tc::smem_desc(sW2 + 2 * q * H * 16, H * 16, 128), ID_T, q > 0);
        }
        if (t + 1 < Kt)
          tc::mma_f16_ss(t_acc1, tc::smem_desc(sA1 + (t + 1) * 2 * PL, PL, 128), tc::smem_desc(sW1, H * 16, 128),
                         ID_T, 0);
        tc::mma_commit(mbar);
      }
    }
    TBP_NOW(tp_e0);
    tc::mbar_wait(mbar, phase);
    phase ^= 1;
    tc::fence_after_sync();
    TBP_NOW(tp_e1);
    TBP_ADD(6, tp_e0, tp_e1);
    // ---- 3. phi and psi ----
    float ps0 = bO[0], ps1 = bO[1], ps2 = bO[2];
    if (r_takes_ld) {
      ps0 = fmaf(WO[0 * NO + C0 + 0], ld0, ps0); ps0 = fmaf(WO[0 * NO + C0 + 1], ld1, ps0); ps0 = fmaf(WO[0 * NO + C0 + 2], ld2, ps0);
      ps1 = fmaf(WO[1 * NO + C0 + 0], ld0, ps1); ps1 = fmaf(WO[1 * NO + C0 + 1], ld1, ps1); ps1 = fmaf(WO[1 * NO + C0 + 2], ld2, ps1);
      ps2 = fmaf(WO[2 * NO + C0 + 0], ld0, ps2); ps2 = fmaf(WO[2 * NO + C0 + 1], ld1, ps2); ps2 = fmaf(WO[2 * NO + C0 + 2], ld2, ps2);
    }
    const float fm = (float)m;
#pragma unroll
    for (int c = 0; c < C0 / 16; ++c) {
      uint32_t v[16];
      tc::tmem_ld16(t_accB + lane_off + c * 16, v);
      tc::tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int o = c * 16 + i;
        const float phi = relu(__uint_as_float(v[i]) + bB[o] + wBn[o] * fm);
        ps0 = fmaf(WO[0 * NO + o], phi, ps0);
        ps1 = fmaf(WO[1 * NO + o], phi, ps1);
        ps2 = fmaf(WO[2 * NO + o], phi, ps2);
      }
    }
    if (pv) { psi[p * 3 + 0] = ps0; psi[p * 3 + 1] = ps1; psi[p * 3 + 2] = ps2; }
    tc::fence_before_sync();
    TBP_NOW(tp_e2);
    TBP_ADD(7, tp_e1, tp_e2);
    tc::bar_sync(bar_id, 128);   // TMEM reads, red[] and perm[] of this tile done before the next
    TBP_NOW(tp_end);
    TBP_ADD(9, tp_t0, tp_end);
  }
    sb = sbn[(it + 1) & 1];   // written before this superblock's barriers, read after them
  }
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc<S::TMEM_COLS>(*tptr);
}

}  // namespace gn
