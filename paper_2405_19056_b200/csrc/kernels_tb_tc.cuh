// kernels_tb_tc.cuh -- the fused T + B + psi kernel on tcgen05.
//
// PAPER.md Eq. eq:SymmetricNN: tau = sum_i h(b_i), h shared; B;
// the psi projection is reading R15.  One warpgroup ("chain") = one 128-pixel
// tile at a time, thread r owns pixel r (= TMEM lane r = MMA row r).  Per tile:
//   1. each thread loads its pixel's K records (16-byte loads) and stores the A1 row
//      [record | 1 1 1 | 0 0] of valid slot k < m into operand plane k; masked slots get
//      all-zero rows (they may hold any bits, NaN/Inf included: reading R4).  e0 is staged
//      as the operand of accB = e0 W_B,e0^T.
//   2. software-pipelined slot rounds t = 0 .. Kt (Kt = the tile's largest valid count):
//        wait for MMA batch t-1;  epilogue 1 of slot t: A2 = ReLU(acc1) -> bf16 (acc1 has b1)
//        issue MMA batch t:       acc2[t&1] = A2 W2^T,  acc1 = A1[t+1] W1ext^T
//        epilogue 2 of slot t-1:  pool += Q(acc2[(t-1)&1] + b2)   (fixed point, see below)
//      acc2 is double-buffered in TMEM so the pool epilogue runs while batch t executes;
//      the critical path per slot is one MMA batch (5 MMAs of N = H) + epilogue 1.
//   3. tau = pool (f16) -> accB += tau W_B,tau^T;  phi = ReLU(accB + b_B + w_Bn n);
//      psi = W_O,d0 phi + W_O,L L_d + b_O  -> HBM (fp32).  Per-fragment activations never
//      reach HBM.
//
// Permutation invariance (reading R5): each fragment's MLP output depends only
// on its own record (every MMA row is an independent dot product), and the pool adds the
// fragments' ReLU outputs as fixed-point integers, Q(v) = round(v 2^12) saturated to
// [0, 2^23), so the sum is exact and independent of the order of the valid slots; the
// output is bit-identical under any permutation without sorting.  The conversion is one
// FFMA against the magic constant 2^23 (+ the bias, pre-scaled): for x in [2^23, 2^24)
// the fp32 bits are 0x4B000000 + round(v 2^12), and the clamps [2^23, 2^24 - 1] are the
// ReLU and the saturation.  Masked rounds clamp to exactly 2^23 (contribution 0).
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

constexpr float TB_QSCALE = 4096.0f;            // pool fixed point: 2^12 per unit
constexpr float TB_QMAGIC = 8388608.0f;         // 2^23
constexpr float TB_QMAX = 16777215.0f;          // 2^24 - 1 (saturation at 2048 - 2^-12)
constexpr uint32_t TB_QBITS = 0x4B000000u;      // bits of 2^23

// Small per-network constants, passed by value so the epilogues read them from the
// constant bank (FFMA operands) instead of shared memory.
struct TbParams {
  float bB[32];          // B bias
  float wBn[32];         // B weight of the count channel n
  float WO[3 * 35];      // [3][C0+3]: output 1x1 over [d0 ; L_d] (L_d part zero if R does not take it)
  float bO[4];
  float q2[64];          // 2^23 + b2 2^12 (fp32-rounded): the FFMA addend of the pool's fixed point
};

template <int K, int H, int C0>
struct TbLayout {
  static constexpr int W1_B = H * 16 * 2;
  static constexpr int W2_B = H * H * 2;
  static constexpr int WBT_B = C0 * H * 2;
  static constexpr int WBE_B = C0 * C0 * 2;
  static constexpr int WIMG_B = W1_B + W2_B + WBT_B + WBE_B;
  static constexpr int OFF_W1 = 0, OFF_W2 = OFF_W1 + W1_B, OFF_WBT = OFF_W2 + W2_B, OFF_WBE = OFF_WBT + WBT_B;
  static constexpr int PL = 128 * 16;                 // one 8-column K-plane of a 128-row operand
  // one chain (= one warpgroup working on its own tile stream):
  static constexpr int CH_A1 = 0;                     // K slots x 2 planes
  static constexpr int CH_A2 = CH_A1 + K * 2 * PL;    // H/8 planes
  static constexpr int CH_A3 = CH_A2 + (H / 8) * PL;  // H/8 planes (tau, f16); the e0 operand aliases it
  static constexpr int SBT = 8;                       // tiles per superblock (pixels sorted by count)
  // superblock sort: perm (SBT*128 u16, kept for the superblock) and wsum (4 warps x (K+2) ints)
  static constexpr int CH_PERM = CH_A3 + (H / 8) * PL;
  static constexpr int CH_SCAN = CH_PERM + SBT * 128 * 2;
  static_assert(C0 <= H, "the e0 operand aliases the tau operand");
  static constexpr int CH_LD = (CH_SCAN + 4 * (K + 2) * 4 + 15) / 16 * 16;   // 128 x float4: psi's L_d part
  static constexpr int CH_B = (CH_LD + 128 * 16 + 127) / 128 * 128;
  static constexpr int OFF_BAR = (WIMG_B + 15) / 16 * 16;   // 4 mbarriers + tmem ptr
  static constexpr int OFF_RED = OFF_BAR + 48;        // 4 chains x 8 ints: per-warp max count, superblock ids
  static constexpr int OFF_CH = (OFF_RED + 128 + 127) / 128 * 128;
  static constexpr int TCOLS = (3 * H + C0 + 31) / 32 * 32;   // TMEM columns per chain: acc1, acc2 x2, accB
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
        const uint16_t* __restrict__ direct, const uint8_t* __restrict__ wimg, const __grid_constant__ TbParams prm,
        float* __restrict__ psi, long P, int* __restrict__ sched) {
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
  const uint32_t t_acc1 = tmem, t_acc2 = tmem + H, t_accB = tmem + 3 * H;   // acc2: two buffers of H
  uint8_t* chs = smem + S::OFF_CH + g * S::CH_B;
  constexpr int NO = C0 + 3;
  static_assert(C0 <= 32 && H <= 64, "TbParams sizes");

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
    TBP_NOW(tp_sb1);
    TBP_ADD(0, tp_sb0, tp_sb1);
#pragma unroll 1
  V nraw[S::NV];   // the next tile's records, loaded while this tile's MMAs run
  for (int v = 0; v < SBT; ++v) {
    TBP_NOW(tp_t0);
    const int pe = perm[v * 128 + r];   // this thread's row of tile v (row | count << 11)
    const long p = q0 + (pe & 2047);
    const bool pv = p < P;
    const int m = pv ? (pe >> 11) : 0;   // min(tcount, K), read once by the superblock sort
    // ---- 1. records -> A1 rows (valid slot k -> plane k; masked slots -> zero rows) ----
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
      TBP_NOW(tp_l1);
      TBP_ADD(12, tp_t0, tp_l1);
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int s0 = 11 * k, wi = s0 >> 1;
        uint32_t w[6];
        if ((s0 & 1) == 0) {
#pragma unroll
          for (int j = 0; j < 5; ++j) w[j] = rw[wi + j];
          w[5] = (rw[wi + 5] & 0xFFFFu) | 0x3F800000u;
        } else {
#pragma unroll
          for (int j = 0; j < 5; ++j) w[j] = __byte_perm(rw[wi + j], rw[wi + j + 1], 0x5432);
          w[5] = (rw[wi + 5] >> 16) | 0x3F800000u;
        }
        const bool ok = k < m;
        const uint32_t dst = sA1 + k * 2 * PL + r * 16;
        tc::sts128(dst, ok ? w[0] : 0u, ok ? w[1] : 0u, ok ? w[2] : 0u, ok ? w[3] : 0u);
        tc::sts128(dst + PL, ok ? w[4] : 0u, ok ? w[5] : 0u, ok ? 0x3F803F80u : 0u, 0u);
      }
      TBP_NOW(tp_l3);
      TBP_ADD(14, tp_l1, tp_l3);
    }
    // the tile's largest count: slots no pixel uses are skipped (they would add 0)
    {
      const int wm = __reduce_max_sync(0xFFFFFFFFu, (unsigned)m);
      if (lane == 0) red[warp] = wm;
    }
    {  // psi's direct-light part W_O,L L_d + b_O, parked in smem across the slot rounds
      float ld0 = 0.f, ld1 = 0.f, ld2 = 0.f;
      if (pv) {
        ld0 = __uint_as_float((uint32_t)__ldg(direct + p * 3 + 0) << 16);
        ld1 = __uint_as_float((uint32_t)__ldg(direct + p * 3 + 1) << 16);
        ld2 = __uint_as_float((uint32_t)__ldg(direct + p * 3 + 2) << 16);
      }
      const float* WO = prm.WO;
      float ps0 = prm.bO[0], ps1 = prm.bO[1], ps2 = prm.bO[2];
      ps0 = fmaf(WO[0 * NO + C0 + 0], ld0, ps0); ps0 = fmaf(WO[0 * NO + C0 + 1], ld1, ps0); ps0 = fmaf(WO[0 * NO + C0 + 2], ld2, ps0);
      ps1 = fmaf(WO[1 * NO + C0 + 0], ld0, ps1); ps1 = fmaf(WO[1 * NO + C0 + 1], ld1, ps1); ps1 = fmaf(WO[1 * NO + C0 + 2], ld2, ps1);
      ps2 = fmaf(WO[2 * NO + C0 + 0], ld0, ps2); ps2 = fmaf(WO[2 * NO + C0 + 1], ld1, ps2); ps2 = fmaf(WO[2 * NO + C0 + 2], ld2, ps2);
      reinterpret_cast<float4*>(chs + S::CH_LD)[r] = make_float4(ps0, ps1, ps2, 0.f);
    }
    // e0 operand in the A3 region (A3 receives tau after the last slot round).
    if (pv) {
      const uint4* e = reinterpret_cast<const uint4*>(e0 + p * C0);
#pragma unroll
      for (int j = 0; j < C0 / 8; ++j) {
        uint4 q = __ldg(e + j);
        tc::sts128(sA3 + j * PL + r * 16, q.x, q.y, q.z, q.w);
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
    TBP_NOW(tp_p0);
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
    TBP_NOW(tp_p1);
    TBP_ADD(13, tp_p0, tp_p1);
    if (S::PREFETCH && v + 1 < SBT) {   // prefetch the next tile's records (latency hidden by the rounds)
      const int pe2 = perm[(v + 1) * 128 + r];
      const long p2 = q0 + (pe2 & 2047);
      load_records(nraw, p2, p2 < P);
    }
    uint32_t pool[H];
#pragma unroll
    for (int j = 0; j < H; ++j) pool[j] = 0;
    // epilogue 2: pool += Q(acc2 + b2) for slot `slot` from acc2 buffer `buf`; masked slots clamp to 0
    auto epi2 = [&](int slot, int buf) {
      const float hi = (slot < m) ? TB_QMAX : TB_QMAGIC;
      uint32_t u[H];
#pragma unroll
      for (int c = 0; c < H / 32; ++c) tc::tmem_ld32(t_acc2 + buf * H + lane_off + c * 32, *reinterpret_cast<uint32_t(*)[32]>(u + 32 * c));
      tc::tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < H; ++i) {
        float x = fmaf(__uint_as_float(u[i]), TB_QSCALE, prm.q2[i]);
        x = fminf(fmaxf(x, TB_QMAGIC), hi);
        pool[i] += __float_as_uint(x);
      }
    };
#pragma unroll 1
    for (int t = 0; t <= Kt; ++t) {
      TBP_NOW(tp_r0);
      tc::mbar_wait(mbar, phase);   // batch t-1: acc2[(t-1)&1] (slot t-1), acc1 (slot t)
      TBP_NOW(tp_r1);
      TBP_ADD(3, tp_r0, tp_r1);
      phase ^= 1;
      tc::fence_after_sync();
      if (t < Kt) {  // epilogue 1 of slot t -> A2
        uint32_t u[H];
#pragma unroll
        for (int c = 0; c < H / 32; ++c) tc::tmem_ld32(t_acc1 + lane_off + c * 32, *reinterpret_cast<uint32_t(*)[32]>(u + 32 * c));
        tc::tmem_ld_wait();
#pragma unroll
        for (int q = 0; q < H / 8; ++q) {
          uint32_t o[4];
#pragma unroll
          for (int i = 0; i < 4; ++i)
            o[i] = tc::cvt_relu_bf16x2(__uint_as_float(u[8 * q + 2 * i]), __uint_as_float(u[8 * q + 2 * i + 1]));
          tc::sts128(sA2 + q * PL + r * 16, o[0], o[1], o[2], o[3]);
        }
      } else if (Kt > 0) {  // last round: the last slot's pool, then tau = pool (f16) -> A3
        epi2(Kt - 1, (Kt - 1) & 1);
        const uint32_t off = (uint32_t)Kt * TB_QBITS;
        const float sc = (POOL == 1 && m > 0) ? (1.f / TB_QSCALE) / (float)m : 1.f / TB_QSCALE;
#pragma unroll
        for (int q = 0; q < H / 8; ++q) {
          uint32_t o[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float lo = (float)(pool[8 * q + 2 * i] - off) * sc;
            const float hv = (float)(pool[8 * q + 2 * i + 1] - off) * sc;
            o[i] = tc::cvt_relu_f16x2(lo, hv);
          }
          tc::sts128(sA3 + q * PL + r * 16, o[0], o[1], o[2], o[3]);
        }
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
        if (t < Kt) {
#pragma unroll
          for (int q = 0; q < H / 16; ++q)
            tc::mma_f16_ss(t_acc2 + (t & 1) * H, tc::smem_desc(sA2 + 2 * q * PL, PL, 128),
                           tc::smem_desc(sW2 + 2 * q * H * 16, H * 16, 128), ID_T, q > 0);
          if (t + 1 < Kt)
            tc::mma_f16_ss(t_acc1, tc::smem_desc(sA1 + (t + 1) * 2 * PL, PL, 128), tc::smem_desc(sW1, H * 16, 128),
                           ID_T, 0);
        } else if (Kt > 0) {
#pragma unroll
          for (int q = 0; q < H / 16; ++q)
            tc::mma_f16_ss(t_accB, tc::smem_desc(sA3 + 2 * q * PL, PL, 128),
                           tc::smem_desc(sWBT + 2 * q * C0 * 16, C0 * 16, 128), ID_BT, 1);
        }
        tc::mma_commit(mbar);
      }
      TBP_NOW(tp_i1);
      TBP_ADD(8, tp_r3, tp_i1);
      if (t >= 1 && t < Kt) epi2(t - 1, (t - 1) & 1);   // overlaps batch t
      TBP_NOW(tp_i2);
      TBP_ADD(15, tp_i1, tp_i2);
    }
    TBP_NOW(tp_e0);
    tc::mbar_wait(mbar, phase);
    phase ^= 1;
    tc::fence_after_sync();
    TBP_NOW(tp_e1);
    TBP_ADD(6, tp_e0, tp_e1);
    // ---- 3. phi and psi ----
    const float4 pl4 = reinterpret_cast<const float4*>(chs + S::CH_LD)[r];
    float ps0 = pl4.x, ps1 = pl4.y, ps2 = pl4.z;
    const float fm = (float)m;
#pragma unroll
    for (int c = 0; c < C0 / 16; ++c) {
      uint32_t u[16];
      tc::tmem_ld16(t_accB + lane_off + c * 16, u);
      tc::tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int o = c * 16 + i;
        const float phi = relu(__uint_as_float(u[i]) + prm.bB[o] + prm.wBn[o] * fm);
        ps0 = fmaf(prm.WO[0 * NO + o], phi, ps0);
        ps1 = fmaf(prm.WO[1 * NO + o], phi, ps1);
        ps2 = fmaf(prm.WO[2 * NO + o], phi, ps2);
      }
    }
    if (pv) { psi[p * 3 + 0] = ps0; psi[p * 3 + 1] = ps1; psi[p * 3 + 2] = ps2; }
    tc::fence_before_sync();
    TBP_NOW(tp_e2);
    TBP_ADD(7, tp_e1, tp_e2);
    tc::bar_sync(bar_id, 128);   // TMEM reads, red[] and operands of this tile done before the next
    TBP_NOW(tp_end);
    TBP_ADD(9, tp_t0, tp_end);
  }
    sb = sbn[(it + 1) & 1];   // written before this superblock's barriers, read after them
  }
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc<S::TMEM_COLS>(*tptr);
}

}  // namespace gn
