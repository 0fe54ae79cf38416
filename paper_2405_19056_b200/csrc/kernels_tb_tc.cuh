// kernels_tb_tc.cuh -- the fused T + B + psi kernel on tcgen05.
//
// PAPER.md Eq. eq:SymmetricNN: tau = sum_i h(b_i), h shared; B;
// the psi projection is reading R15.
//
// Work unit: a tile of 128 pixels.  Pixels are grouped in superblocks of TB_SBT tiles and a
// pre-pass (k_tb_sort) orders each superblock's pixels by their valid count n, so a tile
// runs only as many slot rounds as its own largest count.  Per-pixel results do not depend
// on the row a pixel lands in (every MMA row is an independent dot product), so the
// ordering is a pure schedule.
//
// Operands.  A tile row's K records (K*22 contiguous bytes) are copied by cp.async, with
// zero fill beyond the n valid records, straight into the layer-1 operand as 16-byte K-planes
// (plane i = bytes 16i..16i+15 of every row): record k is the K-window of halfwords
// [11k, 11k+11) and its layer-1 MMA reads planes j = floor(11k/8).. with a copy of W1
// placed at column offset 11k - 8j (8 offset copies; two MMAs when the window crosses a
// third plane).  Masked slots therefore never reach shared memory (reading R4: they may
// hold any bits, NaN/Inf included) and the window's neighbouring columns are zeros or
// finite valid records times zero weights.  The biases enter the accumulators through one
// more MMA per layer (ONES x bias block; for layer 2 also the pool's magic 2^23); A2 is
// written to TMEM (tcgen05.st) and layer 2 reads its A operand from TMEM.
//
// Warp specialisation.  A CTA runs NCH independent "chains"; a chain has three roles, all
// indexed by tile row r = TMEM lane r:
//   E1 (4 warps)  per tile: publish the rows' counts; issue the cp.asyncs of the NEXT
//                 tile's records and e0 (double-buffered operands; completion tracked by
//                 the `loaded` mbarrier, so E1 never waits for global memory);
//                 round t: A2 = ReLU(acc1 + b1) -> bf16 -> TMEM
//                                                    -> MMA: acc2[t&1] = A2 W2^T, acc1 = layer 1 of slot t+1
//                 final: phi = ReLU(accB + b_B + w_Bn n), psi = W_O,d0 phi + W_O,L L_d + b_O -> HBM
//   E2 (4 warps)  pool += Q(acc2[s&1] + b2) for every slot s as its batch completes (acc2
//                 is double-buffered, so this runs beside E1's next slot); then
//                 tau = pool (f16)                   -> MMA: accB = e0 W_B,e0^T + tau W_B,tau^T
//   MMA (1 warp)  one thread issues every tcgen05.mma of the chain, and executes the
//                 generic -> async proxy fence for the operands the others wrote.
// Hand-offs are mbarriers: loaded[b] (cp.async completion of operand buffer b), rdyC (E1 ->
// MMA: counts published), rdyA (E1 -> MMA: A2 written), tstart (E1 -> E2), free2[b] (E2 -> MMA: acc2
// buffer b read), rdyF (E2 -> MMA: tau written), done1 (commit -> E1, batches holding a
// layer-1 MMA), done2[b] (commit -> E2, layer-2 batches into buffer b) and doneF (commit ->
// E1, the accB batch).  Each waiter can be at most one
// phase behind its barrier by construction.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace gn {

#ifdef GN_PROFILE_TB
// clock64 breakdown of chain 0 of CTA 0 (diagnostic build only): counters 0-15 are kept by
// E1's thread 0 (16-31 are reserved for the other roles); accumulated in shared memory (a
// global read-modify-write would itself stall the chain) and flushed at exit
__device__ unsigned long long gn_tb_prof[32];
__shared__ unsigned long long gn_tb_sprof[32];
#define TBP_NOW(v) const long long v = clock64()
#define TBP_ADD(i, a, b) \
  if (threadIdx.x == 0) gn_tb_sprof[i] += (unsigned long long)((b) - (a))
#define TBP_INIT() if (threadIdx.x < 32) gn_tb_sprof[threadIdx.x] = 0
#define TBP_FLUSH() if (blockIdx.x == 0 && threadIdx.x < 32) gn_tb_prof[threadIdx.x] += gn_tb_sprof[threadIdx.x]
#else
#define TBP_INIT()
#define TBP_FLUSH()
#define TBP_NOW(v)
#define TBP_ADD(i, a, b)
#endif

constexpr float TB_QSCALE = 4096.0f;            // pool fixed point: 2^12 per unit
constexpr float TB_QMAGIC = 8388608.0f;         // 2^23
constexpr float TB_QMAX = 16777215.0f;          // 2^24 - 1 (saturation at 2048 - 2^-12)
constexpr uint32_t TB_QBITS = 0x4B000000u;      // bits of 2^23
constexpr int TB_SBT = 32;                      // tiles per superblock (the count sort's window)
constexpr int TB_SBP = TB_SBT * 128;

// Small per-network constants, passed by value so the epilogues read them from the
// constant bank (FFMA operands) instead of shared memory.
struct TbParams {
  float bB[32];          // B bias
  float wBn[32];         // B weight of the count channel n
  float WO[3 * 35];      // [3][C0+3]: output 1x1 over [d0 ; L_d] (L_d part zero if R does not take it)
  float bO[4];
};

// ---------------------------------------------------------------------------------------
// Pre-pass: per superblock of TB_SBP pixels, a counting sort by min(n, K) (absent pixels,
// beyond P, last).  perm[sb*SBP + i] = (pixel offset in the superblock) | (count << 16).
// TB_SBP/8 threads x 8 consecutive pixels (one 8-byte load); the per-thread bin counts are packed
// two 16-bit fields per word and prefix-summed across the block in one pass; the sorted
// superblock is staged in shared memory and written with 16-byte stores.  The order inside
// a bin is deterministic but irrelevant (every MMA row is independent).
template <int K>
__global__ void __launch_bounds__(TB_SBP / 8) k_tb_sort(const uint8_t* __restrict__ tcount, uint32_t* __restrict__ perm,
                                                        long P) {
  constexpr int NT = TB_SBP / 8, NW = NT / 32;   // threads x 8 pixels; per-bin totals <= TB_SBP < 2^16
  static_assert(NT % 32 == 0 && TB_SBP < 65536, "sort block");
  constexpr int NB = K + 2, NV = (NB + 1) / 2;
  __shared__ uint32_t wtot[NW][NV];
  __shared__ uint16_t soff[NT][NB + 1];
  __shared__ __align__(16) uint32_t sperm[TB_SBP];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const long q0 = (long)blockIdx.x * TB_SBP + 8 * t;
  int bin[8];
  if (q0 + 8 <= P && (reinterpret_cast<uintptr_t>(tcount + q0) & 7) == 0) {
    const uint2 u = __ldg(reinterpret_cast<const uint2*>(tcount + q0));
#pragma unroll
    for (int j = 0; j < 8; ++j) bin[j] = min((int)(((j < 4 ? u.x : u.y) >> (8 * (j & 3))) & 0xFF), K);
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j) bin[j] = q0 + j < P ? min((int)__ldg(tcount + q0 + j), K) : K + 1;
  }
  uint32_t own[NV], v[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    uint32_t c = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) c += (bin[j] >> 1) == i ? 1u << (16 * (bin[j] & 1)) : 0u;
    own[i] = v[i] = c;
  }
#pragma unroll
  for (int o = 1; o < 32; o <<= 1)
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, v[i], o);
      if (lane >= o) v[i] += y;
    }
  if (lane == 31)
#pragma unroll
    for (int i = 0; i < NV; ++i) wtot[warp][i] = v[i];
  __syncthreads();
  uint32_t tot[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    uint32_t pre = 0, all = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const uint32_t x = wtot[w][i];
      pre += w < warp ? x : 0u;
      all += x;
    }
    v[i] = v[i] - own[i] + pre;   // exclusive prefix of this thread, per bin
    tot[i] = all;
  }
  int base = 0;
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const int fld = 16 * (b & 1);
    soff[t][b] = (uint16_t)(base + (int)((v[b >> 1] >> fld) & 0xFFFF));
    base += (int)((tot[b >> 1] >> fld) & 0xFFFF);
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    int r = 0;
#pragma unroll
    for (int i = 0; i < j; ++i) r += bin[i] == bin[j] ? 1 : 0;
    sperm[soff[t][bin[j]] + r] = (uint32_t)(8 * t + j) | ((uint32_t)bin[j] << 16);
  }
  __syncthreads();
  uint4* dst = reinterpret_cast<uint4*>(perm + (long)blockIdx.x * TB_SBP);
  dst[2 * t] = reinterpret_cast<const uint4*>(sperm)[2 * t];
  dst[2 * t + 1] = reinterpret_cast<const uint4*>(sperm)[2 * t + 1];
}

template <int K, int H, int C0>
struct TbLayout {
  static constexpr int PL = 128 * 16;                 // one 8-column K-plane of a 128-row operand
  static constexpr int REC_B = K * 22;                // bytes of one pixel's records
  static constexpr bool ASYNC = REC_B % 16 == 0;      // records copied by 16-byte cp.async
  static constexpr int NPL = (REC_B + 15) / 16;       // record planes per row
  static constexpr int A1_PL = NPL + 2;               // + 2 zero planes (a window may reach past the last record)
  static constexpr int W1_B = 8 * 4 * H * 16;         // 8 offset copies x 4 planes x H rows
  static constexpr int W2_B = H * H * 2;
  static constexpr int WBT_B = C0 * H * 2;
  static constexpr int WBE_B = C0 * C0 * 2;
  static constexpr int ONES_B = 128 * 16 * 2;         // bias MMAs: A = ONES (columns 0..3 = 1)
  static constexpr int BB_B = H * 16 * 2;              //            B = [b1 pieces] / [2^23, b2 2^12 pieces]
  static constexpr int WIMG_B = W1_B + W2_B + WBT_B + WBE_B + ONES_B + 2 * BB_B;
  static constexpr int OFF_W1 = 0, OFF_W2 = OFF_W1 + W1_B, OFF_WBT = OFF_W2 + W2_B, OFF_WBE = OFF_WBT + WBT_B;
  static constexpr int OFF_ONES = OFF_WBE + WBE_B, OFF_BB1 = OFF_ONES + ONES_B, OFF_BB2 = OFF_BB1 + BB_B;
  static constexpr int OFF_BAR = (WIMG_B + 15) / 16 * 16;   // per chain 12 mbarrier slots; then the tmem ptr
  static constexpr int OFF_RED = OFF_BAR + 4 * 96 + 16;     // per chain 8 ints: warp max counts, Kt, tile ids
  static constexpr int OFF_CH = (OFF_RED + 4 * 32 + 127) / 128 * 128;
  // one chain: the layer-1 operand is double-buffered (the next tile's records copied during
  // this tile) unless that leaves room for only one chain, where two single-buffered chains
  // fit instead (K = 16: 352-byte records); single-buffered, E2 copies the next tile's records
  // right after this tile's last layer-2 batch, overlapping the tile's tail
  static constexpr int CH_REST = 2 * (C0 / 8) * PL + (H / 8) * PL + 128 + 128 * 8 + 144;
  static constexpr int AVAIL = 232448 - 1024 - OFF_CH;
  static constexpr int A1_NB = (AVAIL / (2 * A1_PL * PL + CH_REST) >= 2 || AVAIL / (A1_PL * PL + CH_REST) < 2) ? 2 : 1;
  static constexpr int CH_A1 = 0;                     // A1_NB buffers x A1_PL planes
  static constexpr int CH_E0 = CH_A1 + A1_NB * A1_PL * PL;      // 2 buffers x C0/8 planes
  static constexpr int CH_TAU = CH_E0 + 2 * (C0 / 8) * PL;      // H/8 planes (f16)
  static constexpr int CH_MROW = CH_TAU + (H / 8) * PL;         // 128 x u8: the rows' valid counts
  static constexpr int CH_NPIX = CH_MROW + 128;                 // 128 x i64: the NEXT tile's pixels (-1: none)
  static constexpr int CH_NCNT = CH_NPIX + 128 * 8;             // 128 x u8 its counts; [128] = a next tile exists
  static constexpr int CH_B = CH_NCNT + 144;
  static constexpr int TCOLS = (3 * H + C0 + H / 2 + 31) / 32 * 32;   // acc1, acc2 x2, accB, A2 (packed)
  static constexpr int NCH_T = 512 / TCOLS;
  static constexpr int NCH_S = (232448 - 1024 - OFF_CH) / CH_B;
  static constexpr int NCH = NCH_T < NCH_S ? (NCH_T < 3 ? NCH_T : 3) : (NCH_S < 3 ? NCH_S : 3);
  static constexpr int SMEM = OFF_CH + NCH * CH_B;
  static constexpr int THREADS = NCH * 288;           // warps: E1 (4/chain), E2 (4/chain), MMA (1/chain)
};

// 16-byte cp.async with zero fill: copies `bytes` (0..16) from src, zeros the rest
__device__ __forceinline__ void cp_async16z(uint32_t dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
}
// arrive on `bar` when all of this thread's prior cp.asyncs have completed
__device__ __forceinline__ void cp_async_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(tc::smem_u32(bar)) : "memory");
}

template <int K, int H, int C0, int POOL>
__global__ void __launch_bounds__(TbLayout<K, H, C0>::THREADS, 1)
k_tb_tc(const uint16_t* __restrict__ tbuf, const uint16_t* __restrict__ e0, const uint16_t* __restrict__ direct,
        const uint8_t* __restrict__ wimg, const __grid_constant__ TbParams prm, const uint32_t* __restrict__ perm,
        float* __restrict__ psi, long P, int* __restrict__ sched) {
  using S = TbLayout<K, H, C0>;
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int NCH = S::NCH;
  constexpr uint32_t PL = S::PL;
  constexpr int NO = C0 + 3;
  static_assert(C0 <= 32 && H <= 64 && H % 32 == 0, "TbParams sizes / epilogue chunks");
  const int wg = threadIdx.x >> 5;
  const int role = wg < 4 * NCH ? 0 : wg < 8 * NCH ? 1 : 2;   // E1, E2, MMA
  const int g = role == 2 ? wg - 8 * NCH : (wg >> 2) % NCH;    // chain
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::OFF_BAR) + 12 * g;
  uint64_t* loaded = bars + 0;     // [2]
  uint64_t* rdyA = bars + 2;
  uint64_t* rdyF = bars + 3;
  uint64_t* free2 = bars + 4;      // [2]
  uint64_t* done1 = bars + 6;
  uint64_t* done2 = bars + 7;      // [2]
  uint64_t* tstart = bars + 9;
  uint64_t* doneF = bars + 10;
  uint64_t* rdyC = bars + 11;      // E1 -> MMA: a tile's counts published (separate from rdyA: E1's
                                   // round 0 may follow at once when layer 1 was issued early)
  uint32_t* tptr = reinterpret_cast<uint32_t*>(smem + S::OFF_BAR + 4 * 96);
  volatile int* red = reinterpret_cast<int*>(smem + S::OFF_RED) + 8 * g;   // [0..3] warp max, [4] Kt, [5..7] tile ids

  TBP_INIT();
  for (int i = threadIdx.x; i < S::WIMG_B / 16; i += blockDim.x)
    reinterpret_cast<int4*>(smem)[i] = reinterpret_cast<const int4*>(wimg)[i];
  for (int c = 0; c < NCH; ++c)   // the zero pad planes of the A1 buffers
    for (int i = threadIdx.x; i < S::A1_NB * 2 * (int)PL / 16; i += blockDim.x) {
      const int b = i / (2 * PL / 16), o = i % (2 * PL / 16);
      reinterpret_cast<int4*>(smem + S::OFF_CH + c * S::CH_B + S::CH_A1 + (b * S::A1_PL + S::NPL) * PL)[o] =
          make_int4(0, 0, 0, 0);
    }
  if (threadIdx.x == 0) {
    for (int c = 0; c < NCH; ++c) {
      uint64_t* b = reinterpret_cast<uint64_t*>(smem + S::OFF_BAR) + 12 * c;
      tc::mbar_init(b + 0, 256); tc::mbar_init(b + 1, 256);   // loaded[2]: E2 (records) + E1 (e0)
      tc::mbar_init(b + 2, 128); tc::mbar_init(b + 3, 128);   // rdyA, rdyF
      tc::mbar_init(b + 4, 128); tc::mbar_init(b + 5, 128);   // free2[2]
      tc::mbar_init(b + 6, 1); tc::mbar_init(b + 7, 1); tc::mbar_init(b + 8, 1);   // done1, done2[2]
      tc::mbar_init(b + 9, 128);                              // tstart
      tc::mbar_init(b + 10, 1);                               // doneF
      tc::mbar_init(b + 11, 128);                             // rdyC
    }
    tc::fence_mbar_init();
  }
  if (threadIdx.x < 32) tc::tmem_alloc<512>(tptr);
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tptr + g * S::TCOLS;
  const uint32_t t_acc1 = tmem, t_acc2 = tmem + H, t_accB = tmem + 3 * H, t_a2 = tmem + 3 * H + C0;
  uint8_t* chs = smem + S::OFF_CH + g * S::CH_B;
  volatile uint8_t* mrow = chs + S::CH_MROW;
  volatile long long* nprow = reinterpret_cast<volatile long long*>(chs + S::CH_NPIX);
  volatile uint8_t* ncnt = chs + S::CH_NCNT;
  const uint32_t sA1 = tc::smem_u32(chs + S::CH_A1), sE0 = tc::smem_u32(chs + S::CH_E0);
  const uint32_t sTAU = tc::smem_u32(chs + S::CH_TAU);
  // copy row r's records of a tile (pixel pp, mm valid records) into operand buffer `buf`, zero
  // fill beyond the valid bytes (E2 issues these for the next tile; E1 for the first)
  auto fill_rec = [&](int r, int buf, long pp, int mm, bool ok) {
    const uint32_t a = sA1 + buf * S::A1_PL * PL + r * 16;
    const int vb = ok ? mm * 22 : 0;            // valid bytes of the row
    if (S::ASYNC) {
      const char* src = ok ? reinterpret_cast<const char*>(tbuf + pp * (K * 11)) : reinterpret_cast<const char*>(tbuf);
#pragma unroll
      for (int i = 0; i < S::NPL; ++i)
        cp_async16z(a + i * PL, src + 16 * i, (uint32_t)min(max(vb - 16 * i, 0), 16));
    } else {   // rows not 16-byte aligned in global memory: through registers
      const uint16_t* src = tbuf + pp * (K * 11);
#pragma unroll
      for (int i = 0; i < S::NPL; ++i) {
        uint32_t w[4];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const int e = 8 * i + 2 * h;
          const uint32_t lo = 2 * e < vb ? __ldg(src + e) : 0u, hi = 2 * e + 2 < vb ? __ldg(src + e + 1) : 0u;
          w[h] = lo | (hi << 16);
        }
        tc::sts128(a + i * PL, w[0], w[1], w[2], w[3]);
      }
    }
  };
  const long ntiles = (P + TB_SBP - 1) / TB_SBP * TB_SBT;

  if (role == 2) {
    // ------------------------------------------------------------------ MMA warp of chain g
    if ((threadIdx.x & 31) == 0) {
      const uint32_t sW1 = tc::smem_u32(smem + S::OFF_W1), sW2 = tc::smem_u32(smem + S::OFF_W2);
      const uint32_t sWBT = tc::smem_u32(smem + S::OFF_WBT), sWBE = tc::smem_u32(smem + S::OFF_WBE);
      constexpr uint32_t ID_T = tc::idesc_f16(128, H, 1, 1);
      constexpr uint32_t ID_BE = tc::idesc_f16(128, C0, 1, 1);
      constexpr uint32_t ID_BT = tc::idesc_f16(128, C0, 0, 0);
      // layer 1 of slot k from operand buffer `buf`: the record's K-window starts in plane
      // j = 11k/8 at column offset o = 11k mod 8 (W1 copy o); a third plane needs a 2nd MMA
      const uint64_t dONES = tc::smem_desc(tc::smem_u32(smem + S::OFF_ONES), PL, 128);
      const uint64_t dBB1 = tc::smem_desc(tc::smem_u32(smem + S::OFF_BB1), H * 16, 128);
      const uint64_t dBB2 = tc::smem_desc(tc::smem_u32(smem + S::OFF_BB2), H * 16, 128);
      auto layer1 = [&](int k, int buf) {
        const int j = (11 * k) >> 3, o = (11 * k) & 7;
        const uint32_t a = sA1 + ((S::A1_NB == 2 ? buf : 0) * S::A1_PL + j) * PL, w = sW1 + o * 4 * H * 16;
        tc::mma_f16_ss(t_acc1, tc::smem_desc(a, PL, 128), tc::smem_desc(w, H * 16, 128), ID_T, 0);
        if (o > 5)
          tc::mma_f16_ss(t_acc1, tc::smem_desc(a + 2 * PL, PL, 128), tc::smem_desc(w + 2 * H * 16, H * 16, 128), ID_T, 1);
        tc::mma_f16_ss(t_acc1, dONES, dBB1, ID_T, 1);   // + b1
      };
      uint32_t aph = 0, cph = 0, fph = 0, lph[2] = {0, 0}, f2ph[2] = {0, 0};
      bool have_l1 = false;   // this tile's first layer-1 batch was issued after the previous tile
      for (int buf = 0;; buf ^= 1) {
        tc::mbar_wait(rdyC, cph); cph ^= 1;        // the tile's counts
        const int Kt = red[4];
        if (Kt < 0) break;
        const bool next_exists = ncnt[128] != 0;   // written with these counts
        if (!have_l1) {   // (always issued, also for Kt = 0: E1 consumes one layer-1 commit per tile)
          tc::mbar_wait(loaded + buf, lph[buf]); lph[buf] ^= 1;   // its records and e0 (cp.async)
          tc::fence_after_sync();
          tc::fence_proxy_async();
          layer1(0, buf);
          tc::mma_commit(done1);
        } else {
          tc::fence_after_sync();
        }
        // accB = e0 W_B,e0^T now (E1 read the previous tile's accB before publishing these
        // counts); the tau part is added after the pool, so the tile's tail holds only it
        const uint32_t e0b = sE0 + buf * (C0 / 8) * PL;
#pragma unroll
        for (int q = 0; q < C0 / 16; ++q)
          tc::mma_f16_ss(t_accB, tc::smem_desc(e0b + 2 * q * PL, PL, 128),
                         tc::smem_desc(sWBE + 2 * q * C0 * 16, C0 * 16, 128), ID_BE, q > 0);
        for (int t = 0; t < Kt; ++t) {
          tc::mbar_wait(rdyA, aph); aph ^= 1;      // A2 of slot t in TMEM (acc1 read)
          if (t >= 2) { tc::mbar_wait(free2 + (t & 1), f2ph[t & 1]); f2ph[t & 1] ^= 1; }   // acc2[t&1] read
          tc::fence_after_sync();
#pragma unroll
          for (int q = 0; q < H / 16; ++q)
            tc::mma_f16_ts(t_acc2 + (t & 1) * H, t_a2 + q * 8, tc::smem_desc(sW2 + 2 * q * H * 16, H * 16, 128), ID_T,
                           q > 0);
          tc::mma_f16_ss(t_acc2 + (t & 1) * H, dONES, dBB2, ID_T, 1);   // + 2^23 + b2 2^12
          if (t + 1 < Kt) { layer1(t + 1, buf); tc::mma_commit(done1); }
          tc::mma_commit(done2 + (t & 1));
        }
        if (Kt >= 2) { tc::mbar_wait(free2 + ((Kt - 2) & 1), f2ph[(Kt - 2) & 1]); f2ph[(Kt - 2) & 1] ^= 1; }
        if (Kt >= 1) { tc::mbar_wait(free2 + ((Kt - 1) & 1), f2ph[(Kt - 1) & 1]); f2ph[(Kt - 1) & 1] ^= 1; }
        tc::mbar_wait(rdyF, fph); fph ^= 1;        // tau written
        tc::fence_after_sync();
        tc::fence_proxy_async();
        if (Kt > 0) {
#pragma unroll
          for (int q = 0; q < H / 16; ++q)
            tc::mma_f16_ss(t_accB, tc::smem_desc(sTAU + 2 * q * PL, PL, 128),
                           tc::smem_desc(sWBT + 2 * q * C0 * 16, C0 * 16, 128), ID_BT, 1);
        }
        tc::mma_commit(doneF);
        // the next tile's first layer-1 batch now: acc1 is free (E1 read this tile's last slot
        // before the tail), so E1's round 0 of the next tile does not wait for it.  Only after a
        // tile with slot rounds: E1's rdyA arrivals then prove it has consumed every earlier
        // layer-1 commit (after a Kt = 0 tile nothing would stop this commit from landing two
        // phases ahead of E1's wait -- the parity would alias)
        have_l1 = next_exists && Kt > 0;
        if (have_l1) {
          tc::mbar_wait(loaded + (buf ^ 1), lph[buf ^ 1]); lph[buf ^ 1] ^= 1;
          tc::fence_after_sync();
          tc::fence_proxy_async();
          layer1(0, buf ^ 1);
          tc::mma_commit(done1);
        }
      }
    }
  } else if (role == 1) {
    // ------------------------------------------------------------------ E2: the pool
    const int r = threadIdx.x & 127, warp = r >> 5;
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    uint32_t tph = 0, d2ph[2] = {0, 0};
    int nbuf = 1;                 // operand buffer of the next tile
    tc::mbar_arrive(loaded + 0);  // the first tile's records are E1's
    for (;;) {
      tc::mbar_wait(tstart, tph); tph ^= 1;
      const int Kt = red[4];
      if (Kt < 0) break;
      const int m = mrow[r];
      // the next tile's records: double-buffered, now into the other operand buffer (its last
      // reader, the tile before this one, has completed: E2 saw its last batch); single-
      // buffered, after this tile's last layer-2 batch (all its layer-1 MMAs have completed)
      const bool has_next = ncnt[128] != 0;
      const long np_next = has_next ? (long)nprow[r] : -1;
      const int nm_next = has_next ? (int)ncnt[r] : 0;
      auto fill_next = [&]() {
        if (has_next) {
          fill_rec(r, S::A1_NB == 2 ? nbuf : 0, np_next, nm_next, np_next >= 0);
          cp_async_arrive(loaded + nbuf);
        }
      };
      if (S::A1_NB == 2) fill_next();
      uint32_t pool[H];
#pragma unroll
      for (int j = 0; j < H; ++j) pool[j] = 0;
#pragma unroll 1
      for (int s = 0; s < Kt; ++s) {
        const int b = s & 1;
        tc::mbar_wait(done2 + b, d2ph[b]); d2ph[b] ^= 1;
        tc::fence_after_sync();
        // pool += Q(a2): acc2 = 2^23 + (W2 a1 + b2) 2^12 (scale folded into W2, magic and bias
        // added by the bias MMA), rounded to an integer in fp32; the clamps are the ReLU and the
        // saturation, and masked slots clamp to exactly 2^23 (0)
        const float hi = (s < m) ? TB_QMAX : TB_QMAGIC;
#pragma unroll
        for (int c = 0; c < H / 32; ++c) {   // two 16-column loads in flight per wait
          uint32_t u[32];
          tc::tmem_ld16(t_acc2 + b * H + lane_off + c * 32, *reinterpret_cast<uint32_t(*)[16]>(u));
          tc::tmem_ld16(t_acc2 + b * H + lane_off + c * 32 + 16, *reinterpret_cast<uint32_t(*)[16]>(u + 16));
          tc::tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float x = fminf(fmaxf(__uint_as_float(u[i]), TB_QMAGIC), hi);
            pool[c * 32 + i] += __float_as_uint(x);
          }
        }
        tc::fence_before_sync();
        tc::mbar_arrive(free2 + b);
      }
      if (S::A1_NB == 1) fill_next();
      nbuf ^= 1;
      if (Kt > 0) {   // tau = pool (f16) -> its operand
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
          tc::sts128(sTAU + q * PL + r * 16, o[0], o[1], o[2], o[3]);
        }
      }
      tc::mbar_arrive(rdyF);   // release; the MMA thread fences the proxies
    }
  } else {
    // ------------------------------------------------------------------ E1: operands, A2, phi, psi
    const int r = threadIdx.x & 127, warp = r >> 5, lane = r & 31;
    const int bar_id = 1 + g;
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    uint32_t d1ph = 0, dfph = 0;
    auto decode = [&](long tl, int pe, long& pp, int& mm, bool& ok) {   // this thread's pixel of tile tl
      pp = tl / TB_SBT * TB_SBP + (pe & 0xFFFF);
      ok = tl < ntiles && pp < P;
      mm = ok ? (pe >> 16) : 0;
    };
    // copy row r's e0 of a tile into operand buffer `buf` (its records: fill_rec, by E2)
    auto fill_e0 = [&](int buf, long pp, bool ok) {
      const uint32_t eb = sE0 + buf * (C0 / 8) * PL + r * 16;
      const uint16_t* es = ok ? e0 + pp * C0 : e0;
#pragma unroll
      for (int j = 0; j < C0 / 8; ++j) cp_async16z(eb + j * PL, es + 8 * j, ok ? 16u : 0u);
      cp_async_arrive(loaded + buf);
    };

    // Tile pipeline: tile ids are claimed three ahead (atomics), the perm entry of the tile
    // after next is loaded one tile ahead, and the next tile's operands are copied during
    // this one, so no global latency sits on a critical path.
    int claim = 0;
    if (r == 0) { red[5] = atomicAdd(sched, 1); red[6] = atomicAdd(sched, 1); claim = atomicAdd(sched, 1); }
    tc::bar_sync(bar_id, 128);
    long tile = red[5], ntile = red[6];
    long p, np;
    int m, nm;
    bool pv, npv;
    decode(tile, tile < ntiles ? (int)__ldg(perm + tile * 128 + r) : 0, p, m, pv);
    if (tile < ntiles) { fill_rec(r, 0, p, m, pv); fill_e0(0, p, pv); }
    decode(ntile, ntile < ntiles ? (int)__ldg(perm + ntile * 128 + r) : 0, np, nm, npv);
    for (int it = 0; tile < ntiles; ++it) {
      TBP_NOW(tp_t0);
      const int buf = it & 1;
      // ---- prologue: publish the counts (and the next tile's pixels, whose records E2 copies);
      // copy the next tile's e0
      mrow[r] = (uint8_t)m;
      nprow[r] = npv ? (long long)np : -1ll;
      ncnt[r] = (uint8_t)nm;
      if (r == 0) ncnt[128] = ntile < ntiles ? 1 : 0;
      {
        const int wm = __reduce_max_sync(0xFFFFFFFFu, (unsigned)m);
        if (lane == 0) red[warp] = wm;
        if (r == 0) { red[5 + (it + 2) % 3] = claim; claim = atomicAdd(sched, 1); }
      }
      tc::bar_sync(bar_id, 128);
      const int Kt = max(max(red[0], red[1]), max(red[2], red[3]));
      const long nntile = red[5 + (it + 2) % 3];
      if (r == 0) red[4] = Kt;
      tc::mbar_arrive(rdyC);
      tc::mbar_arrive(tstart);
      float ld0 = 0.f, ld1 = 0.f, ld2 = 0.f;   // consumed after the slot rounds (latency hidden)
      if (pv) {
        ld0 = __uint_as_float((uint32_t)__ldg(direct + p * 3 + 0) << 16);
        ld1 = __uint_as_float((uint32_t)__ldg(direct + p * 3 + 1) << 16);
        ld2 = __uint_as_float((uint32_t)__ldg(direct + p * 3 + 2) << 16);
      }
      if (ntile < ntiles) fill_e0(buf ^ 1, np, npv);   // buffer buf^1's e0 was last read by the previous tile's accB batch
      const int nnpe = nntile < ntiles ? (int)__ldg(perm + nntile * 128 + r) : 0;   // decoded next iteration
      TBP_NOW(tp_t1);
      TBP_ADD(1, tp_t0, tp_t1);
      TBP_ADD(10, 0, Kt + 1);
      TBP_ADD(11, 0, 1);
      if (Kt == 0) { tc::mbar_wait(done1, d1ph); d1ph ^= 1; }   // the tile's (unused) first layer-1 batch
      // ---- slot rounds: A2 of slot t -> TMEM
#pragma unroll 1
      for (int t = 0; t < Kt; ++t) {
        TBP_NOW(tp_r0);
        tc::mbar_wait(done1, d1ph); d1ph ^= 1;   // batch t-1: acc1 holds slot t
        tc::fence_after_sync();
        TBP_NOW(tp_r1);
        TBP_ADD(3, tp_r0, tp_r1);
        uint32_t u[H];
#pragma unroll
        for (int c = 0; c < H / 32; ++c)
          tc::tmem_ld32(t_acc1 + lane_off + c * 32, *reinterpret_cast<uint32_t(*)[32]>(u + 32 * c));
        tc::tmem_ld_wait();
        uint32_t o[H / 2];
#pragma unroll
        for (int i = 0; i < H / 2; ++i)
          o[i] = tc::cvt_relu_bf16x2(__uint_as_float(u[2 * i]), __uint_as_float(u[2 * i + 1]));   // b1 is in acc1
#pragma unroll
        for (int c = 0; c < H / 32; ++c) tc::tmem_st16(t_a2 + lane_off + 16 * c, o + 16 * c);
        tc::tmem_st_wait();
        tc::fence_before_sync();
        tc::mbar_arrive(rdyA);
        TBP_NOW(tp_r2);
        TBP_ADD(4, tp_r1, tp_r2);
      }
      // ---- final
      TBP_NOW(tp_f0);
      tc::mbar_wait(doneF, dfph); dfph ^= 1;     // accB
      tc::fence_after_sync();
      TBP_NOW(tp_f1);
      TBP_ADD(6, tp_f0, tp_f1);
      const float* WO = prm.WO;
      float ps0 = prm.bO[0], ps1 = prm.bO[1], ps2 = prm.bO[2];
      ps0 = fmaf(WO[0 * NO + C0 + 0], ld0, ps0); ps0 = fmaf(WO[0 * NO + C0 + 1], ld1, ps0); ps0 = fmaf(WO[0 * NO + C0 + 2], ld2, ps0);
      ps1 = fmaf(WO[1 * NO + C0 + 0], ld0, ps1); ps1 = fmaf(WO[1 * NO + C0 + 1], ld1, ps1); ps1 = fmaf(WO[1 * NO + C0 + 2], ld2, ps1);
      ps2 = fmaf(WO[2 * NO + C0 + 0], ld0, ps2); ps2 = fmaf(WO[2 * NO + C0 + 1], ld1, ps2); ps2 = fmaf(WO[2 * NO + C0 + 2], ld2, ps2);
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
          ps0 = fmaf(WO[0 * NO + o], phi, ps0);
          ps1 = fmaf(WO[1 * NO + o], phi, ps1);
          ps2 = fmaf(WO[2 * NO + o], phi, ps2);
        }
      }
      if (pv) { psi[p * 3 + 0] = ps0; psi[p * 3 + 1] = ps1; psi[p * 3 + 2] = ps2; }
      tc::fence_before_sync();
      TBP_NOW(tp_end);
      TBP_ADD(8, tp_f1, tp_end);
      TBP_ADD(9, tp_t0, tp_end);
      // advance the tile pipeline
      tile = ntile; p = np; m = nm; pv = npv;
      ntile = nntile;
      decode(ntile, nnpe, np, nm, npv);
    }
    // stop the MMA warp and E2
    tc::bar_sync(bar_id, 128);
    if (r == 0) red[4] = -1;
    tc::bar_sync(bar_id, 128);
    tc::mbar_arrive(rdyC);
    tc::mbar_arrive(tstart);
  }
  tc::fence_before_sync();
  __syncthreads();
  TBP_FLUSH();
  if (threadIdx.x < 32) tc::tmem_dealloc<512>(*tptr);
}

}  // namespace gn
