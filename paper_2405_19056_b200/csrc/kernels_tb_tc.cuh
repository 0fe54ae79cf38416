// kernels_tb_tc.cuh -- the fused T + B + psi kernel on tcgen05.
//
// PAPER.md Eq. eq:SymmetricNN: tau = sum_i h(b_i), h shared; B;
// the psi projection is reading R15.
//
// Work unit: a tile of 128 pixels (MMA row / TMEM lane r = pixel r).  Pixels are grouped in
// superblocks of TB_SBT tiles and a pre-pass (k_tb_sort) orders each superblock's pixels by
// their valid count n, so a tile runs only as many slot "items" as its largest count.
//
// Slot independence BY CONSTRUCTION (reading R5).  Every record is repacked into its own
// K=16 window: slot s of a row = K-columns [16s, 16s+16) = [11 features, 1, 1, 1, 0, 0], and
// W1's window = [W1 (depth column x 2^-7), b1 as three exact bf16 pieces, 0, 0].  So layer 1
// of EVERY slot is the same single MMA instruction shape over a window at the same column
// offsets (the bias summed inside it), layer 2 the same four TMEM-A MMAs, and the pool an
// exact integer sum: a fragment's contribution does not depend on the slot it arrived in
// (measured in tools/ubench_t2.cu: one K=16 MMA sums its products position-independently;
// round 1's split windows did not).  Masked slots (k >= n) are zero windows written by the
// loader, so their bits (NaN/Inf allowed, reading R4) never reach shared memory.
//
// Pool (R5): a2 = ReLU(W2 a1 + b2) enters as Q = round(a2 * 2^12) via
//   v = sat(acc2 + b2 2^-11)        (W2 pre-scaled by 2^-11: one FFMA.SAT = bias, ReLU and the
//                                    saturation at a2 = 2048)
//   pool += bits(1 + v) - bits(1)   (v + 1 has ulp 2^-23, i.e. 2^-12 in a2 units)
// -- integer adds, so any order of the valid slots gives the same bits.
//
// Warp roles (one CTA per SM, 17 warps):
//   w0       MMA: one thread issues every tcgen05.mma / commit
//   w1..w4   loader: claims tiles, reads the count-sorted perm, the valid records (16-byte
//            loads of the valid prefix only), e0 and L_d; repacks the records into the K=16
//            slot windows (A1, 2 buffers), e0 into its operand (E0, 3 buffers), per-tile meta
//   w5..w8   E1: A2 = bf16(ReLU(acc1)) written back INTO acc1's first H/2 columns (layer 2
//            reads its A operand from TMEM); per tile, one tile late: phi, psi -> HBM
//   w9..w16  E2: two warps per TMEM lane quadrant, H/2 channels each: the fixed-point pool;
//            per tile tau -> f16 -> TMEM (the B MMA's A operand)
// Software pipeline: acc1 and acc2 are 2-deep rings, so layer 1 of item i+1 and E1 of item
// i+1 overlap layer 2 of item i, and E2 of item i overlaps both.  B of tile t (e0 part + tau
// part) is issued after layer 2 of tile t+1's item min(1, Kt-1), E1's phi/psi of tile t right
// after that item's epilogue (the pool of tile t has then had a full item to finish).
// Hand-offs are mbarriers; each waiter is provably at most one phase behind.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace gn {

constexpr uint32_t TB_ONE_BITS = 0x3F800000u;   // bits of 1.0f (the pool's per-fragment offset)
constexpr float TB_VSCALE = 1.0f / 2048.0f;     // a2 -> v = a2 2^-11 (saturation at a2 = 2048)
constexpr float TB_QUNIT = 1.0f / 4096.0f;      // one pool unit = 2^-12
constexpr int TB_SBT = 32;                      // tiles per superblock (the count sort's window)
constexpr int TB_SBP = TB_SBT * 128;

// Small per-network constants, passed by value so the epilogues read them from the
// constant bank (FFMA operands) instead of shared memory.
struct TbParams {
  float bB[32];          // B bias
  float wBn[32];         // B weight of the count channel n
  float WO[3 * 35];      // [3][C0+3]: output 1x1 over [d0 ; L_d] (L_d part zero if R does not take it)
  float bO[4];
  float b2s[64];         // b2 2^-11 (the pool's FFMA.SAT addend)
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

// ---------------------------------------------------------------------------------------
template <int K, int H, int C0>
struct TbLayout {
  static constexpr int PL = 128 * 16;                 // one 8-column K-plane of a 128-row operand
  static constexpr int A1_B = K * 2 * PL;             // a tile's layer-1 operand: slot s = planes 2s, 2s+1
  static constexpr int E0_B = (C0 / 8) * PL;          // a tile's e0 operand
  static constexpr int W1_B = 2 * H * 16;             // [2 planes][H][8]: W1 | b1 pieces | 0
  static constexpr int W2_B = H * H * 2;
  static constexpr int WBE_B = C0 * C0 * 2;
  static constexpr int WBT_B = C0 * H * 2;            // f16
  static constexpr int WIMG_B = W1_B + W2_B + WBE_B + WBT_B;
  static constexpr int OFF_W1 = 0, OFF_W2 = OFF_W1 + W1_B, OFF_WBE = OFF_W2 + W2_B, OFF_WBT = OFF_WBE + WBE_B;
  static constexpr int NA = 2, NE = 3;                // A1 ring, E0 / meta ring
  static constexpr int OFF_A1 = (WIMG_B + 1023) / 1024 * 1024;
  static constexpr int OFF_E0 = OFF_A1 + NA * A1_B;
  // per-tile meta: pixel ids, counts, L_d (E1's psi needs them one tile late), Kt, tile id
  static constexpr int M_PIX = 0, M_LD = 128 * 8, M_CNT = M_LD + 128 * 12, M_KT = M_CNT + 128, META_B = M_KT + 16;
  static constexpr int OFF_META = OFF_E0 + NE * E0_B;
  static constexpr int NBAR = 24;
  static constexpr int OFF_BAR = (OFF_META + NE * META_B + 15) / 16 * 16;
  static constexpr int OFF_MISC = OFF_BAR + NBAR * 8;   // tmem ptr, loader scratch
  static constexpr int SMEM = OFF_MISC + 64;
  static constexpr int NWARP = 17, THREADS = 32 * NWARP;
  static constexpr int T_ACC1 = 0, T_ACC2 = 2 * H, T_ACCB = 4 * H, T_TAU = 4 * H + 2 * C0;   // TMEM columns
  static_assert(T_TAU + H <= 512, "TMEM");
  static_assert(SMEM <= 232448 - 1024, "shared memory");
};

// layer-1 window repack of one record (8 words) from the row's words W starting at halfword 11s
template <int S>
__device__ __forceinline__ void tb_window(const uint32_t* W, bool valid, uint32_t (&o)[8]) {
  constexpr uint32_t ONE = 0x3F80u;   // bf16 1.0
  if ((S & 1) == 0) {
    constexpr int a = 11 * S / 2;
#pragma unroll
    for (int k = 0; k < 5; ++k) o[k] = W[a + k];
    o[5] = (W[a + 5] & 0xFFFFu) | (ONE << 16);
  } else {
    constexpr int a = (11 * S - 1) / 2;
#pragma unroll
    for (int k = 0; k < 5; ++k) o[k] = __byte_perm(W[a + k], W[a + k + 1], 0x5432);
    o[5] = (W[a + 5] >> 16) | (ONE << 16);
  }
  o[6] = ONE | (ONE << 16);
  o[7] = 0;
  if (!valid)
#pragma unroll
    for (int k = 0; k < 8; ++k) o[k] = 0;
}

template <int S, int NS>
struct TbWindows {   // slots S..S+NS-1 of a pass whose words start at the pass's first record
  __device__ __forceinline__ static void run(const uint32_t* W, int m_rel, uint32_t a1, int slot0, int r) {
    if constexpr (NS > 0) {
      uint32_t o[8];
      tb_window<S>(W, S < m_rel, o);
      const uint32_t dst = a1 + (uint32_t)(2 * (slot0 + S)) * (128 * 16) + r * 16;
      tc::sts128(dst, o[0], o[1], o[2], o[3]);
      tc::sts128(dst + 128 * 16, o[4], o[5], o[6], o[7]);
      TbWindows<S + 1, NS - 1>::run(W, m_rel, a1, slot0, r);
    }
  }
};

__device__ __forceinline__ uint32_t tb_ld_nc(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint4 tb_ld_nc4(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ float ffma_sat(float a, float b, float c) {
  float d;
  asm("fma.rn.sat.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// mbarrier phase bits of a small ring, kept in one register (runtime indices would put an
// array in local memory)
template <int V> struct TbInt { static constexpr int value = V; };

struct TbPh {
  uint32_t v = 0;
  __device__ __forceinline__ uint32_t operator[](int i) const { return (v >> i) & 1u; }
  __device__ __forceinline__ void flip(int i) { v ^= 1u << i; }
};

template <int K, int H, int C0, int POOL>
__global__ void __launch_bounds__(TbLayout<K, H, C0>::THREADS, 1)
k_tb_tc(const uint16_t* __restrict__ tbuf, const uint16_t* __restrict__ e0, const uint16_t* __restrict__ direct,
        const uint8_t* __restrict__ wimg, const __grid_constant__ TbParams prm, const uint32_t* __restrict__ perm,
        float* __restrict__ psi, long P, int* __restrict__ sched) {
  using S = TbLayout<K, H, C0>;
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr uint32_t PL = S::PL;
  constexpr int NO = C0 + 3;
  constexpr int LAG = 1;   // B / psi of tile t follow item min(LAG, Kt-1) of tile t+1
  static_assert(C0 <= 32 && (H == 32 || H == 64), "TbParams sizes / epilogue chunks");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::OFF_BAR);
  uint64_t* tileReady = bars + 0;   // [3] loader -> all (4 warp arrivals)
  uint64_t* metaFree = bars + 3;    // [3] MMA commit (B) + E1 (4) + E2 (8) -> loader
  uint64_t* a1Free = bars + 6;      // [2] MMA commit after the tile's last layer-1 MMA -> loader
  uint64_t* done1 = bars + 8;       // [2] commit -> E1 (acc1 ring)
  uint64_t* rdyA = bars + 10;       // [2] E1 (4) -> MMA: A2 in acc1
  uint64_t* done2 = bars + 12;      // [2] commit -> E2 (acc2 ring)
  uint64_t* free2 = bars + 14;      // [2] E2 (8) -> MMA: acc2 read
  uint64_t* tauRdy = bars + 16;     // [2] E2 (8) -> MMA: tau of the tile in TMEM
  uint64_t* doneB = bars + 18;      // [2] commit -> E1 (psi) and E2 (tau buffer reuse)
  uint64_t* accBfree = bars + 20;   // [2] E1 (4) -> MMA: accB read
  uint32_t* tptr = reinterpret_cast<uint32_t*>(smem + S::OFF_MISC);
  volatile int* lred = reinterpret_cast<volatile int*>(smem + S::OFF_MISC + 16);   // [2][4] warp max counts
  volatile int* ids = reinterpret_cast<volatile int*>(smem + S::OFF_MISC + 48);    // [4] claimed tile ids
  auto meta = [&](int e) -> uint8_t* { return smem + S::OFF_META + e * S::META_B; };

  for (int i = threadIdx.x; i < S::WIMG_B / 16; i += blockDim.x)
    reinterpret_cast<int4*>(smem)[i] = reinterpret_cast<const int4*>(wimg)[i];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 3; ++i) { tc::mbar_init(tileReady + i, 4); tc::mbar_init(metaFree + i, 13); }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(a1Free + i, 1); tc::mbar_init(done1 + i, 1); tc::mbar_init(rdyA + i, 4);
      tc::mbar_init(done2 + i, 1); tc::mbar_init(free2 + i, 8); tc::mbar_init(tauRdy + i, 8);
      tc::mbar_init(doneB + i, 1); tc::mbar_init(accBfree + i, 4);
    }
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc<512>(tptr);
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tptr;
  const long ntiles = (P + TB_SBP - 1) / TB_SBP * TB_SBT;

  if (warp == 0) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      const uint32_t sW1 = tc::smem_u32(smem + S::OFF_W1), sW2 = tc::smem_u32(smem + S::OFF_W2);
      const uint32_t sWBE = tc::smem_u32(smem + S::OFF_WBE), sWBT = tc::smem_u32(smem + S::OFF_WBT);
      const uint32_t sA1 = tc::smem_u32(smem + S::OFF_A1), sE0 = tc::smem_u32(smem + S::OFF_E0);
      constexpr uint32_t ID_T = tc::idesc_f16(128, H, 1, 1);
      constexpr uint32_t ID_BE = tc::idesc_f16(128, C0, 1, 1);
      constexpr uint32_t ID_BT = tc::idesc_f16(128, C0, 0, 0);
      const uint64_t dW1 = tc::smem_desc(sW1, H * 16, 128);
      TbPh trph, aph, f2ph, tph, bfph;
      int i1 = 0, i2 = 0;
      auto layer1 = [&](int t, int s) {   // tile t's slot s -> acc1[i1 & 1]
        const uint32_t a = sA1 + (uint32_t)(t & 1) * S::A1_B + (uint32_t)(2 * s) * PL;
        tc::mma_f16_ss(tmem + S::T_ACC1 + (i1 & 1) * H, tc::smem_desc(a, PL, 128), dW1, ID_T, 0);
        tc::mma_commit(done1 + (i1 & 1));
        ++i1;
      };
      auto blend = [&](int u, int Ku) {   // B of tile u: accB = e0 W_B,e0^T + tau W_B,tau^T
        const int ab = u & 1, e = u % 3;
        tc::mbar_wait(accBfree + ab, bfph[ab] ^ 1); bfph.flip(ab);   // E1 read tile u-2's accB
        tc::mbar_wait(tauRdy + ab, tph[ab]); tph.flip(ab);           // E2 wrote tau(u) (even Ku = 0)
        tc::fence_after_sync();
        const uint32_t dB = tmem + S::T_ACCB + ab * C0;
#pragma unroll
        for (int q = 0; q < C0 / 16; ++q)
          tc::mma_f16_ss(dB, tc::smem_desc(sE0 + (uint32_t)e * S::E0_B + 2 * q * PL, PL, 128),
                         tc::smem_desc(sWBE + 2 * q * C0 * 16, C0 * 16, 128), ID_BE, q > 0);
        if (Ku > 0)
#pragma unroll
          for (int q = 0; q < H / 16; ++q)
            tc::mma_f16_ts(dB, tmem + S::T_TAU + ab * (H / 2) + 8 * q,
                           tc::smem_desc(sWBT + 2 * q * C0 * 16, C0 * 16, 128), ID_BT, 1);
        tc::mma_commit(doneB + ab);
        tc::mma_commit(metaFree + e);
      };
      auto peek = [&](int t) -> int {   // wait for tile t's operands, return its Kt (-1: end)
        tc::mbar_wait(tileReady + t % 3, trph[t % 3]); trph.flip(t % 3);
        return *reinterpret_cast<volatile int*>(meta(t % 3) + S::M_KT);
      };
      int t = 0, Kt = peek(0);
      int pend = -1, pendK = 0;
      if (Kt > 0) layer1(0, 0);
      while (Kt >= 0) {
        int Ktn = 0;
        for (int s = 0; s < Kt; ++s) {
          if (s + 1 < Kt) {
            layer1(t, s + 1);
          } else {   // last item of tile t: its A1 buffer is free once these MMAs complete
            tc::mma_commit(a1Free + (t & 1));
            Ktn = peek(t + 1);
            if (Ktn > 0) layer1(t + 1, 0);
          }
          const int b = i2 & 1;
          tc::mbar_wait(rdyA + b, aph[b]); aph.flip(b);              // A2 of item i2 in acc1[b]
          tc::mbar_wait(free2 + b, f2ph[b] ^ 1); f2ph.flip(b);       // E2 read acc2[b] (item i2-2)
          tc::fence_after_sync();
          const uint32_t d2 = tmem + S::T_ACC2 + b * H, a2 = tmem + S::T_ACC1 + b * H;
#pragma unroll
          for (int q = 0; q < H / 16; ++q)
            tc::mma_f16_ts(d2, a2 + 8 * q, tc::smem_desc(sW2 + 2 * q * H * 16, H * 16, 128), ID_T, q > 0);
          tc::mma_commit(done2 + b);
          ++i2;
          if (s == min(LAG, Kt - 1) && pend >= 0) { blend(pend, pendK); pend = -1; }
        }
        if (Kt == 0) {
          tc::mma_commit(a1Free + (t & 1));
          if (pend >= 0) { blend(pend, pendK); pend = -1; }
          Ktn = peek(t + 1);
          if (Ktn > 0) layer1(t + 1, 0);
        }
        pend = t; pendK = Kt;
        ++t;
        Kt = Ktn;
      }
      if (pend >= 0) blend(pend, pendK);
    }
  } else if (warp <= 4) {
    // ---------------------------------------------------------------- loader
    const int r = (warp - 1) * 32 + lane;
    const uint32_t sA1 = tc::smem_u32(smem + S::OFF_A1), sE0 = tc::smem_u32(smem + S::OFF_E0);
    TbPh mfph, afph;
    int claim = 0;
    if (r == 0) { ids[0] = atomicAdd(sched, 1); ids[1] = atomicAdd(sched, 1); claim = atomicAdd(sched, 1); }
    tc::bar_sync(1, 128);
    long tile = ids[0];
    uint32_t pe = tile < ntiles ? __ldg(perm + tile * 128 + r) : 0u;
    for (int t = 0;; ++t) {
      const int e = t % 3, a = t & 1;
      uint8_t* M = meta(e);
      if (tile >= ntiles) {
        tc::mbar_wait(metaFree + e, mfph[e] ^ 1);
        if (r == 0) *reinterpret_cast<volatile int*>(M + S::M_KT) = -1;
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(tileReady + e);
        break;
      }
      const long p = tile / TB_SBT * TB_SBP + (pe & 0xFFFF);
      const bool pv = p < P;
      const int m = pv ? (int)(pe >> 16) : 0;
      // this row's valid records (16-byte loads of the valid prefix only) and e0, L_d
      constexpr bool V16 = (K * 22) % 16 == 0;
      constexpr int PS = K < 8 ? K : 8;             // slots per repack pass
      constexpr int NW = V16 ? PS * 11 / 2 : 1;     // words per pass
      uint32_t W[NW > 1 ? NW : 1];
      const int mv = min(m, PS);
      if constexpr (V16) {
        const uint4* src = reinterpret_cast<const uint4*>(tbuf + p * (K * 11));
        const int nc = (mv * 22 + 15) / 16;
#pragma unroll
        for (int c = 0; c < NW / 4; ++c) {
          const uint4 v = c < nc ? tb_ld_nc4(src + c) : make_uint4(0, 0, 0, 0);
          W[4 * c] = v.x; W[4 * c + 1] = v.y; W[4 * c + 2] = v.z; W[4 * c + 3] = v.w;
        }
      }
      uint4 ev[C0 / 8];
#pragma unroll
      for (int j = 0; j < C0 / 8; ++j) ev[j] = pv ? tb_ld_nc4(e0 + p * C0 + 8 * j) : make_uint4(0, 0, 0, 0);
      float ldv[3] = {0.f, 0.f, 0.f};
      if (pv)
#pragma unroll
        for (int c = 0; c < 3; ++c) ldv[c] = __uint_as_float((uint32_t)__ldg(direct + p * 3 + c) << 16);
      const long ntile = ids[(t + 1) & 3];
      const uint32_t npe = ntile < ntiles ? __ldg(perm + ntile * 128 + r) : 0u;
      // buffers free: meta / E0 of tile t-3, A1 of tile t-2
      tc::mbar_wait(metaFree + e, mfph[e] ^ 1); mfph.flip(e);
      tc::mbar_wait(a1Free + a, afph[a] ^ 1); afph.flip(a);
      const uint32_t a1 = sA1 + (uint32_t)a * S::A1_B;
      if constexpr (V16) {
        TbWindows<0, PS>::run(W, m, a1, 0, r);
        if constexpr (K > 8) {   // second pass: slots 8..15
          const uint4* src = reinterpret_cast<const uint4*>(tbuf + p * (K * 11) + 8 * 11);
          const int m2 = m - 8, nc = m2 > 0 ? (m2 * 22 + 15) / 16 : 0;
#pragma unroll
          for (int c = 0; c < NW / 4; ++c) {
            const uint4 v = c < nc ? tb_ld_nc4(src + c) : make_uint4(0, 0, 0, 0);
            W[4 * c] = v.x; W[4 * c + 1] = v.y; W[4 * c + 2] = v.z; W[4 * c + 3] = v.w;
          }
          TbWindows<0, K - 8>::run(W, m2, a1, 8, r);
        }
      } else {   // rows not 16-byte aligned in global memory: halfword loads (test shapes)
        const uint16_t* src = tbuf + p * (K * 11);
        for (int s = 0; s < K; ++s) {
          uint32_t w[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) w[k] = 0;
          if (s < m) {
            uint32_t h[12];
#pragma unroll
            for (int i = 0; i < 11; ++i) h[i] = __ldg(src + 11 * s + i);
            h[11] = 0x3F80u;
#pragma unroll
            for (int k = 0; k < 6; ++k) w[k] = h[2 * k] | (h[2 * k + 1] << 16);
            w[6] = 0x3F803F80u;
          }
          const uint32_t dst = a1 + (uint32_t)(2 * s) * PL + r * 16;
          tc::sts128(dst, w[0], w[1], w[2], w[3]);
          tc::sts128(dst + PL, w[4], w[5], w[6], w[7]);
        }
      }
#pragma unroll
      for (int j = 0; j < C0 / 8; ++j)
        tc::sts128(sE0 + (uint32_t)e * S::E0_B + j * PL + r * 16, ev[j].x, ev[j].y, ev[j].z, ev[j].w);
      reinterpret_cast<long long*>(M + S::M_PIX)[r] = pv ? (long long)p : -1ll;
      reinterpret_cast<float*>(M + S::M_LD)[3 * r + 0] = ldv[0];
      reinterpret_cast<float*>(M + S::M_LD)[3 * r + 1] = ldv[1];
      reinterpret_cast<float*>(M + S::M_LD)[3 * r + 2] = ldv[2];
      M[S::M_CNT + r] = (uint8_t)m;
      const int wm = __reduce_max_sync(0xFFFFFFFFu, (unsigned)m);
      if (lane == 0) lred[(t & 1) * 4 + warp - 1] = wm;
      if (r == 0) { ids[(t + 2) & 3] = claim; claim = atomicAdd(sched, 1); }
      tc::bar_sync(1, 128);
      if (r == 0) {
        const int* L = const_cast<const int*>(lred) + (t & 1) * 4;
        *reinterpret_cast<volatile int*>(M + S::M_KT) = max(max(L[0], L[1]), max(L[2], L[3]));
      }
      tc::fence_proxy_async();   // this thread's operand writes -> the tensor core's (async) proxy
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(tileReady + e);
      tile = ntile;
      pe = npe;
    }
  } else if (warp <= 8) {
    // ---------------------------------------------------------------- E1: A2, phi, psi
    const int q = warp & 3, r = q * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    TbPh trph, d1ph, dbph;
    int i = 0;
    auto psi_tile = [&](int u) {
      const int ab = u & 1;
      const uint8_t* M = meta(u % 3);
      tc::mbar_wait(doneB + ab, dbph[ab]); dbph.flip(ab);
      tc::fence_after_sync();
      uint32_t v[C0];
#pragma unroll
      for (int c = 0; c < C0 / 16; ++c)
        tc::tmem_ld16(tmem + lane_off + S::T_ACCB + ab * C0 + 16 * c, *reinterpret_cast<uint32_t(*)[16]>(v + 16 * c));
      tc::tmem_ld_wait();
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(accBfree + ab);
      const long long p = reinterpret_cast<const long long*>(M + S::M_PIX)[r];
      const float fm = (float)M[S::M_CNT + r];
      const float* ld = reinterpret_cast<const float*>(M + S::M_LD) + 3 * r;
      const float ld0 = ld[0], ld1 = ld[1], ld2 = ld[2];
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(metaFree + u % 3);
      const float* WO = prm.WO;
      float ps0 = prm.bO[0], ps1 = prm.bO[1], ps2 = prm.bO[2];
      ps0 = fmaf(WO[0 * NO + C0 + 0], ld0, ps0); ps0 = fmaf(WO[0 * NO + C0 + 1], ld1, ps0); ps0 = fmaf(WO[0 * NO + C0 + 2], ld2, ps0);
      ps1 = fmaf(WO[1 * NO + C0 + 0], ld0, ps1); ps1 = fmaf(WO[1 * NO + C0 + 1], ld1, ps1); ps1 = fmaf(WO[1 * NO + C0 + 2], ld2, ps1);
      ps2 = fmaf(WO[2 * NO + C0 + 0], ld0, ps2); ps2 = fmaf(WO[2 * NO + C0 + 1], ld1, ps2); ps2 = fmaf(WO[2 * NO + C0 + 2], ld2, ps2);
#pragma unroll
      for (int o = 0; o < C0; ++o) {
        const float phi = relu(__uint_as_float(v[o]) + prm.bB[o] + prm.wBn[o] * fm);
        ps0 = fmaf(WO[0 * NO + o], phi, ps0);
        ps1 = fmaf(WO[1 * NO + o], phi, ps1);
        ps2 = fmaf(WO[2 * NO + o], phi, ps2);
      }
      if (p >= 0) { psi[p * 3 + 0] = ps0; psi[p * 3 + 1] = ps1; psi[p * 3 + 2] = ps2; }
    };
    int pend = -1;
    for (int t = 0;; ++t) {
      const int e = t % 3;
      tc::mbar_wait(tileReady + e, trph[e]); trph.flip(e);
      const int Kt = *reinterpret_cast<volatile int*>(meta(e) + S::M_KT);
      if (Kt < 0) break;
#pragma unroll 1
      for (int s = 0; s < Kt; ++s) {
        const int b = i & 1;
        tc::mbar_wait(done1 + b, d1ph[b]); d1ph.flip(b);
        tc::fence_after_sync();
        const uint32_t ta = tmem + lane_off + S::T_ACC1 + b * H;
#pragma unroll
        for (int c = 0; c < H / 32; ++c) {
          uint32_t u[32], o[16];
          tc::tmem_ld32(ta + 32 * c, u);
          tc::tmem_ld_wait();
#pragma unroll
          for (int k = 0; k < 16; ++k) o[k] = tc::cvt_relu_bf16x2(__uint_as_float(u[2 * k]), __uint_as_float(u[2 * k + 1]));
          tc::tmem_st16(ta + 16 * c, o);   // A2 over the columns this thread has read (c = 0 first)
        }
        tc::tmem_st_wait();
        tc::fence_before_sync();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(rdyA + b);
        ++i;
        if (s == min(LAG, Kt - 1) && pend >= 0) { psi_tile(pend); pend = -1; }
      }
      if (Kt == 0 && pend >= 0) { psi_tile(pend); pend = -1; }
      pend = t;
    }
    if (pend >= 0) psi_tile(pend);
  } else {
    // ---------------------------------------------------------------- E2: the pool, tau
    constexpr int HC = H / 2;   // channels per warp
    const int q = warp & 3, r = q * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    // the warp's channel half as a compile-time constant, so the b2 addends are constant-bank
    // operands of the FFMA.SAT (no registers)
    auto e2 = [&](auto hc) {
      constexpr int h = decltype(hc)::value;
      TbPh trph, d2ph, dbph;
      int i = 0;
      for (int t = 0;; ++t) {
        const int e = t % 3, ab = t & 1;
        tc::mbar_wait(tileReady + e, trph[e]); trph.flip(e);
        const int Kt = *reinterpret_cast<volatile int*>(meta(e) + S::M_KT);
        if (Kt < 0) break;
        const int m = meta(e)[S::M_CNT + r];
        uint32_t pool[HC];
#pragma unroll
        for (int j = 0; j < HC; ++j) pool[j] = 0;
#pragma unroll 1
        for (int s = 0; s < Kt; ++s) {
          const int b = i & 1;
          tc::mbar_wait(done2 + b, d2ph[b]); d2ph.flip(b);
          tc::fence_after_sync();
          uint32_t u[HC];
          const uint32_t ta = tmem + lane_off + S::T_ACC2 + b * H + h * HC;
#pragma unroll
          for (int c = 0; c < HC / 16; ++c) tc::tmem_ld16(ta + 16 * c, *reinterpret_cast<uint32_t(*)[16]>(u + 16 * c));
          tc::tmem_ld_wait();
          tc::fence_before_sync();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(free2 + b);
          if (s < m) {
#pragma unroll
            for (int j = 0; j < HC; j += 2) {
              const float v0 = ffma_sat(__uint_as_float(u[j]), 1.f, prm.b2s[h * HC + j]);
              const float v1 = ffma_sat(__uint_as_float(u[j + 1]), 1.f, prm.b2s[h * HC + j + 1]);
              const float2 w = __fadd2_rn(make_float2(v0, v1), make_float2(1.f, 1.f));
              pool[j] += __float_as_uint(w.x);
              pool[j + 1] += __float_as_uint(w.y);
            }
          }
          ++i;
        }
        // tau(t) -> TMEM (its buffer's previous reader, B of tile t-2, has completed)
        if (t >= 2) { tc::mbar_wait(doneB + ab, dbph[ab]); dbph.flip(ab); }
        if (Kt > 0) {
          const uint32_t off = (uint32_t)m * TB_ONE_BITS;
          const float sc = (POOL == 1 && m > 0) ? TB_QUNIT / (float)m : TB_QUNIT;
          uint32_t o[HC / 2];
#pragma unroll
          for (int j = 0; j < HC / 2; ++j)
            o[j] = tc::cvt_relu_f16x2((float)(pool[2 * j] - off) * sc, (float)(pool[2 * j + 1] - off) * sc);
          const uint32_t tt = tmem + lane_off + S::T_TAU + ab * (H / 2) + h * (HC / 2);
          if constexpr (HC / 2 == 16) tc::tmem_st16(tt, o);
          else tc::tmem_st8(tt, o);
          tc::tmem_st_wait();
        }
        tc::fence_before_sync();
        __syncwarp();
        if (lane == 0) { tc::mbar_arrive(tauRdy + ab); tc::mbar_arrive(metaFree + e); }
      }
    };
    if (warp < 13) e2(TbInt<0>{});
    else e2(TbInt<1>{});
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

}  // namespace gn
