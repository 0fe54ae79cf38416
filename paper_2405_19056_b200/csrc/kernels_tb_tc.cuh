// kernels_tb_tc.cuh -- the fused T + B + psi kernel on tcgen05.
//
// PAPER.md Eq. eq:SymmetricNN: tau = sum_i h(b_i), h shared; B;
// the psi projection is reading R15.
//
// Work unit: a tile of 128 pixels (MMA row / TMEM lane r = pixel r).  Pixels are grouped in
// superblocks of TB_SBT tiles and a pre-pass (k_tb_sort) orders each superblock's pixels by
// their valid count n, so a tile runs only as many slot "items" as its largest count.
//
// Slot independence BY CONSTRUCTION (reading R5).  Every record gets its own K=16 window: slot s
// of a row = K-columns [16s, 16s+16).  Even slots: [11 features, 0, 1, 1, 1, 0]; odd slots
// (copied from the 4-byte-aligned word before the record): [f, 11 features, 1, 1, 1, 0] where f is
// the previous (valid) record's last feature.  W1's window variants: even = [W1 (depth column x
// 2^-7), 0, b1 as three exact bf16 pieces, 0], odd = [0, W1, b1 pieces, 0].  So layer 1 of EVERY
// slot is ONE MMA whose non-zero products are the same 14 (11 + the bias pieces), summed inside
// one instruction -- position-independently (tools/ubench_t2.cu, Part A: a K=16 MMA's sum does not
// depend on the columns its products sit in; round 1's windows split across two MMAs did) -- then
// the same four TMEM-A layer-2 MMAs, and the pool is an exact integer sum: a fragment's
// contribution does not depend on the slot it arrived in.  Masked slots (k >= n) are zero-filled
// (cp.async with source size 0, or stores), so their bits (NaN/Inf allowed, reading R4) never
// reach shared memory; the odd window's f is a valid record's finite feature times a zero weight.
//
// Pool (R5): a2 = ReLU(W2 a1 + b2) enters as Q = round(a2 * 2^12) via
//   v = sat(acc2 + b2 2^-11)        (W2 pre-scaled by 2^-11: one FADD.SAT = bias, ReLU and the
//                                    saturation at a2 = 2048)
//   pool += bits(1 + v) - bits(1)   (v + 1 has ulp 2^-23, i.e. 2^-12 in a2 units)
// -- integer adds, so any order of the valid slots gives the same bits.
//
// Warp roles (one CTA per SM, 21 warps; the TMEM roles take warp % 4 = their lane quadrant):
//   w0        issuer A (one thread): layer 1 of every item (+ its commit)
//   w1        issuer B (one thread): layer 2 of every item (+ its commit).  One thread issues a
//             tcgen05.mma only every ~50 cycles; two reach the N=64 pipe rate (ubench_multi2)
//   w2        issuer C (one thread): B of every tile, as soon as E2 has written the tile's tau
//   w3..w4    loader (two pixel rows per thread): claims tiles, reads the count-sorted perm,
//             copies the valid records into their K=16 slot windows (A1 ring) and e0 into its
//             operand (E0 ring) by cp.async one tile ahead, writes the per-tile meta
//   w5..w8    psi: one warp per quadrant: phi = ReLU(accB + b_B + w_Bn n), psi -> HBM
//   w9..w12   E1: one warp per quadrant, both channel halves: A2 = bf16(ReLU(acc1)) written back
//             INTO acc1 (layer 2 reads its A operand from TMEM)
//   w13..w20  E2: two warps per quadrant, H/2 channels each: the fixed-point pool, tau -> f16 ->
//             TMEM (the B MMA's A operand)
// Software pipeline: acc1 is a NACC1-deep ring (issuer A runs up to NACC1 - 1 items ahead of
// issuer B), acc2 NACC2-deep; the tensor pipe orders nothing across the issuers, so A writes
// acc1[j % NACC1] only after layer 2 of item j - NACC1 (its previous reader) has completed.  B of tile u is issued
// by C once E2 has pooled the tile; the psi warps and C only consume, so they never hold up the
// item pipeline.
// Hand-offs are mbarriers; each waiter is provably at most one phase behind.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace gn {

#ifdef GN_TB_PROF
// Diagnostic build only (-DGN_TB_PROF): 32-bit clock() intervals accumulated in registers
// (constant indices, so the array is scalarised), flushed once per role by one thread at the
// role's end; summed over CTAs (glassnet_debug_tb_prof).  Indices: tools/tb_breakdown.py.
__device__ unsigned long long gn_tb_prof[40];
#define TBP_DECL() uint32_t tbp_acc[40] = {}
#define TBP_NOW(v) const uint32_t v = (uint32_t)clock()
#define TBP_ADD(i, a) (tbp_acc[i] += (uint32_t)clock() - (a))
#define TBP_CNT(i, n) (tbp_acc[i] += (uint32_t)(n))
#define TBP_FLUSH_IF(c)                                                              \
  if (c) {                                                                           \
    _Pragma("unroll") for (int i_ = 0; i_ < 40; ++i_)                                \
      if (tbp_acc[i_]) atomicAdd(&gn_tb_prof[i_], (unsigned long long)tbp_acc[i_]); \
  }
#else
#define TBP_DECL()
#define TBP_NOW(v)
#define TBP_ADD(i, a)
#define TBP_CNT(i, n)
#define TBP_FLUSH_IF(c)
#endif

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
  float b2s[64];         // b2 2^-11 (the pool's FADD.SAT addend)
  int sigma;             // N1: layer 1 also reads e0 at the pixel (W1,sigma)
};

// ---------------------------------------------------------------------------------------
// Pre-pass: per superblock of TB_SBP pixels, a counting sort by min(n, K) (absent pixels,
// beyond P, last).  perm[sb*SBP + i] = (pixel offset in the superblock) | (count << 16).
// TB_SBP/8 threads x 8 consecutive pixels (one 8-byte load); the per-thread bin counts are packed
// two 16-bit fields per word and prefix-summed across the block in one pass; the sorted
// superblock is staged in shared memory and written with 16-byte stores.  The order inside
// a bin is deterministic but irrelevant (every MMA row is independent).
#ifndef GN_SORT_MINB
#define GN_SORT_MINB 2   // two blocks per SM (<= 64 registers): the sort is latency-bound per block
#endif
template <int K>
__global__ void __launch_bounds__(TB_SBP / 8, GN_SORT_MINB) k_tb_sort(const uint8_t* __restrict__ tcount, uint32_t* __restrict__ perm,
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
  static constexpr int W1_B = 2 * 2 * H * 16;         // [variant][2 planes][H][8] (see the loader)
  static constexpr int W2_B = H * H * 2;
  static constexpr int WBE_B = C0 * C0 * 2;
  static constexpr int WBT_B = C0 * H * 2;            // f16
  static constexpr int W1E_B = H * C0 * 2;            // N1: W1's sigma part [C0/8 planes][H][8]
  static constexpr int WIMG_B = W1_B + W2_B + WBE_B + WBT_B + W1E_B;
  static constexpr int OFF_W1 = 0, OFF_W2 = OFF_W1 + W1_B, OFF_WBE = OFF_W2 + W2_B, OFF_WBT = OFF_WBE + WBE_B;
  static constexpr int OFF_W1E = OFF_WBT + WBT_B;
  // per-tile meta: pixel ids, counts, Kt (the psi warps need them until B(u) has completed)
  static constexpr int M_PIX = 0, M_CNT = 128 * 8, M_KT = M_CNT + 128, META_B = M_KT + 16;
  // CP (K even, so every row's records start 4-byte aligned): each record is copied by 4-byte
  // cp.asyncs straight into its slot window, one tile ahead; otherwise halfword loads + stores
  static constexpr bool CP = K % 2 == 0;
#ifndef GN_TB_NE
#define GN_TB_NE 6
#endif
  static constexpr int NE = CP ? GN_TB_NE : 5;        // E0 / meta ring (tiles the loader may run ahead)
  static constexpr int OFF_A1 = (WIMG_B + 1023) / 1024 * 1024;
  static constexpr int REST = NE * E0_B + NE * META_B + 64 * 8 + 128 + 3072;
  static constexpr int LIMIT = 232448 - 1024;
  // A1 ring: as deep as shared memory allows (the loader runs further ahead over short tiles)
#ifndef GN_TB_NAMAX
#define GN_TB_NAMAX 4
#endif
  static constexpr int NA = GN_TB_NAMAX >= 4 && OFF_A1 + 4 * A1_B + REST <= LIMIT ? 4 : OFF_A1 + 3 * A1_B + REST <= LIMIT ? 3 : 2;
  static constexpr int OFF_E0 = OFF_A1 + NA * A1_B;
  static constexpr int OFF_META = OFF_E0 + NE * E0_B;
  static constexpr int NBAR = 46;
  static constexpr int OFF_BAR = (OFF_META + NE * META_B + 15) / 16 * 16;
  static constexpr int OFF_MISC = OFF_BAR + NBAR * 8;   // tmem ptr, loader scratch, blend queue
  static constexpr int SMEM = OFF_MISC + 128;
#ifndef GN_TB_LW
#define GN_TB_LW 2
#endif
  // warps: 3 MMA issuers, LW loader, 4 psi, 4 E1, 8 E2 (the TMEM roles: warp % 4 = lane quadrant)
#ifndef GN_TB_WA
#define GN_TB_WA 0
#define GN_TB_WB 1
#define GN_TB_WC 2
#endif
  static constexpr int W_A = GN_TB_WA, W_B = GN_TB_WB, W_C = GN_TB_WC;   // warps 0..2, sub-partitions 0..2
  static constexpr int LW = GN_TB_LW, W_LD = 3, W_PSI = W_LD + LW, W_E1 = W_PSI + 4, W_E2 = W_E1 + 4;
  static constexpr int NWARP = W_E2 + 8, THREADS = 32 * NWARP;
  static_assert(LW == 1 || LW == 2 || LW == 4, "loader warps");
  // TMEM columns: acc1 ring of 4 (A2 written over its first H/2 columns), acc2 ring of 2,
  // accB x 1, tau x 3 (f16 pairs; E2 writes tau(u) once B(u-3) has completed)
#ifndef GN_TB_NACC1   // (diagnostic builds may override the ring sizes; the TMEM budget is checked below)
#define GN_TB_NACC1 4
#define GN_TB_NACC2 2
#define GN_TB_NACCB 1
#define GN_TB_NTAU 3
#endif
  static constexpr int NACC1 = GN_TB_NACC1, NACC2 = GN_TB_NACC2, NACCB = GN_TB_NACCB, NTAU = GN_TB_NTAU;
  static constexpr int T_ACC1 = 0, T_ACC2 = NACC1 * H, T_ACCB = T_ACC2 + NACC2 * H, T_TAU = T_ACCB + NACCB * C0;
  static_assert(T_TAU + NTAU * (H / 2) <= 512 && NACC1 <= 4 && NACC2 <= 4 && NACCB <= 2 && NTAU <= 4, "TMEM");
  static_assert(SMEM <= LIMIT, "shared memory");
};

// 4-byte cp.async with zero fill beyond `bytes` (0..4), cached in L1 (a record row's sectors
// serve its 6 copies per slot)
__device__ __forceinline__ void cp_async4z(uint32_t dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
}

// 16-byte cp.async with zero fill: copies `bytes` (0..16) from src, zeros the rest of the 16
__device__ __forceinline__ void cp_async16z(uint32_t dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

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
// FADD.SAT: clamp(a + c, 0, 1) in one instruction; c can be a constant-bank operand (an FFMA
// with an immediate multiplier would need c in a register, i.e. an LDC per use)
__device__ __forceinline__ float fadd_sat(float a, float c) {
  float d;
  asm("add.rn.sat.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(c));
  return d;
}

// mbarrier phase bits of a small ring, kept in one register (runtime indices would put an
// array in local memory)
template <int V> struct TbInt { static constexpr int value = V; };

// diagnostic builds only (-DGN_SENS=role, tools/tb_sens.sh): a busy wait of GN_SENS_CYC cycles in
// one role's per-item (per-tile) path, to see which role the kernel's time is sensitive to
#ifdef GN_SENS
#ifndef GN_SENS_CYC
#define GN_SENS_CYC 300
#endif
#define TB_SENS(role) \
  if (GN_SENS == (role)) { const long long s0_ = clock64(); while (clock64() - s0_ < GN_SENS_CYC) { } }
#else
#define TB_SENS(role)
#endif

struct TbPh {
  uint32_t v = 0;
  __device__ __forceinline__ uint32_t operator[](int i) const { return (v >> i) & 1u; }
  __device__ __forceinline__ void flip(int i) { v ^= 1u << i; }
};

#ifndef GN_TB_MAXNREG
#define GN_TB_MAXNREG 80
#endif
// 21 warps, at most 6 per SM sub-partition: 6 x 32 x 80 registers <= 16,384
template <int K, int H, int C0, int POOL>
__global__ void __maxnreg__(GN_TB_MAXNREG)
k_tb_tc(const uint16_t* __restrict__ tbuf, const uint16_t* __restrict__ e0, const uint16_t* __restrict__ direct,
        const uint8_t* __restrict__ wimg, const __grid_constant__ TbParams prm, const uint32_t* __restrict__ perm,
        float* __restrict__ psi, long P, int* __restrict__ sched) {
  using S = TbLayout<K, H, C0>;
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr uint32_t PL = S::PL;
  constexpr int NO = C0 + 3, NE = S::NE, NA = S::NA;
  static_assert(C0 <= 32 && (H == 32 || H == 64), "TbParams sizes / epilogue chunks");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::OFF_BAR);
  uint64_t* tileReady = bars + 0;   // [NE <= 8] loader -> all (2 warp arrivals)
  uint64_t* metaFree = bars + 8;    // [NE] psi (4) + E2 (8, counts read) -> loader
  uint64_t* done1 = bars + 16;      // [NACC1] issuer A's commit of layer 1 of item i -> E1
  uint64_t* rdyA = bars + 20;       // [NACC1] E1 (4) -> issuer B: A2 of item i in acc1[i % NACC1]
  uint64_t* done2 = bars + 24;      // [4] issuer B's commit of layer 2 of item i -> E2, issuer A
  uint64_t* tauRdy = bars + 28;     // [4] E2 (8) -> issuer C: tau of tile u in TMEM tau[u % NTAU]
  uint64_t* doneB = bars + 32;      // [4] issuer C's commit of B(u) -> psi, E2 (tau[u % NTAU] reuse)
  uint64_t* accBfree = bars + 36;   // [NACCB] psi (4) -> issuer C: accB[u % NACCB] read
  uint64_t* a1Free = bars + 38;     // [NA <= 4] E1 (4): the tile's last layer-1 MMA has completed -> loader
  uint64_t* free2 = bars + 42;      // [NACC2 <= 4] E2 (8) -> issuer B: acc2[i % NACC2] read
  static_assert(NE <= 8 && NA <= 4 && 46 <= S::NBAR, "barrier layout");
  constexpr int NACC1 = S::NACC1;
  uint32_t* tptr = reinterpret_cast<uint32_t*>(smem + S::OFF_MISC);
  volatile int* lred = reinterpret_cast<volatile int*>(smem + S::OFF_MISC + 16);   // [2][4] warp max counts
  volatile int* ids = reinterpret_cast<volatile int*>(smem + S::OFF_MISC + 64);    // [8] claimed tile ids
  volatile int* total = reinterpret_cast<volatile int*>(smem + S::OFF_MISC + 96);  // items in the launch (A -> B)
  auto meta = [&](int t) -> uint8_t* { return smem + S::OFF_META + (t % NE) * S::META_B; };

  TBP_DECL();
  for (int i = threadIdx.x; i < S::WIMG_B / 16; i += blockDim.x)
    reinterpret_cast<int4*>(smem)[i] = reinterpret_cast<const int4*>(wimg)[i];
  if constexpr (S::CP)   // every window's constant columns 12..15 = [1, 1, 1, 0] (the copies never touch them)
    for (int i = threadIdx.x; i < NA * K * 128; i += blockDim.x) {
      const int b = i / (K * 128), k = (i / 128) % K, row = i % 128;
      *reinterpret_cast<uint2*>(smem + S::OFF_A1 + b * S::A1_B + (2 * k + 1) * PL + row * 16 + 8) =
          make_uint2(0x3F803F80u, 0x00003F80u);
    }
  if (threadIdx.x == 0) {
    for (int i = 0; i < NE; ++i) { tc::mbar_init(tileReady + i, S::LW); tc::mbar_init(metaFree + i, 12); }
    for (int i = 0; i < NA; ++i) tc::mbar_init(a1Free + i, 4);
    for (int i = 0; i < NACC1; ++i) { tc::mbar_init(done1 + i, 1); tc::mbar_init(rdyA + i, 4); }
    for (int i = 0; i < 4; ++i) tc::mbar_init(done2 + i, 1);
    for (int i = 0; i < S::NACC2; ++i) tc::mbar_init(free2 + i, 8);
    for (int i = 0; i < S::NACCB; ++i) tc::mbar_init(accBfree + i, 4);
    for (int i = 0; i < 4; ++i) { tc::mbar_init(tauRdy + i, 8); tc::mbar_init(doneB + i, 1); }
    *total = 0x7FFFFFFF;
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc<512>(tptr);
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tptr;
  const long ntiles = (P + TB_SBP - 1) / TB_SBP * TB_SBT;

  if (warp <= 2) {
    // ---------------------------------------------------------------- MMA issuers (one thread each):
    // A = layer 1, B = layer 2, C = the tile-level B.  One thread can issue a tcgen05.mma only
    // every ~50 cycles; two reach the N=64 pipe rate (tools/ubench_multi2.cu).  Across the threads
    // the tensor pipe gives no ordering, so A issues layer 1 of item j into acc1[j % NACC1] only
    // after layer 2 of item j - NACC1 (its previous reader) has COMPLETED (done2 commit).
    const uint32_t sW1 = tc::smem_u32(smem + S::OFF_W1), sW2 = tc::smem_u32(smem + S::OFF_W2);
    const uint32_t sWBE = tc::smem_u32(smem + S::OFF_WBE), sWBT = tc::smem_u32(smem + S::OFF_WBT);
    const uint32_t sW1E = tc::smem_u32(smem + S::OFF_W1E);
    const uint32_t sA1 = tc::smem_u32(smem + S::OFF_A1), sE0 = tc::smem_u32(smem + S::OFF_E0);
    constexpr uint32_t ID_T = tc::idesc_f16(128, H, 1, 1);
    constexpr uint32_t ID_BE = tc::idesc_f16(128, C0, 1, 1);
    constexpr uint32_t ID_BT = tc::idesc_f16(128, C0, 0, 0);
    if (warp == S::W_A && lane == 0) {
      // ------------------------------------------------ issuer A: layer 1 of every item
      const uint64_t dW1 = tc::smem_desc(sW1, H * 16, 128), dW1o = tc::smem_desc(sW1 + 2 * H * 16, H * 16, 128);
      TbPh trph, d2ph;
      TBP_NOW(tot0);
      int ct = 0, cs = 0, cK = 0, nL1 = 0;
      auto peek = [&](int t) -> int {   // wait for tile t's operands, return its Kt (-1: end)
        TBP_NOW(w0);
        tc::mbar_wait(tileReady + t % NE, trph[t % NE]); trph.flip(t % NE);
        TBP_ADD(0, w0);
        TBP_CNT(19, 1);
        return *reinterpret_cast<volatile int*>(meta(t) + S::M_KT);
      };
      cK = peek(0);
      while (cK >= 0) {
        if (cs >= cK) {   // next tile (every tile has >= 1 item: Kt = max(1, max n))
          ++ct;
          cK = peek(ct);
          cs = 0;
          if (cK < 0) break;
        }
        if (nL1 >= NACC1) {   // acc1[nL1 % NACC1]'s previous reader, layer 2 of item nL1-NACC1, has completed
          const int pb = (nL1 - NACC1) & 3;
          TBP_NOW(w1);
          tc::mbar_wait(done2 + pb, d2ph[pb]); d2ph.flip(pb);
          TBP_ADD(2, w1);
          tc::fence_after_sync();
        }
        TB_SENS(1);
        TBP_NOW(l0);
        const uint32_t a = sA1 + (uint32_t)(ct % NA) * S::A1_B + (uint32_t)(2 * cs) * PL;
        tc::mma_f16_ss(tmem + S::T_ACC1 + (nL1 % NACC1) * H, tc::smem_desc(a, PL, 128),
                       (S::CP && (cs & 1)) ? dW1o : dW1, ID_T, 0);
        if (prm.sigma)   // N1: + e0 W1,sigma^T, the same two MMAs for every slot of the pixel
#pragma unroll
          for (int q = 0; q < C0 / 16; ++q)
            tc::mma_f16_ss(tmem + S::T_ACC1 + (nL1 % NACC1) * H,
                           tc::smem_desc(sE0 + (uint32_t)(ct % NE) * S::E0_B + 2 * q * PL, PL, 128),
                           tc::smem_desc(sW1E + 2 * q * H * 16, H * 16, 128), ID_T, 1);
        tc::mma_commit(done1 + nL1 % NACC1);
        TBP_ADD(20, l0);
        TBP_CNT(18, 1);
        ++nL1; ++cs;
      }
      // wake issuer B, which waits for rdyA of item nL1 (it does not exist): first let layer 2 of
      // the last items complete -- their rdyA phases must be fully arrived by E1 before this
      // extra arrival, or it would over-arrive an open phase
      for (int k = (nL1 >= NACC1 ? nL1 - NACC1 : 0); k < nL1; ++k) { tc::mbar_wait(done2 + (k & 3), d2ph[k & 3]); d2ph.flip(k & 3); }
      *total = nL1;
      tc::mbar_arrive_cnt(rdyA + nL1 % NACC1, 4);
      TBP_ADD(4, tot0);
      TBP_FLUSH_IF(true);
    } else if (warp == S::W_B && lane == 0) {
      // ------------------------------------------------ issuer B: layer 2 of every item
      TbPh aph, f2ph;
      TBP_NOW(tot0);
      for (int i = 0;; ++i) {
        const int a3 = i % NACC1, b = i % S::NACC2;
        TBP_NOW(w0);
        tc::mbar_wait(rdyA + a3, aph[a3]); aph.flip(a3);             // A2 of item i in acc1[i % 3]
        TBP_ADD(1, w0);
        if (i >= *total) break;
        TBP_NOW(w1);
        tc::mbar_wait(free2 + b, f2ph[b] ^ 1); f2ph.flip(b);         // E2 read acc2[b] (item i-2)
        TBP_ADD(11, w1);
        tc::fence_after_sync();
        TB_SENS(2);
        const uint32_t d2 = tmem + S::T_ACC2 + b * H, a2 = tmem + S::T_ACC1 + a3 * H;
        TBP_NOW(l2a);
#ifndef GN_ABL_L2
#pragma unroll
        for (int q = 0; q < H / 16; ++q)
          tc::mma_f16_ts(d2, a2 + (q / (H / 32)) * (H / 2) + (q % (H / 32)) * 8,   // A2 half h at column h H/2
                         tc::smem_desc(sW2 + 2 * q * H * 16, H * 16, 128), ID_T, q > 0);
#endif
        tc::mma_commit(done2 + (i & 3));
        TBP_ADD(21, l2a);
      }
      TBP_ADD(22, tot0);
      TBP_FLUSH_IF(true);
    } else if (warp == S::W_C && lane == 0) {
      // ------------------------------------------------ issuer C: B of every tile, as soon as E2 has
      // written its tau: accB = e0 W_B,e0^T + tau W_B,tau^T.  Only the psi warps (accB) and E2 (the
      // tau buffer, after B(u-4)) wait for it, so it never holds up the item chain.
      TbPh trph, tph, bfph;
      TBP_NOW(tot0);
      for (int u = 0;; ++u) {
        TBP_NOW(w0);
        tc::mbar_wait(tileReady + u % NE, trph[u % NE]); trph.flip(u % NE);
        if (*reinterpret_cast<volatile int*>(meta(u) + S::M_KT) < 0) break;
        const int ab = u % S::NACCB;
        tc::mbar_wait(accBfree + ab, bfph[ab] ^ 1); bfph.flip(ab);      // psi read tile u-NACCB's accB
        tc::mbar_wait(tauRdy + (u & 3), tph[u & 3]); tph.flip(u & 3);   // E2 wrote tau(u)
        TBP_ADD(3, w0);
        tc::fence_after_sync();
        TB_SENS(7);
        TBP_NOW(bl0);
        const uint32_t dB = tmem + S::T_ACCB + ab * C0;
#pragma unroll
        for (int q = 0; q < C0 / 16; ++q)
          tc::mma_f16_ss(dB, tc::smem_desc(sE0 + (uint32_t)(u % NE) * S::E0_B + 2 * q * PL, PL, 128),
                         tc::smem_desc(sWBE + 2 * q * C0 * 16, C0 * 16, 128), ID_BE, q > 0);
#pragma unroll
        for (int q = 0; q < H / 16; ++q)
          tc::mma_f16_ts(dB, tmem + S::T_TAU + (u % S::NTAU) * (H / 2) + 8 * q,
                         tc::smem_desc(sWBT + 2 * q * C0 * 16, C0 * 16, 128), ID_BT, 1);
        tc::mma_commit(doneB + (u & 3));
        TBP_ADD(23, bl0);
      }
      TBP_ADD(31, tot0);
      TBP_FLUSH_IF(true);
    }
  } else if (warp < S::W_PSI) {
    // ---------------------------------------------------------------- loader
    // LW warps, LR = 4 / LW pixel rows per thread: rows r0 + RS h of every tile
    constexpr int LR = 4 / S::LW, RS = 32 * S::LW;
    const int r0 = (warp - S::W_LD) * 32 + lane;
    const uint32_t sA1 = tc::smem_u32(smem + S::OFF_A1), sE0 = tc::smem_u32(smem + S::OFF_E0);
    TbPh mfph, afph;
    int claim = 0;
    // tile ids are claimed three ahead by thread 0 (ids ring of 8), perm entries read one tile
    // ahead of the tile whose copies are issued
    if (r0 == 0) {
      ids[0] = atomicAdd(sched, 1); ids[1] = atomicAdd(sched, 1); ids[2] = atomicAdd(sched, 1);
      claim = atomicAdd(sched, 1);
    }
    tc::bar_sync(1, RS);
    auto perm_of = [&](long tl, int r) -> uint32_t { return tl < ntiles ? __ldg(perm + tl * 128 + r) : 0u; };
    auto decode = [&](long tl, uint32_t pe, long& p, int& m) {
      p = tl / TB_SBT * TB_SBP + (pe & 0xFFFF);
      m = (tl < ntiles && p < P) ? (int)(pe >> 16) : 0;
      if (!(tl < ntiles && p < P)) p = -1;
    };
    // CP: issue row r of tile tl's copies into A1 buffer ab and E0 slot es: each valid record by
    // six 4-byte cp.asyncs into its window (columns 0..11; even slots start at the record and
    // zero-fill the column after it, odd slots start one halfword early), e0 by 16-byte cp.asyncs
    // into its K-major planes
    auto issue = [&](long tl, uint32_t pe, int r, int ab, int es) {
      long p; int m;
      decode(tl, pe, p, m);
      const char* src = reinterpret_cast<const char*>(tbuf + (p >= 0 ? p : 0) * (K * 11));
      const uint32_t a1 = sA1 + (uint32_t)ab * S::A1_B + r * 16;
      for (int k = 0; k < m; ++k) {
        const char* rs = src + 22 * k - 2 * (k & 1);
        const uint32_t w0 = a1 + (uint32_t)(2 * k) * PL, w1 = w0 + PL;
        cp_async4z(w0, rs, 4u); cp_async4z(w0 + 4, rs + 4, 4u); cp_async4z(w0 + 8, rs + 8, 4u);
        cp_async4z(w0 + 12, rs + 12, 4u); cp_async4z(w1, rs + 16, 4u);
        cp_async4z(w1 + 4, rs + 20, (k & 1) ? 4u : 2u);
      }
      const uint16_t* es_src = p >= 0 ? e0 + p * C0 : e0;
#pragma unroll
      for (int j = 0; j < C0 / 8; ++j)
        cp_async16z(sE0 + (uint32_t)es * S::E0_B + j * PL + r * 16, es_src + 8 * j, p >= 0 ? 16u : 0u);
    };
    long tile = ids[0], ntile = ids[1];
    uint32_t pe[LR], npe[LR];
#pragma unroll
    for (int h = 0; h < LR; ++h) { pe[h] = perm_of(tile, r0 + RS * h); npe[h] = perm_of(ntile, r0 + RS * h); }
    if constexpr (S::CP) {   // tile 0's copies (its operand slots are fresh: they count as waited)
      if (tile < ntiles)
#pragma unroll
        for (int h = 0; h < LR; ++h) issue(tile, pe[h], r0 + RS * h, 0, 0);
      cp_async_commit();
      mfph.flip(0);
      afph.flip(0);
    }
    TBP_NOW(tot0);
    for (int t = 0;; ++t) {
      const int e = t % NE, a = t % NA;
      uint8_t* M = meta(t);
      if (tile >= ntiles) {   // end marker (CP: this slot was waited for one iteration ago)
        if constexpr (!S::CP) tc::mbar_wait(metaFree + e, mfph[e] ^ 1);
        if (r0 == 0) *reinterpret_cast<volatile int*>(M + S::M_KT) = -1;
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(tileReady + e);
        if constexpr (S::CP) cp_async_wait_all();
        TBP_ADD(7, tot0);
        TBP_FLUSH_IF(r0 == 0);
        break;
      }
      TBP_NOW(ld0);
      long p[LR]; int m[LR];
      uint4 ev[LR][C0 / 8];
#pragma unroll
      for (int h = 0; h < LR; ++h) decode(tile, pe[h], p[h], m[h]);
      if constexpr (S::CP) {
        // the next tile's copies first (its E0 / meta slot: tile t+1-NE's consumers are done; its A1
        // buffer: tile t+1-NA's layer-1 MMAs are done), then this tile's (issued one iteration ago)
        TBP_NOW(w0);
        tc::mbar_wait(metaFree + (t + 1) % NE, mfph[(t + 1) % NE] ^ 1); mfph.flip((t + 1) % NE);
        TBP_ADD(5, w0);
        TBP_NOW(w1);
        tc::mbar_wait(a1Free + (t + 1) % NA, afph[(t + 1) % NA] ^ 1); afph.flip((t + 1) % NA);
        TBP_ADD(6, w1);
        TBP_NOW(is0);
#pragma unroll
        for (int h = 0; h < LR; ++h) {
          if (ntile < ntiles) issue(ntile, npe[h], r0 + RS * h, (t + 1) % NA, (t + 1) % NE);
        }
        cp_async_commit();
        TBP_ADD(30, is0);
        TBP_NOW(cw0);
        cp_async_wait_1();
        TBP_ADD(25, cw0);
      } else {
#pragma unroll
        for (int h = 0; h < LR; ++h) {
#pragma unroll
          for (int j = 0; j < C0 / 8; ++j)
            ev[h][j] = p[h] >= 0 ? tb_ld_nc4(e0 + p[h] * C0 + 8 * j) : make_uint4(0, 0, 0, 0);
        }
        TBP_NOW(w0);
        tc::mbar_wait(metaFree + e, mfph[e] ^ 1); mfph.flip(e);   // meta / E0 of tile t-NE
        TBP_ADD(5, w0);
      }
      TBP_NOW(mt0);
      const long nntile = ids[(t + 2) & 7];   // written before the last bar.sync
      uint32_t nnpe[LR];
#pragma unroll
      for (int h = 0; h < LR; ++h) {
        const int r = r0 + RS * h;
        nnpe[h] = perm_of(nntile, r);
        reinterpret_cast<long long*>(M + S::M_PIX)[r] = p[h] >= 0 ? (long long)p[h] : -1ll;
        M[S::M_CNT + r] = (uint8_t)m[h];
      }
      int mm = m[0];
#pragma unroll
      for (int h = 1; h < LR; ++h) mm = max(mm, m[h]);
      const int wm = __reduce_max_sync(0xFFFFFFFFu, (unsigned)mm);
      if (lane == 0) lred[(t & 1) * 4 + warp - S::W_LD] = wm;
      if (r0 == 0) { ids[(t + 3) & 7] = claim; claim = atomicAdd(sched, 1); }
      TBP_ADD(32, mt0);
      TBP_NOW(w2);
      tc::bar_sync(1, RS);
      TBP_ADD(8, w2);
      TBP_NOW(zf0);
      // Kt >= 1 even for a tile of empty pixels (one item of zero records, pooled by nobody): every
      // tile then advances the item pipeline, which bounds how far a blocked consumer can lag
      // (deadlock freedom of the rings)
      int Kt = 1;
#pragma unroll
      for (int w = 0; w < S::LW; ++w) Kt = max(Kt, (int)lred[(t & 1) * 4 + w]);
      if constexpr (S::CP) {
        // masked slots the tile's items reach: zero columns 0..11 (the constant columns stay)
#pragma unroll
        for (int h = 0; h < LR; ++h) {
          const uint32_t a1 = sA1 + (uint32_t)a * S::A1_B + (r0 + RS * h) * 16;
          for (int k = m[h]; k < Kt; ++k) {
            tc::sts128(a1 + (uint32_t)(2 * k) * PL, 0u, 0u, 0u, 0u);
            asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(a1 + (uint32_t)(2 * k + 1) * PL), "r"(0u), "r"(0u)
                         : "memory");
          }
        }
      } else {
        // halfword loads (K odd: rows not 4-byte aligned); even-slot window layout for all slots
        TBP_NOW(w1);
        tc::mbar_wait(a1Free + a, afph[a] ^ 1); afph.flip(a);     // A1 of tile t-NA
        TBP_ADD(6, w1);
#pragma unroll
        for (int h = 0; h < LR; ++h) {
          const int r = r0 + RS * h;
          const uint32_t a1 = sA1 + (uint32_t)a * S::A1_B + r * 16;
          const uint16_t* src = tbuf + (p[h] >= 0 ? p[h] : 0) * (K * 11);
          for (int k = 0; k < Kt; ++k) {
            uint32_t w[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) w[i] = 0;
            if (k < m[h]) {
              uint32_t hv[12];
#pragma unroll
              for (int i = 0; i < 11; ++i) hv[i] = __ldg(src + 11 * k + i);
              hv[11] = 0;
#pragma unroll
              for (int i = 0; i < 6; ++i) w[i] = hv[2 * i] | (hv[2 * i + 1] << 16);
            }
            w[6] = 0x3F803F80u;   // columns 12, 13 = 1
            w[7] = 0x00003F80u;   // column 14 = 1, column 15 = 0
            tc::sts128(a1 + (uint32_t)(2 * k) * PL, w[0], w[1], w[2], w[3]);
            tc::sts128(a1 + (uint32_t)(2 * k + 1) * PL, w[4], w[5], w[6], w[7]);
          }
#pragma unroll
          for (int j = 0; j < C0 / 8; ++j)
            tc::sts128(sE0 + (uint32_t)e * S::E0_B + j * PL + r * 16, ev[h][j].x, ev[h][j].y, ev[h][j].z, ev[h][j].w);
        }
      }
      TBP_ADD(33, zf0);
      TBP_NOW(fe0);
      if (r0 == 0) *reinterpret_cast<volatile int*>(M + S::M_KT) = Kt;
      TB_SENS(5);
      tc::fence_proxy_async();   // this thread's operand writes (and its waited cp.asyncs) -> async proxy
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(tileReady + e);
      TBP_ADD(34, fe0);
      TBP_ADD(26, ld0);
      tile = ntile; ntile = nntile;
#pragma unroll
      for (int h = 0; h < LR; ++h) { pe[h] = npe[h]; npe[h] = nnpe[h]; }
    }
  } else if (warp < S::W_E1) {
    // ---------------------------------------------------------------- psi
    // one warp per TMEM lane quadrant, all C0 channels of accB: phi = ReLU(accB + b_B + w_Bn n),
    // psi = W_O,d0 phi + W_O,L L_d + b_O (reading R15).  Only consumes: waits for B(u)'s commit,
    // frees accB[u % 2] and the tile's meta slot.
    const int q = warp & 3, r = q * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    TbPh trph, dbph;
    TBP_NOW(tot0);
    for (int u = 0;; ++u) {
      const int e = u % NE, ab = u % S::NACCB;
      TBP_NOW(w0);
      tc::mbar_wait(tileReady + e, trph[e]); trph.flip(e);
      TBP_ADD(29, w0);
      const uint8_t* M = meta(u);
      if (*reinterpret_cast<const volatile int*>(M + S::M_KT) < 0) break;
      // L_d of the pixel, loaded before the wait for B(u) (its latency hides behind the wait)
      const long long p = reinterpret_cast<const long long*>(M + S::M_PIX)[r];
      uint32_t ldr[3] = {0u, 0u, 0u};
      if (p >= 0)
#pragma unroll
        for (int c = 0; c < 3; ++c) ldr[c] = __ldg(direct + p * 3 + c);
      TBP_NOW(w1);
      // one warp polls (sleeping between tries: psi is off the critical path), the four follow
      if (warp == S::W_PSI) tc::mbar_wait_sleep(doneB + (u & 3), dbph[u & 3], 256);
      dbph.flip(u & 3);
      tc::bar_sync(2, 128);
      TBP_ADD(28, w1);
      tc::fence_after_sync();
      uint32_t v[C0];
      if constexpr (C0 == 32) tc::tmem_ld32(tmem + lane_off + S::T_ACCB + ab * C0, *reinterpret_cast<uint32_t(*)[32]>(v));
      else tc::tmem_ld16(tmem + lane_off + S::T_ACCB + ab * C0, *reinterpret_cast<uint32_t(*)[16]>(v));
      tc::tmem_ld_wait();
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(accBfree + ab);
      const float fm = (float)M[S::M_CNT + r];
      const float* WO = prm.WO;
      const float ld0 = __uint_as_float(ldr[0] << 16), ld1 = __uint_as_float(ldr[1] << 16), ld2 = __uint_as_float(ldr[2] << 16);
      float o0 = prm.bO[0], o1 = prm.bO[1], o2 = prm.bO[2];
#pragma unroll
      for (int o = 0; o < C0; ++o) {
        const float phi = relu(__uint_as_float(v[o]) + prm.bB[o] + prm.wBn[o] * fm);
        o0 = fmaf(WO[0 * NO + o], phi, o0);
        o1 = fmaf(WO[1 * NO + o], phi, o1);
        o2 = fmaf(WO[2 * NO + o], phi, o2);
      }
      o0 = fmaf(WO[0 * NO + C0 + 0], ld0, o0); o0 = fmaf(WO[0 * NO + C0 + 1], ld1, o0); o0 = fmaf(WO[0 * NO + C0 + 2], ld2, o0);
      o1 = fmaf(WO[1 * NO + C0 + 0], ld0, o1); o1 = fmaf(WO[1 * NO + C0 + 1], ld1, o1); o1 = fmaf(WO[1 * NO + C0 + 2], ld2, o1);
      o2 = fmaf(WO[2 * NO + C0 + 0], ld0, o2); o2 = fmaf(WO[2 * NO + C0 + 1], ld1, o2); o2 = fmaf(WO[2 * NO + C0 + 2], ld2, o2);
      TB_SENS(6);
      if (p >= 0) { psi[p * 3 + 0] = o0; psi[p * 3 + 1] = o1; psi[p * 3 + 2] = o2; }
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(metaFree + e);
    }
    TBP_ADD(27, tot0);
    TBP_FLUSH_IF(warp == S::W_PSI && lane == 0);
  } else if (warp < S::W_E2) {
    // ---------------------------------------------------------------- E1: A2 = bf16(ReLU(acc1)) -> TMEM
    // one warp per TMEM lane quadrant, the two channel halves in turn; half h writes its A2 (H/4
    // packed columns) over the first columns it has itself read: columns [h H/2, h H/2 + H/4).
    constexpr int HC = H / 2;
    const int q = warp & 3;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    TbPh trph, d1ph;
    int i = 0;
    TBP_NOW(tot0);
    for (int t = 0;; ++t) {
      const int e = t % NE;
      TBP_NOW(w9);
      tc::mbar_wait(tileReady + e, trph[e]); trph.flip(e);
      TBP_ADD(10, w9);
      const int Kt = *reinterpret_cast<volatile int*>(meta(t) + S::M_KT);
      if (Kt < 0) break;
#pragma unroll 1
      for (int s = 0; s < Kt; ++s) {
        const int a3 = i % NACC1;
        TBP_NOW(w0);
        // one warp polls the barrier, the group of 4 E1 warps is released by a named barrier
        if (warp == S::W_E1) tc::mbar_wait(done1 + a3, d1ph[a3]);
        d1ph.flip(a3);
        tc::bar_sync(6, 128);
        TBP_ADD(9, w0);
        TBP_NOW(w1);
        tc::fence_after_sync();
        if (s == Kt - 1 && lane == 0) tc::mbar_arrive(a1Free + t % NA);   // the tile's layer-1 MMAs are done
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t ta = tmem + lane_off + S::T_ACC1 + a3 * H + h * HC;
          uint32_t u[HC], o[HC / 2];
          if constexpr (HC == 32) tc::tmem_ld32(ta, *reinterpret_cast<uint32_t(*)[32]>(u));
          else tc::tmem_ld16(ta, *reinterpret_cast<uint32_t(*)[16]>(u));
          tc::tmem_ld_wait();
#pragma unroll
          for (int k = 0; k < HC / 2; ++k)
            o[k] = tc::cvt_relu_bf16x2(__uint_as_float(u[2 * k]), __uint_as_float(u[2 * k + 1]));
          if constexpr (HC == 32) tc::tmem_st16(ta, o);
          else tc::tmem_st8(ta, o);
        }
        tc::tmem_st_wait();
        tc::fence_before_sync();
        __syncwarp();
        TB_SENS(3);
        if (lane == 0) tc::mbar_arrive(rdyA + a3);
        TBP_ADD(16, w1);
        ++i;
      }
    }
    TBP_ADD(12, tot0);
    TBP_FLUSH_IF(warp == S::W_E1 && lane == 0);
  } else {
    // ---------------------------------------------------------------- E2: the pool, tau
    constexpr int HC = H / 2;   // channels per warp
    const int q = warp & 3, r = q * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    // the warp's channel half as a compile-time constant, so the b2 addends are constant-bank
    // operands of the FADD.SAT (no registers)
    auto e2 = [&](auto hc) {
      constexpr int h = decltype(hc)::value;
      TbPh trph, d2ph, dbph;
      int i = 0;
      TBP_NOW(tot0);
      for (int t = 0;; ++t) {
        const int e = t % NE;
        tc::mbar_wait(tileReady + e, trph[e]); trph.flip(e);
        const int Kt = *reinterpret_cast<volatile int*>(meta(t) + S::M_KT);
        if (Kt < 0) break;
        const int m = meta(t)[S::M_CNT + r];
        uint32_t pool[HC];
#pragma unroll
        for (int j = 0; j < HC; ++j) pool[j] = 0;
#pragma unroll 1
        for (int s = 0; s < Kt; ++s) {
          const int b = i % S::NACC2;
          TBP_NOW(w0);
          tc::mbar_wait(done2 + (i & 3), d2ph[i & 3]);   // every E2 warp polls (no named-barrier hop)
          d2ph.flip(i & 3);
          TBP_ADD(13, w0);
          TBP_NOW(w1);
          tc::fence_after_sync();
          uint32_t u[HC];
          const uint32_t ta = tmem + lane_off + S::T_ACC2 + b * H + h * HC;
#ifdef GN_ABL_TMEM
#pragma unroll
          for (int k = 0; k < HC; ++k) u[k] = (uint32_t)(lane + k + ta);
#else
          if constexpr (HC == 32) tc::tmem_ld32(ta, *reinterpret_cast<uint32_t(*)[32]>(u));
          else
#pragma unroll
          for (int c = 0; c < HC / 16; ++c) tc::tmem_ld16(ta + 16 * c, *reinterpret_cast<uint32_t(*)[16]>(u + 16 * c));
          tc::tmem_ld_wait();
#endif
          TBP_ADD(24, w1);
          tc::fence_before_sync();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(free2 + b);
#ifndef GN_ABL_E2ALU
          if (s < m) {
#else
          if (s < m && m > 100) {   // ablation (diagnostic builds): the pool's arithmetic skipped
#endif
#pragma unroll
            for (int j = 0; j < HC; j += 2) {
              const float v0 = fadd_sat(__uint_as_float(u[j]), prm.b2s[h * HC + j]);
              const float v1 = fadd_sat(__uint_as_float(u[j + 1]), prm.b2s[h * HC + j + 1]);
              const float2 w = __fadd2_rn(make_float2(v0, v1), make_float2(1.f, 1.f));
              pool[j] += __float_as_uint(w.x);
              pool[j + 1] += __float_as_uint(w.y);
            }
          }
          TB_SENS(4);
          ++i;
          TBP_ADD(17, w1);
        }
        // tau(t) -> TMEM, once B of tile t-4 (the last reader of this tau buffer) has completed
        TBP_NOW(w5);
        if (t >= S::NTAU) {   // the last reader of this tau buffer, B(t - NTAU), has completed
          const int uo = (t - S::NTAU) & 3;
          tc::mbar_wait(doneB + uo, dbph[uo]); dbph.flip(uo);
        }
        TBP_ADD(14, w5);
        {
          const uint32_t off = (uint32_t)m * TB_ONE_BITS;
          const float sc = (POOL == 1 && m > 0) ? TB_QUNIT / (float)m : TB_QUNIT;
          uint32_t o[HC / 2];
#pragma unroll
          for (int j = 0; j < HC / 2; ++j)
            o[j] = tc::cvt_relu_f16x2((float)(pool[2 * j] - off) * sc, (float)(pool[2 * j + 1] - off) * sc);
          const uint32_t tt = tmem + lane_off + S::T_TAU + (t % S::NTAU) * (H / 2) + h * (HC / 2);
          if constexpr (HC / 2 == 16) tc::tmem_st16(tt, o);
          else tc::tmem_st8(tt, o);
          tc::tmem_st_wait();
          tc::fence_before_sync();
          __syncwarp();
          if (lane == 0) { tc::mbar_arrive(tauRdy + (t & 3)); tc::mbar_arrive(metaFree + e); }
        }
      }
      TBP_ADD(15, tot0);
      TBP_FLUSH_IF(warp == S::W_E2 && lane == 0);
    };
    if (warp < S::W_E2 + 4) e2(TbInt<0>{});
    else e2(TbInt<1>{});
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

}  // namespace gn
