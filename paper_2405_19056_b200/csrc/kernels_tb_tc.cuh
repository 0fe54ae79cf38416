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
// finite valid records times zero weights.  The layer-1 bias is added in epilogue 1; A2
// is written to TMEM (tcgen05.st) and layer 2 reads its A operand from TMEM.
//
// Streaming pipeline (one per CTA, persistent, tiles handed out dynamically).  Slots are
// numbered globally n = 0, 1, ... over the CTA's tiles; acc1, A2 (TMEM) and acc2 (TMEM)
// are double-buffered by n & 1, and e0, tau (smem) and accB (TMEM) by tile parity, so no
// stage waits for a round trip through another:
//   E1 (8 warps)  per tile: publish the NEXT tile's rows and count in a descriptor ring and
//                 copy its records into the other operand buffer (cp.async, zero fill,
//                 coalesced); per slot n: A2[n&1] = ReLU(acc1[n&1] + b1) -> bf16 (TMEM).
//   MMA (1 warp)  per slot n: L2(n): acc2[n&1] = A2[n&1] W2^T, then L1(n+2): acc1[n&1] =
//                 layer 1 of slot n+2 (acc1[n&1] was just read); per tile, once its tau and
//                 e0 are ready: accB[v&1] = e0 W_B,e0^T + tau W_B,tau^T.  It executes the
//                 generic -> async proxy fence for the operands the others wrote.
//   E2 (8 warps)  per slot: pool += Q(acc2[n&1] + b2); per tile: tau = pool (f16) -> smem.
//   E3 (4 warps)  per tile: e0 -> its operand (cp.async); phi = ReLU(accB + b_B + w_Bn n),
//                 psi = W_O,d0 phi + W_O,L L_d + b_O -> HBM.
// Two threads share a TMEM lane in E1 and E2 (warps w and w+4 take column halves).
// Barriers: desc full/empty (ring of 4 tile descriptors), loadedA[b] / loadedE[b]
// (cp.async completion), a1free[b] (commit: layer 1 of a tile done with its records),
// d1[b] (commit: L1 into acc1[b]), rdyA[b] (E1: acc1[b] read, A2[b] written), d2[b]
// (commit: L2 into acc2[b]), free2[b] (E2: acc2[b] read), rdyF[b] (E2: tau of a tile of
// parity b written), tauF[b] / dF[b] (commit: accB batch done, for E2 / E3), e3free[b]
// (E3: accB[b] read).  Every producer's consecutive arrivals on a barrier are separated
// by a wait that implies its consumer consumed the earlier phase.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace gn {

#ifdef GN_PROFILE_TB
// clock64 breakdown of thread 0 (chain 0, E1) of CTA 0 (diagnostic build only): accumulated
// in shared memory (a global read-modify-write would itself stall the chain) and flushed at exit
__device__ unsigned long long gn_tb_prof[16];
__shared__ unsigned long long gn_tb_sprof[16];
#define TBP_NOW(v) const long long v = clock64()
#define TBP_ADD(i, a, b) \
  if (threadIdx.x == 0) gn_tb_sprof[i] += (unsigned long long)((b) - (a))
#define TBP_ADDM(i, a, b) gn_tb_sprof[i] += (unsigned long long)((b) - (a))
#define TBP_INIT() if (threadIdx.x < 16) gn_tb_sprof[threadIdx.x] = 0
#define TBP_FLUSH() if (blockIdx.x == 0 && threadIdx.x < 16) gn_tb_prof[threadIdx.x] += gn_tb_sprof[threadIdx.x]
#else
#define TBP_ADDM(i, a, b)
#define TBP_INIT()
#define TBP_FLUSH()
#define TBP_NOW(v)
#define TBP_ADD(i, a, b)
#endif

constexpr float TB_QSCALE = 4096.0f;            // pool fixed point: 2^12 per unit
constexpr float TB_QMAGIC = 8388608.0f;         // 2^23
constexpr float TB_QMAX = 16777215.0f;          // 2^24 - 1 (saturation at 2048 - 2^-12)
constexpr uint32_t TB_QBITS = 0x4B000000u;      // bits of 2^23
constexpr int TB_SBT = 8;                       // tiles per superblock (the count sort's window)
constexpr int TB_SBP = TB_SBT * 128;

// Small per-network constants, passed by value so the epilogues read them from the
// constant bank (FFMA operands) instead of shared memory.
struct TbParams {
  float bB[32];          // B bias
  float wBn[32];         // B weight of the count channel n
  float WO[3 * 35];      // [3][C0+3]: output 1x1 over [d0 ; L_d] (L_d part zero if R does not take it)
  float bO[4];
  float q2[64];          // 2^23 + b2 2^12 (fp32-rounded): the FFMA addend of the pool's fixed point
  float b1[64];          // layer-1 bias (added in epilogue 1)
};

// ---------------------------------------------------------------------------------------
// Pre-pass: per superblock of TB_SBP pixels, a stable counting sort by min(n, K) (absent
// pixels, beyond P, last).  perm[sb*SBP + i] = (pixel offset in the superblock) | (count << 11).
template <int K>
__global__ void __launch_bounds__(128) k_tb_sort(const uint8_t* __restrict__ tcount, uint16_t* __restrict__ perm,
                                                 long P) {
  __shared__ int wsum[4][K + 2];
  const int r = threadIdx.x, warp = r >> 5, lane = r & 31;
  const long q0 = (long)blockIdx.x * TB_SBP;
  int mj[TB_SBT];
#pragma unroll
  for (int j = 0; j < TB_SBT; ++j) {
    const long q = q0 + j * 128 + r;
    mj[j] = q < P ? min((int)__ldg(tcount + q), K) : K + 1;
  }
  int cnt[K + 2], incl[K + 2];
#pragma unroll
  for (int b = 0; b < K + 2; ++b) {
    int c = 0;
#pragma unroll
    for (int j = 0; j < TB_SBT; ++j) c += mj[j] == b ? 1 : 0;
    cnt[b] = c;
    int x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xFFFFFFFFu, x, o);
      if (lane >= o) x += y;
    }
    incl[b] = x;
    if (lane == 31) wsum[warp][b] = x;
  }
  __syncthreads();
  int base = 0;
#pragma unroll
  for (int b = 0; b < K + 2; ++b) {
    int woff = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const int v = wsum[w][b];
      woff += w < warp ? v : 0;
      tot += v;
    }
    int pos = base + woff + incl[b] - cnt[b];
#pragma unroll
    for (int j = 0; j < TB_SBT; ++j)
      if (mj[j] == b) perm[q0 + pos++] = (uint16_t)((j * 128 + r) | (b << 11));
    base += tot;
  }
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
  static constexpr int WIMG_B = W1_B + W2_B + WBT_B + WBE_B;
  static constexpr int OFF_W1 = 0, OFF_W2 = OFF_W1 + W1_B, OFF_WBT = OFF_W2 + W2_B, OFF_WBE = OFF_WBT + WBT_B;
  static constexpr int OFF_A1 = (WIMG_B + 127) / 128 * 128;     // 2 buffers x A1_PL planes
  static constexpr int OFF_E0 = OFF_A1 + 2 * A1_PL * PL;         // 2 buffers x C0/8 planes
  static constexpr int OFF_TAU = OFF_E0 + 2 * (C0 / 8) * PL;     // 2 buffers x H/8 planes (f16)
  static constexpr int NDESC = 4;
  static constexpr int OFF_DESC = OFF_TAU + 2 * (H / 8) * PL;    // NDESC x 128 int64 rows
  static constexpr int OFF_DKT = OFF_DESC + NDESC * 128 * 8;     // NDESC int: Kt (-1: end of stream)
  static constexpr int OFF_SCR = OFF_DKT + 16;                   // E1 scratch: 8 warp maxima, 3 tile ids
  static constexpr int OFF_BAR = OFF_SCR + 64;                   // mbarriers
  static constexpr int NBAR = 40;
  static constexpr int OFF_TPTR = OFF_BAR + NBAR * 8;
  static constexpr int SMEM = OFF_TPTR + 16;
  // TMEM columns: acc1[2], A2[2] (packed bf16 pairs), acc2[2], accB[2]
  static constexpr int T_ACC1 = 0, T_A2 = 2 * H, T_ACC2 = 3 * H, T_ACCB = 5 * H;
  static constexpr int TCOLS_USED = 5 * H + 2 * C0;
  static constexpr int TCOLS = TCOLS_USED <= 32 ? 32 : TCOLS_USED <= 64 ? 64 : TCOLS_USED <= 128 ? 128
                             : TCOLS_USED <= 256 ? 256 : 512;
  static constexpr int THREADS = 21 * 32;             // warps 0-7 E1, 8-15 E2, 16-19 E3, 20 MMA
  static_assert(SMEM <= 232448 - 1024, "T kernel shared memory");
};

// 16-byte cp.async with zero fill: copies `bytes` (0..16) from src, zeros the rest
__device__ __forceinline__ void cp_async16z(uint32_t dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
// arrive on `bar` when all of this thread's prior cp.asyncs have completed
__device__ __forceinline__ void cp_async_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(tc::smem_u32(bar)) : "memory");
}
// non-blocking test of a phase (test_wait; try_wait would suspend the thread for a while)
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(tc::smem_u32(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}
#ifdef GN_TB_DEBUG
// hang diagnostics (debug build): a wait that polls ~2^22 times logs (once) who waits on what
// into mapped host memory, then keeps waiting
__device__ int* gn_tb_hang;
__device__ __forceinline__ bool gn_tb_victim() {   // the first CTA whose wait times out logs
  const int prev = atomicCAS(gn_tb_hang + 255, 0, (int)blockIdx.x + 1);
  return prev == 0 || prev == (int)blockIdx.x + 1;
}
#endif
// The phase parities a waiter tracks, one bit per barrier of the CTA's barrier array.
struct Phases {
  uint64_t* bar;
  uint32_t bits = 0;
#ifdef GN_TB_DEBUG
  __device__ void wait(int i) {
    const long long c0 = clock64();
    bool logged = false;
    while (!mbar_try(bar + i, (bits >> i) & 1u))
      if (!logged && clock64() - c0 > (1ll << 31) && (threadIdx.x & 31) == 0 && gn_tb_victim()) {
        logged = true;
        const int k = atomicAdd(gn_tb_hang, 1);
        if (k < 64) {
          gn_tb_hang[1 + 4 * k] = blockIdx.x; gn_tb_hang[2 + 4 * k] = threadIdx.x;
          gn_tb_hang[3 + 4 * k] = i; gn_tb_hang[4 + 4 * k] = (int)bits;
        }
        __threadfence_system();
      }
    bits ^= 1u << i;
  }
#else
  __device__ __forceinline__ void wait(int i) { tc::mbar_wait(bar + i, (bits >> i) & 1u); bits ^= 1u << i; }
#endif
  __device__ __forceinline__ bool ready(int i) const { return mbar_try(bar + i, (bits >> i) & 1u); }
};

template <int K, int H, int C0, int POOL>
__global__ void __launch_bounds__(TbLayout<K, H, C0>::THREADS, 1)
k_tb_tc(const uint16_t* __restrict__ tbuf, const uint16_t* __restrict__ e0, const uint16_t* __restrict__ direct,
        const uint8_t* __restrict__ wimg, const __grid_constant__ TbParams prm, const uint16_t* __restrict__ perm,
        float* __restrict__ psi, long P, int* __restrict__ sched) {
  using S = TbLayout<K, H, C0>;
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr uint32_t PL = S::PL;
  constexpr int NO = C0 + 3;
  constexpr int ND = S::NDESC;
  static_assert(C0 <= 32 && H <= 64 && H % 32 == 0 && C0 % 16 == 0, "TbParams sizes / epilogue chunks");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S::OFF_BAR);
  enum : int { FULL = 0, EMPTY = 4, LOADA = 8, LOADE = 10, A1FREE = 12, D1 = 14, RDYA = 16, D2 = 18, FREE2 = 20,
               RDYF = 22, TAUF = 24, DF = 26, E3FREE = 28 };   // barrier indices ([ND] or [2] each)
  uint64_t* full = bar + FULL;        // [ND]  E1 (256)
  uint64_t* empty = bar + EMPTY;      // [ND]  MMA 1 + E2 256 + E3 128
  uint64_t* loadedA = bar + LOADA;    // [2]   E1 cp.async (256)
  uint64_t* loadedE = bar + LOADE;    // [2]   E3 cp.async (128)
  uint64_t* a1free = bar + A1FREE;    // [2]   commit
  uint64_t* d1 = bar + D1;            // [2]   commit
  uint64_t* rdyA = bar + RDYA;        // [2]   E1 (256)
  uint64_t* d2 = bar + D2;            // [2]   commit
  uint64_t* free2 = bar + FREE2;      // [2]   E2 (256)
  uint64_t* rdyF = bar + RDYF;        // [2]   E2 (256)
  uint64_t* tauF = bar + TAUF;        // [2]   commit
  uint64_t* dF = bar + DF;            // [2]   commit
  uint64_t* e3free = bar + E3FREE;    // [2]   E3 (128)
  volatile long long* drows = reinterpret_cast<long long*>(smem + S::OFF_DESC);   // [ND][128]
  volatile int* dkt = reinterpret_cast<int*>(smem + S::OFF_DKT);                  // [ND]
  volatile int* scr = reinterpret_cast<int*>(smem + S::OFF_SCR);                  // [0..7] warp max, [8..10] tile ids
  uint32_t* tptr = reinterpret_cast<uint32_t*>(smem + S::OFF_TPTR);

  TBP_INIT();
  for (int i = threadIdx.x; i < S::WIMG_B / 16; i += blockDim.x)
    reinterpret_cast<int4*>(smem)[i] = reinterpret_cast<const int4*>(wimg)[i];
  for (int i = threadIdx.x; i < 2 * 2 * (int)PL / 16; i += blockDim.x) {   // the zero pad planes of both A1 buffers
    const int b = i / (2 * PL / 16), o = i % (2 * PL / 16);
    reinterpret_cast<int4*>(smem + S::OFF_A1 + (b * S::A1_PL + S::NPL) * PL)[o] = make_int4(0, 0, 0, 0);
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < ND; ++i) { tc::mbar_init(full + i, 256); tc::mbar_init(empty + i, 1 + 256 + 128); }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(loadedA + i, 256); tc::mbar_init(loadedE + i, 128);
      tc::mbar_init(a1free + i, 1); tc::mbar_init(d1 + i, 1); tc::mbar_init(rdyA + i, 256);
      tc::mbar_init(d2 + i, 1); tc::mbar_init(free2 + i, 256); tc::mbar_init(rdyF + i, 256);
      tc::mbar_init(tauF + i, 1); tc::mbar_init(dF + i, 1); tc::mbar_init(e3free + i, 128);
    }
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc<S::TCOLS>(tptr);
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tptr;
  const uint32_t sA1 = tc::smem_u32(smem + S::OFF_A1), sE0 = tc::smem_u32(smem + S::OFF_E0);
  const uint32_t sTAU = tc::smem_u32(smem + S::OFF_TAU);
  const long ntiles = (P + TB_SBP - 1) / TB_SBP * TB_SBT;
  constexpr int PXB = 32;   // descriptor row: pixel | count << 32, -1 if absent

  if (warp == 20) {
    // ------------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t sW1 = tc::smem_u32(smem + S::OFF_W1), sW2 = tc::smem_u32(smem + S::OFF_W2);
      const uint32_t sWBT = tc::smem_u32(smem + S::OFF_WBT), sWBE = tc::smem_u32(smem + S::OFF_WBE);
      constexpr uint32_t ID_T = tc::idesc_f16(128, H, 1, 1);
      constexpr uint32_t ID_BE = tc::idesc_f16(128, C0, 1, 1);
      constexpr uint32_t ID_BT = tc::idesc_f16(128, C0, 0, 0);
      Phases ph{bar};
      // Kt of the tiles whose descriptors were read, by ring slot (8 bits each, -1: end)
      uint32_t ktc = 0;
      auto ktc_get = [&](int v) -> int { return (int)(int8_t)((ktc >> (8 * (v & (ND - 1)))) & 0xFFu); };
      int vdesc = 0;         // next descriptor to read
      // accB queue: tiles whose layer-2 batches are all issued, accB not yet (FIFO by tile)
      int qhead = 0, qtail = 0;
      uint32_t qkt = 0;      // their counts, by v & 3 (8 bits each)
      auto accB_ready = [&](int v) {
        const int b = v & 1;
        return ph.ready(RDYF + b) && ph.ready(LOADE + b) && (v < 2 || ph.ready(E3FREE + b));
      };
      auto issue_accB = [&](int v) {
        const int b = v & 1;
        ph.wait(RDYF + b); ph.wait(LOADE + b);
        if (v >= 2) ph.wait(E3FREE + b);
        tc::fence_after_sync();
        const uint32_t e0b = sE0 + b * (C0 / 8) * PL, taub = sTAU + b * (H / 8) * PL;
        const uint32_t acc = tmem + S::T_ACCB + b * C0;
#pragma unroll
        for (int q = 0; q < C0 / 16; ++q)
          tc::mma_f16_ss(acc, tc::smem_desc(e0b + 2 * q * PL, PL, 128),
                         tc::smem_desc(sWBE + 2 * q * C0 * 16, C0 * 16, 128), ID_BE, q > 0);
        if (((qkt >> (8 * (v & 3))) & 0xFFu) > 0) {
#pragma unroll
          for (int q = 0; q < H / 16; ++q)
            tc::mma_f16_ss(acc, tc::smem_desc(taub + 2 * q * PL, PL, 128),
                           tc::smem_desc(sWBT + 2 * q * C0 * 16, C0 * 16, 128), ID_BT, 1);
        }
        tc::mma_commit(tauF + b);
        tc::mma_commit(dF + b);
      };
      auto spin_ready = [&](int v) {
#ifdef GN_TB_DEBUG
        const long long c0 = clock64();
        bool logged = false;
        while (!accB_ready(v))
          if (!logged && clock64() - c0 > (1ll << 31) && gn_tb_victim()) {
            logged = true;
            const int k = atomicAdd(gn_tb_hang, 1);
            if (k < 64) {
              gn_tb_hang[1 + 4 * k] = blockIdx.x; gn_tb_hang[2 + 4 * k] = threadIdx.x;
              gn_tb_hang[3 + 4 * k] = 100 + v; gn_tb_hang[4 + 4 * k] = (int)ph.bits;
            }
            __threadfence_system();
          }
#else
        while (!accB_ready(v)) {}
#endif
      };
      auto service = [&]() {   // issue the oldest pending accB batch if its operands are ready
        if (qhead < qtail && accB_ready(qhead)) { issue_accB(qhead); ++qhead; }
      };
#ifdef GN_TB_DEBUG
      int dbg_v1 = 0, dbg_k1 = 0, dbg_v2 = 0, dbg_k2 = 0;
#endif
      auto wait_s = [&](int i) {   // wait on barrier i, issuing pending accB batches meanwhile
#ifdef GN_TB_DEBUG
        const long long c0 = clock64();
        bool logged = false;
        while (!ph.ready(i)) {
          service();
          if (!logged && clock64() - c0 > (1ll << 31) && gn_tb_victim()) {
            logged = true;
            const int k = atomicAdd(gn_tb_hang, 1);
            if (k < 62) {
              gn_tb_hang[1 + 4 * k] = blockIdx.x; gn_tb_hang[2 + 4 * k] = threadIdx.x;
              gn_tb_hang[3 + 4 * k] = i; gn_tb_hang[4 + 4 * k] = (int)ph.bits;
              gn_tb_hang[5 + 4 * k] = blockIdx.x; gn_tb_hang[6 + 4 * k] = -1;
              gn_tb_hang[7 + 4 * k] = (dbg_v1 << 16) | dbg_k1; gn_tb_hang[8 + 4 * k] = (dbg_v2 << 16) | dbg_k2;
              gn_tb_hang[9 + 4 * k] = blockIdx.x; gn_tb_hang[10 + 4 * k] = -2;
              gn_tb_hang[11 + 4 * k] = (qhead << 16) | qtail; gn_tb_hang[12 + 4 * k] = vdesc;
              atomicAdd(gn_tb_hang, 2);
            }
            __threadfence_system();
          }
        }
#else
        while (!ph.ready(i)) service();
#endif
        ph.wait(i);
      };
      // Descriptors are read in tile order (either cursor may read the next one); a tile's
      // descriptor is released (empty) as soon as its last layer-2 batch is issued, so E1 can
      // always publish the tiles the layer-1 cursor runs ahead into.
      auto read_desc = [&]() -> int {
        const int i = vdesc & (ND - 1);
        wait_s(FULL + i);
        const int kt = dkt[i];
        ktc = (ktc & ~(0xFFu << (8 * i))) | ((uint32_t)(kt & 0xFF) << (8 * i));
        ++vdesc;
        return kt;
      };
      auto layer1 = [&](int v, int k, int n) {
        const int j = (11 * k) >> 3, o = (11 * k) & 7;
        const uint32_t a = sA1 + ((v & 1) * S::A1_PL + j) * PL, w = sW1 + o * 4 * H * 16;
        const uint32_t acc = tmem + S::T_ACC1 + (n & 1) * H;
        tc::mma_f16_ss(acc, tc::smem_desc(a, PL, 128), tc::smem_desc(w, H * 16, 128), ID_T, 0);
        if (o > 5)
          tc::mma_f16_ss(acc, tc::smem_desc(a + 2 * PL, PL, 128), tc::smem_desc(w + 2 * H * 16, H * 16, 128), ID_T, 1);
        tc::mma_commit(d1 + (n & 1));
      };
      // layer-1 cursor (tile v1, slot k1) -- a non-blocking state machine: l1_step() returns
      // true when (v1, k1) is an issuable slot (descriptor read, records landed)
      int v1 = 0, k1 = 0, kt1 = 0, n1 = 0;
      bool have1 = false, rec1 = false, end1 = false;
      auto l1_step = [&]() -> bool {
        for (;;) {
          if (end1) return false;
          if (!have1) {
            if (vdesc > v1) kt1 = ktc_get(v1);
            else {
              if (!ph.ready(FULL + (vdesc & (ND - 1)))) return false;
              kt1 = read_desc();
            }
            have1 = true;
            if (kt1 < 0) { end1 = true; return false; }
          }
          if (!rec1) {
            if (!ph.ready(LOADA + (v1 & 1))) return false;
            ph.wait(LOADA + (v1 & 1));
            tc::fence_after_sync();
            rec1 = true;
          }
          if (k1 < kt1) return true;
          tc::mma_commit(a1free + (v1 & 1));   // all of tile v1's layer-1 MMAs issued
          ++v1; k1 = 0; have1 = false; rec1 = false;
        }
      };
      auto l1_issue = [&]() { layer1(v1, k1, n1); ++k1; ++n1; };
      // layer-2 cursor (tile v2, slot k2); global slot n2
      int v2 = 0, k2 = 0, kt2 = 0, n2 = 0;
      bool have2 = false;
      for (;;) {
        if (!have2) {   // the L2 cursor's tile count
          kt2 = (vdesc > v2) ? ktc_get(v2) : read_desc();
          have2 = true;
        }
        if (kt2 < 0) break;
        if (k2 >= kt2) {   // tile v2 done (or empty): queue its accB batch, release its descriptor
          qkt = (qkt & ~(0xFFu << (8 * (v2 & 3)))) | ((uint32_t)kt2 << (8 * (v2 & 3)));
          ++qtail;
          tc::mbar_arrive(empty + (v2 & (ND - 1)));
          ++v2; k2 = 0; have2 = false;
          // the layer-1 cursor never trails: pass (and release) the tiles layer 2 has left
          while (!end1 && v1 < v2)
            if (!l1_step()) service();
          if (qtail - qhead > 2) { spin_ready(qhead); issue_accB(qhead); ++qhead; }
          continue;
        }
        // layer 1 of slot n2 must have been issued (E1 waits for it before signalling rdyA)
        while (n1 <= n2) {
          if (l1_step()) l1_issue();
          else service();
        }
        const int b = n2 & 1;
        TBP_NOW(tm0);
        wait_s(RDYA + b);                         // A2[b] holds slot n2; acc1[b] read
        TBP_NOW(tm1);
        if (n2 >= 2) wait_s(FREE2 + b);           // acc2[b] read (slot n2 - 2)
        TBP_NOW(tm2);
        TBP_ADDM(12, tm0, tm1);
        TBP_ADDM(13, tm1, tm2);
        tc::fence_after_sync();
#pragma unroll
        for (int q = 0; q < H / 16; ++q)
          tc::mma_f16_ts(tmem + S::T_ACC2 + b * H, tmem + S::T_A2 + b * (H / 2) + q * 8,
                         tc::smem_desc(sW2 + 2 * q * H * 16, H * 16, 128), ID_T, q > 0);
        tc::mma_commit(d2 + b);
        TBP_NOW(tm3);
        TBP_ADDM(14, tm2, tm3);
        ++k2; ++n2;
        // layer 1 runs up to two slots ahead (acc1[n & 1] of slot n2 - 1 + 2 was just read)
        while (n1 < n2 + 2 && l1_step()) l1_issue();
        TBP_NOW(tm4);
        TBP_ADDM(15, tm3, tm4);
#ifdef GN_TB_DEBUG
        dbg_v1 = v1; dbg_k1 = k1; dbg_v2 = v2; dbg_k2 = k2;
#endif
        service();
      }
      while (qhead < qtail) { spin_ready(qhead); issue_accB(qhead); ++qhead; }
    }
  } else if (warp >= 16) {
    // ------------------------------------------------------------------ E3: e0, phi, psi
    const int r = threadIdx.x - 16 * 32, q4 = r >> 5;
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    Phases ph{bar};
    for (int v = 0;; ++v) {
      const int i = v & (ND - 1), b = v & 1;
      ph.wait(FULL + i);
      const int kt = dkt[i];
      if (kt < 0) break;
      const long long rw = drows[i * 128 + r];
      {  // e0 of the tile's rows -> operand buffer b (coalesced chunks; last read by accB(v-2))
        constexpr int NC = C0 / 8;
#pragma unroll
        for (int j0 = 0; j0 < NC; ++j0) {
          const int c = j0 * 128 + r, pr = c / NC, j = c % NC;
          const long long x = drows[i * 128 + pr];
          const bool ok = x >= 0;
          const uint16_t* src = ok ? e0 + (x & 0xFFFFFFFFll) * C0 + 8 * j : e0;
          cp_async16z(sE0 + (b * NC + j) * PL + pr * 16, src, ok ? 16u : 0u);
        }
      }
      tc::mbar_arrive(empty + i);
      const bool pv = rw >= 0;
      const long p = pv ? (long)(rw & 0xFFFFFFFFll) : 0;
      const int m = pv ? (int)(rw >> PXB) : 0;
      float ld0 = 0.f, ld1 = 0.f, ld2 = 0.f;
      if (pv) {
        ld0 = __uint_as_float((uint32_t)__ldg(direct + p * 3 + 0) << 16);
        ld1 = __uint_as_float((uint32_t)__ldg(direct + p * 3 + 1) << 16);
        ld2 = __uint_as_float((uint32_t)__ldg(direct + p * 3 + 2) << 16);
      }
      // e0 landed: make it visible to the tensor core (async proxy), then hand it over.  The
      // proxy fence is executed here, by the writer, not by the MMA thread (a fence there would
      // also wait for its in-flight MMAs).
      cp_async_wait_all();
      tc::fence_proxy_async();
      tc::mbar_arrive(loadedE + b);
      ph.wait(DF + b);
      tc::fence_after_sync();
      const float* WO = prm.WO;
      float ps0 = prm.bO[0], ps1 = prm.bO[1], ps2 = prm.bO[2];
      ps0 = fmaf(WO[0 * NO + C0 + 0], ld0, ps0); ps0 = fmaf(WO[0 * NO + C0 + 1], ld1, ps0); ps0 = fmaf(WO[0 * NO + C0 + 2], ld2, ps0);
      ps1 = fmaf(WO[1 * NO + C0 + 0], ld0, ps1); ps1 = fmaf(WO[1 * NO + C0 + 1], ld1, ps1); ps1 = fmaf(WO[1 * NO + C0 + 2], ld2, ps1);
      ps2 = fmaf(WO[2 * NO + C0 + 0], ld0, ps2); ps2 = fmaf(WO[2 * NO + C0 + 1], ld1, ps2); ps2 = fmaf(WO[2 * NO + C0 + 2], ld2, ps2);
      const float fm = (float)m;
#pragma unroll
      for (int c = 0; c < C0 / 16; ++c) {
        uint32_t u[16];
        tc::tmem_ld16(tmem + S::T_ACCB + b * C0 + lane_off + c * 16, u);
        tc::tmem_ld_wait();
#pragma unroll
        for (int ii = 0; ii < 16; ++ii) {
          const int o = c * 16 + ii;
          const float phi = relu(__uint_as_float(u[ii]) + prm.bB[o] + prm.wBn[o] * fm);
          ps0 = fmaf(WO[0 * NO + o], phi, ps0);
          ps1 = fmaf(WO[1 * NO + o], phi, ps1);
          ps2 = fmaf(WO[2 * NO + o], phi, ps2);
        }
      }
      tc::fence_before_sync();
      tc::mbar_arrive(e3free + b);
      if (pv) { psi[p * 3 + 0] = ps0; psi[p * 3 + 1] = ps1; psi[p * 3 + 2] = ps2; }
    }
  } else if (warp >= 8) {
    // ------------------------------------------------------------------ E2: pool, tau
    const int w = warp - 8, q4 = w & 3, hf = w >> 2;   // lane quarter, column half
    const int r = q4 * 32 + lane;
    constexpr int HH = H / 2;                           // columns per thread
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    Phases ph{bar};
    int n = 0;
    for (int v = 0;; ++v) {
      const int i = v & (ND - 1), b = v & 1;
      ph.wait(FULL + i);
      const int kt = dkt[i];
      if (kt < 0) break;
      const long long rw = drows[i * 128 + r];
      tc::mbar_arrive(empty + i);
      const int m = rw >= 0 ? (int)(rw >> PXB) : 0;
      uint32_t pool[HH];
#pragma unroll
      for (int j = 0; j < HH; ++j) pool[j] = 0;
#pragma unroll 1
      for (int s = 0; s < kt; ++s, ++n) {
        const int bb = n & 1;
        ph.wait(D2 + bb);
        tc::fence_after_sync();
        // pool += Q(acc2 + b2): acc2 carries the 2^12 scale (folded into W2), so x = acc2 + q2
        // is 2^23 + (v + b2) 2^12 rounded; masked slots clamp to exactly 2^23 (0)
        const float hi = (s < m) ? TB_QMAX : TB_QMAGIC;
#ifndef GN_ABL_NO_POOL
#pragma unroll
        for (int c = 0; c < HH / 16; ++c) {
          uint32_t u[16];
          tc::tmem_ld16(tmem + S::T_ACC2 + bb * H + lane_off + hf * HH + c * 16, u);
          tc::tmem_ld_wait();
#pragma unroll
          for (int ii = 0; ii < 16; ++ii) {
            float x = __uint_as_float(u[ii]) + prm.q2[hf * HH + c * 16 + ii];
            x = fminf(fmaxf(x, TB_QMAGIC), hi);
            pool[c * 16 + ii] += __float_as_uint(x);
          }
        }
#endif
        tc::fence_before_sync();
        tc::mbar_arrive(free2 + bb);
      }
      if (v >= 2) ph.wait(TAUF + b);   // tau buffer b was read by accB(v-2)
      if (kt > 0) {   // tau = pool (f16) -> operand buffer b, this thread's column half
        const uint32_t off = (uint32_t)kt * TB_QBITS;
        const float sc = (POOL == 1 && m > 0) ? (1.f / TB_QSCALE) / (float)m : 1.f / TB_QSCALE;
        const uint32_t taub = sTAU + b * (H / 8) * PL;
#pragma unroll
        for (int q = 0; q < HH / 8; ++q) {
          uint32_t o[4];
#pragma unroll
          for (int ii = 0; ii < 4; ++ii) {
            const float lo = (float)(pool[8 * q + 2 * ii] - off) * sc;
            const float hv = (float)(pool[8 * q + 2 * ii + 1] - off) * sc;
            o[ii] = tc::cvt_relu_f16x2(lo, hv);
          }
          tc::sts128(taub + (hf * (HH / 8) + q) * PL + r * 16, o[0], o[1], o[2], o[3]);
        }
      }
      tc::fence_proxy_async();     // tau (generic-proxy stores) -> visible to the tensor core
      tc::mbar_arrive(rdyF + b);
    }
  } else {
    // ------------------------------------------------------------------ E1: descriptors, records, A2
    const int q4 = warp & 3, hf = warp >> 2;   // lane quarter, column half
    const int r = q4 * 32 + lane;
    const int t1 = threadIdx.x;                 // 0..255
    constexpr int HH = H / 2;
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    Phases ph{bar};
    auto rowword = [&](long tl, int pe) -> long long {   // row r of tile tl: pixel | count << 32, -1 if absent
      const long long pp = tl / TB_SBT * TB_SBP + (pe & 2047);
      return (tl < ntiles && pp < P) ? (pp | ((long long)(pe >> 11) << PXB)) : -1ll;
    };
    // publish tile v (rows `rw` of this thread's row; `last`: end-of-stream marker) and
    // copy its records into operand buffer v&1 (coalesced: chunk c = i*256 + t1 is 16-byte
    // piece c % NPL of row c / NPL, zero beyond the valid records)
    auto publish = [&](int v, long long rw, bool last) {
      const int i = v & (ND - 1), b = v & 1;
      if (v >= ND) ph.wait(EMPTY + i);            // consumers are done with tile v - ND
      if (hf == 0) drows[i * 128 + r] = rw;
      const int m = rw >= 0 ? (int)(rw >> PXB) : 0;
      const int wm = __reduce_max_sync(0xFFFFFFFFu, (unsigned)m);
      if (lane == 0) scr[warp] = wm;
      tc::bar_sync(1, 256);
      const int kt = last ? -1 : max(max(scr[0], scr[1]), max(scr[2], scr[3]));
      if (t1 == 0) dkt[i] = kt;
      if (!last) {
        if (v >= 2) ph.wait(A1FREE + b);          // tile v-2's layer 1 is done with buffer b
        const uint32_t a = sA1 + b * S::A1_PL * PL;
        for (int c = t1; c < 128 * S::NPL; c += 256) {
          const int pr = c / S::NPL, j = c % S::NPL;
          const long long x = drows[i * 128 + pr];
          const int vb = x >= 0 ? (int)(x >> PXB) * 22 : 0;
          const long pp = x >= 0 ? (long)(x & 0xFFFFFFFFll) : 0;
          if (S::ASYNC) {
            const char* src = reinterpret_cast<const char*>(tbuf + pp * (K * 11)) + 16 * j;
            cp_async16z(a + j * PL + pr * 16, src, (uint32_t)min(max(vb - 16 * j, 0), 16));
          } else {   // rows not 16-byte aligned in global memory: through registers
            const uint16_t* src = tbuf + pp * (K * 11);
            uint32_t w4[4];
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              const int e = 8 * j + 2 * h;
              const uint32_t lo = 2 * e < vb ? __ldg(src + e) : 0u, hi = 2 * e + 2 < vb ? __ldg(src + e + 1) : 0u;
              w4[h] = lo | (hi << 16);
            }
            tc::sts128(a + j * PL + pr * 16, w4[0], w4[1], w4[2], w4[3]);
          }
        }
      }
      tc::bar_sync(1, 256);                       // scr[] read by all before it is rewritten
      tc::mbar_arrive(full + i);
    };

    // Tile pipeline: ids claimed three ahead, the perm entry of the tile after next loaded
    // one tile ahead, the next tile published (records copied) while this one's slots run.
    int claim = 0;
    if (t1 == 0) { scr[8] = atomicAdd(sched, 1); scr[9] = atomicAdd(sched, 1); claim = atomicAdd(sched, 1); }
    tc::bar_sync(1, 256);
    long tile = scr[8], ntile = scr[9];
    long long cur = rowword(tile, tile < ntiles ? (int)__ldg(perm + tile * 128 + r) : 0);
    long long nxt = rowword(ntile, ntile < ntiles ? (int)__ldg(perm + ntile * 128 + r) : 0);
    tc::bar_sync(1, 256);
    publish(0, cur, tile >= ntiles);
    // a published tile's records are confirmed (cp.async landed -> proxy fence -> loadedA) by
    // this group one slot later, so the fence never waits for copies still in flight
    auto confirm = [&](int buf) {
      cp_async_wait_all();
      tc::fence_proxy_async();
      tc::mbar_arrive(loadedA + buf);
    };
    if (tile < ntiles) confirm(0);
    int n = 0, v = 0;
    for (; tile < ntiles; ++v) {
      TBP_NOW(tp_t0);
      const int kt = dkt[v & (ND - 1)];           // written by this group in the previous publish
      // next tile id (claimed two iterations ago) and the one after
      if (t1 == 0) { scr[10] = claim; claim = atomicAdd(sched, 1); }
      tc::bar_sync(1, 256);
      const long nntile = scr[10];
      publish(v + 1, nxt, ntile >= ntiles);
      const int nnpe = nntile < ntiles ? (int)__ldg(perm + nntile * 128 + r) : 0;   // used next iteration
      TBP_NOW(tp_t1);
      TBP_ADD(1, tp_t0, tp_t1);
      TBP_ADD(10, 0, kt + 1);
      TBP_ADD(11, 0, 1);
      const bool nlast = ntile >= ntiles;
      if (kt == 0 && !nlast) confirm((v + 1) & 1);
#pragma unroll 1
      for (int s = 0; s < kt; ++s, ++n) {
        const int bb = n & 1;
        TBP_NOW(tp_r0);
        ph.wait(D1 + bb);                         // L1(n) in acc1[bb] (and L2(n-2) done with A2[bb])
        tc::fence_after_sync();
        TBP_NOW(tp_r1);
        TBP_ADD(3, tp_r0, tp_r1);
#ifndef GN_ABL_NO_EPI1
        uint32_t u[HH];
#pragma unroll
        for (int c = 0; c < HH / 16; ++c)
          tc::tmem_ld16(tmem + S::T_ACC1 + bb * H + lane_off + hf * HH + c * 16, *reinterpret_cast<uint32_t(*)[16]>(u + 16 * c));
        tc::tmem_ld_wait();
        uint32_t o[HH / 2];
#pragma unroll
        for (int ii = 0; ii < HH / 2; ++ii)
          o[ii] = tc::cvt_relu_bf16x2(__uint_as_float(u[2 * ii]) + prm.b1[hf * HH + 2 * ii],
                                      __uint_as_float(u[2 * ii + 1]) + prm.b1[hf * HH + 2 * ii + 1]);
#pragma unroll
        for (int c = 0; c < HH / 16; ++c)
          tc::tmem_st8(tmem + S::T_A2 + bb * (H / 2) + lane_off + hf * (HH / 2) + 8 * c, o + 8 * c);
        tc::tmem_st_wait();
#endif
        tc::fence_before_sync();
        tc::mbar_arrive(rdyA + bb);
        if (s == 0 && !nlast) confirm((v + 1) & 1);   // the next tile's records
        TBP_NOW(tp_r2);
        TBP_ADD(4, tp_r1, tp_r2);
      }
      TBP_NOW(tp_end);
      TBP_ADD(9, tp_t0, tp_end);
      tile = ntile; cur = nxt;
      ntile = nntile;
      nxt = rowword(ntile, nnpe);
    }
    (void)cur;
  }
  tc::fence_before_sync();
  __syncthreads();
  TBP_FLUSH();
  if (warp == 0) tc::tmem_dealloc<S::TCOLS>(*tptr);
}

}  // namespace gn
