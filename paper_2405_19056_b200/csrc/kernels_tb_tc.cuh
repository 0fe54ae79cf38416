// kernels_tb_tc.cuh -- the fused T + B + psi kernel on tcgen05.
//
// PAPER.md Eq. eq:SymmetricNN: tau = sum_i h(b_i), h shared; B;
// the psi projection is reading R15.  One CTA = one 128-pixel tile at a time,
// thread r owns pixel r (= TMEM lane r = MMA row r).  Per tile:
//   1. each thread loads its pixel's K records into registers and sorts the valid ones
//      into the canonical order (reading R5: lexicographic on the storage bits) with a
//      Batcher odd-even merge network; invalid slots become all-ones and sort last.
//   2. per slot s (canonical order):
//        A1 = [record_s | 1 1 1 | 0 0]                      (bf16, 128 x 16)
//        acc = A1 W1ext^T          (bias b1 via the three 1-columns, split hi/mid/lo)
//        A2 = [ReLU(acc) bf16 | 1 1 1 0..]                   (128 x (h+16))
//        acc = A2 W2ext^T          (bias b2 likewise)
//        A3 = ReLU(acc) (/n in mean mode)  f16               (128 x h)
//        accB += A3 W_B,tau^T      -- g = sum is done by the tensor core's accumulation:
//                                      W_B sum_s a2_s = sum_s W_B a2_s (linearity)
//      accB starts as e0 W_B,e0^T.  Invalid slots are all-zero rows (bias columns too),
//      so they add exactly 0; per-fragment activations never leave the SM.
//   3. phi = ReLU(accB + b_B + w_Bn n);  psi = W_O,d0 phi + W_O,L L_d + b_O  -> HBM (fp32).
// A1, A2, A3 and the e0 operand share one 20 KB shared-memory region (their lifetimes do
// not overlap, see the comments at each write), so 4 CTAs (4 independent MMA chains)
// fit on an SM.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace gn {

// Batcher odd-even merge sort network for N = 2^p inputs (compile time).
template <int N>
struct SortNet {
  int a[N * N], b[N * N];
  int n;
  constexpr SortNet() : a(), b(), n(0) {
    for (int p = 1; p < N; p += p)
      for (int k = p; k >= 1; k /= 2)
        for (int j = k % p; j + k <= N - 1; j += 2 * k)
          for (int i = 0; i <= (k - 1 < N - j - k - 1 ? k - 1 : N - j - k - 1); ++i)
            if ((i + j) / (p * 2) == (i + j + k) / (p * 2)) { a[n] = i + j; b[n] = i + j + k; ++n; }
  }
};
constexpr int pow2_ceil(int k) { return k <= 1 ? 1 : 2 * pow2_ceil((k + 1) / 2); }

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
  static constexpr int PL = 128 * 16;          // one 8-column K-plane of a 128-row operand
  static constexpr int OFF_OP = WIMG_B;        // operand region: KA2/8 planes
  // planes of the operand region:  A2 = 0 .. KA2/8-1 ; A3 = 0 .. H/8-1 ; AE = 0 .. C0/8-1 ;
  //                                A1 = the last two planes (H/8, H/8+1)  [>= C0/8 and >= H/8]
  static constexpr int A1_PLANE = H / 8;
  static constexpr int OFF_PAR = OFF_OP + (KA2 / 8) * PL;
  static constexpr int OFF_BAR = (OFF_PAR + NPAR * 4 + 15) / 16 * 16;
  static constexpr int SMEM = OFF_BAR + 16;
  static constexpr int TMEM_COLS = (H + C0) <= 64 ? 64 : ((H + C0) <= 128 ? 128 : 256);
  static constexpr int REC_B = K * 22;          // bytes of one pixel's records
  static constexpr int VW = REC_B % 16 == 0 ? 16 : REC_B % 8 == 0 ? 8 : REC_B % 4 == 0 ? 4 : 2;
  static constexpr int NV = REC_B / VW;
  static constexpr int MINB = K <= 8 ? 4 : 2;
};

struct Frag {                    // one record as the 6 words of an A1 row + its sort key
  uint32_t w[6];                 // ch0|ch1, ch2|ch3, ch4|ch5, ch6|ch7, ch8|ch9, ch10|1.0
  uint64_t key;                  // depth, ch0, ch1, ch2  (16 bits each)
};

__device__ __forceinline__ bool frag_lt(const Frag& x, const Frag& y) {
  if (x.key != y.key) return x.key < y.key;
#pragma unroll
  for (int j = 1; j < 6; ++j)
    if (x.w[j] != y.w[j]) return x.w[j] < y.w[j];
  return false;
}

template <int K, int H, int C0>
__global__ void __launch_bounds__(128, TbLayout<K, H, C0>::MINB)
k_tb_tc(const uint16_t* __restrict__ tbuf, const uint8_t* __restrict__ tcount, const uint16_t* __restrict__ e0,
        const uint16_t* __restrict__ direct, const uint8_t* __restrict__ wimg, const float* __restrict__ params,
        float* __restrict__ psi, long P, int pool, int r_takes_ld) {
  using S = TbLayout<K, H, C0>;
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + S::OFF_BAR);
  uint32_t* tptr = reinterpret_cast<uint32_t*>(smem + S::OFF_BAR + 8);
  const int tid = threadIdx.x, warp = tid >> 5;

  for (int i = tid; i < S::WIMG_B / 16; i += 128)
    reinterpret_cast<int4*>(smem)[i] = reinterpret_cast<const int4*>(wimg)[i];
  float* par = reinterpret_cast<float*>(smem + S::OFF_PAR);
  for (int i = tid; i < S::NPAR; i += 128) par[i] = params[i];
  if (tid == 0) { tc::mbar_init(mbar, 1); tc::fence_mbar_init(); }
  if (warp == 0) tc::tmem_alloc<S::TMEM_COLS>(tptr);
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tptr;
  const uint32_t t_acc = tmem, t_accB = tmem + H;
  const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
  const float* bB = par;
  const float* wBn = par + C0;
  constexpr int NO = C0 + 3;
  const float* WO = par + 2 * C0;
  const float* bO = WO + 3 * NO;

  constexpr uint32_t PL = S::PL;
  const uint32_t sOP = tc::smem_u32(smem + S::OFF_OP);
  const uint32_t sA1 = sOP + S::A1_PLANE * PL;
  const uint32_t sW1 = tc::smem_u32(smem + S::OFF_W1), sW2 = tc::smem_u32(smem + S::OFF_W2);
  const uint32_t sWBT = tc::smem_u32(smem + S::OFF_WBT), sWBE = tc::smem_u32(smem + S::OFF_WBE);
  constexpr uint32_t ID_T = tc::idesc_f16(128, H, 1, 1);
  constexpr uint32_t ID_BE = tc::idesc_f16(128, C0, 1, 1);
  constexpr uint32_t ID_BT = tc::idesc_f16(128, C0, 0, 0);
  constexpr int NP2 = pow2_ceil(K);
  constexpr SortNet<NP2> NET{};
  uint32_t phase = 0;
  const long ntiles = (P + 127) / 128;
  const int r = tid;

  for (long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long p = tile * 128 + r;
    const bool pv = p < P;
    int m = pv ? (int)__ldg(tcount + p) : 0;
    m = m < K ? m : K;
    // ---- 1. records -> registers (this pixel's K*22 contiguous bytes) ----
    uint16_t h[K * 11];
    {
      using V = typename std::conditional<S::VW == 16, uint4,
                typename std::conditional<S::VW == 8, uint2,
                typename std::conditional<S::VW == 4, uint32_t, uint16_t>::type>::type>::type;
      V raw[S::NV];
      if (pv) {
        const V* src = reinterpret_cast<const V*>(tbuf + p * (K * 11));
#pragma unroll
        for (int i = 0; i < S::NV; ++i) raw[i] = __ldg(src + i);
      } else {
#pragma unroll
        for (int i = 0; i < S::NV; ++i) memset(&raw[i], 0, sizeof(V));
      }
      memcpy(h, raw, sizeof(h));
    }
    Frag f[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint16_t* q = h + k * 11;
      if (k < m) {
        f[k].w[0] = q[0] | ((uint32_t)q[1] << 16);
        f[k].w[1] = q[2] | ((uint32_t)q[3] << 16);
        f[k].w[2] = q[4] | ((uint32_t)q[5] << 16);
        f[k].w[3] = q[6] | ((uint32_t)q[7] << 16);
        f[k].w[4] = q[8] | ((uint32_t)q[9] << 16);
        f[k].w[5] = q[10] | (0x3F80u << 16);
        f[k].key = ((uint64_t)q[7] << 48) | ((uint64_t)q[0] << 32) | ((uint64_t)q[1] << 16) | (uint64_t)q[2];
      } else {  // masked slot: any bits may be here (R4) -- replaced, never read
#pragma unroll
        for (int j = 0; j < 6; ++j) f[k].w[j] = 0xFFFFFFFFu;
        f[k].key = ~0ull;
      }
    }
    // ---- canonical order: Batcher network, comparators touching padding skipped ----
#pragma unroll
    for (int c = 0; c < NET.n; ++c) {
      const int ia = NET.a[c], ib = NET.b[c];
      if (ib < K) {
        if (frag_lt(f[ib], f[ia])) { Frag t = f[ia]; f[ia] = f[ib]; f[ib] = t; }
      }
    }
    float ld0 = 0.f, ld1 = 0.f, ld2 = 0.f;
    if (pv) {
      ld0 = __uint_as_float((uint32_t)__ldg(direct + p * 3 + 0) << 16);
      ld1 = __uint_as_float((uint32_t)__ldg(direct + p * 3 + 1) << 16);
      ld2 = __uint_as_float((uint32_t)__ldg(direct + p * 3 + 2) << 16);
    }
    const float inv_m = (pool == 1 && m > 0) ? 1.f / (float)m : 1.f;
    // e0 operand -> planes 0..C0/8-1 (free: the previous tile's last MMA finished, we
    // waited on its commit before its epilogue 3).
    if (pv) {
      const uint4* e = reinterpret_cast<const uint4*>(e0 + p * C0);
#pragma unroll
      for (int j = 0; j < C0 / 8; ++j) {
        uint4 v = __ldg(e + j);
        tc::sts128(sOP + j * PL + r * 16, v.x, v.y, v.z, v.w);
      }
    } else {
#pragma unroll
      for (int j = 0; j < C0 / 8; ++j) tc::sts128(sOP + j * PL + r * 16, 0, 0, 0, 0);
    }
    auto write_A1 = [&](const Frag& g, bool valid) {
      if (valid) {
        tc::sts128(sA1 + r * 16, g.w[0], g.w[1], g.w[2], g.w[3]);
        tc::sts128(sA1 + PL + r * 16, g.w[4], g.w[5], 0x3F803F80u, 0);
      } else {
        tc::sts128(sA1 + r * 16, 0, 0, 0, 0);
        tc::sts128(sA1 + PL + r * 16, 0, 0, 0, 0);
      }
    };
    write_A1(f[0], 0 < m);
    tc::fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      tc::fence_after_sync();
#pragma unroll
      for (int q = 0; q < C0 / 16; ++q)
        tc::mma_f16_ss(t_accB, tc::smem_desc(sOP + 2 * q * PL, PL, 128),
                       tc::smem_desc(sWBE + 2 * q * C0 * 16, C0 * 16, 128), ID_BE, q > 0);
      tc::mma_f16_ss(t_acc, tc::smem_desc(sA1, PL, 128), tc::smem_desc(sW1, H * 16, 128), ID_T, 0);
      tc::mma_commit(mbar);
    }
#pragma unroll
    for (int s = 0; s < K; ++s) {
      tc::mbar_wait(mbar, phase);
      phase ^= 1;
      tc::fence_after_sync();
      // epilogue 1 -> A2 (planes 0..KA2/8-1).  MMA1(s) and the e0 MMA are complete, and
      // MMA3(s-1) was committed with MMA1(s): nothing reads the region any more.
#pragma unroll
      for (int c = 0; c < H / 16; ++c) {
        uint32_t v[16];
        tc::tmem_ld16(t_acc + lane_off + c * 16, v);
        tc::tmem_ld_wait();
        uint32_t w[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) w[i] = tc::cvt_relu_bf16x2(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]));
        tc::sts128(sOP + (2 * c) * PL + r * 16, w[0], w[1], w[2], w[3]);
        tc::sts128(sOP + (2 * c + 1) * PL + r * 16, w[4], w[5], w[6], w[7]);
      }
      {
        const uint32_t one = s < m ? 0x3F80u : 0u;
        tc::sts128(sOP + (H / 8) * PL + r * 16, one | (one << 16), one, 0, 0);
        tc::sts128(sOP + (H / 8 + 1) * PL + r * 16, 0, 0, 0, 0);
      }
      tc::fence_before_sync();
      tc::fence_proxy_async();
      __syncthreads();
      if (tid == 0) {
        tc::fence_after_sync();
#pragma unroll
        for (int q = 0; q < S::KA2 / 16; ++q)
          tc::mma_f16_ss(t_acc, tc::smem_desc(sOP + 2 * q * PL, PL, 128),
                         tc::smem_desc(sW2 + 2 * q * H * 16, H * 16, 128), ID_T, q > 0);
        tc::mma_commit(mbar);
      }
      tc::mbar_wait(mbar, phase);
      phase ^= 1;
      tc::fence_after_sync();
      // epilogue 2 -> A3 (planes 0..H/8-1) and A1(s+1) (planes H/8, H/8+1): MMA2(s) done.
#pragma unroll
      for (int c = 0; c < H / 16; ++c) {
        uint32_t v[16];
        tc::tmem_ld16(t_acc + lane_off + c * 16, v);
        tc::tmem_ld_wait();
        uint32_t w[8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
          w[i] = tc::cvt_relu_f16x2(__uint_as_float(v[2 * i]) * inv_m, __uint_as_float(v[2 * i + 1]) * inv_m);
        tc::sts128(sOP + (2 * c) * PL + r * 16, w[0], w[1], w[2], w[3]);
        tc::sts128(sOP + (2 * c + 1) * PL + r * 16, w[4], w[5], w[6], w[7]);
      }
      if (s + 1 < K) write_A1(f[s + 1 < K ? s + 1 : 0], s + 1 < m);
      tc::fence_before_sync();
      tc::fence_proxy_async();
      __syncthreads();
      if (tid == 0) {
        tc::fence_after_sync();
#pragma unroll
        for (int q = 0; q < H / 16; ++q)
          tc::mma_f16_ss(t_accB, tc::smem_desc(sOP + 2 * q * PL, PL, 128),
                         tc::smem_desc(sWBT + 2 * q * C0 * 16, C0 * 16, 128), ID_BT, 1);
        if (s + 1 < K)
          tc::mma_f16_ss(t_acc, tc::smem_desc(sA1, PL, 128), tc::smem_desc(sW1, H * 16, 128), ID_T, 0);
        tc::mma_commit(mbar);
      }
    }
    tc::mbar_wait(mbar, phase);
    phase ^= 1;
    tc::fence_after_sync();
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
    __syncthreads();   // all epilogue-3 TMEM reads done before the next tile's MMAs
  }
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<S::TMEM_COLS>(tmem);
}

}  // namespace gn
