// kernels_conv_tc.cuh -- NHWC bf16 implicit-GEMM conv3x3 on tcgen05.
//
// out[b][oy][ox][co] = ReLU(bias[co] + sum_{ky,kx,ci} W[co][ky][kx][ci] in[b][s*oy+ky-1][s*ox+kx-1][ci])
// (PAPER.md P:366-383 scene encoder F / rendering network R; reading R10/R12).
//
// GEMM view per CTA tile: M = 128 output pixels of one output row, N = NS output
// channels (a split of C_out), K = 9 taps x C_in.  The A operand is never materialised:
// TMA copies, per 16-channel chunk, the 3 input rows of the tile's halo into shared
// memory (zero fill outside the image = the conv's zero padding) as 32-byte pixel rows in
// the SWIZZLE_32B K-major layout (each pixel's 16 channels are one full 32-byte sector of
// the NHWC input, so every L2 sector is fetched once), and each of the 9 taps is a UMMA
// descriptor shifted by whole pixel rows into that halo (stride 2 uses even/odd
// de-interleaved halos so every tap is affine).
// Weights: either resident in shared memory for the whole persistent kernel (the CTA's
// N-split), or -- when a full-width layer does not fit (WS = 1: F3, R3) -- streamed with the
// halo: each pipeline stage then carries the 16-channel chunk's 9 x 16 x Cout weights too
// (one bulk copy), so N = Cout in one pass instead of re-reading the halo per N-split.
// Warp roles: 0 = TMA producer, 1 = MMA issuer (+TMEM owner),
// 2..5 = epilogue (TMEM -> bias/ReLU -> bf16 NHWC store, or the z projection of R_1);
// GB = 1 (F0 on the full frame): warps 0 and 6.. build the halo from the G-buffer instead.
// Accumulators are double-buffered in TMEM so the epilogue overlaps the next tile.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include "net.h"
#include "tc_ptx.cuh"

namespace gn {
namespace conv {

constexpr int TILE_M = 128;
// bytes of one 8-channel plane of the halo in shared memory (128-byte aligned pieces)
template <int S> struct Halo;
// Stride 1: one TMA box {16 ch, 130 px, RR + 2 rows} over the 4-D view (C, W, H, frame); a
// tile of RR output rows reads RR + 2 input rows.
template <> struct Halo<1> {
  static constexpr int SLOTS = TILE_M + 2;                       // x0-1 .. x0+128
  static constexpr int ROW = SLOTS * 32;                         // one halo row
};
// Stride 2: the halo is de-interleaved into even pixels 2(x0+i) and odd pixels 2(x0+i)-1 so
// every tap is an affine window: one box {16 ch, 1, 128 | 129 px, 3 rows} per parity over the
// 4-D view (C, parity, x/2, frame*rows).
template <> struct Halo<2> {
  static constexpr int EVEN_ROW = TILE_M * 32, ODD_ROW = (TILE_M + 1) * 32;
  static constexpr int ODD_OFF = 3 * EVEN_ROW;                   // 12288: 1024-aligned
  static constexpr int TX = 3 * EVEN_ROW + 3 * ODD_ROW;          // bytes per 16-channel chunk
};

__device__ __forceinline__ void tma_4d(uint32_t dst, const CUtensorMap* m, int c0, int c1, int c2, int c3,
                                       uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(
          dst),
      "l"((uint64_t)m), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(tc::smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_5d(uint32_t dst, const CUtensorMap* m, int c0, int c1, int c2, int c3, int c4,
                                       uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(
          dst),
      "l"((uint64_t)m), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(tc::smem_u32(bar))
      : "memory");
}

struct ConvArgs {
  const uint8_t* wimg;   // resident: [nsplit][9][Cin/8][NS][8]; streamed: [Cin/16][9][2][NS][8] bf16 (K-major planes)
  const float* bias;     // [Cout]
  uint16_t* out;         // [B][Ho][Wo][Cout] bf16 (EPI 0)
  const float* wz;       // [3][Cout] (EPI 1)
  float* zout;           // [B][Ho][Wo][3] (EPI 1)
  int Cin, Cout, Ho, Wo, B, nsplit, nstage;
  // row geometry (row tiles carry one halo row above/below; full frame: 0, 0, Ho)
  int in_row_off;        // input buffer row of global-relative row 0
  int in_rows_buf;       // input buffer rows per frame (stride-2 view stacks frames along rows)
  int out_row_off;       // output buffer row of output row 0
  int out_rows_buf;      // output buffer rows per frame
  const uint16_t* gbuf;  // GB = 1 (F0 on the full frame): [B][H][W][12] bf16, read directly
  const uint16_t* direct;   //                                  [B][H][W][3]
  int Wi;                // input width (GB = 1, 2)
  // N3 super-sampler S (GB = 2 / EPI = 2, full frame): the low-res image [B][Ho/2][Wo/2][3] fp32
  const float* img;      // GB = 2: channels 12..14 of the halo = bf16(img at the covering coarse pixel)
  float b3[3];           // EPI = 2: out = clamp(img(coarse) + S3.W s2 + b3, 0, 1) -> zout
  // N4 object-major T (EPI = 3): a2 = ReLU(acc + b2) of one object, added where it covers the
  // pixel into the exact fixed-point latent tau_q += round(min(a2, qsat) * qscale) (uint32; integer
  // adds commute, so the object order cannot change a bit) and the count tau_n += 1
  const uint8_t* cover;  // [B][Ho][Wo]
  uint32_t* tau_q;       // [B][Ho][Wo][Cout]
  uint32_t* tau_n;       // [B][Ho][Wo]
  float qscale, qsat;
  // row tiles (forward_sharded, boundary rows first): 0 = every row tile of the frame, 1 = only the
  // first and the last row tile (the rows the next halo exchange sends), 2 = only the others
  int edge;
};

// Row tile `i` of the `nrt` a launch covers in edge mode `edge` -> the frame's row-tile index.
__device__ __forceinline__ int edge_row_tile(int i, int nry, int edge) {
  return edge == 0 ? i : edge == 1 ? (i == 0 ? 0 : nry - 1) : 1 + i;
}
__host__ __device__ __forceinline__ int edge_row_tiles(int nry, int edge) {
  return edge == 0 ? nry : edge == 1 ? (nry < 2 ? nry : 2) : (nry > 2 ? nry - 2 : 0);
}

__device__ __forceinline__ void bulk_s2g(void* dst, uint32_t src_smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src_smem), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }

// OST = 1: the epilogue stages each warp's 32 output pixels (32 x NS bf16, contiguous in NHWC)
// in shared memory and writes them with one bulk copy (full, coalesced lines) instead of
// 16-byte per-thread stores that touch every sector twice.
// RR: output rows per tile (stride 1 only): the RR rows share RR + 2 halo rows (each input
// row is read from L2 (RR + 2) / RR times instead of 3 times); RR accumulators of NS columns.
// GB = 1 (F0 only, full frame): the producer warp builds the halo itself from the G-buffer
// and L_d (one pixel row = [G(12), L_d(3), 0], the input normalisation folded into F0's
// weights, exactly) in the same SWIZZLE_32B layout TMA writes, so x16 is never stored.
// GB = 2 (S1 of the N3 super-sampler): the same producer with L_d replaced by the nearest-
// upsampled low-res image (fp32, read at the covering coarse pixel, rounded to bf16).
// EPI = 2 (S2 of N3): the z projection of EPI 1 plus S3's bias and the residual onto the
// nearest-upsampled image, clamped to [0,1], written as the fp32 hi-res output.
constexpr int GB_PRODUCERS = 7;   // GB = 1: warps 0 and 6..11 build the halo
template <int S, int NS, int EPI, int WS = 0, int OST = 0, int RR = 1, int GB = 0>
__global__ void __launch_bounds__(GB ? 32 * (5 + GB_PRODUCERS) : 192, GB ? 2 : 1)
k_conv_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmO, const ConvArgs a) {
  using HL = Halo<S>;
  static_assert(S == 1 || RR == 1, "multi-row tiles are stride-1 only");
  constexpr int TXB = S == 1 ? (RR + 2) * Halo<1>::ROW : Halo<2>::TX;   // bytes the TMA writes per stage
  constexpr int SBA = (TXB + 1023) / 1024 * 1024;   // a stage's halo (swizzled TMA dst: 1024-B aligned)
  constexpr int SBW = WS ? 9 * 2 * NS * 16 : 0;     // a stage's streamed weights (9 taps x 2 K-planes)
  constexpr int SB = SBA + SBW;
  constexpr int ACC = RR * NS;                      // TMEM columns of one tile's accumulators
  constexpr int TMEM_COLS = (2 * ACC) <= 32 ? 32 : (2 * ACC) <= 64 ? 64 : (2 * ACC) <= 128 ? 128 : (2 * ACC) <= 256 ? 256 : 512;
  static_assert(2 * ACC <= 512, "TMEM");
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int Cin = a.Cin, NST = a.nstage;
  const int wbytes = WS ? 0 : 9 * Cin * NS * 2;
  uint8_t* sW = smem;
  uint8_t* sA = smem + ((wbytes + 1023) / 1024) * 1024;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sA + NST * SB);
  uint64_t* full = bars;
  uint64_t* empty = bars + NST;
  uint64_t* tfull = bars + 2 * NST;
  uint64_t* tempty = tfull + 2;
  uint32_t* tptr = reinterpret_cast<uint32_t*>(tempty + 2);
  float* sBias = reinterpret_cast<float*>(tempty + 4);                        // NS floats (EPI 1: + 3 x NS of wz)
  uint8_t* sOut = reinterpret_cast<uint8_t*>(sBias) + ((NS * 4 * (EPI ? 4 : 1) + 127) / 128) * 128;   // OST: [4 warps][2][32][NS] bf16

  const int split = blockIdx.x % a.nsplit;
  if (!WS) {  // resident weights of this split
    const int4* src = reinterpret_cast<const int4*>(a.wimg + (size_t)split * wbytes);
    int4* dst = reinterpret_cast<int4*>(sW);
    for (int i = tid; i < wbytes / 16; i += blockDim.x) dst[i] = __ldg(src + i);
  }
  for (int i = tid; i < NS; i += blockDim.x) sBias[i] = a.bias[split * NS + i];
  if (EPI == 1 || EPI == 2)   // the z projection's weights (EPI 1, 2 run unsplit: NS = Cout)
    for (int i = tid; i < 3 * NS; i += blockDim.x) sBias[NS + i] = a.wz[i];
  if (tid == 0) {
    for (int i = 0; i < NST; ++i) { tc::mbar_init(full + i, GB ? GB_PRODUCERS : 1); tc::mbar_init(empty + i, 1); }
    for (int i = 0; i < 2; ++i) { tc::mbar_init(tfull + i, 1); tc::mbar_init(tempty + i, 128); }
    tc::fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc<TMEM_COLS>(tptr);
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tptr;

  const int ntx = (a.Wo + TILE_M - 1) / TILE_M;
  const int nry = (a.Ho + RR - 1) / RR;             // row tiles per frame
  const int nrt = edge_row_tiles(nry, a.edge);      // row tiles this launch covers
  const long ntiles = (long)a.B * nrt * ntx;
  const int cta = blockIdx.x / a.nsplit, ncta = gridDim.x / a.nsplit;
  const int nchunk = Cin / 16;

  if (GB && (warp == 0 || warp >= 6)) {   // ---------------- G-buffer producers, one 16-channel chunk
    const int pw = warp == 0 ? 0 : warp - 5;
    static_assert(!GB || (S == 1 && WS == 0), "GB: the stride-1 first layer");
    int stage = 0;
    uint32_t ph = 0;
    for (long t = cta; t < ntiles; t += ncta) {
      const int xt = (int)(t % ntx);
      const long r = t / ntx;
      const int oy = edge_row_tile((int)(r % nrt), nry, a.edge) * RR;
      const int b = (int)(r / nrt);
      const int x0 = xt * TILE_M;
      if (lane == 0) tc::mbar_wait(empty + stage, ph ^ 1);
      __syncwarp();
      const uint32_t base = tc::smem_u32(sA + stage * SB);
      // all of this thread's pixels' loads first (up to NPT in flight), then the stores
      constexpr int NSLOT = (RR + 2) * Halo<1>::SLOTS, NPT = (NSLOT + 32 * GB_PRODUCERS - 1) / (32 * GB_PRODUCERS);
      uint32_t w[NPT][8];
#pragma unroll
      for (int k = 0; k < NPT; ++k) {
        const int slot = pw * 32 + lane + k * 32 * GB_PRODUCERS;
        const int y = slot / Halo<1>::SLOTS, sx = slot - y * Halo<1>::SLOTS;
        const int gy = oy - 1 + y, gx = x0 - 1 + sx;
#pragma unroll
        for (int i = 0; i < 8; ++i) w[k][i] = 0;
        if (slot < NSLOT && gy >= 0 && gy < a.in_rows_buf && gx >= 0 && gx < a.Wi) {
          const long p = ((long)b * a.in_rows_buf + gy) * a.Wi + gx;
          const uint2* g = reinterpret_cast<const uint2*>(a.gbuf + p * 12);
          const uint2 g0 = __ldg(g), g1 = __ldg(g + 1), g2 = __ldg(g + 2);
          w[k][0] = g0.x; w[k][1] = g0.y; w[k][2] = g1.x; w[k][3] = g1.y; w[k][4] = g2.x; w[k][5] = g2.y;
          if (GB == 1) {
            const uint16_t* dl = a.direct + p * 3;
            w[k][6] = (uint32_t)__ldg(dl) | ((uint32_t)__ldg(dl + 1) << 16);
            w[k][7] = (uint32_t)__ldg(dl + 2);
          } else {   // nearest up-sampling: the coarse pixel covering (gy, gx)
            const long pc = ((long)b * (a.in_rows_buf >> 1) + (gy >> 1)) * (a.Wi >> 1) + (gx >> 1);
            const float* im = a.img + pc * 3;
            w[k][6] = tc::cvt_bf16x2(__ldg(im), __ldg(im + 1));
            w[k][7] = tc::cvt_bf16x2(__ldg(im + 2), 0.f);
          }
        }
      }
#pragma unroll
      for (int k = 0; k < NPT; ++k) {
        const int slot = pw * 32 + lane + k * 32 * GB_PRODUCERS;
        if (slot < NSLOT) {
          const uint32_t row = base + (uint32_t)slot * 32, sw = (row >> 7) & 1u;   // SWIZZLE_32B
          tc::sts128(row + (sw << 4), w[k][0], w[k][1], w[k][2], w[k][3]);
          tc::sts128(row + ((sw ^ 1u) << 4), w[k][4], w[k][5], w[k][6], w[k][7]);
        }
      }
      tc::fence_proxy_async();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(full + stage);
      if (++stage == NST) { stage = 0; ph ^= 1; }
    }
  } else if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      int stage = 0;
      uint32_t ph = 0;
      for (long t = cta; t < ntiles; t += ncta) {
        const int xt = (int)(t % ntx);
        const long r = t / ntx;
        const int oy = edge_row_tile((int)(r % nrt), nry, a.edge) * RR;
        const int b = (int)(r / nrt);
        const int x0 = xt * TILE_M;
        for (int c = 0; c < nchunk; ++c) {
          tc::mbar_wait(empty + stage, ph ^ 1);
          tc::mbar_arrive_expect_tx(full + stage, TXB + SBW);
          const uint32_t dst = tc::smem_u32(sA + stage * SB);
          if (WS) tc::bulk_g2s(sA + stage * SB + SBA, a.wimg + (size_t)c * SBW, SBW, full + stage);
          const int iy = S * oy - 1 + a.in_row_off;
          if (S == 1) {
            tma_4d(dst, &tmA, 16 * c, x0 - 1, iy, b, full + stage);
          } else {   // frames are stacked along the row dimension: row b*Hbuf + iy (iy = -1: see the MMA)
            const int row = b * a.in_rows_buf + iy;
            tma_4d(dst, &tmA, 16 * c, 0, x0, row, full + stage);
            tma_4d(dst + Halo<2>::ODD_OFF, &tmO, 16 * c, 1, x0 - 1, row, full + stage);
          }
          if (++stage == NST) { stage = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      constexpr uint32_t IDESC = tc::idesc_f16(128, NS, 1, 1);
      const uint32_t sWa = tc::smem_u32(sW), sAa = tc::smem_u32(sA);
      int stage = 0, acc = 0;
      uint32_t ph = 0, aph = 0;
      for (long t = cta; t < ntiles; t += ncta) {
        tc::mbar_wait(tempty + acc, aph ^ 1);
        tc::fence_after_sync();
        const uint32_t d0 = tmem + acc * ACC;
        // stride 2, first output row of a frame: its ky = 0 taps read the zero padding above
        // the image (the stacked view holds the previous frame's last row there): skip them
        bool skip_top = false;
        if (S == 2) {
          const long r = t / ntx;
          skip_top = edge_row_tile((int)(r % nrt), nry, a.edge) == 0 && a.in_row_off == 0;
        }
        bool first = true;
        for (int c = 0; c < nchunk; ++c) {
          tc::mbar_wait(full + stage, ph);
          tc::fence_after_sync();
          const uint32_t base = sAa + stage * SB;
#pragma unroll
          for (int tap = 0; tap < 9; ++tap) {
            const int ky = tap / 3, kx = tap % 3;
            if (S == 2 && ky == 0 && skip_top) continue;
            const uint64_t bd = WS ? tc::smem_desc(base + SBA + tap * 2 * NS * 16, NS * 16, 128)
                                   : tc::smem_desc(sWa + (uint32_t)((tap * (Cin / 8) + 2 * c) * NS * 16), NS * 16, 128);
#pragma unroll
            for (int rr = 0; rr < RR; ++rr) {
              uint32_t aoff;
              if (S == 1) aoff = (rr + ky) * Halo<1>::ROW + kx * 32;
              else if (kx == 1) aoff = ky * Halo<2>::EVEN_ROW;
              else aoff = Halo<2>::ODD_OFF + ky * Halo<2>::ODD_ROW + (kx == 2 ? 32 : 0);
              const uint64_t ad = tc::smem_desc_sw32(base + aoff);
              tc::mma_f16_ss(d0 + rr * NS, ad, bd, IDESC, first ? 0u : 1u);
            }
            first = false;
          }
          tc::mma_commit(empty + stage);
          if (++stage == NST) { stage = 0; ph ^= 1; }
        }
        tc::mma_commit(tfull + acc);
        if (++acc == 2) { acc = 0; aph ^= 1; }
      }
    }
  } else {  // ---------------- epilogue warps 2..5
    const int q = warp & 3;               // TMEM lane quarter of this warp
    const int m = q * 32 + lane;
    const int co0 = split * NS;
    int acc = 0, sb = 0;
    uint32_t aph = 0;
    constexpr uint32_t WBUF = 32 * NS * 2;     // one warp's staged output (OST)
    for (long t = cta; t < ntiles; t += ncta) {
      const int xt = (int)(t % ntx);
      const long r = t / ntx;
      const int oy0 = edge_row_tile((int)(r % nrt), nry, a.edge) * RR;
      const int b = (int)(r / nrt);
      const int px = xt * TILE_M + m;
      const bool pvalid = px < a.Wo;
      tc::mbar_wait(tfull + acc, aph);
      tc::fence_after_sync();
#pragma unroll 1
      for (int rr = 0; rr < RR; ++rr) {
        const int oy = oy0 + rr;
        const bool rvalid = oy < a.Ho;
        const bool valid = pvalid && rvalid;
        const long opix = ((long)b * a.out_rows_buf + oy + a.out_row_off) * a.Wo + px;
        const uint32_t taddr = tmem + acc * ACC + rr * NS + ((uint32_t)(q * 32) << 16);
        const uint32_t stg = tc::smem_u32(sOut) + (q * 2 + sb) * WBUF;
        if (OST) {   // this warp's staging buffer sb: its bulk copy (two rows ago) has read it
          if (lane == 0) bulk_wait_read<1>();
          __syncwarp();
        }
        float z0 = 0.f, z1 = 0.f, z2 = 0.f;
        const bool cov = EPI == 3 && valid && __ldg(a.cover + opix) != 0;
        uint4 tcur[4], tnext[4];   // EPI 3: this and the next chunk's latent (loads one chunk ahead)
        uint4* tq0 = EPI == 3 ? reinterpret_cast<uint4*>(a.tau_q + opix * a.Cout + co0) : nullptr;
        if (EPI == 3 && cov)
#pragma unroll
          for (int j = 0; j < 4; ++j) tnext[j] = tq0[j];
#pragma unroll 1
        for (int c = 0; c < NS / 16; ++c) {
          uint32_t v[16];
          tc::tmem_ld16(taddr + c * 16, v);
          if (EPI == 3 && cov) {
#pragma unroll
            for (int j = 0; j < 4; ++j) tcur[j] = tnext[j];
            if (c + 1 < NS / 16)
#pragma unroll
              for (int j = 0; j < 4; ++j) tnext[j] = tq0[4 * (c + 1) + j];
          }
          tc::tmem_ld_wait();
          float y[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) y[i] = relu(__uint_as_float(v[i]) + sBias[c * 16 + i]);
          if (EPI == 0 && OST) {
            uint32_t w[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) w[i] = tc::cvt_bf16x2(y[2 * i], y[2 * i + 1]);
            const uint32_t dst = stg + lane * (NS * 2) + c * 32;
            tc::sts128(dst, w[0], w[1], w[2], w[3]);
            tc::sts128(dst + 16, w[4], w[5], w[6], w[7]);
          } else if (EPI == 0) {
            if (valid) {
              uint32_t w[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) w[i] = tc::cvt_bf16x2(y[2 * i], y[2 * i + 1]);
              uint4* dst = reinterpret_cast<uint4*>(a.out + opix * a.Cout + co0 + c * 16);
              dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
              dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
            }
          } else if (EPI == 3) {
            if (cov) {   // this thread's pixel, 16 channels: read-modify-write (one writer per pixel)
              uint4* tq = tq0 + 4 * c;
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                uint4 u = tcur[j];
                u.x += __float2uint_rn(fminf(y[4 * j], a.qsat) * a.qscale);
                u.y += __float2uint_rn(fminf(y[4 * j + 1], a.qsat) * a.qscale);
                u.z += __float2uint_rn(fminf(y[4 * j + 2], a.qsat) * a.qscale);
                u.w += __float2uint_rn(fminf(y[4 * j + 3], a.qsat) * a.qscale);
                tq[j] = u;
              }
            }
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const int o = c * 16 + i;
              z0 = fmaf(sBias[NS + o], y[i], z0);
              z1 = fmaf(sBias[2 * NS + o], y[i], z1);
              z2 = fmaf(sBias[3 * NS + o], y[i], z2);
            }
          }
        }
        if (EPI == 1 && valid) {
          a.zout[opix * 3 + 0] = z0; a.zout[opix * 3 + 1] = z1; a.zout[opix * 3 + 2] = z2;
        }
        if (EPI == 3 && cov && split == 0) a.tau_n[opix] += 1u;
        if (EPI == 2 && valid) {   // N3: residual onto the nearest-upsampled image, clamped
          const long pc = ((long)b * (a.out_rows_buf >> 1) + ((oy + a.out_row_off) >> 1)) * (a.Wo >> 1) + (px >> 1);
          const float* im = a.img + pc * 3;
          a.zout[opix * 3 + 0] = fminf(fmaxf(__ldg(im) + (z0 + a.b3[0]), 0.f), 1.f);
          a.zout[opix * 3 + 1] = fminf(fmaxf(__ldg(im + 1) + (z1 + a.b3[1]), 0.f), 1.f);
          a.zout[opix * 3 + 2] = fminf(fmaxf(__ldg(im + 2) + (z2 + a.b3[2]), 0.f), 1.f);
        }
        if (OST) {   // the warp's 32 pixels of this row are contiguous in NHWC: one bulk copy
          tc::fence_proxy_async();
          __syncwarp();
          if (lane == 0) {
            const int px0 = xt * TILE_M + q * 32;
            const int nv = min(32, a.Wo - px0);
            if (nv > 0 && rvalid) {
              const long opix0 = ((long)b * a.out_rows_buf + oy + a.out_row_off) * a.Wo + px0;
              bulk_s2g(a.out + opix0 * a.Cout, stg, (uint32_t)(nv * NS * 2));
            }
            bulk_commit();
          }
          sb ^= 1;
        }
      }
      tc::fence_before_sync();
      tc::mbar_arrive(tempty + acc);
      if (++acc == 2) { acc = 0; aph ^= 1; }
    }
    if (OST && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc<TMEM_COLS>(tmem);
}

}  // namespace conv
}  // namespace gn
