// kernels_simt.cuh -- SIMT (FFMA) GlassNet kernels.
//
// These are the fp32 check-mode kernels (the same graph with FFMA
// math, because 1xTF32 tensor-core operands fail the 1e-4 check) and run on either
// storage type.  Every kernel accumulates in fp32.
#pragma once
#include "common.cuh"

namespace gn {

// 8 consecutive elements (16-byte aligned for bf16, 32-byte for fp32) -> fp32.
__device__ __forceinline__ void load8(const float* p, float v[8]) {
  float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
__device__ __forceinline__ void load8(const __nv_bfloat16* p, float v[8]) {
  uint4 u = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) { float2 f = __bfloat1622float2(h[i]); v[2 * i] = f.x; v[2 * i + 1] = f.y; }
}
__device__ __forceinline__ void store8(float* p, const float v[8]) {
  *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  *reinterpret_cast<float4*>(p + 4) = make_float4(v[4], v[5], v[6], v[7]);
}
__device__ __forceinline__ void store8(__nv_bfloat16* p, const float v[8]) {
  uint4 u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
  *reinterpret_cast<uint4*>(p) = u;
}

// x = [G', L_d, 0] (16 channels).  G' = G with position*2^-3 and depth*2^-7 (reading R9;
// exact in binary floating point, so the stored bf16 x carries no new rounding).
template <typename T>
__global__ void k_prep_x(const T* __restrict__ gbuf, const T* __restrict__ direct, T* __restrict__ x,
                         long P, int norm) {
  long p = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  float v[16];
#pragma unroll
  for (int i = 0; i < 12; ++i) v[i] = to_f(gbuf[p * 12 + i]);
#pragma unroll
  for (int i = 0; i < 3; ++i) v[12 + i] = to_f(direct[p * 3 + i]);
  v[15] = 0.f;
  if (norm) {
    v[0] *= 0.125f; v[1] *= 0.125f; v[2] *= 0.125f;
    v[11] *= 0.0078125f;
  }
  store8(x + p * 16, v);
  store8(x + p * 16 + 8, v + 8);
}

// N2 positional encoding: the features of v are
// v, sin(2^k pi v), cos(2^k pi v) for k < L.  sincospif(v) once (exact argument reduction), then
// the double-angle recurrence sin 2a = 2 sin a cos a, cos 2a = (cos a - sin a)(cos a + sin a):
// the absolute error at most doubles per octave (<= 2^(L-1) x ~1 ulp, ~4e-6 at L = 6), far inside
// bf16 storage rounding and the fp32 check mode's 1e-4.
struct PeIter {
  float s, c;
  __device__ __forceinline__ explicit PeIter(float v) { sincospif(v, &s, &c); }
  __device__ __forceinline__ void next() {
    const float s2 = 2.f * s * c, c2 = (c - s) * (c + s);
    s = s2; c = c2;
  }
};

// N2: x = gamma([G', L_d]) (15 (2L+1) channels, zero-padded to XC).  A block = 32 pixels (one per
// thread); each thread encodes its pixel into shared memory, then the block writes the 32
// contiguous NHWC pixels with 16-byte stores.
template <typename T>
__global__ void __launch_bounds__(32) k_prep_pe(const T* __restrict__ gbuf, const T* __restrict__ direct,
                                                T* __restrict__ x, long P, int norm, int L, int XC) {
  extern __shared__ __align__(16) uint8_t pe_smem[];
  T* st = reinterpret_cast<T*>(pe_smem);
  const long p0 = (long)blockIdx.x * 32;
  const long p = p0 + threadIdx.x;
  const int pe = 2 * L + 1;
  if (p < P) {
    T* o = st + threadIdx.x * XC;
    for (int c = 0; c < 15; ++c) {
      float v = c < 12 ? to_f(gbuf[p * 12 + c]) : to_f(direct[p * 3 + c - 12]);
      if (norm && c < 3) v *= 0.125f;
      if (norm && c == 11) v *= 0.0078125f;
      o[c * pe] = T(v);
      PeIter it(v);
      for (int k = 0; k < L; ++k) {
        o[c * pe + 1 + 2 * k] = T(it.s);
        o[c * pe + 2 + 2 * k] = T(it.c);
        it.next();
      }
    }
    for (int j = 15 * pe; j < XC; ++j) o[j] = T(0.f);
  }
  __syncwarp();
  const long np = (P - p0) < 32 ? (P - p0) : 32;
  const int nvec = (int)(np * XC * sizeof(T) / 16);
  const int4* src = reinterpret_cast<const int4*>(st);
  int4* dst = reinterpret_cast<int4*>(x + p0 * XC);
  for (int i = threadIdx.x; i < nvec; i += 32) dst[i] = src[i];
}

// N3 super-sampler S, SIMT family: x[p] = [G'_hi(12), img(coarse)(3), 0] at the hi-res pixel p
// (nearest up-sampling: the coarse pixel covering it), G' as k_prep_x.  One thread per pixel.
template <typename T>
__global__ void k_prep_ss(const T* __restrict__ gbuf, const float* __restrict__ img, T* __restrict__ x,
                          int W2, int H2, long P2, int norm) {
  long p = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P2) return;
  const int X = (int)(p % W2);
  const long t = p / W2;
  const int Y = (int)(t % H2);
  const long b = t / H2;
  const long pc = (b * (H2 >> 1) + (Y >> 1)) * (W2 >> 1) + (X >> 1);
  float v[16];
#pragma unroll
  for (int i = 0; i < 12; ++i) v[i] = to_f(gbuf[p * 12 + i]);
#pragma unroll
  for (int i = 0; i < 3; ++i) v[12 + i] = to_f(T(img[pc * 3 + i]));   // stored in T like any x
  v[15] = 0.f;
  if (norm) {
    v[0] *= 0.125f; v[1] *= 0.125f; v[2] *= 0.125f;
    v[11] *= 0.0078125f;
  }
  store8(x + p * 16, v);
  store8(x + p * 16 + 8, v + 8);
}

// N3: out = clamp(img(coarse) + r + b3, 0, 1), r = S3.W s2 from k_conv3x3_simt<..., EPI 1>.
__global__ void k_ss_out(const float* __restrict__ img, const float* __restrict__ r, float b30, float b31, float b32,
                         float* __restrict__ out, int W2, int H2, long P2) {
  long p = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P2) return;
  const int X = (int)(p % W2);
  const long t = p / W2;
  const int Y = (int)(t % H2);
  const long b = t / H2;
  const long pc = (b * (H2 >> 1) + (Y >> 1)) * (W2 >> 1) + (X >> 1);
  const float bb[3] = {b30, b31, b32};
#pragma unroll
  for (int c = 0; c < 3; ++c) out[p * 3 + c] = fminf(fmaxf(img[pc * 3 + c] + (r[p * 3 + c] + bb[c]), 0.f), 1.f);
}

// N4 object-major T (reading N4), SIMT side.  x = cover ? [b (depth x 2^-7 with R9), 0 x 5]
// : 0 (16 channels, T) -- the conv input of h's first 3x3 layer.  One thread per pixel.
template <typename T>
__global__ void k_obj_prep(const T* __restrict__ obj, const uint8_t* __restrict__ cover, T* __restrict__ x, long P,
                           int norm) {
  const long p = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  float v[16];
  const bool c = cover[p] != 0;
#pragma unroll
  for (int i = 0; i < 11; ++i) v[i] = c ? to_f(obj[p * 11 + i]) : 0.f;   // select: garbage never read into math
#pragma unroll
  for (int i = 11; i < 16; ++i) v[i] = 0.f;
  if (norm) v[7] *= 0.0078125f;
  store8(x + p * 16, v);
  store8(x + p * 16 + 8, v + 8);
}

// N4, SIMT family: tau_q += round(min(a2, qsat) qscale) and tau_n += 1 where the object covers
// (a2 from k_conv3x3_simt; the same exact fixed-point sum as the tensor-core epilogue).
template <typename T>
__global__ void k_obj_accum(const T* __restrict__ a2, const uint8_t* __restrict__ cover, uint32_t* __restrict__ tau_q,
                            uint32_t* __restrict__ tau_n, long P, int H, float qscale, float qsat) {
  const long p = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P || cover[p] == 0) return;
  for (int j = 0; j < H; j += 8) {
    float v[8];
    load8(a2 + p * H + j, v);
#pragma unroll
    for (int i = 0; i < 8; ++i) tau_q[p * H + j + i] += __float2uint_rn(fminf(v[i], qsat) * qscale);
  }
  tau_n[p] += 1u;
}

// N4: B + psi from the accumulated latent (both families): tau = tau_q / qscale (mean: / n),
// phi = ReLU(W_B [e0; tau; n] + b_B), psi = W_O[:, :c0] phi + W_O[:, c0:] L_d + b_O (R15).
// wb: WB[C0][C0+H+1] bB[C0] WO[3][NO] bO[3] (fp32).
template <typename T, int H, int C0>
__global__ void __launch_bounds__(128) k_b_psi(const T* __restrict__ e0, const uint32_t* __restrict__ tau_q,
                                               const uint32_t* __restrict__ tau_n, const T* __restrict__ direct,
                                               const float* __restrict__ wb, float* __restrict__ psi, long P, int pool,
                                               int r_takes_ld, float inv_qscale) {
  const int NB = C0 + H + 1, NO = C0 + (r_takes_ld ? 3 : 0);
  constexpr int NBP = (C0 + H + 1 + 3) / 4 * 4;   // W_B rows padded to 16 bytes: vector weight loads
  __shared__ __align__(16) float sWB[C0 * NBP];
  __shared__ float sRest[C0 + 3 * (C0 + 3) + 3];   // b_B, W_O, b_O
  for (int i = threadIdx.x; i < C0 * NB; i += blockDim.x) sWB[(i / NB) * NBP + i % NB] = wb[i];
  for (int i = threadIdx.x; i < C0 + 3 * NO + 3; i += blockDim.x) sRest[i] = wb[C0 * NB + i];
  __syncthreads();
  const long p = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const float* bB = sRest;
  const float* WO = bB + C0;
  const float* bO = WO + 3 * NO;
  const float m = (float)tau_n[p];
  float s[H];
#pragma unroll
  for (int j = 0; j < H; ++j) {
    s[j] = (float)tau_q[p * H + j] * inv_qscale;
    if (pool == 1) s[j] = m > 0.f ? __fdiv_rn(s[j], m) : 0.f;
  }
  float ev[C0];
#pragma unroll
  for (int i = 0; i < C0; i += 8) load8(e0 + p * C0 + i, ev + i);
  float ps0 = bO[0], ps1 = bO[1], ps2 = bO[2];
  if (r_takes_ld) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const float l = to_f(direct[p * 3 + i]);
      ps0 = fmaf(WO[0 * NO + C0 + i], l, ps0);
      ps1 = fmaf(WO[1 * NO + C0 + i], l, ps1);
      ps2 = fmaf(WO[2 * NO + C0 + i], l, ps2);
    }
  }
#pragma unroll 2
  for (int o = 0; o < C0; ++o) {
    const float* w = sWB + o * NBP;
    float a = bB[o];
#pragma unroll
    for (int i = 0; i < C0; ++i) a = fmaf(w[i], ev[i], a);
#pragma unroll
    for (int j = 0; j < H; ++j) a = fmaf(w[C0 + j], s[j], a);
    a = fmaf(w[C0 + H], m, a);
    const float phi = relu(a);
    ps0 = fmaf(WO[0 * NO + o], phi, ps0);
    ps1 = fmaf(WO[1 * NO + o], phi, ps1);
    ps2 = fmaf(WO[2 * NO + o], phi, ps2);
  }
  psi[p * 3 + 0] = ps0; psi[p * 3 + 1] = ps1; psi[p * 3 + 2] = ps2;
}

// conv3x3 (cross-correlation, zero pad 1), NHWC.  w: [9][Cin][Cout] fp32.  One thread =
// one output pixel x NJ output channels.  EPI 0: bias + ReLU -> T.  EPI 1 (R_1 only):
// bias + ReLU -> z = Wz y (3 fp32), the projection of reading R15.
template <typename T, int NJ, int EPI>
__global__ void __launch_bounds__(128) k_conv3x3_simt(
    const T* __restrict__ in, int Hi, int Wi, int Cin, const float* __restrict__ w,
    const float* __restrict__ bias, int Cout, int stride, T* __restrict__ out, int Ho, int Wo,
    long npix, const float* __restrict__ wz, float* __restrict__ zout) {
  long q = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= npix) return;
  const int co0 = blockIdx.y * NJ;
  const int ox = (int)(q % Wo);
  const long t = q / Wo;
  const int oy = (int)(t % Ho);
  const long b = t / Ho;
  float acc[NJ];
#pragma unroll
  for (int j = 0; j < NJ; ++j) acc[j] = bias[co0 + j];
  for (int ky = 0; ky < 3; ++ky) {
    const int iy = stride * oy + ky - 1;
    if (iy < 0 || iy >= Hi) continue;
    for (int kx = 0; kx < 3; ++kx) {
      const int ix = stride * ox + kx - 1;
      if (ix < 0 || ix >= Wi) continue;
      const T* ip = in + ((b * Hi + iy) * Wi + ix) * (long)Cin;
      const float* wp = w + (long)(ky * 3 + kx) * Cin * Cout + co0;
      for (int c8 = 0; c8 < Cin; c8 += 8) {
        float v[8];
        load8(ip + c8, v);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float4* wr = reinterpret_cast<const float4*>(wp + (long)(c8 + i) * Cout);
#pragma unroll
          for (int j4 = 0; j4 < NJ / 4; ++j4) {
            float4 ww = __ldg(wr + j4);
            acc[4 * j4 + 0] = fmaf(v[i], ww.x, acc[4 * j4 + 0]);
            acc[4 * j4 + 1] = fmaf(v[i], ww.y, acc[4 * j4 + 1]);
            acc[4 * j4 + 2] = fmaf(v[i], ww.z, acc[4 * j4 + 2]);
            acc[4 * j4 + 3] = fmaf(v[i], ww.w, acc[4 * j4 + 3]);
          }
        }
      }
    }
  }
  if (EPI == 0) {
#pragma unroll
    for (int j = 0; j < NJ; j += 8) {
      float v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = relu(acc[j + i]);
      store8(out + q * Cout + co0 + j, v);
    }
  } else {
    float z0 = 0.f, z1 = 0.f, z2 = 0.f;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      float y = relu(acc[j]);
      z0 = fmaf(wz[j], y, z0);
      z1 = fmaf(wz[NJ + j], y, z1);
      z2 = fmaf(wz[2 * NJ + j], y, z2);
    }
    zout[q * 3 + 0] = z0; zout[q * 3 + 1] = z1; zout[q * 3 + 2] = z2;
  }
}

// Canonical fragment order (reading R5): lexicographic on the storage bit patterns of
// (depth, ch0, ch1, ..., ch10).  Identical records are interchangeable, so the order of
// the VALUES seen by the MLP and the pool is a function of the multiset only.
template <typename T>
__device__ __forceinline__ bool rec_less(const T* a, const T* b) {
  uint32_t x = bits_of(a[7]), y = bits_of(b[7]);
  if (x != y) return x < y;
#pragma unroll 1
  for (int c = 0; c < 11; ++c) {
    x = bits_of(a[c]); y = bits_of(b[c]);
    if (x != y) return x < y;
  }
  return false;
}

// T + B + psi, one thread per pixel (SIMT).
//   tau = [sum over valid fragments (canonical order) of h(b), m]  (Eq. eq:SymmetricNN)
//   phi = ReLU(W_B [e0; tau] + b_B)
//   psi = W_O[:, :c0] phi + W_O[:, c0:] L_d + b_O                    (reading R15)
// wts (fp32): W1[H][NIN] b1[H] W2[H][H] b2[H] WB[C0][C0+H+1] bB[C0] WO[3][NO] bO[3],
// NIN = NR (+ C0 with sigma, N1: h's layer 1 over [record ; e0 at the pixel]); NR = 11, or
// 11 (2 pe_L + 1) with N2's positional encoding of the record (computed here, per fragment)
// SIG (N1) is a template parameter so that without it neither the shared layer-1 part u1 nor e0 is
// live across the fragment loop (register pressure; e0 is loaded for B after the loop).
template <typename T, int H, int C0, bool SIG>
__global__ void __launch_bounds__(128) k_tb_simt(
    const T* __restrict__ tbuf, const uint8_t* __restrict__ tcount, const T* __restrict__ e0,
    const T* __restrict__ direct, const float* __restrict__ wts, float* __restrict__ psi,
    long P, int K, int pool, int r_takes_ld, int norm, int pe_L) {
  constexpr bool sigma = SIG;
  extern __shared__ float sw[];
  const int PE = 2 * pe_L + 1, NR = 11 * PE;
  const int NB = C0 + H + 1, NO = C0 + (r_takes_ld ? 3 : 0), NIN = NR + (sigma ? C0 : 0);
  const int nw = H * NIN + H + H * H + H + C0 * NB + C0 + 3 * NO + 3;
  for (int i = threadIdx.x; i < nw; i += blockDim.x) sw[i] = wts[i];
  if (pe_L) {   // N2: W1 transposed to [NIN][H] so layer 1 reads 4 consecutive outputs per 16-byte load
    __syncthreads();
    float* w1t = sw + ((nw + 3) & ~3);
    for (int i = threadIdx.x; i < H * NIN; i += blockDim.x) w1t[(i % NIN) * H + i / NIN] = sw[i];
  }
  __syncthreads();
  const float* W1 = sw;
  const float* b1 = W1 + H * NIN;
  const float* W2 = b1 + H;
  const float* b2 = W2 + H * H;
  const float* WB = b2 + H;
  const float* bB = WB + C0 * NB;
  const float* WO = bB + C0;
  const float* bO = WO + 3 * NO;

  long p = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  int m = tcount[p];
  m = m < K ? m : K;
  const T* rec = tbuf + p * (long)K * 11;
  // insertion sort of slot indices into the canonical order
  int idx[16];
  for (int k = 0; k < m; ++k) {
    int j = k;
    while (j > 0 && rec_less(rec + k * 11, rec + idx[j - 1] * 11)) { idx[j] = idx[j - 1]; --j; }
    idx[j] = k;
  }
  float ev[C0];
  if (SIG)
#pragma unroll
    for (int i = 0; i < C0; i += 8) load8(e0 + p * C0 + i, ev + i);
  // the layer-1 part every fragment of the pixel shares: b1 (+ W1,sigma e0 with N1)
  float u1[H];
  if (SIG)
#pragma unroll
    for (int o = 0; o < H; ++o) {
      float a = b1[o];
#pragma unroll
      for (int j = 0; j < C0; ++j) a = fmaf(W1[o * NIN + NR + j], ev[j], a);
      u1[o] = a;
    }
  float s[H];
#pragma unroll
  for (int o = 0; o < H; ++o) s[o] = 0.f;
  for (int t = 0; t < m; ++t) {
    const T* r = rec + idx[t] * 11;
    float x[11];
#pragma unroll
    for (int i = 0; i < 11; ++i) x[i] = to_f(r[i]);
    if (norm) x[7] *= 0.0078125f;
    float a1[H];
    if (pe_L == 0) {
#pragma unroll
      for (int o = 0; o < H; ++o) {
        float a = SIG ? u1[o] : b1[o];
#pragma unroll
        for (int i = 0; i < 11; ++i) a = fmaf(W1[o * NIN + i], x[i], a);
        a1[o] = relu(a);
      }
    } else {   // N2: layer 1 over gamma(record), channel by channel (features in index order)
      const float* w1t = sw + ((nw + 3) & ~3);   // [NIN][H]
#pragma unroll
      for (int o = 0; o < H; ++o) a1[o] = SIG ? u1[o] : b1[o];
#pragma unroll 1
      for (int i = 0; i < 11; ++i) {
        const float v = x[i];
        const float4* w = reinterpret_cast<const float4*>(w1t + (i * PE) * H);
#pragma unroll
        for (int o = 0; o < H / 4; ++o) {
          const float4 q = w[o];
          a1[4 * o] = fmaf(q.x, v, a1[4 * o]); a1[4 * o + 1] = fmaf(q.y, v, a1[4 * o + 1]);
          a1[4 * o + 2] = fmaf(q.z, v, a1[4 * o + 2]); a1[4 * o + 3] = fmaf(q.w, v, a1[4 * o + 3]);
        }
        PeIter it(v);
#pragma unroll 1
        for (int k = 0; k < pe_L; ++k) {
          const float4* ws = w + (1 + 2 * k) * (H / 4);
          const float4* wc = w + (2 + 2 * k) * (H / 4);
          const float sn = it.s, cs = it.c;
#pragma unroll
          for (int o = 0; o < H / 4; ++o) {
            const float4 q = ws[o], r = wc[o];
            a1[4 * o] = fmaf(r.x, cs, fmaf(q.x, sn, a1[4 * o]));
            a1[4 * o + 1] = fmaf(r.y, cs, fmaf(q.y, sn, a1[4 * o + 1]));
            a1[4 * o + 2] = fmaf(r.z, cs, fmaf(q.z, sn, a1[4 * o + 2]));
            a1[4 * o + 3] = fmaf(r.w, cs, fmaf(q.w, sn, a1[4 * o + 3]));
          }
          it.next();
        }
      }
#pragma unroll
      for (int o = 0; o < H; ++o) a1[o] = relu(a1[o]);
    }
#pragma unroll 4
    for (int o = 0; o < H; ++o) {
      float a = b2[o];
#pragma unroll
      for (int i = 0; i < H; ++i) a = fmaf(W2[o * H + i], a1[i], a);
      s[o] += relu(a);
    }
  }
  if (pool == 1 && m > 0) {
#pragma unroll
    for (int o = 0; o < H; ++o) s[o] = __fdiv_rn(s[o], (float)m);
  }
  if (!SIG)   // B's e0 input, loaded only now (not live across the fragment loop)
#pragma unroll
    for (int i = 0; i < C0; i += 8) load8(e0 + p * C0 + i, ev + i);
  float ld[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) ld[i] = to_f(direct[p * 3 + i]);
  float ps0 = bO[0], ps1 = bO[1], ps2 = bO[2];
  if (r_takes_ld) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      ps0 = fmaf(WO[0 * NO + C0 + i], ld[i], ps0);
      ps1 = fmaf(WO[1 * NO + C0 + i], ld[i], ps1);
      ps2 = fmaf(WO[2 * NO + C0 + i], ld[i], ps2);
    }
  }
#pragma unroll 2
  for (int o = 0; o < C0; ++o) {
    const float* wb = WB + o * NB;
    float a = bB[o];
#pragma unroll
    for (int i = 0; i < C0; ++i) a = fmaf(wb[i], ev[i], a);
#pragma unroll
    for (int j = 0; j < H; ++j) a = fmaf(wb[C0 + j], s[j], a);
    a = fmaf(wb[C0 + H], (float)m, a);
    const float phi = relu(a);
    ps0 = fmaf(WO[0 * NO + o], phi, ps0);
    ps1 = fmaf(WO[1 * NO + o], phi, ps1);
    ps2 = fmaf(WO[2 * NO + o], phi, ps2);
  }
  psi[p * 3 + 0] = ps0; psi[p * 3 + 1] = ps1; psi[p * 3 + 2] = ps2;
}

// Row geometry of an up2 step: the coarse input may be a row tile with halo rows.
//   fine interior row Y (0..rows_f) is global row grow0_f + Y; its bilinear taps are
//   clamped in GLOBAL coarse rows [0, Hc_full) and read from local buffer row
//   (tap - grow0_c + halo).  Full frame: grow0 = 0, halo = 0, buffers = interior.

// d = up2(y) + skip (bilinear x2, half-pixel, edge clamp, cropped), 8 channels/thread.
template <typename T>
__global__ void k_up2add(const T* __restrict__ y, int w, const T* __restrict__ skip, T* __restrict__ d, int W2,
                         int C, Up2Rows g, long nvec) {
  long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nvec) return;
  const int cv = C / 8;
  const int c8 = (int)(t % cv) * 8;
  long r = t / cv;
  const int X = (int)(r % W2); r /= W2;
  const int Y = (int)(r % g.rows_f);
  const long b = r / g.rows_f;
  int ya, yb, xa, xb; float wya, wyb, wxa, wxb;
  up2_taps(g.grow0_f + Y, g.Hc_full, ya, yb, wya, wyb);
  ya += g.halo - g.grow0_c;
  yb += g.halo - g.grow0_c;
  up2_taps(X, w, xa, xb, wxa, wxb);
  const long yb0 = b * g.rows_c_buf;
  float v00[8], v01[8], v10[8], v11[8], sk[8], o[8];
  load8(y + ((yb0 + ya) * w + xa) * C + c8, v00);
  load8(y + ((yb0 + ya) * w + xb) * C + c8, v01);
  load8(y + ((yb0 + yb) * w + xa) * C + c8, v10);
  load8(y + ((yb0 + yb) * w + xb) * C + c8, v11);
  const long q = ((b * g.rows_f_buf + Y + g.halo) * W2 + X) * C + c8;
  load8(skip + q, sk);
#pragma unroll
  for (int i = 0; i < 8; ++i)
    o[i] = (wya * wxa) * v00[i] + (wya * wxb) * v01[i] + (wyb * wxa) * v10[i] + (wyb * wxb) * v11[i] + sk[i];
  store8(d + q, o);
}

// out = sigmoid(up2(z) + psi): the level-0 skip-add and output 1x1 rewritten with the
// 3-channel projections (reading R15; exact in real arithmetic by linearity).
__global__ void k_output(const float* __restrict__ z, int w, const float* __restrict__ psi,
                         float* __restrict__ out, int W, Up2Rows g, long P) {
  long p = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const int X = (int)(p % W);
  long r = p / W;
  const int Y = (int)(r % g.rows_f);
  const long b = r / g.rows_f;
  int ya, yb, xa, xb; float wya, wyb, wxa, wxb;
  up2_taps(g.grow0_f + Y, g.Hc_full, ya, yb, wya, wyb);
  ya += g.halo - g.grow0_c;
  yb += g.halo - g.grow0_c;
  up2_taps(X, w, xa, xb, wxa, wxb);
  const long zb0 = b * g.rows_c_buf;
  const float* z00 = z + ((zb0 + ya) * w + xa) * 3;
  const float* z01 = z + ((zb0 + ya) * w + xb) * 3;
  const float* z10 = z + ((zb0 + yb) * w + xa) * 3;
  const float* z11 = z + ((zb0 + yb) * w + xb) * 3;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    float l = (wya * wxa) * z00[c] + (wya * wxb) * z01[c] + (wyb * wxa) * z10[c] + (wyb * wxb) * z11[c];
    l += psi[p * 3 + c];
    out[p * 3 + c] = 1.f / (1.f + expf(-l));
  }
}

}  // namespace gn
