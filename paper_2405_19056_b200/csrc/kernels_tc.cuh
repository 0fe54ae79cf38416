// kernels_tc.cuh -- tcgen05 tensor-core kernels for bf16 mode.
//
// k_tb_tc: the fused T + B + psi kernel; its design is documented at
// the top of kernels_tb_tc.cuh.  This file holds the host-side packing and launchers.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <vector>

#include "kernels_conv_tc.cuh"
#include "kernels_ew.cuh"
#include "kernels_tb_tc.cuh"
#include "net.h"
#include "tc_ptx.cuh"

namespace gn {

// ------------------------------------------------------------------------ host side
// Weights-level description of one conv layer (packed once per handle).
struct TcConv {
  bool used = false;
  int S = 1, Cin = 0, Cout = 0, NS = 0, nsplit = 1, nstage = 2, epi = 0, ws = 0, ost = 0;   // ws: weights streamed, ost: staged output
  int rr = 1;                    // output rows per tile (stride 1)
  size_t smem = 0;
  int ctas_per_sm = 1;
  uint8_t* wimg = nullptr;
  const float* bias = nullptr;
  const float* wz = nullptr;     // EPI 1/2 projection weights [3][Cout] (nullptr: the handle's R15 wz)
};

// One conv layer in one execution geometry (buffers, row offsets, tensor maps).
struct ConvGeom {
  int Hi_buf = 0, Wi = 0, Ho = 0, Wo = 0, in_row_off = 0, out_row_off = 0, out_rows_buf = 0;
  CUtensorMap mA, mO;
  uint16_t* out = nullptr;
  float* zout = nullptr;
};

// An execution geometry: the full frame (halo = 0, batch up to max_batch) or one rank's
// row tile of a single frame (halo = 1: every activation buffer carries one extra row
// above and below its interior rows; at the frame's top/bottom these stay zero).
struct Geom {
  int halo = 0, L = 0, Bmax = 1;
  int rows[4] = {}, W[4] = {}, grow0[4] = {}, Hfull[4] = {};
  void *x16 = nullptr, *e[4] = {}, *y[4] = {}, *dd[4] = {};
  float *psi = nullptr, *z = nullptr;
  ConvGeom cg[8];                 // [l] = F_l, [4+l] = R_l
  std::vector<void*> owned;       // buffers allocated for this geometry (tiles)
  size_t bytes = 0;
};

struct TcState {
  uint8_t* tb_wimg = nullptr;   // T+B weight image (K-major, no-swizzle planes)
  cudaStream_t sort_st = nullptr;   // the count sort runs here, beside the F encoder
  cudaEvent_t ev_fwd = nullptr, ev_sorted = nullptr;
  // row tiles: T runs on its own stream right after F0 (it needs no halo), overlapping the rest
  // of the encoder/decoder and their halo exchanges; the output stage waits for it
  cudaStream_t tb_st = nullptr;
  cudaEvent_t ev_e0 = nullptr, ev_tb = nullptr;
  TbParams tb_prm;              // bB, wBn, WO (c0+3 wide), bO (kernel parameters)
  TcConv conv[8];               // [l] = F_l, [4+l] = R_l
  Geom full;                    // the handle's own workspace
  Geom* tile = nullptr;         // row-tile geometry (forward_sharded)
  TcConv ssconv[2];             // N3 super-sampler: S1 (GB = 2), S2 (EPI = 2)
  ConvGeom ssg[2];
  TcConv objconv[2];            // N4 object-major h: T1 (16 -> h), T2 (h -> h, EPI = 3 accumulate)
  ConvGeom objg[2];
  int* sched = nullptr;         // T kernel's dynamic tile counter
  uint32_t* perm = nullptr;     // T kernel's count-sorted pixel order (k_tb_sort), one entry per pixel
  long perm_cap = 0;
  int tile_nranks = 0, tile_rank = -1;
};

static inline uint16_t h_bf16(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  u = (u + 0x7FFFu + ((u >> 16) & 1u)) >> 16;
  return (uint16_t)u;
}
static inline float h_bf16f(uint16_t b) {
  uint32_t u = (uint32_t)b << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}
static inline uint16_t h_f16(float f) {
  __half h = __float2half_rn(f);
  uint16_t u;
  memcpy(&u, &h, 2);
  return u;
}

// K-major, SWIZZLE_NONE operand image: plane j (K columns 8j..8j+7) holds all N rows.
static void pack_kmajor(const std::vector<float>& W, int N, int Kc, bool f16, std::vector<uint8_t>& out) {
  const size_t base = out.size();
  out.resize(base + (size_t)N * Kc * 2);
  uint16_t* o = reinterpret_cast<uint16_t*>(out.data() + base);
  for (int j = 0; j < Kc / 8; ++j)
    for (int n = 0; n < N; ++n)
      for (int kk = 0; kk < 8; ++kk) {
        const float v = W[(size_t)n * Kc + 8 * j + kk];
        o[((size_t)j * N + n) * 8 + kk] = f16 ? h_f16(v) : h_bf16(v);
      }
}

// b = hi + mid + lo with each piece bf16 (exact for normal fp32 b).
static void split3(float b, float& hi, float& mid, float& lo) {
  hi = h_bf16f(h_bf16(b));
  double r = (double)b - hi;
  mid = h_bf16f(h_bf16((float)r));
  r -= mid;
  lo = h_bf16f(h_bf16((float)r));
}

inline int tc_pack_weights(glassnet* net, const float* T1W, const float* T1b, const float* T2W, const float* T2b,
                           const std::vector<const float*>& FW, const std::vector<const float*>& Fb,
                           const float* BW, const float* Bb, const std::vector<const float*>& RW,
                           const std::vector<const float*>& Rb, const float* OW, const float* Ob) {
  (void)FW; (void)Fb; (void)RW; (void)Rb;
  const glassnet_dims& d = net->d;
  const int H = d.t_hidden, C0 = d.widths[0];
  const bool norm = (d.flags & GLASSNET_FLAG_INPUT_NORM) != 0;
  const bool ld = (d.flags & GLASSNET_FLAG_R_TAKES_LD) != 0;
  TcState* s = new TcState();
  net->tc_state = s;
  auto rb = [](float v) { return h_bf16f(h_bf16(v)); };
  std::vector<uint8_t> img;
  // W1 as K=16 windows [H][16], two variants (kernels_tb_tc.cuh): even = the record's 11 weights
  // (depth column x 2^-7 when normalising; bf16-exact) at columns 0..10, odd = at columns 1..11;
  // both: b1 as three exact bf16 pieces at columns 12..14 (the record window carries 1.0 there)
  const bool sig = (d.flags & GLASSNET_FLAG_SIGMA_COND) != 0;
  // N1: T1.W rows are [record weights ; sigma weights].  With N2 (positional encoding) T runs on
  // the SIMT kernel and these windows are not used.
  const int nin = gn_rec_in(d) + (sig ? C0 : 0);
  for (int v = 0; v < 2; ++v) {
    std::vector<float> w1((size_t)H * 16, 0.f);
    for (int n = 0; n < H; ++n) {
      for (int i = 0; i < 11; ++i) w1[(size_t)n * 16 + v + i] = rb(T1W[n * nin + i]) * ((norm && i == 7) ? 0.0078125f : 1.f);
      split3(T1b[n], w1[(size_t)n * 16 + 12], w1[(size_t)n * 16 + 13], w1[(size_t)n * 16 + 14]);
    }
    pack_kmajor(w1, H, 16, false, img);
  }
  // W2 [H][H], scaled by 2^-11 (exact: a power of two), so acc2 = (W2 a1) 2^-11 and the pool's
  // FADD.SAT with b2 2^-11 is ReLU + saturation at a2 = 2048 in one instruction
  std::vector<float> w2((size_t)H * H, 0.f);
  for (int o = 0; o < H; ++o)
    for (int i = 0; i < H; ++i) w2[(size_t)o * H + i] = rb(T2W[o * H + i]) * TB_VSCALE;
  pack_kmajor(w2, H, H, false, img);
  const int NB = C0 + H + 1;
  std::vector<float> wbt((size_t)C0 * H), wbe((size_t)C0 * C0);
  for (int o = 0; o < C0; ++o) {
    for (int j = 0; j < H; ++j) wbt[(size_t)o * H + j] = rb(BW[(size_t)o * NB + C0 + j]);
    for (int i = 0; i < C0; ++i) wbe[(size_t)o * C0 + i] = rb(BW[(size_t)o * NB + i]);
  }
  pack_kmajor(wbe, C0, C0, false, img);
  pack_kmajor(wbt, C0, H, true, img);   // f16: tau is an f16 operand (reading R19)
  {   // N1: W1's sigma part [H][C0] (layer 1 += e0 W1,sigma^T: two more MMAs per item from the
      // tile's e0 operand); zeros (and unused) without GLASSNET_FLAG_SIGMA_COND
    std::vector<float> w1e((size_t)H * C0, 0.f);
    if (sig)
      for (int n = 0; n < H; ++n)
        for (int j = 0; j < C0; ++j) w1e[(size_t)n * C0 + j] = rb(T1W[n * nin + 11 + j]);
    pack_kmajor(w1e, H, C0, false, img);
  }
  TbParams& prm = s->tb_prm;
  memset(&prm, 0, sizeof prm);
  for (int o = 0; o < C0; ++o) prm.bB[o] = Bb[o];
  for (int o = 0; o < C0; ++o) prm.wBn[o] = rb(BW[(size_t)o * NB + C0 + H]);
  const int NO = C0 + (ld ? 3 : 0);
  for (int j = 0; j < 3; ++j)
    for (int i = 0; i < C0 + 3; ++i) prm.WO[j * (C0 + 3) + i] = i < NO ? rb(OW[(size_t)j * NO + i]) : 0.f;
  for (int j = 0; j < 3; ++j) prm.bO[j] = Ob[j];
  for (int o = 0; o < H; ++o) prm.b2s[o] = T2b[o] * TB_VSCALE;
  prm.sigma = sig ? 1 : 0;
  s->perm_cap = ((long)d.max_batch * d.height * d.width + TB_SBP - 1) / TB_SBP * TB_SBP;
  if (cudaMalloc(&s->tb_wimg, img.size()) != cudaSuccess || cudaMalloc(&s->sched, sizeof(int)) != cudaSuccess ||
      cudaMalloc(&s->perm, s->perm_cap * sizeof(uint32_t)) != cudaSuccess)
    return gn_fail(GLASSNET_ERR_OUT_OF_MEMORY, "tc weight alloc");
  cudaMemcpy(s->tb_wimg, img.data(), img.size(), cudaMemcpyHostToDevice);
  net->w_bytes += img.size() + sizeof(TbParams);
  return 0;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// Halo tensor maps over an NHWC bf16 activation [B][Hbuf][W][C] (zero fill out of bounds).
static int make_halo_maps(int S, ConvGeom& G, void* in, int B, int C, int rr) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return gn_fail(GLASSNET_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r;
  if (S == 1) {
    // (C, x, row, frame): a box of {16 channels, 130 px, rr + 2 rows} = 32-byte pixel rows
    const cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)G.Wi, (cuuint64_t)G.Hi_buf, (cuuint64_t)B};
    const cuuint64_t str[3] = {(cuuint64_t)C * 2, (cuuint64_t)G.Wi * C * 2, (cuuint64_t)G.Hi_buf * G.Wi * C * 2};
    const cuuint32_t box[4] = {16, conv::Halo<1>::SLOTS, (cuuint32_t)(rr + 2), 1};
    r = enc(&G.mA, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, in, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    G.mO = G.mA;
  } else {
    // (C, parity, x/2, frame*rows)
    const cuuint64_t dims[4] = {(cuuint64_t)C, 2, (cuuint64_t)G.Wi / 2, (cuuint64_t)G.Hi_buf * B};
    const cuuint64_t str[3] = {(cuuint64_t)C * 2, (cuuint64_t)C * 4, (cuuint64_t)G.Wi * C * 2};
    const cuuint32_t boxE[4] = {16, 1, conv::TILE_M, 3};
    const cuuint32_t boxO[4] = {16, 1, conv::TILE_M + 1, 3};
    r = enc(&G.mA, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, in, dims, str, boxE, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r == CUDA_SUCCESS)
      r = enc(&G.mO, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, in, dims, str, boxO, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (r != CUDA_SUCCESS) return gn_fail(GLASSNET_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return 0;
}

static size_t conv_smem(int S, int Cin, int NS, int nstage, int ws = 0, int ost = 0, int rr = 1, int epi = 0) {
  const size_t tx = S == 1 ? (size_t)(rr + 2) * conv::Halo<1>::ROW : conv::Halo<2>::TX;
  const size_t sb = (tx + 1023) / 1024 * 1024 + (ws ? (size_t)9 * 2 * NS * 16 : 0);
  const size_t w = ws ? 0 : (((size_t)9 * Cin * NS * 2 + 1023) / 1024) * 1024;
  const size_t bias = ((size_t)NS * 4 * (epi ? 4 : 1) + 127) / 128 * 128;   // bias (+ the z projection's 3 x NS)
  return w + nstage * sb + (2 * nstage + 4) * 8 + bias + (ost ? (size_t)4 * 2 * 32 * NS * 2 : 0) + 128;
}

// One conv layer: choose the N split so the split's weights stay resident, pack them.
static int setup_conv(glassnet* net, TcConv& L, int S, const float* W, const float* bias, int cin_real, int Cin,
                      int Cout, int epi, const float* in_scale = nullptr) {
  constexpr size_t LIMIT = 232448 - 1024;
  L.used = true; L.S = S; L.Cin = Cin; L.Cout = Cout; L.epi = epi;
  int NS = Cout;
  // full width with resident weights if they fit; else full width with the weights streamed
  // per channel chunk (no N-split: an N-split re-reads the halo and multiplies the MMA count)
  L.ws = (conv_smem(S, Cin, Cout, 2, 0, 0, 1, epi) > LIMIT && Cout <= 256 && conv_smem(S, Cin, Cout, 2, 1, 0, 1, epi) <= LIMIT && epi == 0 &&
          !getenv("GN_CONV_NO_STREAM")) ? 1 : 0;
  if (!L.ws)
    while (NS > 16 && conv_smem(S, Cin, NS, 2, 0, 0, 1, epi) > LIMIT) NS /= 2;
  if (conv_smem(S, Cin, NS, 2, L.ws, 0, 1, epi) > LIMIT || (epi >= 1 && NS != Cout))
    return gn_fail(GLASSNET_ERR_UNSUPPORTED, "conv %d->%d does not fit shared memory", Cin, Cout);
  L.NS = NS;
  L.nsplit = Cout / NS;
  // multi-row tiles (stride 1): as many rows (4, 2) as TMEM (2 x rr x NS columns) and shared
  // memory (>= 2 stages) allow
  L.rr = 1;
  if (S == 1)
    for (int rr : {4, 2})
      if (2 * rr * NS <= 512 && conv_smem(S, Cin, NS, 2, L.ws, 0, rr, epi) <= LIMIT) { L.rr = rr; break; }
  if (const char* e = getenv("GN_CONV_RR")) if (S == 1) L.rr = atoi(e);
  L.nstage = 4;
  if (const char* e = getenv("GN_CONV_NSTAGE")) L.nstage = atoi(e);   // diagnostic: pipeline depth cap
  while (L.nstage > 2 && conv_smem(S, Cin, NS, L.nstage, L.ws, 0, L.rr, epi) > LIMIT) --L.nstage;
  // staged (bulk-copied) output when it fits without giving up pipeline depth
  L.ost = (epi == 0 && !L.ws && conv_smem(S, Cin, NS, L.nstage, L.ws, 1, L.rr, epi) <= LIMIT && !getenv("GN_CONV_NO_OST"))
              ? 1 : 0;
  L.smem = conv_smem(S, Cin, NS, L.nstage, L.ws, L.ost, L.rr, epi);
  const int acc2 = 2 * L.rr * NS;
  const int tcols = acc2 <= 32 ? 32 : acc2 <= 64 ? 64 : acc2 <= 128 ? 128 : acc2 <= 256 ? 256 : 512;
  // a tcgen05.mma issue blocks its thread for about one MMA, so two CTAs per SM (two MMA
  // issuers) beat a deeper pipeline: trade stages for a second CTA when TMEM allows it
  if (2 * tcols <= 512)
    for (int ns = L.nstage; ns >= 2; --ns)
      if (2 * (conv_smem(S, Cin, NS, ns, L.ws, L.ost, L.rr, epi) + 1024) <= 232448) {
        L.nstage = ns;
        L.smem = conv_smem(S, Cin, NS, ns, L.ws, L.ost, L.rr, epi);
        break;
      }
  L.ctas_per_sm = (int)(232448 / (L.smem + 1024));
  if (L.ctas_per_sm > 2) L.ctas_per_sm = 2;
  if (L.ctas_per_sm * tcols > 512) L.ctas_per_sm = 512 / tcols;
  if (L.ctas_per_sm < 1) L.ctas_per_sm = 1;
  // weights: resident [split][tap][Cin/8][NS][8]; streamed [Cin/16][tap][2][NS][8] (one
  // contiguous block per 16-channel chunk) -- bf16
  std::vector<uint16_t> img((size_t)L.nsplit * 9 * Cin * NS, 0);
  for (int sp = 0; sp < L.nsplit; ++sp)
    for (int t = 0; t < 9; ++t)
      for (int j = 0; j < Cin / 8; ++j)
        for (int n = 0; n < NS; ++n)
          for (int kk = 0; kk < 8; ++kk) {
            const int co = sp * NS + n, ci = 8 * j + kk;
            const float v = ci < cin_real ? W[((size_t)co * 9 + t) * cin_real + ci] * (in_scale ? in_scale[ci] : 1.f)
                                          : 0.f;
            const size_t idx = L.ws ? (((((size_t)(j / 2) * 9 + t) * 2 + (j % 2)) * NS + n) * 8 + kk)
                                    : (((((size_t)sp * 9 + t) * (Cin / 8) + j) * NS + n) * 8 + kk);
            img[idx] = h_bf16(v);
          }
  if (cudaMalloc(&L.wimg, img.size() * 2) != cudaSuccess)
    return gn_fail(GLASSNET_ERR_OUT_OF_MEMORY, "conv weight image");
  cudaMemcpy(L.wimg, img.data(), img.size() * 2, cudaMemcpyHostToDevice);
  net->w_bytes += img.size() * 2;
  L.bias = bias;
  return 0;
}

inline int tc_setup_convs(glassnet* net, const std::vector<const float*>& FW, const std::vector<const float*>& RW) {
  TcState* s = reinterpret_cast<TcState*>(net->tc_state);
  const glassnet_dims& d = net->d;
  const int L = d.levels;
  const int* c = d.widths;
  // F0's weights carry the input normalisation (reading R9: position x 2^-3, depth x 2^-7 --
  // powers of two, so bf16(W) x scale is exact and each MMA product equals the one on the
  // normalised input bit for bit): F0 then reads the raw G-buffer (full frame: directly, no
  // x16; row tiles: x16 built without normalisation)
  float sc0[16];
  for (int i = 0; i < 16; ++i) sc0[i] = 1.f;
  if (d.flags & GLASSNET_FLAG_INPUT_NORM) { sc0[0] = sc0[1] = sc0[2] = 0.125f; sc0[11] = 0.0078125f; }
  // N2: F0 reads the stored gamma(x) (normalised before the encoding: no weight scale)
  int rc = gn_pe_L(d) ? setup_conv(net, s->conv[0], 1, FW[0], net->convB[0], gn_x_in(d), gn_x_ch(d), c[0], 0)
                      : setup_conv(net, s->conv[0], 1, FW[0], net->convB[0], 15, 16, c[0], 0, sc0);
  for (int l = 1; l < L && !rc; ++l) rc = setup_conv(net, s->conv[l], 2, FW[l], net->convB[l], c[l - 1], c[l - 1], c[l], 0);
  for (int l = L - 1; l >= 1 && !rc; --l)
    rc = setup_conv(net, s->conv[4 + l], 1, RW[l], net->convB[4 + l], c[l], c[l], c[l - 1], l == 1 ? 1 : 0);
  return rc;
}

// Fill the per-layer conv geometry of G (buffers already set).
static int geom_convs(glassnet* net, Geom& G) {
  TcState* s = reinterpret_cast<TcState*>(net->tc_state);
  const int L = G.L, h = G.halo;
  const int* c = net->d.widths;
  auto set = [&](int idx, int lin, int S, void* in, int cin, int lout, void* out, float* zout) {
    ConvGeom& g = G.cg[idx];
    g.Hi_buf = G.rows[lin] + 2 * h; g.Wi = G.W[lin];
    g.Ho = G.rows[lout]; g.Wo = G.W[lout];
    g.in_row_off = h; g.out_row_off = h; g.out_rows_buf = G.rows[lout] + 2 * h;
    g.out = reinterpret_cast<uint16_t*>(out);
    g.zout = zout;
    return make_halo_maps(S, g, in, G.Bmax, cin, s->conv[idx].rr);
  };
  int rc = set(0, 0, 1, G.x16, gn_x_ch(net->d), 0, G.e[0], nullptr);
  for (int l = 1; l < L && !rc; ++l) rc = set(l, l - 1, 2, G.e[l - 1], c[l - 1], l, G.e[l], nullptr);
  for (int l = L - 1; l >= 1 && !rc; --l) {
    void* in = (l == L - 1) ? G.e[L - 1] : G.dd[l];
    rc = set(4 + l, l, 1, in, c[l], l, l == 1 ? nullptr : G.y[l], l == 1 ? G.z : nullptr);
  }
  (void)s;
  return rc;
}

// The handle's full-frame geometry over its own workspace.
inline int tc_setup_full_geom(glassnet* net) {
  TcState* s = reinterpret_cast<TcState*>(net->tc_state);
  Geom& G = s->full;
  const glassnet_dims& d = net->d;
  G.halo = 0; G.L = d.levels; G.Bmax = d.max_batch;
  for (int l = 0; l < d.levels; ++l) {
    G.rows[l] = d.height >> l; G.W[l] = d.width >> l; G.grow0[l] = 0; G.Hfull[l] = d.height >> l;
    G.e[l] = net->e[l]; G.y[l] = net->y[l]; G.dd[l] = net->dd[l];
  }
  G.x16 = net->x16; G.psi = net->psi; G.z = net->z;
  return geom_convs(net, G);
}

// N3 super-sampler S on the tensor cores: S1 = k_conv_tc<..., GB = 2> (its producers build the
// [G'_hi, bf16(up_nearest(img)), 0] halo), S2 = k_conv_tc<..., EPI = 2> (projection, residual,
// clamp in the epilogue): the hi-res input x and the residual r never reach HBM, only s1 does.
inline int tc_setup_ss(glassnet* net, const float* S1W, const float* S2W) {
  TcState* s = reinterpret_cast<TcState*>(net->tc_state);
  const glassnet_dims& d = net->d;
  const int c0 = d.widths[0];
  float sc0[16];
  for (int i = 0; i < 16; ++i) sc0[i] = 1.f;
  if (d.flags & GLASSNET_FLAG_INPUT_NORM) { sc0[0] = sc0[1] = sc0[2] = 0.125f; sc0[11] = 0.0078125f; }
  int rc = setup_conv(net, s->ssconv[0], 1, S1W, net->ssB[0], 15, 16, c0, 0, sc0);
  if (!rc) rc = setup_conv(net, s->ssconv[1], 1, S2W, net->ssB[1], c0, c0, c0, 2);
  if (rc) return rc;
  s->ssconv[1].wz = net->ss_wz;
  for (int i = 0; i < 2 && !rc; ++i) {
    ConvGeom& g = s->ssg[i];
    g.Hi_buf = 2 * d.height; g.Wi = 2 * d.width; g.Ho = 2 * d.height; g.Wo = 2 * d.width;
    g.in_row_off = 0; g.out_row_off = 0; g.out_rows_buf = 2 * d.height;
    g.out = i == 0 ? reinterpret_cast<uint16_t*>(net->ss_s1) : nullptr;
    g.zout = nullptr;   // S2: the caller's out_hi, set per call
    // S1's producers build the halo themselves (the map, over s1, is valid but unused); S2 reads s1
    rc = make_halo_maps(1, g, net->ss_s1, d.max_batch, c0, s->ssconv[i].rr);
  }
  return rc;
}


// Row-tile geometry for rank `rank` of `nranks` (one frame, halo rows, own buffers).
inline int tc_setup_tile_geom(glassnet* net, int nranks, int rank, int row0, int rows0) {
  TcState* s = reinterpret_cast<TcState*>(net->tc_state);
  if (s->tile && s->tile_nranks == nranks && s->tile_rank == rank) return 0;
  if (s->tile) { for (void* q : s->tile->owned) cudaFree(q); delete s->tile; s->tile = nullptr; }
  const glassnet_dims& d = net->d;
  const int L = d.levels;
  const int* c = d.widths;
  Geom* G = new Geom();
  G->halo = 1; G->L = L; G->Bmax = 1;
  for (int l = 0; l < L; ++l) {
    G->rows[l] = rows0 >> l; G->W[l] = d.width >> l; G->grow0[l] = row0 >> l; G->Hfull[l] = d.height >> l;
  }
  auto alloc = [&](size_t bytes) -> void* {
    void* q = nullptr;
    if (cudaMalloc(&q, bytes) != cudaSuccess) return nullptr;
    cudaMemset(q, 0, bytes);
    G->owned.push_back(q);
    G->bytes += bytes;
    return q;
  };
  bool ok = (G->x16 = alloc((size_t)(G->rows[0] + 2) * G->W[0] * gn_x_ch(d) * 2)) != nullptr;
  for (int l = 0; l < L && ok; ++l) ok = (G->e[l] = alloc((size_t)(G->rows[l] + 2) * G->W[l] * c[l] * 2)) != nullptr;
  for (int l = 2; l < L && ok; ++l) ok = (G->y[l] = alloc((size_t)(G->rows[l] + 2) * G->W[l] * c[l - 1] * 2)) != nullptr;
  for (int l = 1; l < L - 1 && ok; ++l) ok = (G->dd[l] = alloc((size_t)(G->rows[l] + 2) * G->W[l] * c[l] * 2)) != nullptr;
  if (ok) ok = (G->z = (float*)alloc((size_t)(G->rows[1] + 2) * G->W[1] * 3 * 4)) != nullptr;
  if (ok) ok = (G->psi = (float*)alloc((size_t)G->rows[0] * G->W[0] * 3 * 4)) != nullptr;
  if (!ok) {
    for (void* q : G->owned) cudaFree(q);
    delete G;
    return gn_fail(GLASSNET_ERR_OUT_OF_MEMORY, "row-tile workspace");
  }
  int rc = geom_convs(net, *G);
  if (rc) { for (void* q : G->owned) cudaFree(q); delete G; return rc; }
  s->tile = G;
  s->tile_nranks = nranks;
  s->tile_rank = rank;
  return 0;
}

template <int S, int NS, int EPI, int WS, int OST, int RR, int GB = 0>
static void launch_conv_k(glassnet* net, const TcConv& L, const ConvGeom& G, int B, cudaStream_t st,
                          const void* gbuf = nullptr, const void* direct = nullptr, const float* img = nullptr,
                          const float* b3 = nullptr, const uint8_t* cover = nullptr, int edge = 0) {
  auto kfn = conv::k_conv_tc<S, NS, EPI, WS, OST, RR, GB>;
  const long ntiles = (long)B * conv::edge_row_tiles((G.Ho + RR - 1) / RR, edge) * ((G.Wo + conv::TILE_M - 1) / conv::TILE_M);
  if (ntiles == 0) return;   // edge mode 2 of a tile with <= 2 row tiles: nothing inside
  static int smem_set = -1;   // the attribute is set once per instantiation and size (not per launch)
  if (smem_set < (int)L.smem) {
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.smem);
    smem_set = (int)L.smem;
  }
  conv::ConvArgs a;
  a.wimg = L.wimg; a.bias = L.bias; a.out = G.out; a.wz = L.wz ? L.wz : net->wz; a.zout = G.zout;
  a.img = img;
  for (int i = 0; i < 3; ++i) a.b3[i] = b3 ? b3[i] : 0.f;
  a.cover = cover; a.tau_q = net->tau_q; a.tau_n = net->tau_n; a.qscale = net->qscale; a.qsat = net->qsat;
  a.edge = edge;
  a.Cin = L.Cin; a.Cout = L.Cout; a.Ho = G.Ho; a.Wo = G.Wo; a.B = B; a.nsplit = L.nsplit; a.nstage = L.nstage;
  a.in_row_off = G.in_row_off; a.out_row_off = G.out_row_off; a.out_rows_buf = G.out_rows_buf;
  a.in_rows_buf = G.Hi_buf;
  a.gbuf = reinterpret_cast<const uint16_t*>(gbuf); a.direct = reinterpret_cast<const uint16_t*>(direct); a.Wi = G.Wi;
  long per_split = (long)net->num_sms * L.ctas_per_sm / L.nsplit;
  if (per_split > ntiles) per_split = ntiles;
  if (per_split < 1) per_split = 1;
  kfn<<<(unsigned)(per_split * L.nsplit), GB ? 32 * (5 + conv::GB_PRODUCERS) : 192, L.smem, st>>>(G.mA, G.mO, a);
}

static int launch_conv(glassnet* net, const TcConv& L, const ConvGeom& G, int B, cudaStream_t st,
                       const void* gbuf = nullptr, const void* direct = nullptr, const float* img = nullptr,
                       const float* b3 = nullptr, const uint8_t* cover = nullptr, int edge = 0) {
  if (L.epi == 3) {   // N4: h's second conv, accumulated into the fixed-point latent where covered
#define CONV_E3(NS_, RR_)                                                                                \
    if (L.S == 1 && L.NS == NS_ && L.ws == 0 && L.ost == 0 && L.rr == RR_) {                            \
      launch_conv_k<1, NS_, 3, 0, 0, RR_>(net, L, G, B, st, nullptr, nullptr, nullptr, nullptr, cover); \
      return 0;                                                                                         \
    }
    CONV_E3(32, 1) CONV_E3(32, 2) CONV_E3(32, 4) CONV_E3(64, 1) CONV_E3(64, 2) CONV_E3(64, 4)
#undef CONV_E3
    return gn_fail(GLASSNET_ERR_UNSUPPORTED, "object conv: NS=%d rr=%d", L.NS, L.rr);
  }
  if (gbuf && img) {   // N3 S1: the hi-res G-buffer + the nearest-upsampled image
#define CONV_GB2(NS_, OST_, RR_)                                                                         \
    if (L.S == 1 && L.NS == NS_ && L.epi == 0 && L.ws == 0 && L.ost == OST_ && L.rr == RR_) {           \
      launch_conv_k<1, NS_, 0, 0, OST_, RR_, 2>(net, L, G, B, st, gbuf, nullptr, img);                 \
      return 0;                                                                                         \
    }
    CONV_GB2(16, 0, 4) CONV_GB2(16, 1, 4) CONV_GB2(32, 0, 4) CONV_GB2(32, 1, 4)
    CONV_GB2(16, 0, 2) CONV_GB2(16, 1, 2) CONV_GB2(32, 0, 2) CONV_GB2(32, 1, 2)
#undef CONV_GB2
    return gn_fail(GLASSNET_ERR_UNSUPPORTED, "S1 from the G-buffer: NS=%d ost=%d rr=%d", L.NS, L.ost, L.rr);
  }
  if (img) {   // N3 S2: the residual epilogue
#define CONV_E2(NS_, RR_)                                                                                \
    if (L.S == 1 && L.NS == NS_ && L.epi == 2 && L.ws == 0 && L.ost == 0 && L.rr == RR_) {              \
      launch_conv_k<1, NS_, 2, 0, 0, RR_>(net, L, G, B, st, nullptr, nullptr, img, b3);                 \
      return 0;                                                                                         \
    }
    CONV_E2(16, 1) CONV_E2(16, 2) CONV_E2(16, 4) CONV_E2(32, 1) CONV_E2(32, 2) CONV_E2(32, 4)
#undef CONV_E2
    return gn_fail(GLASSNET_ERR_UNSUPPORTED, "S2: NS=%d rr=%d", L.NS, L.rr);
  }
  if (gbuf) {   // F0 straight from the G-buffer (full frame)
#define CONV_GB(NS_, OST_, RR_)                                                                          \
    if (L.S == 1 && L.NS == NS_ && L.epi == 0 && L.ws == 0 && L.ost == OST_ && L.rr == RR_) {           \
      launch_conv_k<1, NS_, 0, 0, OST_, RR_, 1>(net, L, G, B, st, gbuf, direct);                       \
      return 0;                                                                                         \
    }
    CONV_GB(16, 0, 4) CONV_GB(16, 1, 4) CONV_GB(32, 0, 4) CONV_GB(32, 1, 4)
    CONV_GB(16, 0, 2) CONV_GB(16, 1, 2) CONV_GB(32, 0, 2) CONV_GB(32, 1, 2)
#undef CONV_GB
    return gn_fail(GLASSNET_ERR_UNSUPPORTED, "F0 from the G-buffer: NS=%d ost=%d rr=%d", L.NS, L.ost, L.rr);
  }
#define CONV_K(S_, NS_, E_, WS_, OST_, RR_)                                                              \
  if (L.S == S_ && L.NS == NS_ && L.epi == E_ && L.ws == WS_ && L.ost == OST_ && L.rr == RR_) {         \
    launch_conv_k<S_, NS_, E_, WS_, OST_, RR_>(net, L, G, B, st, nullptr, nullptr, nullptr, nullptr,     \
                                               nullptr, edge);                                          \
    return 0;                                                                                           \
  }
#define CONV_S1(NS_, RR_) CONV_K(1, NS_, 0, 0, 0, RR_) CONV_K(1, NS_, 0, 0, 1, RR_) CONV_K(1, NS_, 1, 0, 0, RR_)
  CONV_S1(16, 1) CONV_S1(16, 2) CONV_S1(16, 4) CONV_S1(32, 1) CONV_S1(32, 2) CONV_S1(32, 4)
  CONV_S1(64, 1) CONV_S1(64, 2) CONV_S1(64, 4) CONV_S1(128, 1) CONV_S1(128, 2) CONV_S1(256, 1)
  CONV_K(1, 64, 0, 1, 0, 1) CONV_K(1, 64, 0, 1, 0, 2) CONV_K(1, 64, 0, 1, 0, 4)
  CONV_K(1, 128, 0, 1, 0, 1) CONV_K(1, 128, 0, 1, 0, 2) CONV_K(1, 256, 0, 1, 0, 1)
  CONV_K(2, 16, 0, 0, 0, 1) CONV_K(2, 32, 0, 0, 0, 1) CONV_K(2, 64, 0, 0, 0, 1) CONV_K(2, 128, 0, 0, 0, 1)
  CONV_K(2, 256, 0, 0, 0, 1) CONV_K(2, 16, 0, 0, 1, 1) CONV_K(2, 32, 0, 0, 1, 1) CONV_K(2, 64, 0, 0, 1, 1)
  CONV_K(2, 128, 0, 0, 1, 1) CONV_K(2, 64, 0, 1, 0, 1) CONV_K(2, 128, 0, 1, 0, 1) CONV_K(2, 256, 0, 1, 0, 1)
#undef CONV_S1
#undef CONV_K
  return gn_fail(GLASSNET_ERR_UNSUPPORTED, "conv variant S=%d NS=%d epi=%d ws=%d ost=%d rr=%d", L.S, L.NS, L.epi, L.ws,
                 L.ost, L.rr);
}

inline int tc_supersample(glassnet* net, const float* img, const void* gbuf_hi, float* out_hi, int B, cudaStream_t st) {
  TcState* s = reinterpret_cast<TcState*>(net->tc_state);
  int rc = launch_conv(net, s->ssconv[0], s->ssg[0], B, st, gbuf_hi, nullptr, img);
  net->prof.mark("ss_S1", st);
  if (rc) return rc;
  ConvGeom g = s->ssg[1];
  g.zout = out_hi;
  rc = launch_conv(net, s->ssconv[1], g, B, st, nullptr, nullptr, img, net->ss_b3);
  net->prof.mark("ss_S2", st);
  return rc;
}

// N4 object-major h on the tensor cores: T1 = k_conv_tc over the 16-channel object input (x built
// by k_obj_prep), T2 = k_conv_tc EPI = 3 whose epilogue adds ReLU(acc + b2) into the exact
// fixed-point latent tau_q where the object covers (a2 never reaches HBM).
inline int tc_setup_objects(glassnet* net, const float* T1W, const float* T2W) {
  TcState* s = reinterpret_cast<TcState*>(net->tc_state);
  const glassnet_dims& d = net->d;
  const int h = d.t_hidden;
  int rc = setup_conv(net, s->objconv[0], 1, T1W, net->objB[0], 11, 16, h, 0);
  if (!rc) rc = setup_conv(net, s->objconv[1], 1, T2W, net->objB[1], h, h, h, 3);
  for (int i = 0; i < 2 && !rc; ++i) {
    ConvGeom& g = s->objg[i];
    g.Hi_buf = d.height; g.Wi = d.width; g.Ho = d.height; g.Wo = d.width;
    g.in_row_off = 0; g.out_row_off = 0; g.out_rows_buf = d.height;
    g.out = i == 0 ? reinterpret_cast<uint16_t*>(net->obj_h1) : nullptr;
    g.zout = nullptr;
    rc = make_halo_maps(1, g, i == 0 ? net->obj_x : net->obj_h1, d.max_batch, i == 0 ? 16 : h, s->objconv[i].rr);
  }
  return rc;
}

inline int tc_objects_convs(glassnet* net, const uint8_t* cover, int B, cudaStream_t st) {
  TcState* s = reinterpret_cast<TcState*>(net->tc_state);
  int rc = launch_conv(net, s->objconv[0], s->objg[0], B, st);
  net->prof.mark("obj_h1", st);
  if (rc) return rc;
  rc = launch_conv(net, s->objconv[1], s->objg[1], B, st, nullptr, nullptr, nullptr, nullptr, cover);
  net->prof.mark("obj_h2_accum", st);
  return rc;
}

inline bool tc_supported(const glassnet_dims& d) {
  for (int l = 0; l < d.levels; ++l)   // the elementwise kernels index channel vectors with shifts
    if (d.widths[l] & (d.widths[l] - 1)) return false;
  return (d.t_hidden == 32 || d.t_hidden == 64) && (d.widths[0] == 16 || d.widths[0] == 32);
}

inline void tc_release(glassnet* net) {
  TcState* s = reinterpret_cast<TcState*>(net->tc_state);
  if (!s) return;
  if (s->tb_wimg) cudaFree(s->tb_wimg);
  for (auto& c : s->conv) if (c.wimg) cudaFree(c.wimg);
  if (s->tile) { for (void* q : s->tile->owned) cudaFree(q); delete s->tile; }
  if (s->sched) cudaFree(s->sched);
  if (s->perm) cudaFree(s->perm);
  if (s->sort_st) cudaStreamDestroy(s->sort_st);
  if (s->tb_st) cudaStreamDestroy(s->tb_st);
  if (s->ev_e0) cudaEventDestroy(s->ev_e0);
  if (s->ev_tb) cudaEventDestroy(s->ev_tb);
  if (s->ev_fwd) cudaEventDestroy(s->ev_fwd);
  if (s->ev_sorted) cudaEventDestroy(s->ev_sorted);
  delete s;
  net->tc_state = nullptr;
}

template <int K, int H, int C0, int POOL>
static int launch_tb_tc_kp(glassnet* net, const __nv_bfloat16* tbuf, const uint8_t* tcount, const __nv_bfloat16* e0,
                           const __nv_bfloat16* direct, float* psi, long P, cudaStream_t st) {
  using S = TbLayout<K, H, C0>;
  TcState* s = reinterpret_cast<TcState*>(net->tc_state);
  const long nsb = (P + TB_SBP - 1) / TB_SBP;
  if (nsb * TB_SBP > s->perm_cap) return gn_fail(GLASSNET_ERR_INVALID_ARGUMENT, "T kernel: %ld pixels exceed the workspace", P);
  (void)tcount;
  cudaStreamWaitEvent(st, s->ev_sorted, 0);   // k_tb_sort (tc_launch_sort) ran beside the encoder
  auto kfn = k_tb_tc<K, H, C0, POOL>;
  static bool attr = false;   // once per instantiation (not per launch)
  if (!attr) {
    if (cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, S::SMEM) != cudaSuccess)
      return gn_fail(GLASSNET_ERR_CUDA, "T kernel: shared memory attribute");
    attr = true;
  }
  const long ntiles = nsb * TB_SBT;
  long grid = net->num_sms;   // persistent: one CTA (the whole TMEM) per SM
  if (grid > ntiles) grid = ntiles;
  cudaMemsetAsync(s->sched, 0, sizeof(int), st);
  kfn<<<(unsigned)grid, S::THREADS, S::SMEM, st>>>(
      reinterpret_cast<const uint16_t*>(tbuf), reinterpret_cast<const uint16_t*>(e0),
      reinterpret_cast<const uint16_t*>(direct), s->tb_wimg, s->tb_prm, s->perm, psi, P, s->sched);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return gn_fail(GLASSNET_ERR_CUDA, "T kernel launch: %s", cudaGetErrorString(e));
  return 0;
}

template <int K, int H, int C0>
static int launch_tb_tc_k(glassnet* net, const __nv_bfloat16* tbuf, const uint8_t* tcount, const __nv_bfloat16* e0,
                          const __nv_bfloat16* direct, float* psi, long P, cudaStream_t st) {
  if (net->d.pool == GLASSNET_POOL_MEAN) return launch_tb_tc_kp<K, H, C0, 1>(net, tbuf, tcount, e0, direct, psi, P, st);
  return launch_tb_tc_kp<K, H, C0, 0>(net, tbuf, tcount, e0, direct, psi, P, st);
}

template <int H, int C0>
static int launch_tb_tc_h(glassnet* net, const __nv_bfloat16* tbuf, const uint8_t* tcount, const __nv_bfloat16* e0,
                          const __nv_bfloat16* direct, float* psi, long P, cudaStream_t st) {
  switch (net->d.k_slots) {
#define KCASE(k) case k: return launch_tb_tc_k<k, H, C0>(net, tbuf, tcount, e0, direct, psi, P, st);
#ifdef GN_DIAG_K8_ONLY   // diagnostic builds: the bench configuration only (fast to compile)
    KCASE(8)
#else
    KCASE(1) KCASE(2) KCASE(3) KCASE(4) KCASE(5) KCASE(6) KCASE(7) KCASE(8)
    KCASE(9) KCASE(10) KCASE(11) KCASE(12) KCASE(13) KCASE(14) KCASE(15) KCASE(16)
#endif
#undef KCASE
  }
  return gn_fail(GLASSNET_ERR_UNSUPPORTED, "k_slots");
}

// The T kernel's count-sort pre-pass reads only the input counts, so it runs on its own stream
// at the start of the forward, overlapping the F encoder; the T launch waits for it.
inline int tc_launch_sort(glassnet* net, const uint8_t* tcount, long P, cudaStream_t st) {
  TcState* s = reinterpret_cast<TcState*>(net->tc_state);
  if (!s->sort_st) {
    if (cudaStreamCreateWithFlags(&s->sort_st, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&s->ev_fwd, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&s->ev_sorted, cudaEventDisableTiming) != cudaSuccess)
      return gn_fail(GLASSNET_ERR_CUDA, "sort stream / events");
  }
  const long nsb = (P + TB_SBP - 1) / TB_SBP;
  if (nsb * TB_SBP > s->perm_cap) return gn_fail(GLASSNET_ERR_INVALID_ARGUMENT, "T kernel: %ld pixels exceed the workspace", P);
  cudaEventRecord(s->ev_fwd, st);               // after the previous forward's T kernel read perm
  cudaStreamWaitEvent(s->sort_st, s->ev_fwd, 0);
  switch (net->d.k_slots) {
#define KCASE(k) case k: k_tb_sort<k><<<(unsigned)nsb, TB_SBP / 8, 0, s->sort_st>>>(tcount, s->perm, P); break;
#ifdef GN_DIAG_K8_ONLY
    KCASE(8)
#else
    KCASE(1) KCASE(2) KCASE(3) KCASE(4) KCASE(5) KCASE(6) KCASE(7) KCASE(8)
    KCASE(9) KCASE(10) KCASE(11) KCASE(12) KCASE(13) KCASE(14) KCASE(15) KCASE(16)
#endif
#undef KCASE
    default: return gn_fail(GLASSNET_ERR_UNSUPPORTED, "k_slots");
  }
  cudaEventRecord(s->ev_sorted, s->sort_st);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return gn_fail(GLASSNET_ERR_CUDA, "count sort launch: %s", cudaGetErrorString(e));
  return 0;
}

inline int tc_launch_tb(glassnet* net, const __nv_bfloat16* tbuf, const uint8_t* tcount, const __nv_bfloat16* e0,
                        const __nv_bfloat16* direct, float* psi, long P, cudaStream_t st) {
  const int H = net->d.t_hidden, C0 = net->d.widths[0];
  if (H == 64 && C0 == 32) return launch_tb_tc_h<64, 32>(net, tbuf, tcount, e0, direct, psi, P, st);
  if (H == 32 && C0 == 16) return launch_tb_tc_h<32, 16>(net, tbuf, tcount, e0, direct, psi, P, st);
  if (H == 32 && C0 == 32) return launch_tb_tc_h<32, 32>(net, tbuf, tcount, e0, direct, psi, P, st);
  if (H == 64 && C0 == 16) return launch_tb_tc_h<64, 16>(net, tbuf, tcount, e0, direct, psi, P, st);
  return gn_fail(GLASSNET_ERR_UNSUPPORTED, "tensor-core T kernel: (t_hidden, widths[0]) = (%d, %d)", H, C0);
}

}  // namespace gn
