// glassnet.cu -- the C ABI (include/glassnet.h): validation, weight repack, workspace,
// and the per-batch kernel chain.  PAPER.md §3.4 defines the network; the
// layer-by-layer graph and every reading are in DESIGN.md.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/glassnet.h"
#include "kernels_simt.cuh"
#include "kernels_tc.cuh"
#include "net.h"

namespace {
thread_local std::string g_err;
}

int gn_fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CUDA_TRY(x)                                                                        \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess)                                                                 \
      return gn_fail(GLASSNET_ERR_CUDA, "%s failed: %s", #x, cudaGetErrorString(e_));      \
  } while (0)

extern "C" const char* glassnet_last_error(void) { return g_err.c_str(); }

// ------------------------------------------------------------------------ validation
static int validate_dims(const glassnet_dims* d) {
  if (!d) return gn_fail(GLASSNET_ERR_INVALID_ARGUMENT, "dims is NULL");
  if (d->abi_version != GLASSNET_ABI_VERSION)
    return gn_fail(GLASSNET_ERR_INVALID_ARGUMENT, "abi_version %d != %d", d->abi_version,
                   GLASSNET_ABI_VERSION);
  if (d->levels < 2 || d->levels > 4)
    return gn_fail(GLASSNET_ERR_INVALID_ARGUMENT, "levels must be 2..4 (got %d)", d->levels);
  if (d->height < 1 || d->width < 1 || d->max_batch < 1)
    return gn_fail(GLASSNET_ERR_INVALID_ARGUMENT, "height/width/max_batch must be >= 1");
  if (d->k_slots < 1) return gn_fail(GLASSNET_ERR_INVALID_ARGUMENT, "k_slots must be >= 1");
  if (d->k_slots > 16) return gn_fail(GLASSNET_ERR_UNSUPPORTED, "k_slots > 16 is not implemented");
  if (d->precision != GLASSNET_BF16 && d->precision != GLASSNET_FP32)
    return gn_fail(GLASSNET_ERR_INVALID_ARGUMENT, "precision must be GLASSNET_BF16 or GLASSNET_FP32");
  if (d->pool != GLASSNET_POOL_SUM && d->pool != GLASSNET_POOL_MEAN)
    return gn_fail(GLASSNET_ERR_INVALID_ARGUMENT, "pool must be GLASSNET_POOL_SUM or _MEAN");
  const int u = 1 << (d->levels - 1);
  if (d->height % u || d->width % u)
    return gn_fail(GLASSNET_ERR_UNSUPPORTED, "height and width must be multiples of 2^(levels-1)=%d", u);
  for (int l = 0; l < d->levels; ++l)
    if (d->widths[l] < 16 || d->widths[l] > 256 || d->widths[l] % 16)
      return gn_fail(GLASSNET_ERR_UNSUPPORTED, "widths[%d]=%d must be a multiple of 16 in [16,256]", l,
                     d->widths[l]);
  if (d->widths[0] > 32)
    return gn_fail(GLASSNET_ERR_UNSUPPORTED, "widths[0] > 32 is not implemented");
  if (d->t_hidden != 16 && d->t_hidden != 32 && d->t_hidden != 64)
    return gn_fail(GLASSNET_ERR_UNSUPPORTED, "t_hidden must be 16, 32 or 64");
  if (gn_pe_L(*d) > 10) return gn_fail(GLASSNET_ERR_INVALID_ARGUMENT, "positional encoding L_pe must be <= 10");
  if (d->flags & ~(0x1Fu | (0xFu << 8)))
    return gn_fail(GLASSNET_ERR_INVALID_ARGUMENT, "unknown flag bits 0x%x", d->flags & ~(0x1Fu | (0xFu << 8)));
  if ((d->flags & GLASSNET_FLAG_OBJECTS) && ((d->flags & GLASSNET_FLAG_SIGMA_COND) || gn_pe_L(*d)))
    return gn_fail(GLASSNET_ERR_UNSUPPORTED, "GLASSNET_FLAG_OBJECTS with SIGMA_COND or POSENC is not implemented");
  return GLASSNET_OK;
}

extern "C" size_t glassnet_weight_count(const glassnet_dims* d) {
  if (validate_dims(d) != GLASSNET_OK) return 0;
  const int h = d->t_hidden, L = d->levels;
  const int* c = d->widths;
  const int nin = gn_rec_in(*d) + ((d->flags & GLASSNET_FLAG_SIGMA_COND) ? d->widths[0] : 0);   // N1: [record ; e0]
  const int taps = (d->flags & GLASSNET_FLAG_OBJECTS) ? 9 : 1;   // N4: h's layers are 3x3 convs
  size_t n = (size_t)h * taps * nin + h + (size_t)h * taps * h + h;
  int cin = gn_x_in(*d);   // N2: 15 (2 L_pe + 1)
  for (int l = 0; l < L; ++l) { n += (size_t)c[l] * 9 * cin + c[l]; cin = c[l]; }
  n += (size_t)c[0] * (c[0] + h + 1) + c[0];
  for (int l = L - 1; l >= 1; --l) n += (size_t)c[l - 1] * 9 * c[l] + c[l - 1];
  const int nO = c[0] + ((d->flags & GLASSNET_FLAG_R_TAKES_LD) ? 3 : 0);
  n += (size_t)3 * nO + 3;
  if (d->flags & GLASSNET_FLAG_SUPERSAMPLE) {   // N3: S1, S2, S3 with s = c0
    const size_t sw = (size_t)c[0];
    n += sw * 9 * 15 + sw + sw * 9 * sw + sw + 3 * sw + 3;
  }
  return n;
}

// ------------------------------------------------------------------------ create
static float round_bf16(float v) { return __bfloat162float(__float2bfloat16_rn(v)); }

template <typename X>
static int dev_upload(X** dst, const std::vector<X>& v, size_t* acc) {
  CUDA_TRY(cudaMalloc((void**)dst, v.size() * sizeof(X)));
  CUDA_TRY(cudaMemcpy(*dst, v.data(), v.size() * sizeof(X), cudaMemcpyHostToDevice));
  *acc += v.size() * sizeof(X);
  return GLASSNET_OK;
}

extern "C" int glassnet_create(const float* weights, size_t n_weights, const glassnet_dims* dims,
                               int device, glassnet_t* out) {
  if (!out) return gn_fail(GLASSNET_ERR_INVALID_ARGUMENT, "out is NULL");
  *out = nullptr;
  int rc = validate_dims(dims);
  if (rc) return rc;
  if (!weights) return gn_fail(GLASSNET_ERR_INVALID_ARGUMENT, "weights is NULL");
  const size_t need = glassnet_weight_count(dims);
  if (n_weights != need)
    return gn_fail(GLASSNET_ERR_INVALID_ARGUMENT, "n_weights=%zu but dims need %zu", n_weights, need);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return gn_fail(GLASSNET_ERR_CUDA, "no CUDA device (this library has no CPU path)");
  if (device < 0 || device >= ndev)
    return gn_fail(GLASSNET_ERR_INVALID_ARGUMENT, "device %d out of range [0,%d)", device, ndev);
  CUDA_TRY(cudaSetDevice(device));
  cudaDeviceProp prop;
  CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return gn_fail(GLASSNET_ERR_UNSUPPORTED, "device %d is sm_%d%d; this library is built for sm_100a",
                   device, prop.major, prop.minor);

  glassnet* net = new glassnet();
  net->d = *dims;
  net->dev = device;
  net->num_sms = prop.multiProcessorCount;
  net->tc = (dims->precision == GLASSNET_BF16);
  const glassnet_dims& d = *dims;
  const int L = d.levels, h = d.t_hidden;
  const int* c = d.widths;
  const bool bf = d.precision == GLASSNET_BF16;
  const bool ld = (d.flags & GLASSNET_FLAG_R_TAKES_LD) != 0;
  auto W = [&](float v) { return bf ? round_bf16(v) : v; };

  // ---- parse the blob (documented order) ----
  const float* p = weights;
  std::vector<const float*> FW(L), Fb(L), RW(L), Rb(L);
  const bool sig = (d.flags & GLASSNET_FLAG_SIGMA_COND) != 0;
  const int nin = gn_rec_in(d) + (sig ? c[0] : 0);
  const bool objm = (d.flags & GLASSNET_FLAG_OBJECTS) != 0;
  const int taps = objm ? 9 : 1;   // N4: T1.W [h][3][3][11], T2.W [h][3][3][h]
  const float *T1W = p; p += (size_t)h * taps * nin; const float* T1b = p; p += h;
  const float *T2W = p; p += (size_t)h * taps * h; const float* T2b = p; p += h;
  const int XIN = gn_x_in(d), XC = gn_x_ch(d);   // N2: F0's input channels (real, stored)
  int cin = XIN;
  for (int l = 0; l < L; ++l) { FW[l] = p; p += (size_t)c[l] * 9 * cin; Fb[l] = p; p += c[l]; cin = c[l]; }
  const int NB = c[0] + h + 1;
  const float* BW = p; p += (size_t)c[0] * NB; const float* Bb = p; p += c[0];
  for (int l = L - 1; l >= 1; --l) { RW[l] = p; p += (size_t)c[l - 1] * 9 * c[l]; Rb[l] = p; p += c[l - 1]; }
  const int NO = c[0] + (ld ? 3 : 0);
  const float* OW = p; p += (size_t)3 * NO; const float* Ob = p; p += 3;
  const bool ss = (d.flags & GLASSNET_FLAG_SUPERSAMPLE) != 0;
  const float *S1W = nullptr, *S1b = nullptr, *S2W = nullptr, *S2b = nullptr, *S3W = nullptr, *S3b = nullptr;
  if (ss) {   // N3 (blob tail): S1.W[s][3][3][15] S1.b S2.W[s][3][3][s] S2.b S3.W[3][s] S3.b, s = c0
    S1W = p; p += (size_t)c[0] * 9 * 15; S1b = p; p += c[0];
    S2W = p; p += (size_t)c[0] * 9 * c[0]; S2b = p; p += c[0];
    S3W = p; p += (size_t)3 * c[0]; S3b = p;
  }

  // ---- SIMT packs ----
  std::vector<float> tb;
  for (int i = 0; i < h * taps * nin; ++i) tb.push_back(W(T1W[i]));
  for (int i = 0; i < h; ++i) tb.push_back(T1b[i]);
  for (int i = 0; i < h * taps * h; ++i) tb.push_back(W(T2W[i]));
  for (int i = 0; i < h; ++i) tb.push_back(T2b[i]);
  net->wb_off = tb.size();
  for (int i = 0; i < c[0] * NB; ++i) tb.push_back(W(BW[i]));
  for (int i = 0; i < c[0]; ++i) tb.push_back(Bb[i]);
  for (int i = 0; i < 3 * NO; ++i) tb.push_back(W(OW[i]));
  for (int i = 0; i < 3; ++i) tb.push_back(Ob[i]);
  rc = dev_upload(&net->w_tb, tb, &net->w_bytes);
  if (rc) { glassnet_destroy(net); return rc; }
  // conv: OHWI [co][ky][kx][ci] -> [tap][ci_pad][co]
  auto pack_conv = [&](const float* src, int co_n, int ci_n, int ci_pad, std::vector<float>& dst) {
    dst.assign((size_t)9 * ci_pad * co_n, 0.f);
    for (int co = 0; co < co_n; ++co)
      for (int t = 0; t < 9; ++t)
        for (int ci = 0; ci < ci_n; ++ci)
          dst[((size_t)t * ci_pad + ci) * co_n + co] = W(src[((size_t)co * 9 + t) * ci_n + ci]);
  };
  std::vector<float> tmp;
  for (int l = 0; l < L; ++l) {
    const int ci = l == 0 ? XIN : c[l - 1], cip = l == 0 ? XC : c[l - 1];
    pack_conv(FW[l], c[l], ci, cip, tmp);
    if ((rc = dev_upload(&net->convW[l], tmp, &net->w_bytes))) { glassnet_destroy(net); return rc; }
    std::vector<float> bb(Fb[l], Fb[l] + c[l]);
    if ((rc = dev_upload(&net->convB[l], bb, &net->w_bytes))) { glassnet_destroy(net); return rc; }
  }
  for (int l = L - 1; l >= 1; --l) {
    pack_conv(RW[l], c[l - 1], c[l], c[l], tmp);
    if ((rc = dev_upload(&net->convW[4 + l], tmp, &net->w_bytes))) { glassnet_destroy(net); return rc; }
    std::vector<float> bb(Rb[l], Rb[l] + c[l - 1]);
    if ((rc = dev_upload(&net->convB[4 + l], bb, &net->w_bytes))) { glassnet_destroy(net); return rc; }
  }
  std::vector<float> wz((size_t)3 * c[0]);
  for (int o = 0; o < 3; ++o)
    for (int i = 0; i < c[0]; ++i) wz[(size_t)o * c[0] + i] = W(OW[(size_t)o * NO + i]);
  if ((rc = dev_upload(&net->wz, wz, &net->w_bytes))) { glassnet_destroy(net); return rc; }
  if (objm) {   // N4: h's convs for the SIMT family (T1 over the 16-channel object input)
    pack_conv(T1W, h, 11, 16, tmp);
    if ((rc = dev_upload(&net->objW[0], tmp, &net->w_bytes))) { glassnet_destroy(net); return rc; }
    pack_conv(T2W, h, h, h, tmp);
    if ((rc = dev_upload(&net->objW[1], tmp, &net->w_bytes))) { glassnet_destroy(net); return rc; }
    std::vector<float> b1(T1b, T1b + h), b2(T2b, T2b + h);
    if ((rc = dev_upload(&net->objB[0], b1, &net->w_bytes)) || (rc = dev_upload(&net->objB[1], b2, &net->w_bytes))) {
      glassnet_destroy(net);
      return rc;
    }
    net->qscale = bf ? 4096.f : 1048576.f;   // 2^12 (R5's format) / 2^20 (fp32 check mode)
    net->qsat = bf ? 2048.f : 256.f;
  }
  if (ss) {
    pack_conv(S1W, c[0], 15, 16, tmp);
    if ((rc = dev_upload(&net->ssW[0], tmp, &net->w_bytes))) { glassnet_destroy(net); return rc; }
    pack_conv(S2W, c[0], c[0], c[0], tmp);
    if ((rc = dev_upload(&net->ssW[1], tmp, &net->w_bytes))) { glassnet_destroy(net); return rc; }
    std::vector<float> b1(S1b, S1b + c[0]), b2(S2b, S2b + c[0]), w3((size_t)3 * c[0]);
    for (size_t i = 0; i < w3.size(); ++i) w3[i] = W(S3W[i]);
    if ((rc = dev_upload(&net->ssB[0], b1, &net->w_bytes)) || (rc = dev_upload(&net->ssB[1], b2, &net->w_bytes)) ||
        (rc = dev_upload(&net->ss_wz, w3, &net->w_bytes))) { glassnet_destroy(net); return rc; }
    for (int i = 0; i < 3; ++i) net->ss_b3[i] = S3b[i];
  }

  // ---- workspace (independent of K: the T stage streams fragments) ----
  const size_t es = bf ? 2 : 4;
  const size_t B = (size_t)d.max_batch;
  size_t ws = 0;
  auto alloc = [&](void** ptr, size_t bytes) -> int {
    if (cudaMalloc(ptr, bytes) != cudaSuccess)
      return gn_fail(GLASSNET_ERR_OUT_OF_MEMORY, "cudaMalloc(%zu) failed", bytes);
    ws += bytes;
    return GLASSNET_OK;
  };
  size_t Hl[4], Wl[4];
  for (int l = 0; l < L; ++l) { Hl[l] = (size_t)d.height >> l; Wl[l] = (size_t)d.width >> l; }
  const size_t P0 = Hl[0] * Wl[0];
  rc = alloc(&net->x16, B * P0 * XC * es);
  for (int l = 0; l < L && !rc; ++l) rc = alloc(&net->e[l], B * Hl[l] * Wl[l] * c[l] * es);
  if (!rc) rc = alloc((void**)&net->psi, B * P0 * 3 * sizeof(float));
  for (int l = 1; l < L && !rc; ++l) rc = alloc(&net->y[l], B * Hl[l] * Wl[l] * c[l - 1] * es);
  for (int l = 1; l < L - 1 && !rc; ++l) rc = alloc(&net->dd[l], B * Hl[l] * Wl[l] * c[l] * es);
  if (!rc) rc = alloc((void**)&net->z, B * Hl[1] * Wl[1] * 3 * sizeof(float));
  if (ss && !rc) rc = alloc(&net->ss_s1, B * 4 * P0 * c[0] * es);
  if (objm && !rc) rc = alloc(&net->obj_x, B * P0 * 16 * es);
  if (objm && !rc) rc = alloc(&net->obj_h1, B * P0 * h * es);
  if (objm && !rc) rc = alloc(&net->obj_a2, B * P0 * h * es);
  if (objm && !rc) rc = alloc((void**)&net->tau_q, B * P0 * h * sizeof(uint32_t));
  if (objm && !rc) rc = alloc((void**)&net->tau_n, B * P0 * sizeof(uint32_t));
  if (ss && !rc) rc = alloc(&net->ss_x, B * 4 * P0 * 16 * es);      // SIMT family only: x and r stored
  if (ss && !rc) rc = alloc((void**)&net->ss_r, B * 4 * P0 * 3 * sizeof(float));
  if (rc) { glassnet_destroy(net); return rc; }
  net->ws_bytes = ws;
  // ---- tensor-core packs (bf16 mode) ----
  if (bf && gn::tc_supported(d)) {
    rc = gn::tc_pack_weights(net, T1W, T1b, T2W, T2b, FW, Fb, BW, Bb, RW, Rb, OW, Ob);
    if (!rc) rc = gn::tc_setup_convs(net, FW, RW);
    if (!rc) rc = gn::tc_setup_full_geom(net);
    if (!rc && ss) rc = gn::tc_setup_ss(net, S1W, S2W);
    if (!rc && objm) rc = gn::tc_setup_objects(net, T1W, T2W);
    if (rc) { glassnet_destroy(net); return rc; }
  }
  net->tc = bf && gn::tc_supported(d);
  *out = net;
  return GLASSNET_OK;
}

extern "C" void glassnet_destroy(glassnet_t net) {
  if (!net) return;
  cudaSetDevice(net->dev);
  void* ptrs[] = {net->w_tb, net->wz, net->x16, net->psi, net->z, net->st_g, net->st_d, net->st_t,
                  net->st_n, net->st_o, net->ssW[0], net->ssW[1], net->ssB[0], net->ssB[1], net->ss_wz,
                  net->ss_s1, net->ss_x, net->ss_r, net->objW[0], net->objW[1], net->objB[0], net->objB[1],
                  net->obj_x, net->obj_h1, net->obj_a2, net->tau_q, net->tau_n};
  for (void* q : ptrs) if (q) cudaFree(q);
  if (net->st_in) cudaStreamDestroy(net->st_in);
  if (net->st_out) cudaStreamDestroy(net->st_out);
  for (int i = 0; i < 8; ++i) { if (net->convW[i]) cudaFree(net->convW[i]); if (net->convB[i]) cudaFree(net->convB[i]); }
  for (int i = 0; i < 4; ++i) { if (net->e[i]) cudaFree(net->e[i]); if (net->y[i]) cudaFree(net->y[i]); if (net->dd[i]) cudaFree(net->dd[i]); }
  gn::tc_release(net);
  for (auto e : net->prof.ev) cudaEventDestroy(e);
  delete net;
}

extern "C" size_t glassnet_workspace_bytes(glassnet_t net) { return net ? net->ws_bytes : 0; }
extern "C" size_t glassnet_weight_bytes(glassnet_t net) { return net ? net->w_bytes : 0; }

extern "C" int glassnet_set_kernel_family(glassnet_t net, int tensor_cores) {
  if (!net) return gn_fail(GLASSNET_ERR_INVALID_ARGUMENT, "net is NULL");
  if (tensor_cores && net->d.precision != GLASSNET_BF16)
    return gn_fail(GLASSNET_ERR_UNSUPPORTED, "tensor-core kernels need GLASSNET_BF16 (fp32 check mode is FFMA)");
  if (tensor_cores && !gn::tc_supported(net->d))
    return gn_fail(GLASSNET_ERR_UNSUPPORTED, "no tensor-core kernels for t_hidden=%d widths[0]=%d", net->d.t_hidden,
                   net->d.widths[0]);
  net->tc = tensor_cores != 0;
  return GLASSNET_OK;
}

extern "C" int glassnet_launches_per_forward(glassnet_t net, int32_t batch) {
  if (!net) return 0;
  const int L = net->d.levels;
  (void)batch;
  // prep (SIMT family only), F_0..F_{L-1}, T (+ its count-sort pre-pass on the tensor-core
  // family), R_{L-1}..R_1, up2add at levels L-2..1, output
  return (net->tc ? 0 : 1) + L + (net->tc ? 2 : 1) + (L - 1) + (L - 2) + 1;   // (tc: F0 reads the G-buffer)
}

// ------------------------------------------------------------------------ forward (SIMT family)
static inline unsigned nblk(long n, int b) { return (unsigned)((n + b - 1) / b); }
static const char* kConvNames[8] = {"conv_F0", "conv_F1", "conv_F2", "conv_F3", "", "conv_R1", "conv_R2", "conv_R3"};

static gn::Up2Rows full_rows(int rows_f, int rows_c) {
  gn::Up2Rows g;
  g.rows_f = rows_f; g.rows_f_buf = rows_f; g.grow0_f = 0;
  g.rows_c_buf = rows_c; g.grow0_c = 0; g.Hc_full = rows_c; g.halo = 0;
  return g;
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per kernel and size, not per launch.
static void smem_attr_once(const void* kfn, int smem) {
  static std::mutex mu;
  static std::vector<std::pair<const void*, int>> done;
  std::lock_guard<std::mutex> g(mu);
  for (auto& e : done)
    if (e.first == kfn) {
      if (e.second >= smem) return;
      cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      e.second = smem;
      return;
    }
  cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  done.emplace_back(kfn, smem);
}

// T + B + psi on the SIMT kernel (FFMA): the fp32 check mode, the SIMT family, and -- with N2's
// positional encoding -- the tensor-core family's T stage (h's layer 1 over 11 (2L+1) encoded
// features per record has no tensor-core kernel here).
template <typename T>
static void launch_tb_simt(glassnet* net, const T* tbuf, const uint8_t* tcount, const T* e0, const T* direct, float* psi,
                           long P0, cudaStream_t st) {
  const glassnet_dims& d = net->d;
  const int K = d.k_slots, h = d.t_hidden;
  const int* c = d.widths;
  const bool norm = (d.flags & GLASSNET_FLAG_INPUT_NORM) != 0;
  const bool ld = (d.flags & GLASSNET_FLAG_R_TAKES_LD) != 0;
  const int NB = c[0] + h + 1, NO = c[0] + (ld ? 3 : 0);
  const bool sig = (d.flags & GLASSNET_FLAG_SIGMA_COND) != 0;
  const size_t nw = h * (gn_rec_in(d) + (sig ? c[0] : 0)) + h + h * h + h + c[0] * NB + c[0] + 3 * NO + 3;
  // (+ N2: a transposed copy of W1, 16-byte aligned)
  const size_t smem = sizeof(float) * (gn_pe_L(d) ? (nw + 3) / 4 * 4 + h * (gn_rec_in(d) + (sig ? c[0] : 0)) : nw);
  const unsigned g = nblk(P0, 128);
#define TB_LAUNCH(HH, CC)                                                                                      \
  {                                                                                                            \
    auto kfn = sig ? gn::k_tb_simt<T, HH, CC, true> : gn::k_tb_simt<T, HH, CC, false>;                        \
    smem_attr_once((const void*)kfn, (int)smem);                                                              \
    kfn<<<g, 128, smem, st>>>(tbuf, tcount, e0, direct, net->w_tb, psi, P0, K, d.pool, ld, norm, gn_pe_L(d)); \
  }
  if (h == 64 && c[0] == 32) TB_LAUNCH(64, 32)
  else if (h == 64 && c[0] == 16) TB_LAUNCH(64, 16)
  else if (h == 32 && c[0] == 32) TB_LAUNCH(32, 32)
  else if (h == 32 && c[0] == 16) TB_LAUNCH(32, 16)
  else if (h == 16 && c[0] == 32) TB_LAUNCH(16, 32)
  else TB_LAUNCH(16, 16)
#undef TB_LAUNCH
}

// N4: B + psi from tau_q / tau_n (kernels_simt.cuh k_b_psi), both families.
template <typename T>
static void launch_b_psi(glassnet* net, const T* e0, const T* direct, float* psi, long P0, cudaStream_t st) {
  const glassnet_dims& d = net->d;
  const int h = d.t_hidden, c0 = d.widths[0];
  const int ld = (d.flags & GLASSNET_FLAG_R_TAKES_LD) ? 1 : 0;
  const float* wb = net->w_tb + net->wb_off;
  const unsigned g = nblk(P0, 128);
  const float iq = 1.f / net->qscale;
#define BP_LAUNCH(HH, CC) \
  gn::k_b_psi<T, HH, CC><<<g, 128, 0, st>>>(e0, net->tau_q, net->tau_n, direct, wb, psi, P0, d.pool, ld, iq);
  if (h == 64 && c0 == 32) BP_LAUNCH(64, 32)
  else if (h == 64 && c0 == 16) BP_LAUNCH(64, 16)
  else if (h == 32 && c0 == 32) BP_LAUNCH(32, 32)
  else if (h == 32 && c0 == 16) BP_LAUNCH(32, 16)
  else if (h == 16 && c0 == 32) BP_LAUNCH(16, 32)
  else BP_LAUNCH(16, 16)
#undef BP_LAUNCH
}

template <typename T>
static int forward_simt(glassnet* net, const T* gbuf, const T* direct, const T* tbuf, const uint8_t* tcount,
                        float* out, int B, cudaStream_t st) {
  const glassnet_dims& d = net->d;
  const int L = d.levels;
  const int* c = d.widths;
  const bool norm = (d.flags & GLASSNET_FLAG_INPUT_NORM) != 0;
  int Hl[4], Wl[4];
  for (int l = 0; l < L; ++l) { Hl[l] = d.height >> l; Wl[l] = d.width >> l; }
  const long P0 = (long)B * Hl[0] * Wl[0];
  T* x16 = (T*)net->x16;
  const int XC = gn_x_ch(d);
  net->prof.mark(nullptr, st);
  if (gn_pe_L(d))   // N2: x = gamma([G', L_d])
    gn::k_prep_pe<T><<<nblk(P0, 32), 32, 32 * XC * sizeof(T), st>>>(gbuf, direct, x16, P0, norm, gn_pe_L(d), XC);
  else
    gn::k_prep_x<T><<<nblk(P0, 256), 256, 0, st>>>(gbuf, direct, x16, P0, norm);
  net->prof.mark("prep_x", st);
  auto conv = [&](const T* in, int l_in, int cin, int wi, int cout, int stride, T* o, int epi) {
    const int Ho = Hl[l_in] / stride, Wo = Wl[l_in] / stride;
    const long npix = (long)B * Ho * Wo;
    const int nj = cout >= 32 ? 32 : 16;
    dim3 grid(nblk(npix, 128), cout / nj);
    const float* w = net->convW[wi];
    const float* bb = net->convB[wi];
    if (epi == 0) {
      if (nj == 32)
        gn::k_conv3x3_simt<T, 32, 0><<<grid, 128, 0, st>>>(in, Hl[l_in], Wl[l_in], cin, w, bb, cout, stride, o, Ho, Wo, npix, nullptr, nullptr);
      else
        gn::k_conv3x3_simt<T, 16, 0><<<grid, 128, 0, st>>>(in, Hl[l_in], Wl[l_in], cin, w, bb, cout, stride, o, Ho, Wo, npix, nullptr, nullptr);
    } else {
      if (nj == 32)
        gn::k_conv3x3_simt<T, 32, 1><<<grid, 128, 0, st>>>(in, Hl[l_in], Wl[l_in], cin, w, bb, cout, stride, nullptr, Ho, Wo, npix, net->wz, net->z);
      else
        gn::k_conv3x3_simt<T, 16, 1><<<grid, 128, 0, st>>>(in, Hl[l_in], Wl[l_in], cin, w, bb, cout, stride, nullptr, Ho, Wo, npix, net->wz, net->z);
    }
    net->prof.mark(kConvNames[wi], st);
  };
  T* e[4];
  for (int l = 0; l < L; ++l) e[l] = (T*)net->e[l];
  conv(x16, 0, XC, 0, c[0], 1, e[0], 0);
  for (int l = 1; l < L; ++l) conv(e[l - 1], l - 1, c[l - 1], l, c[l], 2, e[l], 0);
  if (d.flags & GLASSNET_FLAG_OBJECTS)   // N4: B + psi over the streamed latent
    launch_b_psi<T>(net, e[0], direct, net->psi, P0, st);
  else
    launch_tb_simt<T>(net, tbuf, tcount, e[0], direct, net->psi, P0, st);
  net->prof.mark("T_B_psi", st);
  // R: d_{L-1} = e_{L-1}
  const T* dcur = e[L - 1];
  for (int l = L - 1; l >= 2; --l) {
    T* yl = (T*)net->y[l];
    conv(dcur, l, c[l], 4 + l, c[l - 1], 1, yl, 0);
    T* dn = (T*)net->dd[l - 1];
    const long nvec = (long)B * Hl[l - 1] * Wl[l - 1] * (c[l - 1] / 8);
    gn::k_up2add<T><<<nblk(nvec, 256), 256, 0, st>>>(yl, Wl[l], e[l - 1], dn, Wl[l - 1], c[l - 1],
                                                    full_rows(Hl[l - 1], Hl[l]), nvec);
    net->prof.mark("up2add", st);
    dcur = dn;
  }
  conv(dcur, 1, c[1], 4 + 1, c[0], 1, nullptr, 1);  // R_1 -> z (3 fp32 at level 1)
  gn::k_output<<<nblk(P0, 256), 256, 0, st>>>(net->z, Wl[1], net->psi, out, Wl[0], full_rows(Hl[0], Hl[1]), P0);
  net->prof.mark("output", st);
  CUDA_TRY(cudaGetLastError());
  return GLASSNET_OK;
}

// ------------------------------------------------------------------------ forward (tensor-core family)
namespace gn {

int tc_steps(const glassnet* net, Step* out, int max, bool tile) {
  const int L = net->d.levels;
  int n = 0;
  auto push = [&](int kind, int idx, int edge = 0) { if (n < max) out[n] = Step{kind, idx, edge}; ++n; };
  if (tile) {
    // Row tile, boundary rows first: every CONV / UP whose output is exchanged runs as
    // [first/last rows; EXCH of its output (comm stream); the other rows], so the halo transfer
    // overlaps the interior; T (no halo) runs on its own stream once e0 is complete.
    // Only producers at the two finest levels are split: their interior runs long enough to cover
    // an exchange, while at the coarse levels the extra launch costs more than the latency it
    // hides (tools/tile_times.py: splitting all nine costs 0.65 -> 0.78 ms of rank compute at N = 8).
    // One rank alone has no neighbour to exchange with: no split.  GN_TILE_SPLIT=0 / 2 (env): none / all.
    const TcState* ts = reinterpret_cast<const TcState*>(net->tc_state);
    static const int pol = getenv("GN_TILE_SPLIT") ? atoi(getenv("GN_TILE_SPLIT")) : 1;
    const bool multi = ts && ts->tile_nranks > 1;
    auto split = [&](int kind, int idx, int tensor, int out_level) {
      if (!multi || pol == 0 || (pol == 1 && out_level > 1)) { push(kind, idx); push(ST_EXCH, tensor); return; }
      push(kind, idx, 1); push(ST_EXCH, tensor); push(kind, idx, 2);
    };
    push(ST_PREP, 0);
    push(ST_EXCH, TEN_X);
    split(ST_CONV, 0, TEN_E + 0, 0);
    push(ST_TB, 0);
    for (int l = 1; l < L; ++l) split(ST_CONV, l, TEN_E + l, l);
    split(ST_CONV, 4 + L - 1, L - 1 >= 2 ? TEN_Y + L - 1 : TEN_Z, L - 1);
    for (int l = L - 1; l >= 2; --l) {
      split(ST_UP, l, TEN_D + l - 1, l - 1);
      split(ST_CONV, 4 + l - 1, l - 1 >= 2 ? TEN_Y + l - 1 : TEN_Z, l - 1);
    }
    push(ST_OUT, 0);
    return n;
  }
  push(ST_PREP, 0);
  push(ST_EXCH, TEN_X);
  push(ST_CONV, 0);
  if (tile) push(ST_TB, 0);   // launched on its own stream: overlaps F1.. and the halo exchanges
  for (int l = 1; l < L; ++l) { push(ST_EXCH, TEN_E + l - 1); push(ST_CONV, l); }
  if (!tile) push(ST_TB, 0);
  push(ST_EXCH, TEN_E + L - 1);
  push(ST_CONV, 4 + L - 1);
  for (int l = L - 1; l >= 2; --l) {
    push(ST_EXCH, TEN_Y + l);
    push(ST_UP, l);
    push(ST_EXCH, TEN_D + l - 1);
    push(ST_CONV, 4 + l - 1);
  }
  push(ST_EXCH, TEN_Z);
  push(ST_OUT, 0);
  return n;
}

int tc_prepare_tile(glassnet* net, int nranks, int rank, int row0, int rows) {
  return tc_setup_tile_geom(net, nranks, rank, row0, rows);
}

static Geom& geom_of(glassnet* net, bool tile) {
  TcState* s = reinterpret_cast<TcState*>(net->tc_state);
  return tile ? *s->tile : s->full;
}

int tc_tensor_rows(glassnet* net, bool tile, int tensor, char** base, size_t* row_bytes, int* rows) {
  Geom& G = geom_of(net, tile);
  const int* c = net->d.widths;
  int l = 0;
  size_t ch = 0, es = 2;
  void* p = nullptr;
  if (tensor == TEN_X) { l = 0; ch = gn_x_ch(net->d); p = G.x16; }
  else if (tensor >= TEN_E && tensor < TEN_E + 4) { l = tensor - TEN_E; ch = c[l]; p = G.e[l]; }
  else if (tensor >= TEN_Y && tensor < TEN_Y + 4) { l = tensor - TEN_Y; ch = c[l - 1]; p = G.y[l]; }
  else if (tensor >= TEN_D && tensor < TEN_D + 4) { l = tensor - TEN_D; ch = c[l]; p = G.dd[l]; }
  else if (tensor == TEN_Z) { l = 1; ch = 3; es = 4; p = G.z; }
  if (!p) return gn_fail(GLASSNET_ERR_INVALID_ARGUMENT, "tensor %d has no buffer", tensor);
  *base = reinterpret_cast<char*>(p);
  *row_bytes = (size_t)G.W[l] * ch * es;
  *rows = G.rows[l];
  return 0;
}

int tc_run_step(glassnet* net, bool tile, const Step& sp, const void* gbuf, const void* direct, const void* tbuf,
                const uint8_t* tcount, float* out, int B, cudaStream_t st) {
  TcState* s = reinterpret_cast<TcState*>(net->tc_state);
  Geom& G = geom_of(net, tile);
  const glassnet_dims& d = net->d;
  const int* c = d.widths;
  const int h = G.halo;
  const long P0 = (long)B * G.rows[0] * G.W[0];
  typedef __nv_bfloat16 bf;
  switch (sp.kind) {
    case ST_PREP: {
      if (d.flags & GLASSNET_FLAG_OBJECTS) {   // N4: no records to sort; F0 reads the G-buffer
        if (!tile) return 0;
        bf* x = (bf*)G.x16 + (size_t)h * G.W[0] * 16;
        const dim3 grid((unsigned)((G.W[0] + 255) / 256), (unsigned)G.rows[0], (unsigned)B);
        ew::k_prep_x<<<grid, 256, 0, st>>>((const bf*)gbuf, (const bf*)direct, x, G.W[0], G.rows[0], 0);
        net->prof.mark("prep_x", st);
        return 0;
      }
      if (gn_pe_L(d)) {   // N2: x = gamma([G', L_d]) stored (XC channels) for F0's TMA halo; T runs SIMT
        const int XC = gn_x_ch(d);
        bf* x = (bf*)G.x16 + (size_t)h * G.W[0] * XC;
        k_prep_pe<bf><<<nblk(P0, 32), 32, 32 * XC * sizeof(bf), st>>>((const bf*)gbuf, (const bf*)direct, x, P0,
                                                           (d.flags & GLASSNET_FLAG_INPUT_NORM) ? 1 : 0, gn_pe_L(d), XC);
        net->prof.mark("prep_x", st);
        return 0;
      }
      {   // T's count sort, on its own stream beside the encoder (kernels_tc.cuh)
        const int rc = tc_launch_sort(net, tcount, P0, st);
        if (rc) return rc;
      }
      // the full frame's F0 reads the G-buffer itself (k_conv_tc<..., GB = 1>); a row tile
      // builds x16 (with its halo rows exchanged) -- unnormalised: F0's weights carry R9
      if (!tile) return 0;
      bf* x = (bf*)G.x16 + (size_t)h * G.W[0] * 16;
      const dim3 grid((unsigned)((G.W[0] + 255) / 256), (unsigned)G.rows[0], (unsigned)B);
      ew::k_prep_x<<<grid, 256, 0, st>>>((const bf*)gbuf, (const bf*)direct, x, G.W[0], G.rows[0], 0);
      net->prof.mark("prep_x", st);
      return 0;
    }
    case ST_CONV: {
      int rc = (!tile && sp.idx == 0 && !gn_pe_L(d))
                   ? launch_conv(net, s->conv[0], G.cg[0], B, st, gbuf, direct)
                   : launch_conv(net, s->conv[sp.idx], G.cg[sp.idx], B, st, nullptr, nullptr, nullptr, nullptr, nullptr,
                                 sp.edge);
      net->prof.mark(kConvNames[sp.idx], st);
      return rc;
    }
    case ST_TB: {
      const bf* e0 = (const bf*)G.e[0] + (size_t)h * G.W[0] * c[0];
      if (d.flags & GLASSNET_FLAG_OBJECTS) {   // N4: B + psi over the streamed latent
        if (tile) return gn_fail(GLASSNET_ERR_UNSUPPORTED, "row tiles with GLASSNET_FLAG_OBJECTS");
        launch_b_psi<bf>(net, e0, (const bf*)direct, G.psi, P0, st);
        net->prof.mark("T_B_psi", st);
        return 0;
      }
      if (gn_pe_L(d)) {   // N2: T over the encoded records on the SIMT kernel (same stream order)
        launch_tb_simt<bf>(net, (const bf*)tbuf, tcount, e0, (const bf*)direct, G.psi, P0, st);
        net->prof.mark("T_B_psi", st);
        return 0;
      }
      if (!tile) {
        int rc = tc_launch_tb(net, (const bf*)tbuf, tcount, e0, (const bf*)direct, G.psi, P0, st);
        net->prof.mark("T_B_psi", st);
        return rc;
      }
      // row tile: T needs e0's interior rows only (no halo) -> its own stream after F0
      if (!s->tb_st &&
          (cudaStreamCreateWithFlags(&s->tb_st, cudaStreamNonBlocking) != cudaSuccess ||
           cudaEventCreateWithFlags(&s->ev_e0, cudaEventDisableTiming) != cudaSuccess ||
           cudaEventCreateWithFlags(&s->ev_tb, cudaEventDisableTiming) != cudaSuccess))
        return gn_fail(GLASSNET_ERR_CUDA, "T stream / events");
      cudaEventRecord(s->ev_e0, st);
      cudaStreamWaitEvent(s->tb_st, s->ev_e0, 0);
      net->prof.mark(nullptr, s->tb_st);
      int rc = tc_launch_tb(net, (const bf*)tbuf, tcount, e0, (const bf*)direct, G.psi, P0, s->tb_st);
      net->prof.mark("T_B_psi", s->tb_st);
      cudaEventRecord(s->ev_tb, s->tb_st);
      net->prof.mark(nullptr, st);   // the main stream's stages time from here
      return rc;
    }
    case ST_UP: {
      const int l = sp.idx;
      Up2Rows g;
      g.rows_f = G.rows[l - 1]; g.rows_f_buf = G.rows[l - 1] + 2 * h; g.grow0_f = G.grow0[l - 1];
      g.rows_c_buf = G.rows[l] + 2 * h; g.grow0_c = G.grow0[l]; g.Hc_full = G.Hfull[l]; g.halo = h;
      const int cv = c[l - 1] / 8, lcv = __builtin_ctz((unsigned)cv);
      const int rf = G.rows[l - 1];
      int ny = rf;   // edge 1: rows 0 and rf-1; edge 2: rows 1..rf-2
      if (sp.edge == 1) { ny = rf < 2 ? rf : 2; g.yoff = 0; g.ystep = rf > 1 ? rf - 1 : 1; }
      if (sp.edge == 2) { ny = rf > 2 ? rf - 2 : 0; g.yoff = 1; g.ystep = 1; }
      if (ny == 0) return 0;
      const dim3 grid((unsigned)(((long)(G.W[l - 1] / 2) * cv + 255) / 256), (unsigned)ny, (unsigned)B);
      ew::k_up2add<<<grid, 256, 0, st>>>((const bf*)G.y[l], G.W[l], (const bf*)G.e[l - 1], (bf*)G.dd[l - 1],
                                         G.W[l - 1], c[l - 1], lcv, g);
      net->prof.mark("up2add", st);
      return 0;
    }
    case ST_OUT: {
      Up2Rows g;
      g.rows_f = G.rows[0]; g.rows_f_buf = G.rows[0] + 2 * h; g.grow0_f = G.grow0[0];
      g.rows_c_buf = G.rows[1] + 2 * h; g.grow0_c = G.grow0[1]; g.Hc_full = G.Hfull[1]; g.halo = h;
      const dim3 grid((unsigned)((G.W[0] / 2 + 255) / 256), (unsigned)G.rows[0], (unsigned)B);
      if (tile && !gn_pe_L(d) && !(d.flags & GLASSNET_FLAG_OBJECTS)) cudaStreamWaitEvent(st, s->ev_tb, 0);   // psi from T's stream
      ew::k_output<<<grid, 256, 0, st>>>(G.z, G.W[1], G.psi, out, G.W[0], g);
      net->prof.mark("output", st);
      return 0;
    }
    default:
      return 0;   // ST_EXCH: the caller's transport
  }
}

}  // namespace gn

static int forward_tc(glassnet* net, const void* gbuf, const void* direct, const void* tbuf, const uint8_t* tcount,
                      float* out, int B, cudaStream_t st) {
  gn::Step steps[64];
  const int n = gn::tc_steps(net, steps, 64);
  net->prof.mark(nullptr, st);
  for (int i = 0; i < n; ++i) {
    int rc = gn::tc_run_step(net, false, steps[i], gbuf, direct, tbuf, tcount, out, B, st);
    if (rc) return rc;
  }
  CUDA_TRY(cudaGetLastError());
  return GLASSNET_OK;
}

static int check_ptr(const void* p, const char* name) {
  if (!p) return gn_fail(GLASSNET_ERR_INVALID_ARGUMENT, "%s is NULL", name);
  if ((uintptr_t)p % 16) return gn_fail(GLASSNET_ERR_INVALID_ARGUMENT, "%s is not 16-byte aligned", name);
  return GLASSNET_OK;
}

extern "C" int glassnet_forward(glassnet_t net, const void* gbuf, const void* direct, const void* tbuf,
                                const uint8_t* tcount, float* out, int32_t batch, glassnet_stream_t stream) {
  if (!net) return gn_fail(GLASSNET_ERR_INVALID_ARGUMENT, "net is NULL");
  int rc;
  if ((rc = check_ptr(gbuf, "gbuf")) || (rc = check_ptr(direct, "direct")) || (rc = check_ptr(tbuf, "tbuf")) ||
      (rc = check_ptr(out, "out")))
    return rc;
  if (!tcount) return gn_fail(GLASSNET_ERR_INVALID_ARGUMENT, "tcount is NULL");
  if (batch < 1 || batch > net->d.max_batch)
    return gn_fail(GLASSNET_ERR_INVALID_ARGUMENT, "batch=%d outside [1, max_batch=%d]", batch, net->d.max_batch);
  if (net->d.flags & GLASSNET_FLAG_OBJECTS)
    return gn_fail(GLASSNET_ERR_UNSUPPORTED, "GLASSNET_FLAG_OBJECTS handle: use glassnet_objects_begin/add/finish");
  CUDA_TRY(cudaSetDevice(net->dev));
  cudaStream_t st = (cudaStream_t)stream;
  if (net->d.precision == GLASSNET_FP32)
    return forward_simt<float>(net, (const float*)gbuf, (const float*)direct, (const float*)tbuf, tcount, out, batch, st);
  if (net->tc) return forward_tc(net, gbuf, direct, tbuf, tcount, out, batch, st);
  return forward_simt<__nv_bfloat16>(net, (const __nv_bfloat16*)gbuf, (const __nv_bfloat16*)direct,
                                     (const __nv_bfloat16*)tbuf, tcount, out, batch, st);
}

extern "C" int glassnet_forward_host(glassnet_t net, const void* gbuf, const void* direct, const void* tbuf,
                                     const uint8_t* tcount, float* out, int32_t batch, glassnet_stream_t stream) {
  if (!net) return gn_fail(GLASSNET_ERR_INVALID_ARGUMENT, "net is NULL");
  if (!gbuf || !direct || !tbuf || !tcount || !out)
    return gn_fail(GLASSNET_ERR_INVALID_ARGUMENT, "a host buffer is NULL");
  if (batch < 1 || batch > net->d.max_batch)
    return gn_fail(GLASSNET_ERR_INVALID_ARGUMENT, "batch=%d outside [1, max_batch=%d]", batch, net->d.max_batch);
  CUDA_TRY(cudaSetDevice(net->dev));
  const glassnet_dims& d = net->d;
  const size_t es = d.precision == GLASSNET_BF16 ? 2 : 4;
  const size_t P = (size_t)d.height * d.width;
  const size_t MB = (size_t)d.max_batch;
  if (!net->st_g) {  // device staging, allocated once per handle on first use (all or nothing)
    void *g = nullptr, *dd = nullptr, *t = nullptr, *n = nullptr, *o = nullptr;
    const bool ok = cudaMalloc(&g, MB * P * 12 * es) == cudaSuccess && cudaMalloc(&dd, MB * P * 3 * es) == cudaSuccess &&
                    cudaMalloc(&t, MB * P * d.k_slots * 11 * es) == cudaSuccess && cudaMalloc(&n, MB * P) == cudaSuccess &&
                    cudaMalloc(&o, MB * P * 3 * sizeof(float)) == cudaSuccess;
    if (!ok) {
      for (void* q : {g, dd, t, n, o}) if (q) cudaFree(q);
      cudaGetLastError();
      return gn_fail(GLASSNET_ERR_OUT_OF_MEMORY, "forward_host staging buffers");
    }
    net->st_g = g; net->st_d = dd; net->st_t = t; net->st_n = n; net->st_o = (float*)o;
  }
  if (!net->st_in) {
    CUDA_TRY(cudaStreamCreateWithFlags(&net->st_in, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&net->st_out, cudaStreamNonBlocking));
  }
  // Pipelined in chunks of frames: the copy-in of chunk i+1 (stream st_in) and the copy-out of
  // chunk i-1 (st_out) overlap the forward of chunk i (the caller's stream); chunks use
  // disjoint frame ranges of the staging buffers, and frames are independent (R21), so the
  // result equals one whole-batch forward bit for bit.  On any error the function still
  // drains all three streams (no copy may touch the caller's buffers after it returns) and
  // destroys its events.
  cudaStream_t st = (cudaStream_t)stream;
  const int CF = batch < 4 ? batch : 4;
  const int nch = (batch + CF - 1) / CF;
  std::vector<cudaEvent_t> ev_in(nch, nullptr), ev_c(nch, nullptr);
  cudaEvent_t ev0 = nullptr;
  int rc = GLASSNET_OK;
  cudaError_t ce = cudaSuccess;
  auto ck = [&](cudaError_t e, const char* what) {
    if (e != cudaSuccess && ce == cudaSuccess) { ce = e; rc = gn_fail(GLASSNET_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e)); }
    return ce == cudaSuccess;
  };
  for (int i = 0; i < nch && ce == cudaSuccess; ++i) {
    ck(cudaEventCreateWithFlags(&ev_in[i], cudaEventDisableTiming), "event");
    ck(cudaEventCreateWithFlags(&ev_c[i], cudaEventDisableTiming), "event");
  }
  if (ck(cudaEventCreateWithFlags(&ev0, cudaEventDisableTiming), "event") &&
      ck(cudaEventRecord(ev0, st), "event record"))   // the copies follow earlier work on the caller's stream
    ck(cudaStreamWaitEvent(net->st_in, ev0, 0), "stream wait");
  for (int i = 0; i < nch && rc == GLASSNET_OK; ++i) {
    const size_t f0 = (size_t)i * CF, nf = (size_t)((i + 1) * CF <= batch ? CF : batch - i * CF);
    const char* hg = (const char*)gbuf + f0 * P * 12 * es;
    const char* hd = (const char*)direct + f0 * P * 3 * es;
    const char* ht = (const char*)tbuf + f0 * P * d.k_slots * 11 * es;
    char* dg = (char*)net->st_g + f0 * P * 12 * es;
    char* dd = (char*)net->st_d + f0 * P * 3 * es;
    char* dt = (char*)net->st_t + f0 * P * d.k_slots * 11 * es;
    uint8_t* dn = (uint8_t*)net->st_n + f0 * P;
    float* dout = net->st_o + f0 * P * 3;
    if (!(ck(cudaMemcpyAsync(dg, hg, nf * P * 12 * es, cudaMemcpyHostToDevice, net->st_in), "H2D") &&
          ck(cudaMemcpyAsync(dd, hd, nf * P * 3 * es, cudaMemcpyHostToDevice, net->st_in), "H2D") &&
          ck(cudaMemcpyAsync(dt, ht, nf * P * d.k_slots * 11 * es, cudaMemcpyHostToDevice, net->st_in), "H2D") &&
          ck(cudaMemcpyAsync(dn, tcount + f0 * P, nf * P, cudaMemcpyHostToDevice, net->st_in), "H2D") &&
          ck(cudaEventRecord(ev_in[i], net->st_in), "event record") && ck(cudaStreamWaitEvent(st, ev_in[i], 0), "wait")))
      break;
    rc = glassnet_forward(net, dg, dd, dt, dn, dout, (int32_t)nf, stream);
    if (rc) break;
    if (!(ck(cudaEventRecord(ev_c[i], st), "event record") && ck(cudaStreamWaitEvent(net->st_out, ev_c[i], 0), "wait") &&
          ck(cudaMemcpyAsync(out + f0 * P * 3, dout, nf * P * 3 * sizeof(float), cudaMemcpyDeviceToHost, net->st_out),
             "D2H")))
      break;
  }
  const cudaError_t e1 = cudaStreamSynchronize(net->st_in), e2 = cudaStreamSynchronize(net->st_out),
                    e3 = cudaStreamSynchronize(st);
  for (int i = 0; i < nch; ++i) {
    if (ev_in[i]) cudaEventDestroy(ev_in[i]);
    if (ev_c[i]) cudaEventDestroy(ev_c[i]);
  }
  if (ev0) cudaEventDestroy(ev0);
  if (rc) return rc;
  CUDA_TRY(e1 != cudaSuccess ? e1 : e2 != cudaSuccess ? e2 : e3);
  return GLASSNET_OK;
}

// ------------------------------------------------------------------------ N4 object-major T
static int objects_check(glassnet* net, int32_t batch) {
  if (!net) return gn_fail(GLASSNET_ERR_INVALID_ARGUMENT, "net is NULL");
  if (!(net->d.flags & GLASSNET_FLAG_OBJECTS))
    return gn_fail(GLASSNET_ERR_UNSUPPORTED, "the handle was created without GLASSNET_FLAG_OBJECTS");
  if (batch < 1 || batch > net->d.max_batch)
    return gn_fail(GLASSNET_ERR_INVALID_ARGUMENT, "batch=%d outside [1, max_batch=%d]", batch, net->d.max_batch);
  CUDA_TRY(cudaSetDevice(net->dev));
  return GLASSNET_OK;
}

extern "C" int glassnet_objects_begin(glassnet_t net, int32_t batch, glassnet_stream_t stream) {
  int rc = objects_check(net, batch);
  if (rc) return rc;
  const size_t P = (size_t)batch * net->d.height * net->d.width;
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(cudaMemsetAsync(net->tau_q, 0, P * net->d.t_hidden * sizeof(uint32_t), st));
  CUDA_TRY(cudaMemsetAsync(net->tau_n, 0, P * sizeof(uint32_t), st));
  return GLASSNET_OK;
}

template <typename T>
static int objects_add_simt(glassnet* net, const T* obj, const uint8_t* cover, int B, cudaStream_t st) {
  const glassnet_dims& d = net->d;
  const int H = d.height, W = d.width, h = d.t_hidden;
  const long P = (long)B * H * W;
  T* x = (T*)net->obj_x;
  T* h1 = (T*)net->obj_h1;
  T* a2 = (T*)net->obj_a2;
  net->prof.mark(nullptr, st);
  gn::k_obj_prep<T><<<nblk(P, 256), 256, 0, st>>>(obj, cover, x, P, (d.flags & GLASSNET_FLAG_INPUT_NORM) ? 1 : 0);
  net->prof.mark("obj_prep", st);
  const int nj = h >= 32 ? 32 : 16;
  const dim3 grid(nblk(P, 128), h / nj);
  if (nj == 32) {
    gn::k_conv3x3_simt<T, 32, 0><<<grid, 128, 0, st>>>(x, H, W, 16, net->objW[0], net->objB[0], h, 1, h1, H, W, P, nullptr, nullptr);
    gn::k_conv3x3_simt<T, 32, 0><<<grid, 128, 0, st>>>(h1, H, W, h, net->objW[1], net->objB[1], h, 1, a2, H, W, P, nullptr, nullptr);
  } else {
    gn::k_conv3x3_simt<T, 16, 0><<<grid, 128, 0, st>>>(x, H, W, 16, net->objW[0], net->objB[0], h, 1, h1, H, W, P, nullptr, nullptr);
    gn::k_conv3x3_simt<T, 16, 0><<<grid, 128, 0, st>>>(h1, H, W, h, net->objW[1], net->objB[1], h, 1, a2, H, W, P, nullptr, nullptr);
  }
  net->prof.mark("obj_h", st);
  gn::k_obj_accum<T><<<nblk(P, 256), 256, 0, st>>>(a2, cover, net->tau_q, net->tau_n, P, h, net->qscale, net->qsat);
  net->prof.mark("obj_accum", st);
  CUDA_TRY(cudaGetLastError());
  return GLASSNET_OK;
}

extern "C" int glassnet_objects_add(glassnet_t net, const void* obj, const uint8_t* cover, int32_t batch,
                                    glassnet_stream_t stream) {
  int rc = objects_check(net, batch);
  if (rc) return rc;
  if ((rc = check_ptr(obj, "obj"))) return rc;
  if (!cover) return gn_fail(GLASSNET_ERR_INVALID_ARGUMENT, "cover is NULL");
  cudaStream_t st = (cudaStream_t)stream;
  if (net->d.precision == GLASSNET_FP32) return objects_add_simt<float>(net, (const float*)obj, cover, batch, st);
  if (!net->tc) return objects_add_simt<__nv_bfloat16>(net, (const __nv_bfloat16*)obj, cover, batch, st);
  const long P = (long)batch * net->d.height * net->d.width;
  net->prof.mark(nullptr, st);
  gn::k_obj_prep<__nv_bfloat16><<<nblk(P, 256), 256, 0, st>>>((const __nv_bfloat16*)obj, cover,
                                                              (__nv_bfloat16*)net->obj_x, P,
                                                              (net->d.flags & GLASSNET_FLAG_INPUT_NORM) ? 1 : 0);
  net->prof.mark("obj_prep", st);
  rc = gn::tc_objects_convs(net, cover, batch, st);
  if (rc) return rc;
  CUDA_TRY(cudaGetLastError());
  return GLASSNET_OK;
}

extern "C" int glassnet_objects_finish(glassnet_t net, const void* gbuf, const void* direct, float* out, int32_t batch,
                                       glassnet_stream_t stream) {
  int rc = objects_check(net, batch);
  if (rc) return rc;
  if ((rc = check_ptr(gbuf, "gbuf")) || (rc = check_ptr(direct, "direct")) || (rc = check_ptr(out, "out"))) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  if (net->d.precision == GLASSNET_FP32)
    return forward_simt<float>(net, (const float*)gbuf, (const float*)direct, nullptr, nullptr, out, batch, st);
  if (net->tc) return forward_tc(net, gbuf, direct, nullptr, nullptr, out, batch, st);
  return forward_simt<__nv_bfloat16>(net, (const __nv_bfloat16*)gbuf, (const __nv_bfloat16*)direct, nullptr, nullptr,
                                     out, batch, st);
}

// ------------------------------------------------------------------------ N3 super-sampler
template <typename T>
static int supersample_simt(glassnet* net, const float* img, const T* gbuf_hi, float* out_hi, int B, cudaStream_t st) {
  const glassnet_dims& d = net->d;
  const int H2 = 2 * d.height, W2 = 2 * d.width, c0 = d.widths[0];
  const long P2 = (long)B * H2 * W2;
  T* x = (T*)net->ss_x;
  T* s1 = (T*)net->ss_s1;
  net->prof.mark(nullptr, st);
  gn::k_prep_ss<T><<<nblk(P2, 256), 256, 0, st>>>(gbuf_hi, img, x, W2, H2, P2, (d.flags & GLASSNET_FLAG_INPUT_NORM) ? 1 : 0);
  net->prof.mark("ss_prep", st);
  const dim3 g1(nblk(P2, 128), c0 / 16), g2(nblk(P2, 128), 1);
  gn::k_conv3x3_simt<T, 16, 0><<<g1, 128, 0, st>>>(x, H2, W2, 16, net->ssW[0], net->ssB[0], c0, 1, s1, H2, W2, P2,
                                                  nullptr, nullptr);
  net->prof.mark("ss_S1", st);
  if (c0 == 32)
    gn::k_conv3x3_simt<T, 32, 1><<<g2, 128, 0, st>>>(s1, H2, W2, c0, net->ssW[1], net->ssB[1], c0, 1, nullptr, H2, W2,
                                                    P2, net->ss_wz, net->ss_r);
  else
    gn::k_conv3x3_simt<T, 16, 1><<<g2, 128, 0, st>>>(s1, H2, W2, c0, net->ssW[1], net->ssB[1], c0, 1, nullptr, H2, W2,
                                                    P2, net->ss_wz, net->ss_r);
  net->prof.mark("ss_S2", st);
  gn::k_ss_out<<<nblk(P2, 256), 256, 0, st>>>(img, net->ss_r, net->ss_b3[0], net->ss_b3[1], net->ss_b3[2], out_hi, W2,
                                             H2, P2);
  net->prof.mark("ss_out", st);
  CUDA_TRY(cudaGetLastError());
  return GLASSNET_OK;
}

extern "C" int glassnet_supersample(glassnet_t net, const float* img, const void* gbuf_hi, float* out_hi, int32_t batch,
                                    glassnet_stream_t stream) {
  if (!net) return gn_fail(GLASSNET_ERR_INVALID_ARGUMENT, "net is NULL");
  if (!(net->d.flags & GLASSNET_FLAG_SUPERSAMPLE))
    return gn_fail(GLASSNET_ERR_UNSUPPORTED, "the handle was created without GLASSNET_FLAG_SUPERSAMPLE");
  int rc;
  if ((rc = check_ptr(img, "img")) || (rc = check_ptr(gbuf_hi, "gbuf_hi")) || (rc = check_ptr(out_hi, "out_hi")))
    return rc;
  if (batch < 1 || batch > net->d.max_batch)
    return gn_fail(GLASSNET_ERR_INVALID_ARGUMENT, "batch=%d outside [1, max_batch=%d]", batch, net->d.max_batch);
  const size_t P = (size_t)batch * net->d.height * net->d.width;
  if ((const char*)out_hi < (const char*)(img + 3 * P) && (const char*)img < (const char*)(out_hi + 12 * P))
    return gn_fail(GLASSNET_ERR_INVALID_ARGUMENT, "out_hi overlaps img");
  CUDA_TRY(cudaSetDevice(net->dev));
  cudaStream_t st = (cudaStream_t)stream;
  if (net->d.precision == GLASSNET_FP32)
    return supersample_simt<float>(net, img, (const float*)gbuf_hi, out_hi, batch, st);
  if (net->tc) {
    net->prof.mark(nullptr, st);
    rc = gn::tc_supersample(net, img, gbuf_hi, out_hi, batch, st);
    if (rc) return rc;
    CUDA_TRY(cudaGetLastError());
    return GLASSNET_OK;
  }
  return supersample_simt<__nv_bfloat16>(net, img, (const __nv_bfloat16*)gbuf_hi, out_hi, batch, st);
}

extern "C" int glassnet_debug_psi(glassnet_t net, float* dst, int32_t batch, glassnet_stream_t stream) {
  if (!net || !dst) return gn_fail(GLASSNET_ERR_INVALID_ARGUMENT, "net or dst is NULL");
  if (batch < 1 || batch > net->d.max_batch)
    return gn_fail(GLASSNET_ERR_INVALID_ARGUMENT, "batch=%d outside [1, max_batch=%d]", batch, net->d.max_batch);
  CUDA_TRY(cudaSetDevice(net->dev));
  CUDA_TRY(cudaMemcpyAsync(dst, net->psi, (size_t)batch * net->d.height * net->d.width * 3 * sizeof(float),
                           cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  return GLASSNET_OK;
}

// ------------------------------------------------------------------------ profiling
extern "C" int glassnet_profile_begin(glassnet_t net, int32_t max_launches) {
  if (!net || max_launches < 2) return gn_fail(GLASSNET_ERR_INVALID_ARGUMENT, "bad profile_begin args");
  CUDA_TRY(cudaSetDevice(net->dev));
  StageProfiler& p = net->prof;
  for (auto e : p.ev) cudaEventDestroy(e);
  p.ev.assign((size_t)max_launches, nullptr);
  p.stage.assign((size_t)max_launches, -1);
  for (auto& e : p.ev) CUDA_TRY(cudaEventCreate(&e));
  p.used = 0;
  p.dropped = 0;
  p.on = true;
  return GLASSNET_OK;
}

extern "C" int glassnet_profile_end(glassnet_t net, int32_t max_stages, char* names, double* total_ms,
                                    int32_t* launches, int32_t* n_stages) {
  if (!net) return gn_fail(GLASSNET_ERR_INVALID_ARGUMENT, "net is NULL");
  StageProfiler& p = net->prof;
  p.on = false;
  if (p.dropped)
    return gn_fail(GLASSNET_ERR_INVALID_ARGUMENT, "profile: %zu stage marks exceeded the %zu reserved by profile_begin",
                   p.dropped, p.ev.size());
  std::vector<double> tot(p.names.size(), 0.0);
  std::vector<int> cnt(p.names.size(), 0);
  if (p.used) CUDA_TRY(cudaEventSynchronize(p.ev[p.used - 1]));
  for (size_t i = 1; i < p.used; ++i) {
    if (p.stage[i] < 0) continue;
    float ms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&ms, p.ev[i - 1], p.ev[i]));
    tot[p.stage[i]] += ms;
    cnt[p.stage[i]] += 1;
  }
  const int n = (int)p.names.size();
  if (n_stages) *n_stages = n;
  for (int i = 0; i < n && i < max_stages; ++i) {
    if (names) { strncpy(names + 32 * i, p.names[i].c_str(), 31); names[32 * i + 31] = 0; }
    if (total_ms) total_ms[i] = tot[i];
    if (launches) launches[i] = cnt[i];
  }
  for (auto e : p.ev) cudaEventDestroy(e);
  p.ev.clear(); p.stage.clear(); p.names.clear(); p.used = 0;
  return GLASSNET_OK;
}

// ------------------------------------------------------------------------ tiles
extern "C" int glassnet_tile_rows(const glassnet_dims* dims, int32_t nranks, int32_t rank, int32_t* row0,
                                  int32_t* rows) {
  int rc = validate_dims(dims);
  if (rc) return rc;
  if (nranks < 1 || rank < 0 || rank >= nranks || !row0 || !rows)
    return gn_fail(GLASSNET_ERR_INVALID_ARGUMENT, "bad nranks/rank/out pointers");
  const int u = 1 << (dims->levels - 1);
  const long U = dims->height / u;
  const long a = U * rank / nranks, b = U * (rank + 1) / nranks;
  if (b <= a) return gn_fail(GLASSNET_ERR_INVALID_ARGUMENT, "too many ranks (%d) for %ld row units", nranks, U);
  *row0 = (int32_t)(a * u);
  *rows = (int32_t)((b - a) * u);
  return GLASSNET_OK;
}

#ifdef GN_TB_PROF
extern "C" int glassnet_debug_tb_prof(unsigned long long* out40, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out40, gn::gn_tb_prof, 40 * sizeof(unsigned long long));
  if (reset) {
    unsigned long long z[40] = {};
    cudaMemcpyToSymbol(gn::gn_tb_prof, z, sizeof z);
  }
  return 0;
}
#endif

#ifdef GN_MBAR_WATCHDOG
static unsigned int* gn_wd_host = nullptr;
// diagnostic: map a host log the mbarrier watchdog writes before it traps (read after a failure)
extern "C" int glassnet_debug_watchdog(unsigned int* out8, int init) {
  if (init) {
    if (!gn_wd_host) {
      if (cudaHostAlloc((void**)&gn_wd_host, 64, cudaHostAllocMapped) != cudaSuccess) return -1;
      unsigned int* dptr = nullptr;
      cudaHostGetDevicePointer((void**)&dptr, gn_wd_host, 0);
      cudaMemcpyToSymbol(gn::gn_wd_log, &dptr, sizeof dptr);
    }
    memset(gn_wd_host, 0, 64);
    return 0;
  }
  for (int i = 0; i < 8; ++i) out8[i] = gn_wd_host ? ((volatile unsigned int*)gn_wd_host)[i] : 0u;
  return 0;
}
#endif

