// net.h -- the handle behind glassnet_t (library-internal).
#pragma once
#include <cstddef>
#include <cstdint>
#include <vector>

#include "../../include/glassnet.h"

int gn_fail(int code, const char* fmt, ...);

// N2 positional encoding: L_pe, channels per encoded input channel, the encoded widths of a
// record (h's layer-1 input) and of x (F0's input), and x's stored width (padded to 16).
inline int gn_pe_L(const glassnet_dims& d) { return GLASSNET_POSENC_OF(d.flags); }
inline int gn_pe(const glassnet_dims& d) { return 2 * gn_pe_L(d) + 1; }
inline int gn_rec_in(const glassnet_dims& d) { return 11 * gn_pe(d); }
inline int gn_x_in(const glassnet_dims& d) { return 15 * gn_pe(d); }
inline int gn_x_ch(const glassnet_dims& d) { return (gn_x_in(d) + 15) / 16 * 16; }

#include <cuda_runtime.h>
#include <string>

// Optional per-stage timing with CUDA events on the launching stream (bench.py's
// roofline): when enabled, an event is recorded after every launch.
struct StageProfiler {
  bool on = false;
  std::vector<cudaEvent_t> ev;
  std::vector<int> stage;           // stage id of the interval ending at ev[i] (-1 = start)
  std::vector<std::string> names;
  size_t used = 0;
  int id(const char* n) {
    for (size_t i = 0; i < names.size(); ++i) if (names[i] == n) return (int)i;
    names.push_back(n);
    return (int)names.size() - 1;
  }
  size_t dropped = 0;         // marks beyond the capacity given to profile_begin
  void mark(const char* n, cudaStream_t st) {
    if (!on) return;
    if (used >= ev.size()) { ++dropped; return; }
    stage[used] = n ? id(n) : -1;
    cudaEventRecord(ev[used++], st);
  }
};

struct glassnet;
namespace gn {
// The tensor-core forward as a list of steps (glassnet.cu).  The full frame runs them
// back to back; a row tile (forward_sharded, comm.cu) exchanges halo rows at EXCH steps.
enum StepKind { ST_PREP = 0, ST_CONV = 1, ST_TB = 2, ST_UP = 3, ST_OUT = 4, ST_EXCH = 5 };
enum TensorId { TEN_X = 0, TEN_E = 1, TEN_Y = 5, TEN_D = 9, TEN_Z = 13 };   // TEN_E + l, ...
// CONV: conv slot (l = F_l, 4+l = R_l); UP: level; EXCH: tensor.  edge (row tiles, boundary rows
// first): 0 = every row, 1 = only the first / last rows (what the next EXCH sends), 2 = the rest
// (runs while that EXCH is in flight).
struct Step { int kind; int idx; int edge = 0; };
// tile = true: the row-tile order (T right after F0, on its own stream; see tc_run_step)
int tc_steps(const struct ::glassnet* net, Step* out, int max, bool tile = false);
int tc_prepare_tile(struct ::glassnet* net, int nranks, int rank, int row0, int rows);
int tc_run_step(struct ::glassnet* net, bool tile, const Step& s, const void* gbuf, const void* direct, const void* tbuf,
                const uint8_t* tcount, float* out, int B, cudaStream_t st);
// rows of a tensor in the geometry: buffer base, bytes per row, interior rows (halo rows
// are at buffer rows 0 and rows+1)
int tc_tensor_rows(struct ::glassnet* net, bool tile, int tensor, char** base, size_t* row_bytes, int* rows);
}  // namespace gn

struct glassnet {
  glassnet_dims d{};
  int dev = 0;
  int num_sms = 148;
  bool tc = false;          // bf16 mode: tensor-core kernel family
  // SIMT weight packs (fp32; W tensors pre-rounded to bf16 values in bf16 mode)
  float* w_tb = nullptr;    // W1 b1 W2 b2 WB bB WO bO
  float* convW[8] = {};     // [l] = F_l, [4+l] = R_l ; layout [tap][ci][co]
  float* convB[8] = {};
  float* wz = nullptr;      // [3][c0] = W_O[:, :c0]
  // workspace (per max_batch)
  void* x16 = nullptr;      // [B][H][W][16]
  void* e[4] = {};          // encoder features
  float* psi = nullptr;     // [B][H][W][3]   (reading R15)
  void* y[4] = {};          // y_l at level l
  void* dd[4] = {};         // d_l (1 <= l <= L-2)
  float* z = nullptr;       // [B][H/2][W/2][3]
  // N3 super-sampler S (GLASSNET_FLAG_SUPERSAMPLE): SIMT packs [tap][ci][co], biases, S3.W, S3.b
  float* ssW[2] = {};
  float* ssB[2] = {};
  float* ss_wz = nullptr;   // [3][c0]
  float ss_b3[3] = {};
  void* ss_s1 = nullptr;    // [B][2H][2W][c0]
  void* ss_x = nullptr;     // [B][2H][2W][16]  (SIMT family)
  float* ss_r = nullptr;    // [B][2H][2W][3]   (SIMT family)
  // N4 object-major T (GLASSNET_FLAG_OBJECTS)
  float* objW[2] = {};      // SIMT conv packs of T1 (16 -> h), T2 (h -> h), [tap][ci][co]
  float* objB[2] = {};
  void* obj_x = nullptr;    // [B][H][W][16]   an object's conv input
  void* obj_h1 = nullptr;   // [B][H][W][h]    its first layer
  void* obj_a2 = nullptr;   // [B][H][W][h]    its second layer (SIMT family only)
  uint32_t* tau_q = nullptr;   // [B][H][W][h] fixed-point latent
  uint32_t* tau_n = nullptr;   // [B][H][W]    covering objects
  size_t wb_off = 0;        // offset of W_B in w_tb
  float qscale = 4096.f, qsat = 2048.f;
  size_t ws_bytes = 0, w_bytes = 0;
  // staging for glassnet_forward_host
  void *st_g = nullptr, *st_d = nullptr, *st_t = nullptr, *st_n = nullptr;
  float* st_o = nullptr;
  cudaStream_t st_in = nullptr, st_out = nullptr;   // forward_host's copy streams (created on first use)
  // tensor-core state (kernels_tc.cuh)
  void* tc_state = nullptr;
  StageProfiler prof;
};
