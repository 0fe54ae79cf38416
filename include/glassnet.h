/*
 * glassnet.h -- C ABI of the B200-native GlassNet inference forward pass
 * (arXiv 2405.19056; PAPER.md = /root/reference/PAPER.md, "P:n" = its line n).
 *
 * The operation (one frame; §3.4 "Rendering Model", and
 * Eq. eq:SymmetricNN; widths from BASELINE.json configs[0]/[1] since the
 * paper gives none; every reading is listed in DESIGN.md "Readings"):
 *
 *   x      = [G', L_d]                     G' = G with position*2^-3, depth*2^-7 (R9)
 *   e_0    = ReLU(conv3x3_s1(x))            scene encoder F
 *   e_l    = ReLU(conv3x3_s2(e_{l-1}))      l = 1..L-1
 *   tau    = [ sum_{k < min(n,K)} h(b_k), n ]   T, Eq. eq:SymmetricNN; h = ReLU MLP 11->h->h
 *   phi    = ReLU(W_B [e_0; tau] + b_B)     blending network B
 *   d_{L-1}= e_{L-1};  y_l = ReLU(conv3x3_s1(d_l));  d_{l-1} = up2(y_l) + skip_{l-1}
 *            (skip_0 = phi, else e_{l-1})   rendering network R
 *   out    = sigmoid(W_O [d_0; L_d] + b_O)  fp32 RGB in [0,1]
 *
 * Every stage runs in this library's own sm_100a CUDA kernels.  There is no CPU
 * fallback: a missing device or an unsupported shape is an error.
 *
 * Tensors (all dense, NHWC, caller-owned, >= 16-byte aligned device pointers unless a
 * function says "host"):
 *   gbuf   [B][H][W][12]   pos xyz, normal xyz, albedo rgb, roughness, metallic, depth
 *   direct [B][H][W][3]    L_d (raw, un-normalised)
 *   tbuf   [B][H][W][K][11] per slot: normal xyz, colour rgb, alpha, depth, direct rgb;
 *                          UNSORTED; slots k >= tcount may hold any bits (NaN/Inf ok)
 *   tcount [B][H][W] uint8 valid slots per pixel; values > K are clamped to K
 *   out    [B][H][W][3] fp32
 * gbuf/direct/tbuf element type = dims.precision (GLASSNET_BF16: bfloat16 bits,
 * GLASSNET_FP32: float).
 *
 * Weights: one little-endian fp32 host blob, in this order (conv weights OHWI,
 * cross-correlation, tap (ky,kx) reads offset (ky-1,kx-1)):
 *   (with GLASSNET_FLAG_POSENC(L): every "11" below is 11(2L+1) and F0's "15" is 15(2L+1))
 *   (with GLASSNET_FLAG_OBJECTS: T1.W[h][3][3][11], T2.W[h][3][3][h] -- h's two 3x3 convolutions)
 *   T1.W[h][11] T1.b[h] T2.W[h][h] T2.b[h]   (GLASSNET_FLAG_SIGMA_COND: T1.W[h][11 + c0] --
 *                                             the paper's h(b_i, sigma), Eq. eq:SymmetricNN
 *                                             P:308-316, layer 1 over [record ; e0 at the
 *                                             pixel])
 *   F0.W[c0][3][3][15] F0.b ... F_{L-1}.W[c_{L-1}][3][3][c_{L-2}] F_{L-1}.b
 *   B.W[c0][c0+h+1] B.b[c0]                 concat order [e0, tau_sum, n]
 *   R_{L-1}.W[c_{L-2}][3][3][c_{L-1}] R_{L-1}.b ... R_1.W[c0][3][3][c1] R_1.b
 *   O.W[3][c0+3] O.b[3]                     concat order [d0, L_d]
 *   (GLASSNET_FLAG_SUPERSAMPLE only, s = c0:)
 *   S1.W[s][3][3][15] S1.b[s] S2.W[s][3][3][s] S2.b[s] S3.W[3][s] S3.b[3]   (glassnet_supersample)
 * In GLASSNET_BF16 mode the W tensors are rounded RNE to bf16; biases stay fp32.
 *
 * Errors: every function returns GLASSNET_OK (0) or an error code; the message
 * (naming the violated invariant) is in glassnet_last_error() (thread-local).
 * Validation is synchronous and happens before anything is enqueued.  Asynchronous
 * device faults surface as GLASSNET_ERR_CUDA on a later call or at the caller's sync.
 */
#ifndef GLASSNET_H_
#define GLASSNET_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GLASSNET_ABI_VERSION 1

enum { GLASSNET_OK = 0, GLASSNET_ERR_INVALID_ARGUMENT = 1, GLASSNET_ERR_UNSUPPORTED = 2,
       GLASSNET_ERR_CUDA = 3, GLASSNET_ERR_NCCL = 4, GLASSNET_ERR_OUT_OF_MEMORY = 5 };
enum { GLASSNET_BF16 = 0, GLASSNET_FP32 = 1 };          /* storage + math mode         */
enum { GLASSNET_POOL_SUM = 0, GLASSNET_POOL_MEAN = 1 };  /* g of Eq. eq:SymmetricNN     */
enum { GLASSNET_FLAG_R_TAKES_LD = 1u << 0,               /* reading R15, default on     */
       GLASSNET_FLAG_INPUT_NORM = 1u << 1,               /* reading R9, default on      */
       GLASSNET_FLAG_SIGMA_COND = 1u << 2,               /* N1, default off: h(b, sigma) */
       GLASSNET_FLAG_SUPERSAMPLE = 1u << 3,              /* N3, default off: the x2 super-sampler S */
       GLASSNET_FLAG_OBJECTS = 1u << 4 };                /* N4, default off: object-major T (below) */
/* N2 (default off): positional encoding with L_pe = 1..10 frequencies of every input channel
 * (§3.4 P:373-375 "All the inputs use positional encoding by Mildenhall et al.";
 * SPEC.md S:395-403): gamma(v) = (v, sin(2^0 pi v), cos(2^0 pi v), ..., sin(2^(L-1) pi v),
 * cos(2^(L-1) pi v)) per channel, channels in input order, applied after the R9 normalisation
 * to x (15 -> 15(2L+1) channels, F0's input) and to every record (11 -> 11(2L+1), h's layer-1
 * input).  Stored in flags bits 8..11. */
#define GLASSNET_FLAG_POSENC(L) ((uint32_t)(L) << 8)
#define GLASSNET_POSENC_OF(flags) ((int)(((flags) >> 8) & 15u))

typedef struct glassnet* glassnet_t;
typedef struct glassnet_comm* glassnet_comm_t;
typedef void* glassnet_stream_t;                         /* a cudaStream_t (0 = legacy) */

typedef struct {
  int32_t abi_version;   /* = GLASSNET_ABI_VERSION                                  */
  int32_t height, width; /* full frame; multiples of 2^(levels-1)                   */
  int32_t max_batch;     /* workspace is sized for this many frames                 */
  int32_t k_slots;       /* K, 1..16                                                */
  int32_t levels;        /* L, 2..4                                                 */
  int32_t widths[4];     /* c_0..c_{L-1}, multiples of 16, <= 256                   */
  int32_t t_hidden;      /* h, multiple of 16, <= 64                                */
  int32_t precision;     /* GLASSNET_BF16 | GLASSNET_FP32                           */
  int32_t pool;          /* GLASSNET_POOL_*                                         */
  uint32_t flags;        /* GLASSNET_FLAG_*                                         */
} glassnet_dims;

/* Number of fp32 values in the weight blob for these dims (0 if dims are invalid). */
size_t glassnet_weight_count(const glassnet_dims* dims);

/* Create a handle on CUDA device `device`: validates dims, copies + repacks the host
 * weight blob (n_weights fp32 values, caller keeps ownership) into device memory and
 * allocates the workspace for dims->max_batch frames.  The workspace size does not
 * depend on K (the transparency stage streams fragments). */
int glassnet_create(const float* weights, size_t n_weights, const glassnet_dims* dims,
                    int device, glassnet_t* out);

/* Enqueue one forward pass of `batch` frames (1..max_batch) on `stream`.  All pointers
 * are device pointers with the layouts above.  No host sync, no allocation.  A handle
 * must not run two forwards concurrently. */
int glassnet_forward(glassnet_t net, const void* gbuf, const void* direct, const void* tbuf,
                     const uint8_t* tcount, float* out, int32_t batch, glassnet_stream_t stream);

/* Same as glassnet_forward but with HOST buffers (pinned for best speed): copies the
 * inputs host->device, runs the forward on `stream`, copies `out` back and synchronises
 * before returning (the end-to-end user call).  Pipelined in chunks of up to 4 frames:
 * the copies run on the handle's own two copy streams and overlap the forward of the
 * neighbouring chunk; the result is bitwise the whole-batch forward's (frames are
 * independent).  Host buffers must stay valid until the call returns. */
int glassnet_forward_host(glassnet_t net, const void* gbuf, const void* direct,
                          const void* tbuf, const uint8_t* tcount, float* out, int32_t batch,
                          glassnet_stream_t stream);

/* Device bytes owned by the handle: workspace (activations) and repacked weights. */
size_t glassnet_workspace_bytes(glassnet_t net);
size_t glassnet_weight_bytes(glassnet_t net);

/* Number of kernel launches one glassnet_forward of `batch` frames enqueues
 * (glassnet_forward_sharded's row tile adds one: the x16 input stage for its halo exchange). */
int glassnet_launches_per_forward(glassnet_t net, int32_t batch);

/* Select the kernel family for bf16 mode: 1 = tcgen05 tensor-core kernels (default
 * when built for sm_100a), 0 = SIMT FFMA kernels (the fp32-check-mode kernels run on
 * bf16 storage).  Both are this library's CUDA; used by tests to cross-check. */
int glassnet_set_kernel_family(glassnet_t net, int tensor_cores);

/* Per-stage device timing (CUDA events recorded on the launching stream after every
 * launch).  begin: allocate room for max_launches events and start recording.
 * end: synchronise, then report per stage (up to max_stages) its name (32 bytes each,
 * NUL-terminated), total milliseconds and launch count; *n_stages = stages seen. */
int glassnet_profile_begin(glassnet_t net, int32_t max_launches);
int glassnet_profile_end(glassnet_t net, int32_t max_stages, char* names, double* total_ms,
                         int32_t* launches, int32_t* n_stages);

/* Test / diagnostic: copy (device to device, on `stream`) the psi intermediate of the last
 * glassnet_forward -- psi = W_O,d0 phi + W_O,L L_d + b_O, [batch][H][W][3] fp32 (reading
 * R15), the only place the transparency latent tau reaches memory -- into the caller's
 * device buffer `dst`.  Bitwise checks of T (slot permutation invariance, Eq.
 * eq:SymmetricNN P:303-318, table:OrderLoss P:666-679) compare it across forwards. */
int glassnet_debug_psi(glassnet_t net, float* dst, int32_t batch, glassnet_stream_t stream);

/* N3 -- the x2 super-sampling network S (§3.4: "A
 * multi-layer CNN is used as a super-sampling network that super-samples the result at x2 the
 * original resolution", fed with the cheaply rasterised high-resolution G-buffer; the
 * architecture is unstated, so SPEC.md S:434-439's form, reading N3):
 *   u = up_nearest(img);  x = [G'_hi, u] (15 ch, G' normalised as above when INPUT_NORM)
 *   s1 = ReLU(conv3x3_s1(x; S1));  s2 = ReLU(conv3x3_s1(s1; S2));  r = S3.W s2 + S3.b
 *   out_hi = clamp(u + r, 0, 1)
 * Needs a handle created with GLASSNET_FLAG_SUPERSAMPLE (the blob then ends with S's weights,
 * hidden width s = widths[0]; the workspace adds the hi-res activations for max_batch frames).
 *   img     [B][H][W][3]        fp32 device (e.g. glassnet_forward's out)
 *   gbuf_hi [B][2H][2W][12]     device, element type = dims.precision, layout as gbuf
 *   out_hi  [B][2H][2W][3]      fp32 device, may not alias img
 * Enqueued on `stream`; no host sync, no allocation.  Errors as above (UNSUPPORTED without
 * the flag). */
int glassnet_supersample(glassnet_t net, const float* img, const void* gbuf_hi, float* out_hi, int32_t batch,
                         glassnet_stream_t stream);

/* N4 -- object-major transparency buffers with a spatial h, streamed one object at a time
 * (one (w, h, c) buffer per transparent object; P:366-368:
 * T is a "multi-layer CNN without down-sampling"; "the model can operate on a single
 * buffer of each transparent object, and then add it to the summed latent representation" --
 * constant memory in the number of objects).  Needs a handle created with GLASSNET_FLAG_OBJECTS
 * (not combinable with SIGMA_COND or POSENC; glassnet_forward then returns UNSUPPORTED):
 *   a_i = ReLU(conv3x3(ReLU(conv3x3(x_i; T1)); T2)),  x_i = cover_i ? b_i' : 0 (b_i' = R9-normalised)
 *   tau = [ sum over covering objects of a_i , number of covering objects ]
 * accumulated as an exact fixed-point integer sum (round(a_i * 2^12) in bf16 mode, 2^20 in fp32
 * check mode; uint32 per channel), so the order of the objects cannot change a bit.
 *   begin:  tau := 0 for `batch` frames.
 *   add:    obj [B][H][W][11] (element type = dims.precision; uncovered pixels may hold any bits),
 *           cover [B][H][W] uint8 (nonzero = the object covers the pixel); adds this object.
 *   finish: gbuf, direct, out as glassnet_forward; runs F, B (over tau), R and the output.
 * All device pointers, enqueued on `stream`, no allocation.  Calls on one handle must be ordered
 * begin, add*, finish on one stream. */
int glassnet_objects_begin(glassnet_t net, int32_t batch, glassnet_stream_t stream);
int glassnet_objects_add(glassnet_t net, const void* obj, const uint8_t* cover, int32_t batch,
                         glassnet_stream_t stream);
int glassnet_objects_finish(glassnet_t net, const void* gbuf, const void* direct, float* out, int32_t batch,
                            glassnet_stream_t stream);

/* ---- row-tile sharding (one process per GPU, NCCL point-to-point halos) ---- */

/* ncclGetUniqueId into id[128] (rank 0 calls it and broadcasts the bytes). */
int glassnet_get_unique_id(uint8_t id[128]);
/* ncclCommInitRank on the current device; collective over nranks processes. */
int glassnet_comm_create(const uint8_t id[128], int32_t nranks, int32_t rank,
                         glassnet_comm_t* out);
void glassnet_comm_destroy(glassnet_comm_t comm);
/* Rows [row0, row0+rows) of the full frame owned by `rank` of `nranks`: rows are split
 * in units of u = 2^(levels-1); rank r gets units [floor(rU/N), floor((r+1)U/N)). */
int glassnet_tile_rows(const glassnet_dims* dims, int32_t nranks, int32_t rank, int32_t* row0,
                       int32_t* rows);
/* Collective forward of ONE frame split in row tiles: each rank passes its tile's
 * rows (pointers cover rows [row0,row0+rows) of gbuf/direct/tbuf/tcount/out).  The
 * result equals glassnet_forward's rows bitwise (reading R22). */
int glassnet_forward_sharded(glassnet_t net, glassnet_comm_t comm, const void* gbuf,
                             const void* direct, const void* tbuf, const uint8_t* tcount,
                             float* out, glassnet_stream_t stream);

/* Single-device emulation of the row-tile decomposition (tests and diagnostics): nets[r]
 * is rank r's handle (all on one device, same dims), pointer arrays give each rank's tile.
 * Runs exactly the per-rank steps of glassnet_forward_sharded, rank by rank, with the
 * halo rows moved by device-to-device copies instead of NCCL. */
int glassnet_forward_sharded_local(glassnet_t* nets, int32_t nranks, const void* const* gbuf,
                                   const void* const* direct, const void* const* tbuf,
                                   const uint8_t* const* tcount, float* const* out,
                                   glassnet_stream_t stream);

void glassnet_destroy(glassnet_t net);
const char* glassnet_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* GLASSNET_H_ */
