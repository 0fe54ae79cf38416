// comm.cu -- NCCL bootstrap for row-tile sharding (PL2/PL3).
// Point-to-point only; the unique id travels over the caller's torch process group.
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstring>

#include "../../include/glassnet.h"
#include "net.h"

struct glassnet_comm {
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  cudaStream_t cs = nullptr;                  // halo exchanges run here, beside the interior rows
  cudaEvent_t ev_b = nullptr, ev_x = nullptr;  // boundary rows written / exchange done
};

extern "C" int glassnet_get_unique_id(uint8_t id[128]) {
  if (!id) return gn_fail(GLASSNET_ERR_INVALID_ARGUMENT, "id is NULL");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId u;
  ncclResult_t r = ncclGetUniqueId(&u);
  if (r != ncclSuccess) return gn_fail(GLASSNET_ERR_NCCL, "ncclGetUniqueId: %s", ncclGetErrorString(r));
  memcpy(id, &u, 128);
  return GLASSNET_OK;
}

extern "C" int glassnet_comm_create(const uint8_t id[128], int32_t nranks, int32_t rank, glassnet_comm_t* out) {
  if (!id || !out) return gn_fail(GLASSNET_ERR_INVALID_ARGUMENT, "id/out is NULL");
  if (nranks < 1 || rank < 0 || rank >= nranks)
    return gn_fail(GLASSNET_ERR_INVALID_ARGUMENT, "rank %d of %d", rank, nranks);
  ncclUniqueId u;
  memcpy(&u, id, 128);
  glassnet_comm* c = new glassnet_comm();
  ncclResult_t r = ncclCommInitRank(&c->comm, nranks, u, rank);
  if (r != ncclSuccess) {
    delete c;
    return gn_fail(GLASSNET_ERR_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
  }
  c->nranks = nranks;
  c->rank = rank;
  if (cudaStreamCreateWithFlags(&c->cs, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_b, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_x, cudaEventDisableTiming) != cudaSuccess) {
    glassnet_comm_destroy(c);
    return gn_fail(GLASSNET_ERR_CUDA, "comm stream / events");
  }
  *out = c;
  return GLASSNET_OK;
}

extern "C" void glassnet_comm_destroy(glassnet_comm_t c) {
  if (!c) return;
  if (c->comm) ncclCommDestroy(c->comm);
  if (c->cs) cudaStreamDestroy(c->cs);
  if (c->ev_b) cudaEventDestroy(c->ev_b);
  if (c->ev_x) cudaEventDestroy(c->ev_x);
  delete c;
}

// Row-tile forward: the tensor-core step list with halo rows exchanged at EXCH steps.
// Rank r sends its first interior row up (to r-1) and its last interior row down (to
// r+1) and receives the neighbours' rows into its halo rows; frame-edge halos stay zero.
// Boundary rows first (gn::tc_steps, tile order): a producer's first/last rows are computed,
// the exchange of them runs on the comm stream (after an event on the main stream), and the
// producer's other rows run on the main stream meanwhile; the next step that reads the
// exchanged rows (anything but an edge-2 step or T) first waits for the exchange's event.  The
// exchange writes only the halo rows and reads only the boundary rows, which the edge-2 launch
// neither reads nor writes.
static int run_tile_steps(glassnet_t net, glassnet_comm* c, const void* gbuf, const void* direct, const void* tbuf,
                          const uint8_t* tcount, float* out, cudaStream_t st,
                          int (*exch)(void*, glassnet_t, int, cudaStream_t), void* ctx) {
  gn::Step steps[96];
  const int n = gn::tc_steps(net, steps, 96, true);
  if (n > 96) return gn_fail(GLASSNET_ERR_UNSUPPORTED, "tile step list");
  net->prof.mark(nullptr, st);
  bool pending = false;
  for (int i = 0; i < n; ++i) {
    const gn::Step& sp = steps[i];
    int rc;
    if (sp.kind == gn::ST_EXCH) {
      if (pending && cudaStreamWaitEvent(c->cs, c->ev_x, 0) != cudaSuccess) return gn_fail(GLASSNET_ERR_CUDA, "wait");
      if (cudaEventRecord(c->ev_b, st) != cudaSuccess || cudaStreamWaitEvent(c->cs, c->ev_b, 0) != cudaSuccess)
        return gn_fail(GLASSNET_ERR_CUDA, "exchange event");
      rc = exch(ctx, net, sp.idx, c->cs);
      if (!rc && cudaEventRecord(c->ev_x, c->cs) != cudaSuccess) return gn_fail(GLASSNET_ERR_CUDA, "exchange event");
      pending = true;
    } else {
      if (pending && sp.edge != 2 && sp.kind != gn::ST_TB) {
        if (cudaStreamWaitEvent(st, c->ev_x, 0) != cudaSuccess) return gn_fail(GLASSNET_ERR_CUDA, "exchange wait");
        pending = false;
      }
      rc = gn::tc_run_step(net, true, sp, gbuf, direct, tbuf, tcount, out, 1, st);
    }
    if (rc) return rc;
  }
  if (pending && cudaStreamWaitEvent(st, c->ev_x, 0) != cudaSuccess) return gn_fail(GLASSNET_ERR_CUDA, "exchange wait");
  return GLASSNET_OK;
}

static int check_tile_args(glassnet_t net, int nranks, int rank, int* row0, int* rows) {
  if (!net) return gn_fail(GLASSNET_ERR_INVALID_ARGUMENT, "net is NULL");
  if (net->d.precision != GLASSNET_BF16 || !net->tc)
    return gn_fail(GLASSNET_ERR_UNSUPPORTED, "row-tile sharding runs the bf16 tensor-core family only");
  int rc = glassnet_tile_rows(&net->d, nranks, rank, row0, rows);
  if (rc) return rc;
  if (cudaSetDevice(net->dev) != cudaSuccess) return gn_fail(GLASSNET_ERR_CUDA, "cudaSetDevice");
  return gn::tc_prepare_tile(net, nranks, rank, *row0, *rows);
}

static int nccl_exch(void* ctx, glassnet_t net, int tensor, cudaStream_t st) {
  glassnet_comm* c = reinterpret_cast<glassnet_comm*>(ctx);
  char* base;
  size_t rb;
  int rows;
  int rc = gn::tc_tensor_rows(net, true, tensor, &base, &rb, &rows);
  if (rc) return rc;
  ncclResult_t r = ncclGroupStart();
  if (c->rank > 0) {
    if (r == ncclSuccess) r = ncclSend(base + rb, rb, ncclUint8, c->rank - 1, c->comm, st);
    if (r == ncclSuccess) r = ncclRecv(base, rb, ncclUint8, c->rank - 1, c->comm, st);
  }
  if (c->rank < c->nranks - 1) {
    if (r == ncclSuccess) r = ncclSend(base + rb * rows, rb, ncclUint8, c->rank + 1, c->comm, st);
    if (r == ncclSuccess) r = ncclRecv(base + rb * (rows + 1), rb, ncclUint8, c->rank + 1, c->comm, st);
  }
  ncclResult_t r2 = ncclGroupEnd();
  if (r != ncclSuccess || r2 != ncclSuccess)
    return gn_fail(GLASSNET_ERR_NCCL, "halo exchange: %s", ncclGetErrorString(r != ncclSuccess ? r : r2));
  return GLASSNET_OK;
}

extern "C" int glassnet_forward_sharded(glassnet_t net, glassnet_comm_t comm, const void* gbuf, const void* direct,
                                        const void* tbuf, const uint8_t* tcount, float* out,
                                        glassnet_stream_t stream) {
  if (!comm) return gn_fail(GLASSNET_ERR_INVALID_ARGUMENT, "comm is NULL");
  if (!gbuf || !direct || !tbuf || !tcount || !out)
    return gn_fail(GLASSNET_ERR_INVALID_ARGUMENT, "a tile pointer is NULL");
  int row0, rows;
  int rc = check_tile_args(net, comm->nranks, comm->rank, &row0, &rows);
  if (rc) return rc;
  rc = run_tile_steps(net, comm, gbuf, direct, tbuf, tcount, out, (cudaStream_t)stream, nccl_exch, comm);
  if (rc) return rc;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return gn_fail(GLASSNET_ERR_CUDA, "forward_sharded: %s", cudaGetErrorString(e));
  return GLASSNET_OK;
}

// ---- single-device emulation of the row-tile decomposition (tests / diagnostics) ----
extern "C" int glassnet_forward_sharded_local(glassnet_t* nets, int32_t nranks, const void* const* gbuf,
                                              const void* const* direct, const void* const* tbuf,
                                              const uint8_t* const* tcount, float* const* out,
                                              glassnet_stream_t stream) {
  if (!nets || nranks < 1 || !gbuf || !direct || !tbuf || !tcount || !out)
    return gn_fail(GLASSNET_ERR_INVALID_ARGUMENT, "bad forward_sharded_local arguments");
  cudaStream_t st = (cudaStream_t)stream;
  for (int r = 0; r < nranks; ++r) {
    int row0, rows;
    int rc = check_tile_args(nets[r], nranks, r, &row0, &rows);
    if (rc) return rc;
    if (nets[r]->dev != nets[0]->dev)
      return gn_fail(GLASSNET_ERR_INVALID_ARGUMENT, "forward_sharded_local needs all handles on one device");
  }
  gn::Step steps[96];
  const int n = gn::tc_steps(nets[0], steps, 96, true);
  if (n > 96) return gn_fail(GLASSNET_ERR_UNSUPPORTED, "tile step list");
  for (int r = 0; r < nranks; ++r) nets[r]->prof.mark(nullptr, st);
  for (int i = 0; i < n; ++i) {
    if (steps[i].kind != gn::ST_EXCH) {
      for (int r = 0; r < nranks; ++r) {
        int rc = gn::tc_run_step(nets[r], true, steps[i], gbuf[r], direct[r], tbuf[r], tcount[r], out[r], 1, st);
        if (rc) return rc;
      }
      continue;
    }
    // halo rows by device copies: rank r's row 0 <- rank r-1's last interior row,
    // rank r's row rows+1 <- rank r+1's first interior row
    for (int r = 0; r < nranks; ++r) {
      char* base;
      size_t rb;
      int rows;
      int rc = gn::tc_tensor_rows(nets[r], true, steps[i].idx, &base, &rb, &rows);
      if (rc) return rc;
      if (r > 0) {
        char* pb; size_t prb; int prows;
        gn::tc_tensor_rows(nets[r - 1], true, steps[i].idx, &pb, &prb, &prows);
        if (cudaMemcpyAsync(base, pb + prb * prows, rb, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
          return gn_fail(GLASSNET_ERR_CUDA, "halo copy");
      }
      if (r < nranks - 1) {
        char* nb; size_t nrb; int nrows;
        gn::tc_tensor_rows(nets[r + 1], true, steps[i].idx, &nb, &nrb, &nrows);
        if (cudaMemcpyAsync(base + rb * (rows + 1), nb + nrb, rb, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
          return gn_fail(GLASSNET_ERR_CUDA, "halo copy");
      }
    }
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return gn_fail(GLASSNET_ERR_CUDA, "forward_sharded_local: %s", cudaGetErrorString(e));
  return GLASSNET_OK;
}
