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
  *out = c;
  return GLASSNET_OK;
}

extern "C" void glassnet_comm_destroy(glassnet_comm_t c) {
  if (!c) return;
  if (c->comm) ncclCommDestroy(c->comm);
  delete c;
}

extern "C" int glassnet_forward_sharded(glassnet_t net, glassnet_comm_t comm, const void* gbuf, const void* direct,
                                        const void* tbuf, const uint8_t* tcount, float* out,
                                        glassnet_stream_t stream) {
  (void)net; (void)comm; (void)gbuf; (void)direct; (void)tbuf; (void)tcount; (void)out; (void)stream;
  return gn_fail(GLASSNET_ERR_UNSUPPORTED, "forward_sharded: not implemented yet");
}
