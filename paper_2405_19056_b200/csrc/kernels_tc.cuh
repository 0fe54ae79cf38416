// kernels_tc.cuh -- tcgen05 tensor-core kernels (bf16 mode).  Placeholder until the
// tcgen05 family lands: bf16 mode runs the SIMT family.
#pragma once
#include <cuda_bf16.h>
#include <vector>

#include "net.h"

namespace gn {

inline int tc_pack_weights(glassnet*, const float*, const float*, const float*, const float*,
                           const std::vector<const float*>&, const std::vector<const float*>&,
                           const float*, const float*, const std::vector<const float*>&,
                           const std::vector<const float*>&, const float*, const float*) {
  return 0;
}
inline int tc_setup(glassnet* net) { net->tc = false; return 0; }
inline void tc_release(glassnet*) {}
inline int tc_launches(glassnet*, int) { return 0; }
inline int tc_forward(glassnet* net, const __nv_bfloat16*, const __nv_bfloat16*, const __nv_bfloat16*,
                      const uint8_t*, float*, int, cudaStream_t) {
  return gn_fail(GLASSNET_ERR_UNSUPPORTED, "tensor-core family not built");
}

}  // namespace gn
