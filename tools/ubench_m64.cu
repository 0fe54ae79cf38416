// ubench_m64.cu -- where does an M=64 (cta_group::1) tcgen05.mma put its 64 accumulator rows in
// TMEM, and can two M=64 accumulators share columns in different lanes?  (not part of the
// product; de-risks "64-row tiles, four chains" in DESIGN.md §6.1)
// A (64 x 16, K-major): A[r][0] = r + 1, else 0.  B (64 x 16): B[n][0] = 1.  So D[r][n] = r + 1.
// TMEM columns 0..63 are first filled with -1 by every warp; after the MMA (D at lane offset
// `loff`, column 0) each of the 4 warps reads its 32 lanes of column 0 and column 5.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2405_19056_b200/csrc tools/ubench_m64.cu
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace gn;

__global__ void k_m64(float* out, int loff, int two) {
  __shared__ __align__(1024) uint16_t sA[2 * 64 * 8];   // 2 K-planes x 64 rows x 8
  __shared__ __align__(1024) uint16_t sB[2 * 64 * 8];
  __shared__ uint64_t bar;
  __shared__ uint32_t tptr;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 2 * 64 * 8; i += blockDim.x) {
    const int plane = i / (64 * 8), row = (i / 8) % 64, k = i % 8;
    const bool c0 = plane == 0 && k == 0;
    sA[i] = c0 ? __bfloat16_as_ushort(__float2bfloat16((float)(row + 1))) : 0;
    sB[i] = c0 ? __bfloat16_as_ushort(__float2bfloat16(1.f)) : 0;
  }
  if (tid == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  if (warp == 0) tc::tmem_alloc<64>(&tptr);
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tptr;
  {   // fill all 128 lanes x 64 columns with -1
    uint32_t v[32];
    for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(-1.f);
    tc::tmem_st32(tmem + ((uint32_t)(warp * 32) << 16), v);
    tc::tmem_st32(tmem + ((uint32_t)(warp * 32) << 16) + 32, v);
    tc::tmem_st_wait();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if (tid == 0) {
    constexpr uint32_t ID = tc::idesc_f16(64, 64, 1, 1);
    const uint64_t ad = tc::smem_desc(tc::smem_u32(sA), 64 * 16, 128), bd = tc::smem_desc(tc::smem_u32(sB), 64 * 16, 128);
    tc::mma_f16_ss(tmem + ((uint32_t)loff << 16), ad, bd, ID, 0);
    if (two) tc::mma_f16_ss(tmem + ((uint32_t)(loff + 16) << 16), ad, bd, ID, 0);   // a second M=64 D
    tc::mma_commit(&bar);
    tc::mbar_wait(&bar, 0);
  }
  __syncthreads();
  tc::fence_after_sync();
  uint32_t v[16];
  tc::tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16), v);
  tc::tmem_ld_wait();
  out[tid] = __uint_as_float(v[0]);
  out[128 + tid] = __uint_as_float(v[5]);
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<64>(tmem);
}

int main() {
  float* d;
  cudaMalloc(&d, 256 * sizeof(float));
  float h[256];
  const int cases[3][2] = {{0, 0}, {16, 0}, {0, 1}};
  for (auto& c : cases) {
    cudaMemset(d, 0, 256 * sizeof(float));
    k_m64<<<1, 128>>>(d, c[0], c[1]);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("D lane offset %d%s (%s)\n", c[0], c[1] ? " + a second M=64 MMA at lane offset +16" : "", cudaGetErrorString(e));
    for (int q = 0; q < 4; ++q) {
      printf("  lanes %3d-%3d col0:", q * 32, q * 32 + 31);
      for (int l = 0; l < 32; ++l) printf(" %g", h[q * 32 + l]);
      printf("\n");
    }
    printf("  (col5, lanes 0-31):");
    for (int l = 0; l < 32; ++l) printf(" %g", h[128 + l]);
    printf("\n");
  }
  return 0;
}
