// ubench_tc2.cu -- do MMA batches issued by different warps (different accumulators) overlap?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Ipaper_2405_19056_b200/csrc tools/ubench_tc2.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include "tc_ptx.cuh"
using namespace gn;

// NB warps issue the T-kernel round batch each into its own TMEM columns; time until all done.
__global__ void k(long long* out, int nb, int nrep, int mode) {
  __shared__ __align__(1024) uint8_t smem[40 * 1024];
  __shared__ uint64_t bar[4];
  __shared__ uint32_t tptr;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 40 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (tid == 0) { for (int i = 0; i < 4; ++i) tc::mbar_init(&bar[i], 1); tc::fence_mbar_init(); }
  if (warp == 0) tc::tmem_alloc<512>(&tptr);
  tc::fence_proxy_async(); tc::fence_before_sync(); __syncthreads(); tc::fence_after_sync();
  const uint32_t tmem = tptr;
  const uint32_t sA = tc::smem_u32(smem), sB = tc::smem_u32(smem + 32768);
  uint32_t phase = 0;
  long long acc = 0;
  for (int rep = 0; rep < nrep; ++rep) {
    __syncthreads();
    long long c0 = clock64();
    if (warp < nb && (tid & 31) == 0) {
      tc::fence_after_sync();
      const uint32_t base = tmem + warp * 160;
      const int nbatch = mode == 1 ? nb : 1;   // mode 1: warp 0 issues all batches
      if (mode == 0 || warp == 0) {
        for (int bb = 0; bb < nbatch; ++bb) {
          const uint32_t bs = (mode == 1) ? tmem + bb * 160 : base;
          for (int q = 0; q < 4; ++q)
            tc::mma_f16_ss(bs + 128, tc::smem_desc(sA + q * 4096, 2048, 128), tc::smem_desc(sB, 512, 128), tc::idesc_f16(128, 32, 0, 0), 1);
          for (int q = 0; q < 5; ++q)
            tc::mma_f16_ss(bs + 64, tc::smem_desc(sA + q * 4096, 2048, 128), tc::smem_desc(sB + (q % 2) * 2048, 1024, 128), tc::idesc_f16(128, 64, 1, 1), q > 0);
          tc::mma_f16_ss(bs, tc::smem_desc(sA, 2048, 128), tc::smem_desc(sB, 1024, 128), tc::idesc_f16(128, 64, 1, 1), 0);
          if (mode == 1) tc::mma_commit(&bar[bb]);
        }
        if (mode == 0) tc::mma_commit(&bar[warp]);
      }
    }
    for (int w = 0; w < nb; ++w) tc::mbar_wait(&bar[w], phase);
    phase ^= 1;
    long long c1 = clock64();
    acc += c1 - c0;
  }
  if (tid == 0) out[0] = acc / nrep;
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}
int main() {
  long long* d; cudaMalloc(&d, 64);
  for (int mode = 0; mode < 2; ++mode)
    for (int nb = 1; nb <= 3; ++nb) {
      k<<<1, 128>>>(d, nb, 50, mode);
      long long h; cudaError_t e = cudaDeviceSynchronize(); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      printf("mode=%d (%s) batches=%d: %lld cyc  (%s)\n", mode, mode ? "one issuer" : "one issuer per warp", nb, h, cudaGetErrorString(e));
    }
  return 0;
}
