// ubench_commit.cu -- is tcgen05.commit blocking for the issuing thread?  (not part of the
// product)  Issue NM MMAs (M=128 N=64 K=16), then time (a) the issue loop, (b) the commit
// instruction itself, (c) until the mbarrier completes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2405_19056_b200/csrc tools/ubench_commit.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace gn;

__global__ void k_commit(long long* out, int nm, int chain) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[2];
  __shared__ uint32_t tptr;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (tid == 0) { tc::mbar_init(&bar[0], 1); tc::mbar_init(&bar[1], 1); tc::fence_mbar_init(); }
  if (warp == 0) tc::tmem_alloc<512>(&tptr);
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tptr;
  constexpr uint32_t ID = tc::idesc_f16(128, 64, 1, 1);
  const uint32_t sA = tc::smem_u32(smem), sB = tc::smem_u32(smem + 65536);
  if (tid == 0) {
    long long t[4] = {0, 0, 0, 0};
    uint32_t ph = 0;
    for (int rep = 0; rep < 64; ++rep) {
      const long long c0 = clock64();
      for (int q = 0; q < nm; ++q)
        tc::mma_f16_ss(tmem + (chain ? 0 : (q & 7) * 64), tc::smem_desc(sA + (q & 7) * 4096, 2048, 128),
                       tc::smem_desc(sB + (q & 7) * 2048, 1024, 128), ID, chain ? (q > 0) : 0);
      const long long c1 = clock64();
      tc::mma_commit(&bar[0]);
      const long long c2 = clock64();
      tc::mbar_wait(&bar[0], ph); ph ^= 1;
      const long long c3 = clock64();
      t[0] += c1 - c0; t[1] += c2 - c1; t[2] += c3 - c2;
    }
    out[4 * blockIdx.x + 0] = t[0] / 64; out[4 * blockIdx.x + 1] = t[1] / 64; out[4 * blockIdx.x + 2] = t[2] / 64;
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

int main() {
  long long* d;
  cudaMalloc(&d, 4 * 256 * sizeof(long long));
  long long h[4 * 256];
  cudaFuncSetAttribute(k_commit, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int chain = 0; chain < 2; ++chain)
    for (int nm : {1, 4, 8, 16}) {
      k_commit<<<148, 128, 100 * 1024>>>(d, nm, chain);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(h, d, 4 * 148 * sizeof(long long), cudaMemcpyDeviceToHost);
      double a = 0, b = 0, c = 0;
      for (int i = 0; i < 148; ++i) { a += h[4 * i]; b += h[4 * i + 1]; c += h[4 * i + 2]; }
      printf("%s NM=%2d: issue %6.0f  commit %6.0f  until complete %6.0f cycles (%s)\n",
             chain ? "same D (accumulate chain)" : "distinct D                ", nm, a / 148, b / 148, c / 148,
             cudaGetErrorString(e));
    }
  return 0;
}
