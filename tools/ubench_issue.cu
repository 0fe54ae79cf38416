// ubench_issue.cu -- issue cost of the T kernel's per-slot MMA batch (not part of the product):
// 4 TS MMAs (A from TMEM, N=64, K=16 each) + commit + 1-2 SS MMAs (N=64) + commit, back to back
// from one thread; cycles per batch, measured at the issuing thread.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2405_19056_b200/csrc tools/ubench_issue.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace gn;

__global__ void k_issue(long long* out, int nrep, int mode) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[4];
  __shared__ uint32_t tptr;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (tid == 0) { for (int i = 0; i < 4; ++i) tc::mbar_init(&bar[i], 1); tc::fence_mbar_init(); }
  if (warp == 0) tc::tmem_alloc<512>(&tptr);
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tptr;
  constexpr uint32_t ID = tc::idesc_f16(128, 64, 1, 1);
  const uint32_t sA = tc::smem_u32(smem), sW2 = tc::smem_u32(smem + 65536), sW1 = tc::smem_u32(smem + 65536 + 8192);
  if (tid == 0) {
    long long c0 = clock64();
    for (int it = 0; it < nrep; ++it) {
      const int b = it & 1;
      if (mode >= 4) {   // an already-completed mbarrier wait (+ fence) before each batch
        tc::mbar_wait(&bar[3], 1);
        if (mode == 5) tc::fence_after_sync();
      }
      if (mode != 2)
        for (int q = 0; q < 4; ++q)
          tc::mma_f16_ts(tmem + 192 + b * 64, tmem + 128 + b * 32 + q * 8, tc::smem_desc(sW2 + 2 * q * 1024, 1024, 128), ID, q > 0);
      if (mode != 3) tc::mma_commit(&bar[0]);
      if (mode != 1) {
        const int j = (it * 11 / 8) % 8;
        tc::mma_f16_ss(tmem + b * 64, tc::smem_desc(sA + j * 2048, 2048, 128), tc::smem_desc(sW1 + (it & 7) * 4096, 1024, 128), ID, 0);
      }
      if (mode != 3) tc::mma_commit(&bar[1]);
    }
    tc::mma_commit(&bar[2]);
    tc::mbar_wait(&bar[2], 0);
    out[blockIdx.x] = clock64() - c0;
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

int main() {
  long long* d;
  cudaMalloc(&d, 256 * sizeof(long long));
  long long h[256];
  const int nsm = 148, nrep = 2000;
  cudaFuncSetAttribute(k_issue, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  const char* names[] = {"4 TS + commit + 1 SS + commit", "4 TS + commits only", "1 SS + commits only", "4 TS + 1 SS, no commits",
                         "mode0 + completed mbar wait", "mode0 + mbar wait + fence"};
  for (int mode = 0; mode < 6; ++mode) {
    k_issue<<<nsm, 128, 140 * 1024>>>(d, nrep, mode);
    k_issue<<<nsm, 128, 140 * 1024>>>(d, nrep, mode);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, nsm * sizeof(long long), cudaMemcpyDeviceToHost);
    double s = 0;
    for (int i = 0; i < nsm; ++i) s += h[i];
    printf("%-34s %7.1f cyc/batch (%s)\n", names[mode], s / nsm / nrep, cudaGetErrorString(e));
  }
  return 0;
}
