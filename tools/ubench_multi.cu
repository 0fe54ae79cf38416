// ubench_multi.cu -- does MMA throughput per SM scale with the number of issuing threads
// (warps)?  (not part of the product)  NW warps, lane 0 of each issues NREP back-to-back
// M=128 N=64 K=16 SS MMAs (changing operands) into its own TMEM accumulator.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2405_19056_b200/csrc tools/ubench_multi.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace gn;

template <int N>
__global__ void k_multi(long long* out, int nrep, int nw, int commit_every) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[8];
  __shared__ uint32_t tptr;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (tid == 0) { for (int i = 0; i < 8; ++i) tc::mbar_init(&bar[i], 1); tc::fence_mbar_init(); }
  if (warp == 0) tc::tmem_alloc<512>(&tptr);
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tptr;
  constexpr uint32_t ID = tc::idesc_f16(128, N, 1, 1);
  const uint32_t sA = tc::smem_u32(smem), sB = tc::smem_u32(smem + 65536);
  __syncthreads();
  long long c0 = clock64();
  if ((tid & 31) == 0 && warp < nw) {
    for (int q = 0; q < nrep; ++q) {
      tc::mma_f16_ss(tmem + warp * N, tc::smem_desc(sA + ((q + warp) & 7) * 4096, 2048, 128),
                     tc::smem_desc(sB + (q & 7) * N * 32, N * 16, 128), ID, 1);
      if (commit_every && (q % commit_every) == commit_every - 1) tc::mma_commit(&bar[4 + warp % 4]);
    }
    tc::mma_commit(&bar[warp]);
    tc::mbar_wait(&bar[warp], 0);
  }
  __syncthreads();
  if (tid == 0) out[blockIdx.x] = clock64() - c0;
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

template <int N>
void run(int nw, int ce) {
  long long* d;
  cudaMalloc(&d, 256 * sizeof(long long));
  long long h[256];
  const int nsm = 148, nrep = 2048;
  auto k = k_multi<N>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  k<<<nsm, 256, 140 * 1024>>>(d, nrep, nw, ce);
  k<<<nsm, 256, 140 * 1024>>>(d, nrep, nw, ce);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d, nsm * sizeof(long long), cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < nsm; ++i) s += h[i];
  s /= nsm;
  printf("N=%3d issuing warps %d commit every %d: %6.1f cyc per MMA (SM aggregate), ideal %5.1f (%s)\n", N, nw, ce,
         s / (nrep * (double)nw), N / 2.0, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  for (int nw : {1, 2, 4}) run<64>(nw, 0);
  for (int nw : {1, 2, 4}) run<64>(nw, 5);
  for (int nw : {1, 2}) run<128>(nw, 0);
  return 0;
}
