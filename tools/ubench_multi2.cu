// ubench_multi2.cu -- aggregate tcgen05.mma issue rate per SM with 1/2/4 issuing threads in
// different warps (sub-partitions), TS and SS, N=64 and N=32 (not part of the product)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2405_19056_b200/csrc tools/ubench_multi2.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace gn;

template <int TS, int N>
__global__ void k(long long* out, int nrep, int nw) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[4];
  __shared__ uint32_t tptr;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (tid == 0) { for (int i = 0; i < 4; ++i) tc::mbar_init(&bar[i], 1); tc::fence_mbar_init(); }
  if (warp == 0) tc::tmem_alloc<512>(&tptr);
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tptr;
  constexpr uint32_t ID = tc::idesc_f16(128, N, 1, 1);
  const uint32_t sA = tc::smem_u32(smem), sB = sA + 32768;
  __syncthreads();
  const long long c0 = clock64();
  if ((tid & 31) == 0 && warp < nw) {
    const uint32_t d = tmem + warp * 64;
    for (int q = 0; q < nrep; ++q) {
      const uint64_t bd = tc::smem_desc(sB + (q & 3) * 2 * N * 16, N * 16, 128);
      if (TS)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
                     "r"(tmem + 256 + warp * 32 + (q & 3) * 8), "l"(bd), "r"(ID), "r"(1u));
      else
        tc::mma_f16_ss(d, tc::smem_desc(sA + ((q + warp) & 7) * 4096, 2048, 128), bd, ID, 1);
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

template <int TS, int N>
void run(int nw) {
  long long* d;
  cudaMalloc(&d, 256 * sizeof(long long));
  long long h[256];
  const int nrep = 2048;
  auto kk = k<TS, N>;
  cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  kk<<<148, 128, 100 * 1024>>>(d, nrep, nw);
  kk<<<148, 128, 100 * 1024>>>(d, nrep, nw);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d, 148 * sizeof(long long), cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < 148; ++i) s += h[i];
  s /= 148;
  printf("%s N=%3d issuing warps %d: %6.1f cyc per MMA (SM aggregate), ideal %5.1f (%s)\n", TS ? "TS" : "SS", N, nw,
         s / (nrep * (double)nw), N / 2.0, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  for (int nw : {1, 2, 3, 4}) run<1, 64>(nw);
  for (int nw : {1, 2, 4}) run<0, 64>(nw);
  for (int nw : {1, 2, 4}) run<1, 32>(nw);
  for (int nw : {1, 2}) run<1, 128>(nw);
  return 0;
}
