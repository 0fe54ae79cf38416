// ubench_issue2.cu -- what does a thread pay, after issuing tcgen05.mma, for a shared-memory load,
// an mbarrier test on a completed barrier, and a commit?  (not part of the product)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2405_19056_b200/csrc tools/ubench_issue2.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace gn;

template <int NM>
__global__ void k(long long* out, int nrep) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, bar2, done;
  __shared__ uint32_t tptr;
  __shared__ volatile int val[32];
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 32 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (tid < 32) val[tid] = tid;
  if (tid == 0) { tc::mbar_init(&bar, 1); tc::mbar_init(&bar2, 1); tc::mbar_init(&done, 1); tc::fence_mbar_init(); }
  if (warp == 0) tc::tmem_alloc<512>(&tptr);
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tptr;
  if (tid == 0) {
    tc::mbar_arrive(&bar2);   // completes phase 0
    constexpr uint32_t ID = tc::idesc_f16(128, 64, 1, 1);
    const uint32_t sB = tc::smem_u32(smem);
    long long s_mma = 0, s_lds = 0, s_test = 0, s_commit = 0;
    int acc = 0;
    uint32_t ph = 0;
    for (int q = 0; q < nrep; ++q) {
      long long a = clock64();
#pragma unroll
      for (int m = 0; m < NM; ++m)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem + (q & 1) * 64),
                     "r"(tmem + 448 + m * 8), "l"(tc::smem_desc(sB + m * 2048, 1024, 128)), "r"(ID), "r"((uint32_t)(m > 0)));
      long long b = clock64();
      acc += val[q & 31];
      long long c = clock64();
      acc += tc::mbar_test(&bar2, 0) ? 1 : 0;
      long long d = clock64();
      tc::mma_commit(&bar);
      long long e = clock64();
      tc::mbar_wait(&bar, ph); ph ^= 1;
      s_mma += b - a; s_lds += c - b; s_test += d - c; s_commit += e - d;
    }
    out[blockIdx.x * 4 + 0] = s_mma; out[blockIdx.x * 4 + 1] = s_lds; out[blockIdx.x * 4 + 2] = s_test;
    out[blockIdx.x * 4 + 3] = s_commit;
    if (acc == 12345) out[0] = 0;
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

template <int NM>
void run() {
  long long* d;
  cudaMalloc(&d, 148 * 4 * sizeof(long long));
  const int nrep = 1000;
  cudaFuncSetAttribute(k<NM>, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
  k<NM><<<148, 128, 40 * 1024>>>(d, nrep);
  k<NM><<<148, 128, 40 * 1024>>>(d, nrep);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148 * 4];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  double s[4] = {0, 0, 0, 0};
  for (int b = 0; b < 148; ++b)
    for (int i = 0; i < 4; ++i) s[i] += h[b * 4 + i];
  printf("%d MMAs issued: issue %.1f, then LDS %.1f, mbarrier test %.1f, commit %.1f cycles (%s)\n", NM,
         s[0] / 148 / nrep, s[1] / 148 / nrep, s[2] / 148 / nrep, s[3] / 148 / nrep, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<1>();
  run<2>();
  run<4>();
  return 0;
}
