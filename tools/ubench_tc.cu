// ubench_tc.cu -- latency microbenchmark for the tcgen05 building blocks used by the
// T kernel (not part of the product).  One CTA of 128 threads; clock64 deltas.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2405_19056_b200/csrc tools/ubench_tc.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace gn;

__global__ void k_ubench(long long* out, int nrep, int mode) {
  __shared__ __align__(1024) uint8_t smem[40 * 1024];
  __shared__ uint64_t bar;
  __shared__ uint32_t tptr;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 40 * 1024 / 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (tid == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  if (warp == 0) tc::tmem_alloc<256>(&tptr);
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tptr;
  const uint32_t sA = tc::smem_u32(smem), sB = tc::smem_u32(smem + 32768);
  uint32_t phase = 0;
  long long t_mma1 = 0, t_mma5 = 0, t_mma10 = 0, t_ld = 0, t_sync = 0, t_fence = 0;
  long long c0, c1;
  for (int rep = 0; rep < nrep; ++rep) {
    if (mode & 1) {
    // (1) one MMA M=128 N=64 K=16 : issue -> mbarrier completion seen by all threads
    __syncthreads();
    c0 = clock64();
    if (tid == 0) {
      tc::fence_after_sync();
      tc::mma_f16_ss(tmem, tc::smem_desc(sA, 2048, 128), tc::smem_desc(sB, 1024, 128), tc::idesc_f16(128, 64, 1, 1), 0);
      tc::mma_commit(&bar);
    }
    tc::mbar_wait(&bar, phase); phase ^= 1;
    c1 = clock64();
    t_mma1 += c1 - c0;
    }
    if (mode & 2) {
    // (2) five MMAs (the T2 batch, N=64, K=80)
    __syncthreads();
    c0 = clock64();
    if (tid == 0) {
      for (int q = 0; q < 5; ++q)
        tc::mma_f16_ss(tmem, tc::smem_desc(sA + q * 4096, 2048, 128), tc::smem_desc(sB + (q % 2) * 2048, 1024, 128),
                       tc::idesc_f16(128, 64, 1, 1), q > 0);
      tc::mma_commit(&bar);
    }
    tc::mbar_wait(&bar, phase); phase ^= 1;
    c1 = clock64();
    t_mma5 += c1 - c0;
    }
    if (mode & 4) {
    // (3) ten MMAs N=128
    __syncthreads();
    c0 = clock64();
    if (tid == 0) {
      for (int q = 0; q < 10; ++q)
        tc::mma_f16_ss(tmem, tc::smem_desc(sA + (q % 5) * 4096, 2048, 128), tc::smem_desc(sB, 2048, 128),
                       tc::idesc_f16(128, 128, 1, 1), q > 0);
      tc::mma_commit(&bar);
    }
    tc::mbar_wait(&bar, phase); phase ^= 1;
    c1 = clock64();
    t_mma10 += c1 - c0;
    }
    if (mode & 32) {   // the T-kernel round batch: 4x (f16, N=32) + 5x (bf16, N=64) + 1x (bf16, N=64)
    __syncthreads();
    c0 = clock64();
    if (tid == 0) {
      for (int q = 0; q < 4; ++q)
        tc::mma_f16_ss(tmem + 128, tc::smem_desc(sA + q * 4096, 2048, 128), tc::smem_desc(sB, 512, 128),
                       tc::idesc_f16(128, 32, 0, 0), 1);
      for (int q = 0; q < 5; ++q)
        tc::mma_f16_ss(tmem + 64, tc::smem_desc(sA + q * 4096, 2048, 128), tc::smem_desc(sB + (q % 2) * 2048, 1024, 128),
                       tc::idesc_f16(128, 64, 1, 1), q > 0);
      tc::mma_f16_ss(tmem, tc::smem_desc(sA, 2048, 128), tc::smem_desc(sB, 1024, 128), tc::idesc_f16(128, 64, 1, 1), 0);
      tc::mma_commit(&bar);
    }
    tc::mbar_wait(&bar, phase); phase ^= 1;
    c1 = clock64();
    t_mma1 += c1 - c0;
    }
    tc::fence_after_sync();
    if (mode & 8) {
    // (4) TMEM load of 64 columns (2 x x32) + wait
    c0 = clock64();
    uint32_t v[32], w[32];
    tc::tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16), v);
    tc::tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + 32, w);
    tc::tmem_ld_wait();
    c1 = clock64();
    t_ld += c1 - c0;
    uint32_t acc = 0;
    for (int i = 0; i < 32; ++i) acc += v[i] ^ w[i];
    out[6 + tid] = acc;
    }
    uint32_t acc = tid;
    // (5) STS + fence.proxy.async + tcgen05 fence + bar.sync
    c0 = clock64();
    tc::sts128(sA + 8192 + tid * 16, acc, acc, acc, acc);
    tc::fence_before_sync();
    tc::fence_proxy_async();
    __syncthreads();
    c1 = clock64();
    t_fence += c1 - c0;
    c0 = clock64();
    __syncthreads();
    c1 = clock64();
    t_sync += c1 - c0;
  }
  if (tid == 0) {
    out[0] = t_mma1 / nrep; out[1] = t_mma5 / nrep; out[2] = t_mma10 / nrep;
    out[3] = t_ld / nrep; out[4] = t_fence / nrep; out[5] = t_sync / nrep;
  }
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<256>(tmem);
}

int main() {
  long long* d;
  cudaMalloc(&d, 8 * 256);
  cudaMemset(d, 0, 8 * 256);
  int mode = 0;
  if (const char* m = getenv("MODE")) mode = atoi(m);
  k_ubench<<<1, 128>>>(d, 100, mode);
  long long h[6];
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  printf("err=%s\n", cudaGetErrorString(e));
  printf("mma1(N64,K16) issue->observed: %lld cyc\nmma5(N64,K80): %lld cyc\nmma10(N128,K160): %lld cyc\n"
         "tmem ld 64 cols + wait: %lld cyc\nsts+fences+bar: %lld cyc\nbar.sync: %lld cyc\n",
         h[0], h[1], h[2], h[3], h[4], h[5]);
  return 0;
}
