// ubench_contention.cu -- does a stream of tcgen05.mma slow down concurrent tcgen05.ld
// (TMEM reads) and st.shared (operand writes) from other warps?  (not part of the product)
// One CTA per SM: warp 4 lane 0 issues back-to-back M=128 N=64 K=16 MMAs (SS) into TMEM
// columns [256, 320) while warps 0-3 time NREP iterations of (a) 2x tcgen05.ld.32x32b.x32 +
// wait on columns [0, 64), or (b) 8x st.shared.v4 of a 128-row operand plane + bar.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2405_19056_b200/csrc tools/ubench_contention.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace gn;

__global__ void k_cont(long long* out, int nrep, int mode, int mma_on) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tptr;
  __shared__ volatile int stop;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (tid == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); stop = 0; }
  if (warp == 0) tc::tmem_alloc<512>(&tptr);
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tptr;
  if (warp == 4) {
    if ((tid & 31) == 0 && mma_on) {
      const uint32_t sA = tc::smem_u32(smem), sB = tc::smem_u32(smem + 32768);
      constexpr uint32_t ID = tc::idesc_f16(128, 64, 1, 1);
      long n = 0;
      while (!stop) {
        for (int q = 0; q < 16; ++q)
          tc::mma_f16_ss(tmem + 256, tc::smem_desc(sA + (q & 7) * 4096, 2048, 128),
                         tc::smem_desc(sB + (q & 7) * 2048, 1024, 128), ID, 1);
        n += 16;
      }
      tc::mma_commit(&bar);
      tc::mbar_wait(&bar, 0);
      out[1024 + blockIdx.x] = n;
    }
  } else {
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    const uint32_t sW = tc::smem_u32(smem + 65536);
    uint32_t acc = 0;
    for (int i = 0; i < 64; ++i) __nanosleep(100);
    tc::bar_sync(1, 128);
    const long long c0 = clock64();
    for (int i = 0; i < nrep; ++i) {
      if (mode == 0) {
        uint32_t a[32], b[32];
        tc::tmem_ld32(tmem + lane_off, a);
        tc::tmem_ld32(tmem + lane_off + 32, b);
        tc::tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) acc += a[j] ^ b[j];
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) tc::sts128(sW + q * 2048 + tid * 16, acc, q, i, tid);
        tc::fence_proxy_async();
        tc::bar_sync(1, 128);
      }
    }
    const long long c1 = clock64();
    tc::bar_sync(1, 128);
    if (tid == 0) { out[blockIdx.x] = c1 - c0; stop = 1; }
    if (acc == 0x12345) out[2000] = acc;
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

int main() {
  long long* d;
  cudaMalloc(&d, 4096 * sizeof(long long));
  long long h[4096];
  const int nsm = 148, nrep = 2000;
  cudaFuncSetAttribute(k_cont, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int mode = 0; mode < 2; ++mode)
    for (int on = 0; on < 2; ++on) {
      k_cont<<<nsm, 160, 100 * 1024>>>(d, nrep, mode, on);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(h, d, 4096 * sizeof(long long), cudaMemcpyDeviceToHost);
      double s = 0, nm = 0;
      for (int i = 0; i < nsm; ++i) { s += h[i]; nm += h[1024 + i]; }
      s /= nsm; nm /= nsm;
      printf("%s  MMA stream %s: %7.1f cyc/iter  (MMAs issued per SM %.0f -> %.1f cyc/MMA) %s\n",
             mode == 0 ? "2x tcgen05.ld.x32 + wait" : "8x STS.128 + fence + bar", on ? "ON " : "off",
             s / nrep, on ? nm : 0.0, on ? s / nm : 0.0, cudaGetErrorString(e));
    }
  return 0;
}
