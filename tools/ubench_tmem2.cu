// ubench_tmem2.cu -- TMEM load bandwidth with many warps and loads in flight, alone and beside an
// MMA stream (not part of the product).  Decides how many epilogue warps / loads in flight the T
// kernel needs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2405_19056_b200/csrc tools/ubench_tmem2.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace gn;

__device__ __forceinline__ void ld64(uint32_t taddr, uint32_t (&r)[64]) {
  tc::tmem_ld32(taddr, *reinterpret_cast<uint32_t(*)[32]>(r));
  tc::tmem_ld32(taddr + 32, *reinterpret_cast<uint32_t(*)[32]>(r + 32));
}

// NW warps (warp w reads lanes of quadrant w%4), each iteration: F loads of 32 columns, one wait
template <int F, bool MMA>
__global__ void k_tm(long long* out, int nrep, int nw, unsigned* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tptr;
  __shared__ uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 32 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (tid == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  if (warp == 0) tc::tmem_alloc<512>(&tptr);
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tptr;
  long long c0 = clock64();
  unsigned acc = 0;
  if (warp < nw) {
    const uint32_t base = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) % 2 * 128;
    for (int q = 0; q < nrep; ++q) {
      uint32_t r[F][32];
#pragma unroll
      for (int f = 0; f < F; ++f) tc::tmem_ld32(base + 32 * f, r[f]);
      tc::tmem_ld_wait();
#pragma unroll
      for (int f = 0; f < F; ++f)
#pragma unroll
        for (int k = 0; k < 32; ++k) acc += r[f][k];
    }
  } else if (MMA && warp == nw && lane == 0) {
    // an N=64 TS MMA stream into columns 384.. (A from TMEM columns 448..)
    constexpr uint32_t ID = tc::idesc_f16(128, 64, 1, 1);
    const uint32_t sB = tc::smem_u32(smem);
    for (int q = 0; q < nrep * 4; ++q)
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem + 384),
                   "r"(tmem + 448 + (q & 3) * 8), "l"(tc::smem_desc(sB + (q & 3) * 2048, 1024, 128)), "r"(ID), "r"(1));
    tc::mma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    out[blockIdx.x * 64 + 63] = clock64() - c0;
  }
  long long c1 = clock64();
  if (lane == 0 && warp < nw) out[blockIdx.x * 64 + warp] = c1 - c0;
  if (acc == 0x12345) sink[0] = acc;
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

template <int F, bool MMA>
void run(int nw) {
  long long* d;
  unsigned* sink;
  cudaMalloc(&d, 148 * 64 * sizeof(long long));
  cudaMalloc(&sink, 4);
  cudaMemset(d, 0, 148 * 64 * sizeof(long long));
  const int nrep = 512;
  auto k = k_tm<F, MMA>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const int threads = 32 * (nw + (MMA ? 1 : 0));
  k<<<148, threads, 64 * 1024>>>(d, nrep, nw, sink);
  k<<<148, threads, 64 * 1024>>>(d, nrep, nw, sink);
  cudaError_t e = cudaDeviceSynchronize();
  static long long h[148 * 64];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int b = 0; b < 148; ++b)
    for (int w = 0; w < nw; ++w) mx += h[b * 64 + w];
  mx /= 148.0 * nw;
  const double bytes = (double)nw * nrep * F * 32 * 32 * 4;
  double mm = 0;
  for (int b = 0; b < 148; ++b) mm += h[b * 64 + 63];
  mm /= 148.0;
  printf("warps %2d loads-in-flight %d (x32 cols) %s: %6.1f B/clk/SM  (%.0f cyc per warp-iteration)  MMA %.1f cyc/instr %s\n", nw, F,
         MMA ? "+MMA stream" : "           ", bytes / mx, mx / nrep, MMA ? mm / (nrep * 4) : 0.0, cudaGetErrorString(e));
  cudaFree(d);
  cudaFree(sink);
}

int main() {
  for (int nw : {4, 8, 12, 16}) { run<1, false>(nw); run<2, false>(nw); run<4, false>(nw); }
  for (int nw : {0, 4, 8, 12, 16}) { run<2, true>(nw); }
  return 0;
}
