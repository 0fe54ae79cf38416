// ubench_mma.cu -- tcgen05 MMA throughput microbenchmark (not part of the product).
// One CTA per SM (grid = #SMs), one thread issues NREP back-to-back M=128 K=16 MMAs
// of width N into one TMEM accumulator, commit, wait; cycles per MMA vs the ideal N/2.
// Modes: SS (A and B in shared memory) and TS (A in TMEM).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2405_19056_b200/csrc tools/ubench_mma.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace gn;

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(acc));
}

template <int N, int TS, int SPREAD>
__global__ void k_tput(long long* out, int nrep) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tptr;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (tid == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  if (warp == 0) tc::tmem_alloc<512>(&tptr);
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tptr;
  const uint32_t sA = tc::smem_u32(smem), sB = tc::smem_u32(smem + 32768);
  constexpr uint32_t ID = tc::idesc_f16(128, N, 1, 1);
  long long c0 = 0, c1 = 0;
  if (tid == 0) {
    // warm
    for (int q = 0; q < 8; ++q) tc::mma_f16_ss(tmem, tc::smem_desc(sA, 2048, 128), tc::smem_desc(sB, N * 16, 128), ID, q > 0);
    tc::mma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    c0 = clock64();
    for (int q = 0; q < nrep; ++q) {
      // SPREAD: cycle the A operand over 8 K-steps of a 128x128 tile (as a real K loop does)
      const uint32_t ao = SPREAD ? (q & 7) * 2 * 2048 : 0;
      const uint32_t bo = SPREAD ? (q & 7) * 2 * N * 16 : 0;
      if (TS) mma_ts(tmem + 256, tmem + (q & 7) * 8, tc::smem_desc(sB + bo, N * 16, 128), ID, 1);
      else tc::mma_f16_ss(tmem + (N <= 256 ? 0 : 0), tc::smem_desc(sA + ao, 2048, 128),
                          tc::smem_desc(sB + bo, N * 16, 128), ID, 1);
    }
    tc::mma_commit(&bar);
    tc::mbar_wait(&bar, 1);
    c1 = clock64();
    out[blockIdx.x] = c1 - c0;
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

template <int N, int TS, int SPREAD>
void run(const char* name, int nsm) {
  long long* d;
  cudaMalloc(&d, nsm * sizeof(long long));
  const int nrep = 2048;
  auto k = k_tput<N, TS, SPREAD>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  k<<<nsm, 128, 100 * 1024>>>(d, nrep);
  k<<<nsm, 128, 100 * 1024>>>(d, nrep);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[256];
  cudaMemcpy(h, d, nsm * sizeof(long long), cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < nsm; ++i) s += h[i];
  s /= nsm;
  printf("%-28s N=%3d  %7.1f cyc/MMA  ideal %5.1f  eff %5.1f%%  (%s)\n", name, N, s / nrep, N / 2.0,
         100.0 * (N / 2.0) / (s / nrep), cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  int nsm = 148;
  run<32, 0, 0>("SS same-operand", nsm);
  run<64, 0, 0>("SS same-operand", nsm);
  run<128, 0, 0>("SS same-operand", nsm);
  run<256, 0, 0>("SS same-operand", nsm);
  run<32, 0, 1>("SS K-loop operands", nsm);
  run<64, 0, 1>("SS K-loop operands", nsm);
  run<128, 0, 1>("SS K-loop operands", nsm);
  run<256, 0, 1>("SS K-loop operands", nsm);
  run<32, 1, 1>("TS (A in TMEM)", nsm);
  run<64, 1, 1>("TS (A in TMEM)", nsm);
  run<128, 1, 1>("TS (A in TMEM)", nsm);
  run<256, 1, 1>("TS (A in TMEM)", nsm);
  return 0;
}
