// ubench_pingpong.cu -- hand-off latency between warps of one CTA (not part of the product):
// warp 0 lane 0 and warp 1 lane 0 bounce a token through two mbarriers NREP times; cycles per
// round trip (= 2 hand-offs).  Modes: try_wait loop, test_wait spin, try_wait with a suspend-time
// hint, and the tcgen05.commit path (the waiter's partner commits instead of arriving).  With
// `busy` extra warps spinning on an unrelated barrier, to see the cost of pollers.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2405_19056_b200/csrc tools/ubench_pingpong.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace gn;

__device__ __forceinline__ void wait_mode(uint64_t* bar, uint32_t ph, int mode) {
  const uint32_t a = tc::smem_u32(bar);
  if (mode == 1) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "LAB_T:\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra LAB_T;\n\t}" ::"r"(a), "r"(ph) : "memory");
  } else if (mode == 2) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "LAB_H:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@!P1 bra LAB_H;\n\t}" ::"r"(a), "r"(ph), "r"(20) : "memory");
  } else {
    tc::mbar_wait(bar, ph);
  }
}

__global__ void k_pp(long long* out, int nrep, int mode, int commit) {
  __shared__ uint64_t bar[3];
  __shared__ uint32_t tptr;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    tc::mbar_init(&bar[0], 1); tc::mbar_init(&bar[1], 1); tc::mbar_init(&bar[2], 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc<32>(&tptr);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if (warp == 0 && lane == 0) {
    const long long c0 = clock64();
    for (int i = 0; i < nrep; ++i) {
      tc::mbar_arrive(&bar[0]);
      wait_mode(&bar[1], i & 1, mode);
    }
    out[blockIdx.x] = clock64() - c0;
  } else if (warp == 1 && lane == 0) {
    for (int i = 0; i < nrep; ++i) {
      wait_mode(&bar[0], i & 1, mode);
      if (commit) tc::mma_commit(&bar[1]);
      else tc::mbar_arrive(&bar[1]);
    }
  } else if (warp >= 2) {
    if (lane == 0) wait_mode(&bar[2], 0, mode);   // never completes until the end
  }
  if (warp == 0) {
    __syncwarp();
  }
  if (tid == 0) tc::mbar_arrive(&bar[2]);
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<32>(tptr);
}

int main() {
  long long* d;
  cudaMalloc(&d, 256 * sizeof(long long));
  long long h[256];
  const int nsm = 148, nrep = 4000;
  const char* mn[] = {"try_wait loop", "test_wait spin", "try_wait + hint 20ns"};
  for (int commit = 0; commit < 2; ++commit)
    for (int busy = 0; busy < 2; ++busy)
      for (int mode = 0; mode < 3; ++mode) {
        const int threads = busy ? 18 * 32 : 64;
        k_pp<<<nsm, threads>>>(d, nrep, mode, commit);
        k_pp<<<nsm, threads>>>(d, nrep, mode, commit);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, d, nsm * sizeof(long long), cudaMemcpyDeviceToHost);
        double s = 0;
        for (int i = 0; i < nsm; ++i) s += h[i];
        printf("%-22s %-14s %-12s %7.1f cyc/round trip (%s)\n", mn[mode], commit ? "commit back" : "arrive back",
               busy ? "+16 pollers" : "alone", s / nsm / nrep, cudaGetErrorString(e));
      }
  return 0;
}
