// ubench_tmem.cu -- TMEM read throughput, A-collector reuse, M=64 and f16-accumulator
// layout probes for tcgen05 (not part of the product).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2405_19056_b200/csrc tools/ubench_tmem.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

#include "tc_ptx.cuh"

using namespace gn;

// (1) TMEM read throughput: NW warps, each loads 32 lanes x 32 columns (4 KB) per iteration
__global__ void k_tmem_rd(long long* out, int nrep, int x16) {
  __shared__ uint32_t tptr;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tc::tmem_alloc<512>(&tptr);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t t = tptr + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 64;
  uint32_t acc = 0;
  __syncthreads();
  long long c0 = clock64();
  for (int i = 0; i < nrep; ++i) {
    uint32_t v[32];
    if (x16) {
      uint32_t a[16], b[16];
      tc::tmem_ld16(t, a);
      tc::tmem_ld16(t + 16, b);
      tc::tmem_ld_wait();
      for (int j = 0; j < 16; ++j) acc += a[j] ^ b[j];
    } else {
      tc::tmem_ld32(t, v);
      tc::tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 32; ++j) acc += v[j];
    }
  }
  __syncthreads();
  long long c1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = c1 - c0;
  if (acc == 0x1234567) out[1000] = acc;
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tptr);
}

__device__ __forceinline__ void mma_coll(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, int which) {
  if (which == 0)
    asm volatile("tcgen05.mma.cta_group::1.kind::f16.collector::a::fill [%0], %1, %2, %3, 1;" ::"r"(d), "l"(a), "l"(b), "r"(idesc));
  else if (which == 1)
    asm volatile("tcgen05.mma.cta_group::1.kind::f16.collector::a::use [%0], %1, %2, %3, 1;" ::"r"(d), "l"(a), "l"(b), "r"(idesc));
  else
    asm volatile("tcgen05.mma.cta_group::1.kind::f16.collector::a::lastuse [%0], %1, %2, %3, 1;" ::"r"(d), "l"(a), "l"(b), "r"(idesc));
}

// (2) A reuse: groups of 3 MMAs sharing A (different B, different D), with/without collector hints
template <int N, int M, int COLL>
__global__ void k_reuse(long long* out, int nrep) {
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
  const uint32_t sA = tc::smem_u32(smem), sB = tc::smem_u32(smem + 65536);
  constexpr uint32_t ID = tc::idesc_f16(M, N, 1, 1);
  if (tid == 0) {
    long long c0 = clock64();
    for (int q = 0; q < nrep; ++q) {
      const uint64_t ad = tc::smem_desc(sA + (q & 7) * 4096, 2048, 128);
      for (int j = 0; j < 3; ++j) {
        const uint64_t bd = tc::smem_desc(sB + (j * 3 + (q & 1)) * 2 * N * 16, N * 16, 128);
        const uint32_t d = tmem + j * (N <= 128 ? N : 128);
        if (COLL) mma_coll(d, ad, bd, ID, j == 0 ? 0 : j == 1 ? 1 : 2);
        else tc::mma_f16_ss(d, ad, bd, ID, 1);
      }
    }
    tc::mma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    out[blockIdx.x] = clock64() - c0;
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

// (3) f16 accumulator layout: A = all 1.0 (f16 0x3c00), B row n = value (n+1) in channel 0 only.
// D[m][n] = n+1.  Dump TMEM columns 0..15 of lane 0 as raw 32-bit words.
__global__ void k_f16_layout(uint32_t* out) {
  __shared__ __align__(1024) uint8_t smem[16384];
  __shared__ uint64_t bar;
  __shared__ uint32_t tptr;
  const int tid = threadIdx.x, warp = tid >> 5;
  uint16_t* s16 = reinterpret_cast<uint16_t*>(smem);
  // A: 128 x 16 f16 (K-major interleaved: 8-row core matrices 128 B, LBO = 2048 between K halves)
  for (int i = tid; i < 128 * 16; i += blockDim.x) s16[i] = 0x3c00;   // 1.0
  // B: 64 x 16 at offset 4096: row n, k -> value (n+1) if k == 0 else 0
  for (int i = tid; i < 64 * 16; i += blockDim.x) {
    // interleaved layout: plane (k/8) at + (k/8)*1024, row group n/8 at *128, row n%8 *16, k%8 *2
    const int pl = i / 512, rem = i % 512, n = rem / 8, k = rem % 8;
    const int kk = pl * 8 + k;
    const float v = kk == 0 ? (float)(n + 1) : 0.f;
    s16[2048 + i] = __half_as_ushort(__float2half(v));
  }
  if (tid == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  if (warp == 0) tc::tmem_alloc<64>(&tptr);
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tptr;
  if (tid == 0) {
    const uint32_t id = tc::idesc_f16(128, 64, 0, 0) & ~(3u << 4);   // c_format = F16
    tc::mma_f16_ss(tmem, tc::smem_desc(tc::smem_u32(smem), 2048, 128), tc::smem_desc(tc::smem_u32(smem + 4096), 1024, 128),
                   id, 0);
    tc::mma_commit(&bar);
  }
  tc::mbar_wait(&bar, 0);
  tc::fence_after_sync();
  uint32_t v[32];
  tc::tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16), v);
  tc::tmem_ld_wait();
  if (tid == 0)
    for (int j = 0; j < 32; ++j) out[j] = v[j];
  uint32_t p[16];
  // packed load variant
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(p[0]), "=r"(p[1]), "=r"(p[2]), "=r"(p[3]), "=r"(p[4]), "=r"(p[5]), "=r"(p[6]), "=r"(p[7]),
        "=r"(p[8]), "=r"(p[9]), "=r"(p[10]), "=r"(p[11]), "=r"(p[12]), "=r"(p[13]), "=r"(p[14]), "=r"(p[15])
      : "r"(tmem + ((uint32_t)(warp * 32) << 16)));
  tc::tmem_ld_wait();
  if (tid == 0)
    for (int j = 0; j < 16; ++j) out[32 + j] = p[j];
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<64>(tmem);
}

int main() {
  long long* d;
  cudaMalloc(&d, 2048 * sizeof(long long));
  long long h[256];
  const int nsm = 148;
  for (int x16 = 0; x16 < 2; ++x16)
    for (int nw : {4, 8, 16, 32}) {
      const int nrep = 4096;
      k_tmem_rd<<<nsm, nw * 32>>>(d, nrep, x16);
      k_tmem_rd<<<nsm, nw * 32>>>(d, nrep, x16);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(h, d, nsm * sizeof(long long), cudaMemcpyDeviceToHost);
      double s = 0;
      for (int i = 0; i < nsm; ++i) s += h[i];
      s /= nsm;
      printf("TMEM read %s  warps=%2d  %.1f B/clk/SM  (%s)\n", x16 ? "2x x16" : "x32   ", nw,
             (double)nw * 4096.0 * nrep / s, cudaGetErrorString(e));
    }
  auto reuse = [&](auto k, const char* name, double ideal) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    const int nrep = 1024;
    k<<<nsm, 128, 160 * 1024>>>(d, nrep);
    k<<<nsm, 128, 160 * 1024>>>(d, nrep);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, nsm * sizeof(long long), cudaMemcpyDeviceToHost);
    double s = 0;
    for (int i = 0; i < nsm; ++i) s += h[i];
    s /= nsm;
    printf("%-40s %7.1f cyc/MMA  ideal %5.1f  (%s)\n", name, s / (3.0 * nrep), ideal, cudaGetErrorString(e));
  };
  reuse(k_reuse<32, 128, 0>, "3xB per A, N=32 M=128 no hint", 16);
  reuse(k_reuse<32, 128, 1>, "3xB per A, N=32 M=128 collector", 16);
  reuse(k_reuse<64, 128, 0>, "3xB per A, N=64 M=128 no hint", 32);
  reuse(k_reuse<64, 128, 1>, "3xB per A, N=64 M=128 collector", 32);
  reuse(k_reuse<128, 128, 0>, "3xB per A, N=128 M=128 no hint", 64);
  reuse(k_reuse<128, 128, 1>, "3xB per A, N=128 M=128 collector", 64);
  reuse(k_reuse<256, 64, 0>, "3xB per A, N=256 M=64 no hint", 64);
  reuse(k_reuse<128, 64, 0>, "3xB per A, N=128 M=64 no hint", 32);
  uint32_t* du;
  cudaMalloc(&du, 64 * 4);
  k_f16_layout<<<1, 128>>>(du);
  cudaError_t e = cudaDeviceSynchronize();
  uint32_t hu[64];
  cudaMemcpy(hu, du, 64 * 4, cudaMemcpyDeviceToHost);
  printf("f16-D layout (%s): x32 cols:", cudaGetErrorString(e));
  for (int j = 0; j < 32; ++j) printf(" %08x", hu[j]);
  printf("\n  pack::16b x16:");
  for (int j = 0; j < 16; ++j) printf(" %08x", hu[32 + j]);
  printf("\n");
  return 0;
}
