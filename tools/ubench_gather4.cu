// ubench_gather4.cu -- TMA tile::gather4 on sm_100a: semantics (swizzle, negative / out-of-range
// coordinates) and throughput for the T kernel's record windows.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_gather4 tools/ubench_gather4.cu -lcuda
// Part A: one CTA gathers 32-byte windows (16 halfwords at column 11k-5) of 128 rows of a
//         [R][88] u16 tensor into a SWIZZLE_32B tile and prints / checks the layout.
// Part B: 148 CTAs x many tiles of random rows: time per gather4 and bytes/s.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1); } } while (0)

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void arrive_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@P1 bra D;\n\tbra W;\n\tD:\n\t}" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void gather4c(uint32_t dst, const CUtensorMap* m, int c, int r0, int r1, int r2, int r3, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
      ::"r"(dst), "l"(m), "r"(c), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(su32(b)) : "memory");
}
__device__ __forceinline__ void gather4(uint32_t dst, const CUtensorMap* m, int c, int r0, int r1, int r2, int r3, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
      ::"r"(dst), "l"(m), "r"(c), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(su32(b)) : "memory");
}

__device__ __forceinline__ void tile2d(uint32_t dst, const CUtensorMap* m, int c, int r, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(dst), "l"(m), "r"(c), "r"(r), "r"(su32(b)) : "memory");
}
__global__ void kP(const __grid_constant__ CUtensorMap map, uint16_t* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  if (threadIdx.x == 0) {
    arrive_tx(&bar, 4 * 32);
    for (int i = 0; i < 4; ++i) tile2d(su32(sm + i * 128), &map, 0, i * 3, &bar);
  }
  mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < 64; i += blockDim.x) out[i] = reinterpret_cast<uint16_t*>(sm)[(i / 16) * 64 + i % 16];
}
__global__ void kA(const __grid_constant__ CUtensorMap map, const int* rows, int nslot, uint16_t* out, int coff, int bw) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  if (threadIdx.x == 0) {
    arrive_tx(&bar, nslot * 128 * bw * 2);
    for (int k = 0; k < nslot; ++k)
      for (int i = 0; i < 32; ++i)
        if (coff == 0 && bw == 99) gather4c(su32(sm + k * 256 * bw + i * 8 * bw), &map, 11 * k - coff, rows[4 * i], rows[4 * i + 1], rows[4 * i + 2], rows[4 * i + 3], &bar);
        else gather4(su32(sm + k * 256 * bw + i * 8 * bw), &map, 11 * k - coff, rows[4 * i], rows[4 * i + 1], rows[4 * i + 2], rows[4 * i + 3], &bar);
  }
  mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < nslot * 2048; i += blockDim.x) out[i] = reinterpret_cast<uint16_t*>(sm)[i];
}

// Part B: each CTA loads `tiles` tiles of nslot windows x 128 random rows, double-buffered
__global__ void kB(const __grid_constant__ CUtensorMap map, const int* rows, int R, int tiles, int nslot, int nthr, unsigned* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[2];
  if (threadIdx.x == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  unsigned acc = 0;
  const int per = 32 / nthr;
  for (int t = 0; t < tiles; ++t) {
    const int b = t & 1;
    if (t >= 2) mbar_wait(&bar[b], ((t - 2) >> 1) & 1);
    __syncthreads();
    if (threadIdx.x < nthr) {
      if (threadIdx.x == 0) arrive_tx(&bar[b], nslot * 128 * 32);
      const int* rr = rows + ((long)(blockIdx.x * tiles + t) * 128) % ((long)R - 128);
      for (int k = 0; k < nslot; ++k)
        for (int i = threadIdx.x * per; i < threadIdx.x * per + per; ++i)
          gather4(su32(sm + b * 65536 + k * 4096 + i * 128), &map, 11 * k - 5, rr[4 * i], rr[4 * i + 1], rr[4 * i + 2], rr[4 * i + 3], &bar[b]);
    }
  }
  for (int t = tiles - 2; t < tiles; ++t) if (t >= 0) mbar_wait(&bar[t & 1], (t >> 1) & 1);
  acc += sm[threadIdx.x];
  if (acc == 0x12345) sink[0] = acc;
}

int main(int argc, char** argv) {
  const int swz = argc > 1 ? atoi(argv[1]) : 1, bw = argc > 2 ? atoi(argv[2]) : 16, partB = argc > 3 ? atoi(argv[3]) : 0;
  const CUtensorMapSwizzle SW[4] = {CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_SWIZZLE_128B};
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q));
  EncodeTiledFn enc = (EncodeTiledFn)fp;
  const long R = 1L << 22;   // rows (pixels) of 88 u16 = 176 B: 738 MB
  uint16_t* dT;
  CK(cudaMalloc(&dT, R * 176));
  std::vector<uint16_t> h(R * 88);
  for (long r = 0; r < R; ++r)
    for (int c = 0; c < 88; ++c) h[r * 88 + c] = (uint16_t)(((r & 0xFF) << 8) | c);
  CK(cudaMemcpy(dT, h.data(), R * 176, cudaMemcpyHostToDevice));
  CUtensorMap map;
  const long RM = argc > 6 ? atol(argv[6]) : R;
  const cuuint64_t dims[2] = {88, (cuuint64_t)RM};
  const cuuint64_t str[1] = {176};
  const cuuint32_t box[2] = {(cuuint32_t)bw, 1};
  const cuuint32_t es[2] = {1, 1};
  CUresult cr = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, dT, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    SW[swz], CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("swizzle %d box %d: encode %d\n", swz, bw, (int)cr);
  {
    uint16_t* dP; CK(cudaMalloc(&dP, 128));
    CK(cudaFuncSetAttribute(kP, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
    kP<<<1, 128, 64 * 1024>>>(map, dP);
    CK(cudaDeviceSynchronize());
    uint16_t hp[64]; CK(cudaMemcpy(hp, dP, 128, cudaMemcpyDeviceToHost));
    printf("plain tile:"); for (int i = 0; i < 20; ++i) printf(" %04x", hp[i]); printf("\n");
  }
  // Part A
  std::vector<int> rows(128);
  for (int i = 0; i < 128; ++i) rows[i] = (i * 7919 + 13) % 1000;
  const int safe = argc > 4 ? atoi(argv[4]) : 0;
  if (!safe) { rows[5] = (int)R; rows[6] = (int)R + 77; }   // out of range -> zeros?
  int* dR;
  CK(cudaMalloc(&dR, 128 * 4));
  CK(cudaMemcpy(dR, rows.data(), 128 * 4, cudaMemcpyHostToDevice));
  const int ns = 8;
  uint16_t* dO;
  CK(cudaMalloc(&dO, ns * 4096));
  CK(cudaFuncSetAttribute(kA, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
  if (argc > 5 && atoi(argv[5])) {   // launch as a 1-CTA cluster
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = 64 * 1024;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = 1; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, kA, map, (const int*)dR, safe ? 4 : ns, dO, safe ? 0 : 5, bw));
  } else {
    kA<<<1, 128, 64 * 1024>>>(map, dR, safe ? 4 : ns, dO, safe ? 0 : 5, bw);
  }
  CK(cudaDeviceSynchronize());
  std::vector<uint16_t> o(ns * 2048);
  CK(cudaMemcpy(o.data(), dO, ns * 4096, cudaMemcpyDeviceToHost));
  // expected value of (slot k, tile row i, window column j)
  auto expv = [&](int k, int i, int j) -> int {
    const long r = rows[i];
    const int c = 11 * k - 5 + j;
    if (r >= R || c < 0 || c >= 88) return 0;
    return (int)(((r & 0xFF) << 8) | c);
  };
  // hypothesis: SWIZZLE_32B = 16-byte chunk index ^= address bit 7 (row i at 32 i: bit 7 = (i >> 2) & 1)
  long bad_sw = 0, bad_lin = 0;
  for (int k = 0; k < ns; ++k)
    for (int i = 0; i < 128; ++i)
      for (int j = 0; j < 16; ++j) {
        const int e = expv(k, i, j);
        const int ch = j >> 3, w = j & 7;
        const int sw = (k * 2048) + i * 16 + (((ch ^ ((i >> 2) & 1))) * 8) + w;
        const int lin = (k * 2048) + i * 16 + j;
        bad_sw += o[sw] != e;
        bad_lin += o[lin] != e;
      }
  printf("part A: mismatches swizzle32-hypothesis %ld, linear %ld (of %d)\n", bad_sw, bad_lin, ns * 2048);
  for (int i = 0; i < 8; ++i) {
    printf("row %d (src %d):", i, rows[i]);
    for (int j = 0; j < 16; ++j) printf(" %04x", o[2048 * 1 + i * 16 + j]);
    printf("\n");
  }
  if (!partB) return 0;
  // Part B: random rows
  std::vector<int> rr(R);
  srand(1);
  for (long i = 0; i < R; ++i) rr[i] = (int)(((long)rand() * 7 + rand()) % R);
  int* dRR;
  CK(cudaMalloc(&dRR, R * 4));
  CK(cudaMemcpy(dRR, rr.data(), R * 4, cudaMemcpyHostToDevice));
  unsigned* sink;
  CK(cudaMalloc(&sink, 4));
  CK(cudaFuncSetAttribute(kB, cudaFuncAttributeMaxDynamicSharedMemorySize, 130 * 1024));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int nthr : {1, 4, 32})
    for (int nsl : {4, 8}) {
      const int tiles = 400;
      kB<<<148, 128, 130 * 1024>>>(map, dRR, (int)R, 4, nsl, nthr, sink);
      cudaEventRecord(a);
      kB<<<148, 128, 130 * 1024>>>(map, dRR, (int)R, tiles, nsl, nthr, sink);
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double ninst = 148.0 * tiles * nsl * 32, bytes = ninst * 128;
      printf("part B: issuing threads %2d, slots %d: %.3f ms, %.1f ns per tile per SM, %.2f cycles/gather4/SM (1.965 GHz), %.0f GB/s delivered\n",
             nthr, nsl, ms, ms * 1e6 / tiles, ms * 1e-3 * 1.965e9 / (ninst / 148), bytes / ms / 1e6);
    }
  return 0;
}
