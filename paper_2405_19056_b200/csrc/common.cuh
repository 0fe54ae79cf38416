// common.cuh -- small device helpers shared by the GlassNet kernels (product path).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace gn {

__device__ __forceinline__ float to_f(float v) { return v; }
__device__ __forceinline__ float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }

template <typename T> __device__ __forceinline__ T from_f(float v);
template <> __device__ __forceinline__ float from_f<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}

// Raw storage bits of one element (for the canonical fragment order).
__device__ __forceinline__ uint32_t bits_of(float v) { return __float_as_uint(v); }
__device__ __forceinline__ uint32_t bits_of(__nv_bfloat16 v) {
  return (uint32_t)__bfloat16_as_ushort(v);
}

__device__ __forceinline__ float relu(float v) { return v > 0.f ? v : 0.f; }

// Bilinear x2 (half-pixel, edge clamp) source taps for fine index J of a coarse axis of
// length n ("up-sampling"; reading R14 in DESIGN.md).
__device__ __forceinline__ void up2_taps(int J, int n, int& a, int& b, float& wa, float& wb) {
  int i = J >> 1;
  if ((J & 1) == 0) { a = i > 0 ? i - 1 : 0; b = i; wa = 0.25f; wb = 0.75f; }
  else { a = i; b = i + 1 < n ? i + 1 : n - 1; wa = 0.75f; wb = 0.25f; }
}

struct Up2Rows {
  int rows_f, rows_f_buf, grow0_f;   // fine level (skip, d, psi, out)
  int rows_c_buf, grow0_c, Hc_full;  // coarse level (y or z)
  int halo;
  int yoff = 0, ystep = 1;           // fine row of grid row j = j * ystep + yoff (row tiles: edge rows first)
};

}  // namespace gn
