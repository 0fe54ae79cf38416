// synth_dev.cu -- device twin of synth/__init__.py's seeded input generator (HARNESS).
//
// Same counter hash, same exact fp64 arithmetic (compiled with -fmad=false so no mul+add
// is contracted), same rounding (fp64 -> fp32 RNE -> bf16 RNE): the values are bitwise
// identical to the numpy generator (pinned by tests/test_synth_gpu.py).  Holds none of
// the method's arithmetic.  Used by bench.py and the full-size GPU tests to fill
// multi-GB batches quickly.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__host__ uint64_t splitmix64_h(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ double u24(uint64_t h) { return (double)(h >> 40) * 0x1p-24; }

__device__ double gauss(uint64_t key, uint64_t base, int d) {
  double s = 0.0;
  for (int k = 0; k < 3; ++k) {
    uint64_t h = splitmix64(key ^ (base | (uint64_t)(d + k)));
    for (int sh = 0; sh < 64; sh += 16) {
      double f = (double)((h >> sh) & 0xFFFFull);
      s = s + (f + 0.5) / 65536.0;
    }
  }
  return s - 6.0;
}

__device__ double exp_ieee(double x) {
  const double C[14] = {1.0, 1.0, 0.5, 0.16666666666666666, 0.041666666666666664,
                        0.008333333333333333, 0.001388888888888889, 0.0001984126984126984,
                        2.48015873015873e-05, 2.7557319223985893e-06, 2.755731922398589e-07,
                        2.505210838544172e-08, 2.08767569878681e-09, 1.6059043836821613e-10};
  double k = floor(x * 1.4426950408889634 + 0.5);
  double r = (x - k * 0.6931471803691238) - k * 1.9082149292705877e-10;
  double p = C[13];
  for (int j = 12; j >= 0; --j) p = p * r + C[j];
  return ldexp(p, (int)k);
}

__device__ void normal3(uint64_t key, uint64_t base, int d0, double out[3]) {
  double z[3];
  for (int c = 0; c < 3; ++c) z[c] = gauss(key, base, d0 + 3 * c);
  double n2 = (z[0] * z[0] + z[1] * z[1]) + z[2] * z[2];
  double nrm = sqrt(n2);
  if (nrm < 1e-12) { out[0] = 0.0; out[1] = 0.0; out[2] = 1.0; return; }
  for (int c = 0; c < 3; ++c) out[c] = z[c] / nrm;
}

__device__ __forceinline__ double lognormal(uint64_t key, uint64_t base, int d) {
  return exp_ieee(-1.0 + gauss(key, base, d));
}

template <typename T> __device__ __forceinline__ T store(double v);
template <> __device__ __forceinline__ float store<float>(double v) { return __double2float_rn(v); }
template <> __device__ __forceinline__ __nv_bfloat16 store<__nv_bfloat16>(double v) {
  return __float2bfloat16_rn(__double2float_rn(v));
}

struct Keys { uint64_t g, d, t, n; };

template <typename T>
__global__ void k_synth(Keys keys, int frame0, int nframes, int H, int W, int K, int y0, int y1,
                        T* gbuf, T* direct, T* tbuf, uint8_t* tcount, const uint8_t* mask) {
  const long rows = y1 - y0;
  const long npx = (long)nframes * rows * W;
  long q = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= npx) return;
  const int x = (int)(q % W);
  const long t = q / W;
  const int y = y0 + (int)(t % rows);
  const long f = frame0 + t / rows;
  const uint64_t base = ((uint64_t)f * (uint64_t)H * (uint64_t)W + (uint64_t)y * W + x) << 10;
  // gbuf: pos, normal, albedo, roughness, metallic, depth
  T* g = gbuf + q * 12;
  for (int c = 0; c < 3; ++c) g[c] = store<T>(-10.0 + 20.0 * u24(splitmix64(keys.g ^ (base | (uint64_t)c))));
  double nv[3];
  normal3(keys.g, base, 3, nv);
  for (int c = 0; c < 3; ++c) g[3 + c] = store<T>(nv[c]);
  for (int c = 0; c < 3; ++c) g[6 + c] = store<T>(u24(splitmix64(keys.g ^ (base | (uint64_t)(12 + c)))));
  g[9] = store<T>(u24(splitmix64(keys.g ^ (base | 15ull))));
  g[10] = store<T>(u24(splitmix64(keys.g ^ (base | 16ull))));
  g[11] = store<T>(0.1 + 99.9 * u24(splitmix64(keys.g ^ (base | 17ull))));
  // direct light: lognormal(-1, 1)
  for (int c = 0; c < 3; ++c) direct[q * 3 + c] = store<T>(lognormal(keys.d, base, 3 * c));
  // transparency records
  for (int k = 0; k < K; ++k) {
    T* r = tbuf + (q * K + k) * 11;
    const int d = k * 32;
    normal3(keys.t, base, d, nv);
    for (int c = 0; c < 3; ++c) r[c] = store<T>(nv[c]);
    for (int c = 0; c < 3; ++c) r[3 + c] = store<T>(u24(splitmix64(keys.t ^ (base | (uint64_t)(d + 9 + c)))));
    r[6] = store<T>(0.05 + 0.9 * u24(splitmix64(keys.t ^ (base | (uint64_t)(d + 12)))));
    r[7] = store<T>(0.1 + 99.9 * u24(splitmix64(keys.t ^ (base | (uint64_t)(d + 13)))));
    for (int c = 0; c < 3; ++c) r[8 + c] = store<T>(lognormal(keys.t, base, d + 14 + 3 * c));
  }
  // count
  const uint64_t hn = splitmix64(keys.n ^ base) >> 40;
  uint64_t n;
  if (mask == nullptr) n = (hn * (uint64_t)(K + 1)) >> 24;
  else n = mask[(long)y * W + x] ? 1 + ((hn * (uint64_t)K) >> 24) : 0;
  tcount[q] = (uint8_t)n;
}

}  // namespace

// precision: 0 = bf16, 1 = fp32.  Fills frames [frame0, frame0+nframes), rows [y0,y1),
// all columns.  mask (optional, device, [H][W] u8) selects c2's covered pixels.
extern "C" int glassnet_synth_fill(int precision, uint64_t seed, int frame0, int nframes, int H, int W, int K,
                                   int y0, int y1, void* gbuf, void* direct, void* tbuf, uint8_t* tcount,
                                   const uint8_t* mask, void* stream) {
  Keys keys{splitmix64_h(seed * 16 + 1), splitmix64_h(seed * 16 + 2), splitmix64_h(seed * 16 + 3),
            splitmix64_h(seed * 16 + 4)};
  const long npx = (long)nframes * (y1 - y0) * W;
  const unsigned blocks = (unsigned)((npx + 127) / 128);
  cudaStream_t st = (cudaStream_t)stream;
  if (precision == 0)
    k_synth<__nv_bfloat16><<<blocks, 128, 0, st>>>(keys, frame0, nframes, H, W, K, y0, y1, (__nv_bfloat16*)gbuf,
                                                  (__nv_bfloat16*)direct, (__nv_bfloat16*)tbuf, tcount, mask);
  else
    k_synth<float><<<blocks, 128, 0, st>>>(keys, frame0, nframes, H, W, K, y0, y1, (float*)gbuf, (float*)direct,
                                          (float*)tbuf, tcount, mask);
  return (int)cudaGetLastError();
}
