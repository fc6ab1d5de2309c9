// init.cu — K12: counter-hash synthetic values on device.
//
// Same generator as sidp_inputs/gen.py, implemented independently:
//   key = seed ^ (tensor << 56) ^ (layer << 44) ^ idx ;  h = splitmix64(key)
//   weight = ((h >> 56) - 128) * 2^-7 * 2^-floor(log2(K)/2); gain = 1 + ((h >> 60) - 8) * 2^-7
//   bias = ((h >> 56) - 128) * 2^-7 * 2^-3; unit = ((h >> 56) - 128) * 2^-7
// Values are exact in bf16, so the GPU copy is bit-identical to the logical tensor.
#include "../common.cuh"
#include "../kernels.h"

namespace sidp {

namespace {

constexpr int kTensorWGate = 6;   // sidp_inputs.gen.WGATE
constexpr int kTensorWUp = 7;     // sidp_inputs.gen.WUP
constexpr int64_t kTStride = 1 << 17;

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ float gen_value(uint64_t seed, int tensor, int layer, uint64_t idx,
                                           int kind, float wscale) {
  const uint64_t h = splitmix64(seed ^ ((uint64_t)tensor << 56) ^ ((uint64_t)layer << 44) ^ idx);
  const float lvl = (float)((int)(h >> 56) - 128) * 0.0078125f;   // 2^-7
  switch (kind) {
    case GEN_WEIGHT: return lvl * wscale;
    case GEN_GAIN: return 1.0f + (float)((int)(h >> 60) - 8) * 0.0078125f;
    case GEN_BIAS: return lvl * 0.125f;
    default: return lvl;
  }
}

__global__ void gen_kernel(GenArgs a, float wscale) {
  const int64_t total = a.rows * a.cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / a.cols, c = e % a.cols;
    int tensor = a.tensor;
    int64_t lrow = a.row0 + r;
    if (a.row_map == 1) {            // packed gate/up: 16-row group g = [gate 8g.. | up 8g..]
      const int64_t pr = a.row0 + r;
      const int64_t g = pr / 16, i = pr % 16;
      tensor = i < 8 ? kTensorWGate : kTensorWUp;
      lrow = g * 8 + (i & 7);
    }
    const uint64_t idx = (uint64_t)(lrow * a.lcols + c);
    a.dst[r * a.ld + c] = f_to_bf16(gen_value(a.seed, tensor, a.layer, idx, a.kind, wscale));
  }
}

__global__ void gen_kv_kernel(bf16* cache, int B, int nkv, int smax, int hd, int T, int64_t b0,
                              uint64_t seed, int tensor, int layer) {
  const int64_t total = (int64_t)B * nkv * T * hd;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int d = (int)(e % hd);
    int64_t rest = e / hd;
    const int t = (int)(rest % T);
    rest /= T;
    const int g = (int)(rest % nkv);
    const int64_t b = rest / nkv;
    const uint64_t idx = (uint64_t)((((b0 + b) * kTStride + t) * nkv + g) * hd + d);
    cache[((b * nkv + g) * (int64_t)smax + t) * hd + d] =
        f_to_bf16(gen_value(seed, tensor, layer, idx, GEN_UNIT, 1.0f));
  }
}

int grid_for(int64_t n) {
  int64_t g = (n + 255) / 256;
  return (int)(g < 148 * 32 ? (g < 1 ? 1 : g) : 148 * 32);
}

}  // namespace

cudaError_t gen_launch(const GenArgs& a, cudaStream_t s) {
  if (a.rows <= 0 || a.cols <= 0) return cudaSuccess;
  int k = a.scale_k > 0 ? a.scale_k : 1;
  int lg = 31 - __builtin_clz((unsigned)k);
  float wscale = ldexpf(1.0f, -(lg / 2));
  gen_kernel<<<grid_for(a.rows * a.cols), 256, 0, s>>>(a, wscale);
  return cudaGetLastError();
}

cudaError_t gen_kv_launch(bf16* cache, int B, int nkv, int smax, int hd, int T, int64_t b0,
                          uint64_t seed, int tensor, int layer, cudaStream_t s) {
  const int64_t n = (int64_t)B * nkv * T * hd;
  if (n <= 0) return cudaSuccess;
  gen_kv_kernel<<<grid_for(n), 256, 0, s>>>(cache, B, nkv, smax, hd, T, b0, seed, tensor, layer);
  return cudaGetLastError();
}

}  // namespace sidp
