// norm.cu — RMSNorm, embedding gather, argmax finalisation.
// HBM-bound row kernels: 16-byte vector loads, fp32 statistics, one bf16 rounding.
#include "../common.cuh"
#include "../kernels.h"

namespace sidp {

namespace {

// y = bf16( x * rsqrt(mean(x^2) + eps) * g ), one CTA per row, h % 8 == 0.  The row is read
// once: up to kVec 16-byte vectors per thread are loaded up front (all in flight together) and
// kept in registers for the scaling pass (h <= 256 * 8 * kVec = 8192 covers every north_star
// model); longer rows take the strided loop.
constexpr int kNormThreads = 256, kVec = 4;

__global__ void __launch_bounds__(kNormThreads) rmsnorm_kernel(const bf16* __restrict__ x, int ldx,
                                                               const bf16* __restrict__ g, float eps,
                                                               bf16* __restrict__ y, int ldy, int h) {
  pdl_trigger();
  pdl_wait();
  const int row = blockIdx.x;
  const bf16* xr = x + (size_t)row * ldx;
  bf16* yr = y + (size_t)row * ldy;
  const int nvec = h / 8;
  const bool cached = nvec <= kNormThreads * kVec;
  uint4 v[kVec];
  float ss = 0.0f;
  if (cached) {
#pragma unroll
    for (int i = 0; i < kVec; ++i) {
      const int k = threadIdx.x + i * kNormThreads;
      v[i] = k < nvec ? *reinterpret_cast<const uint4*>(xr + k * 8) : make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (int i = 0; i < kVec; ++i) {
      const bf16* e = reinterpret_cast<const bf16*>(&v[i]);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float f = bf16_to_f(e[q]);
        ss += f * f;
      }
    }
  } else {
    for (int k = threadIdx.x; k < nvec; k += kNormThreads) {
      const uint4 raw = *reinterpret_cast<const uint4*>(xr + k * 8);
      const bf16* e = reinterpret_cast<const bf16*>(&raw);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float f = bf16_to_f(e[q]);
        ss += f * f;
      }
    }
  }
  __shared__ float red[32];
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < (kNormThreads >> 5) ? red[threadIdx.x] : 0.0f;
    t = warp_sum(t);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  const float r = rsqrtf(red[0] / (float)h + eps);
  auto scale = [&](const uint4& raw, int k) {
    const uint4 graw = *reinterpret_cast<const uint4*>(g + k * 8);
    const bf16* e = reinterpret_cast<const bf16*>(&raw);
    const bf16* ge = reinterpret_cast<const bf16*>(&graw);
    uint4 out;
    bf16* o = reinterpret_cast<bf16*>(&out);
#pragma unroll
    for (int q = 0; q < 8; ++q) o[q] = f_to_bf16(bf16_to_f(e[q]) * r * bf16_to_f(ge[q]));
    *reinterpret_cast<uint4*>(yr + k * 8) = out;
  };
  if (cached) {
#pragma unroll
    for (int i = 0; i < kVec; ++i) {
      const int k = threadIdx.x + i * kNormThreads;
      if (k < nvec) scale(v[i], k);
    }
  } else {
    for (int k = threadIdx.x; k < nvec; k += kNormThreads)
      scale(*reinterpret_cast<const uint4*>(xr + k * 8), k);
  }
}

__global__ void embed_kernel(const bf16* __restrict__ E, int h, const int32_t* __restrict__ tok,
                             bf16* __restrict__ x) {
  pdl_trigger();
  pdl_wait();
  const int row = blockIdx.x;
  const uint4* src = reinterpret_cast<const uint4*>(E + (size_t)tok[row] * h);
  uint4* dst = reinterpret_cast<uint4*>(x + (size_t)row * h);
  for (int v = threadIdx.x; v < h / 8; v += blockDim.x) dst[v] = src[v];
}

__global__ void argmax_finalize_kernel(const unsigned long long* packed, int32_t* next,
                                       int32_t* pos_out, const int32_t* pos, int rows) {
  pdl_trigger();
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < rows) {
    next[i] = (int32_t)(0xFFFFFFFFu - (uint32_t)(packed[i] & 0xFFFFFFFFull));
    if (pos_out) pos_out[i] = pos[i] + 1;
  }
}

__global__ void argmax_reset_kernel(unsigned long long* packed, int rows) {
  pdl_trigger();
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < rows) packed[i] = 0ull;
}

}  // namespace

cudaError_t rmsnorm_launch(const bf16* x, int ldx, const bf16* g, float eps, bf16* y, int ldy,
                           int rows, int h, cudaStream_t s) {
  if (rows <= 0) return cudaSuccess;
  if (h % 8) return cudaErrorInvalidValue;
  return launch_pdl(rmsnorm_kernel, dim3(rows), dim3(kNormThreads), 0, s, x, ldx, g, eps, y, ldy, h);
}

cudaError_t embed_launch(const bf16* E, int h, const int32_t* tokens, bf16* x, int rows,
                         cudaStream_t s) {
  if (rows <= 0) return cudaSuccess;
  return launch_pdl(embed_kernel, dim3(rows), dim3(128), 0, s, E, h, tokens, x);
}

cudaError_t argmax_finalize_launch(const unsigned long long* packed, int32_t* next,
                                   int32_t* pos_out, const int32_t* pos, int rows, cudaStream_t s) {
  if (rows <= 0) return cudaSuccess;
  return launch_pdl(argmax_finalize_kernel, dim3((rows + 255) / 256), dim3(256), 0, s, packed, next,
                    pos_out, pos, rows);
}

cudaError_t argmax_reset_launch(unsigned long long* packed, int rows, cudaStream_t s) {
  if (rows <= 0) return cudaSuccess;
  return launch_pdl(argmax_reset_kernel, dim3((rows + 255) / 256), dim3(256), 0, s, packed, rows);
}

cudaError_t norm_preload() {
  cudaFuncAttributes fa;
  cudaError_t e = cudaSuccess;
  if (cudaFuncGetAttributes(&fa, rmsnorm_kernel) != cudaSuccess) e = cudaGetLastError();
  if (cudaFuncGetAttributes(&fa, embed_kernel) != cudaSuccess) e = cudaGetLastError();
  if (cudaFuncGetAttributes(&fa, argmax_finalize_kernel) != cudaSuccess) e = cudaGetLastError();
  if (cudaFuncGetAttributes(&fa, argmax_reset_kernel) != cudaSuccess) e = cudaGetLastError();
  return e;
}

}  // namespace sidp
