// norm.cu — RMSNorm, embedding gather, argmax finalisation.
// HBM-bound row kernels: 16-byte vector loads, fp32 statistics, one bf16 rounding.
#include <algorithm>
#include <cstdlib>

#include "../common.cuh"
#include "../kernels.h"

namespace sidp {

namespace {

__device__ __forceinline__ float2 bf16x2_to_f2(uint32_t w) {
  __nv_bfloat162 h;
  memcpy(&h, &w, 4);
  return __bfloat1622float2(h);
}
__device__ __forceinline__ uint32_t f2_to_bf16x2(float a, float b) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  uint32_t w;
  memcpy(&w, &h, 4);
  return w;
}

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

// Deferred stream-K fix-up + residual + RMSNorm, one CTA per row (see resid_norm_launch), one
// thread per 8-feature vector (h <= 8 * 640; longer rows loop).  Per vector the fp32 partial
// slices of its tile are summed in slice order, the bf16 residual added in fp32 and the sum
// rounded once to bf16 (x_out, the residual stream); the norm statistics use the rounded
// x_out, exactly as rmsnorm_kernel on a stored x_out.  The slice loads of a vector are issued
// together (unrolled, predicated): the kernel is bound by their L2 round trips otherwise.
constexpr int kFixSeg = 4;
__global__ void __launch_bounds__(640, 2) resid_norm_kernel(
    const PartialSrc ps, const bf16* __restrict__ resid, int ldr, bf16* xout, int ldx,
    const bf16* __restrict__ g, float eps, bf16* __restrict__ u, int ldu, int h, int rows,
    int late_trigger) {
  if (!late_trigger) pdl_trigger();
  pdl_wait();
  const int nvec = h / 8;
  const size_t slice = (size_t)ps.M * ps.N;
  __shared__ float red[32];
  // rows are walked by a grid of at most one CTA per SM, so the CTAs fit beside the next
  // kernel's early-launched (PDL) CTAs instead of queueing behind them
  for (int row = blockIdx.x; row < rows; row += gridDim.x) {
  const float* wrow = ps.ws + (size_t)row * ps.N;
  float ss = 0.0f;
  for (int k = threadIdx.x; k < nvec; k += blockDim.x) {
    const int n = k * 8;
    const int nseg = ps.nseg[partial_tile(ps, row, n)];
    const float* src = wrow + n;
    const uint4 rr = *reinterpret_cast<const uint4*>(resid + (size_t)row * ldr + n);
    float4 lo[kFixSeg], hi[kFixSeg];
#pragma unroll
    for (int q = 0; q < kFixSeg; ++q) {
      lo[q] = hi[q] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (q < nseg) {
        lo[q] = __ldcg(reinterpret_cast<const float4*>(src + q * slice));
        hi[q] = __ldcg(reinterpret_cast<const float4*>(src + q * slice + 4));
      }
    }
    float4 al = make_float4(0.f, 0.f, 0.f, 0.f), ah = al;
#pragma unroll
    for (int q = 0; q < kFixSeg; ++q) {   // slice order; slices past nseg add +0
      al.x += lo[q].x; al.y += lo[q].y; al.z += lo[q].z; al.w += lo[q].w;
      ah.x += hi[q].x; ah.y += hi[q].y; ah.z += hi[q].z; ah.w += hi[q].w;
    }
    for (int q = kFixSeg; q < nseg; ++q) {
      const float4 x0 = __ldcg(reinterpret_cast<const float4*>(src + q * slice));
      const float4 x1 = __ldcg(reinterpret_cast<const float4*>(src + q * slice + 4));
      al.x += x0.x; al.y += x0.y; al.z += x0.z; al.w += x0.w;
      ah.x += x1.x; ah.y += x1.y; ah.z += x1.z; ah.w += x1.w;
    }
    const float2 r0 = bf16x2_to_f2(rr.x), r1 = bf16x2_to_f2(rr.y), r2 = bf16x2_to_f2(rr.z),
                 r3 = bf16x2_to_f2(rr.w);
    const uint4 out = make_uint4(f2_to_bf16x2(al.x + r0.x, al.y + r0.y), f2_to_bf16x2(al.z + r1.x, al.w + r1.y),
                                 f2_to_bf16x2(ah.x + r2.x, ah.y + r2.y), f2_to_bf16x2(ah.z + r3.x, ah.w + r3.y));
    *reinterpret_cast<uint4*>(xout + (size_t)row * ldx + n) = out;
    const float2 o0 = bf16x2_to_f2(out.x), o1 = bf16x2_to_f2(out.y), o2 = bf16x2_to_f2(out.z),
                 o3 = bf16x2_to_f2(out.w);
    ss += o0.x * o0.x + o0.y * o0.y + o1.x * o1.x + o1.y * o1.y + o2.x * o2.x + o2.y * o2.y +
          o3.x * o3.x + o3.y * o3.y;
  }
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0f;
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
    *reinterpret_cast<uint4*>(u + (size_t)row * ldu + k * 8) = out;
  };
  // re-read this thread's own x_out vectors (L1/L2 hits)
  for (int k = threadIdx.x; k < nvec; k += blockDim.x)
    scale(*reinterpret_cast<const uint4*>(xout + (size_t)row * ldx + k * 8), k);
  __syncthreads();   // red is reused by the next row
  }
  if (late_trigger) pdl_trigger();
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

cudaError_t resid_norm_launch(const PartialSrc& ps, const bf16* resid, int ldr, bf16* xout, int ldx,
                              const bf16* g, float eps, bf16* u, int ldu, int rows, int h,
                              cudaStream_t s) {
  if (rows <= 0) return cudaSuccess;
  if (h % 8 || ps.ws == nullptr || ps.N != h || rows > ps.M) return cudaErrorInvalidValue;
  const int threads = std::min(640, (h / 8 + 31) / 32 * 32);
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  // SIDP_FIX_GRID: 0 = one CTA per row; else at most one CTA per SM (default)
  static const int grid_mode = getenv("SIDP_FIX_GRID") ? atoi(getenv("SIDP_FIX_GRID")) : 1;
  static const int late = getenv("SIDP_FIX_LATE_TRIGGER") ? atoi(getenv("SIDP_FIX_LATE_TRIGGER")) : 0;
  const int grid = grid_mode ? std::min(rows, sms) : rows;
  return launch_pdl(resid_norm_kernel, dim3(grid), dim3(threads), 0, s, ps, resid, ldr, xout, ldx,
                    g, eps, u, ldu, h, rows, late);
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
  if (cudaFuncGetAttributes(&fa, resid_norm_kernel) != cudaSuccess) e = cudaGetLastError();
  if (cudaFuncGetAttributes(&fa, argmax_finalize_kernel) != cudaSuccess) e = cudaGetLastError();
  if (cudaFuncGetAttributes(&fa, argmax_reset_kernel) != cudaSuccess) e = cudaGetLastError();
  return e;
}

}  // namespace sidp
