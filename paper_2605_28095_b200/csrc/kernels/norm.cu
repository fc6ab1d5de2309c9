// norm.cu — RMSNorm, embedding gather, argmax finalisation.
// HBM-bound row kernels: 16-byte vector loads, fp32 statistics, one bf16 rounding.
#include <algorithm>
#include <cstdlib>

#include "../common.cuh"
#include "../fixup.cuh"
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

// CaS requester, round trip 1 (see cas_send_norm_launch): the rmsnorm_kernel arithmetic with the
// row's u and x stored into the owner's staging row [u | x] (a peer VA), then the last CTA to
// finish posts the arrival flag with release semantics at system scope.
__global__ void __launch_bounds__(kNormThreads) cas_send_norm_kernel(const CasSendArgs a) {
  pdl_trigger();
  pdl_wait();
  if (a.wait.n) {   // the owner served its previous round trip: its staging slots are free
    if (threadIdx.x == 0) flags_wait(a.wait.p, a.wait.n, a.wait.value, a.wait.timeout_ns, a.wait.err, a.wait.base);
    __syncthreads();
  }
  const int h = a.h, nvec = h / 8;
  const bool cached = nvec <= kNormThreads * kVec;
  for (int row = blockIdx.x; row < a.rows; row += gridDim.x) {
    const bf16* xr = a.x + (size_t)row * a.ldx;
    bf16* ur = a.dst + (size_t)row * a.ldd;
    bf16* xd = ur + h;
    // the row read once (kept in registers, as rmsnorm_kernel; same summation order, so u is
    // bitwise the replicated path's) and forwarded to the owner while the statistics reduce
    uint4 v[kVec];
    float ss = 0.0f;
    auto acc = [&](const uint4& raw) {
      const bf16* e = reinterpret_cast<const bf16*>(&raw);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float f = bf16_to_f(e[q]);
        ss += f * f;
      }
    };
    if (cached) {
#pragma unroll
      for (int i = 0; i < kVec; ++i) {
        const int k = threadIdx.x + i * kNormThreads;
        v[i] = k < nvec ? *reinterpret_cast<const uint4*>(xr + k * 8) : make_uint4(0u, 0u, 0u, 0u);
      }
#pragma unroll
      for (int i = 0; i < kVec; ++i) {
        const int k = threadIdx.x + i * kNormThreads;
        if (k < nvec) *reinterpret_cast<uint4*>(xd + k * 8) = v[i];
        acc(v[i]);
      }
    } else {
      for (int k = threadIdx.x; k < nvec; k += kNormThreads) {
        const uint4 raw = *reinterpret_cast<const uint4*>(xr + k * 8);
        *reinterpret_cast<uint4*>(xd + k * 8) = raw;
        acc(raw);
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
    const float r = rsqrtf(red[0] / (float)h + a.eps);
    auto scale = [&](const uint4& raw, int k) {
      const uint4 graw = *reinterpret_cast<const uint4*>(a.g + k * 8);
      const bf16* e = reinterpret_cast<const bf16*>(&raw);
      const bf16* ge = reinterpret_cast<const bf16*>(&graw);
      uint4 out;
      bf16* o = reinterpret_cast<bf16*>(&out);
#pragma unroll
      for (int q = 0; q < 8; ++q) o[q] = f_to_bf16(bf16_to_f(e[q]) * r * bf16_to_f(ge[q]));
      *reinterpret_cast<uint4*>(ur + k * 8) = out;
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
    __syncthreads();   // red[] reused by the next row
  }
  __syncthreads();
  if (threadIdx.x == 0) {   // the CTA counted in with an acq_rel gpu-scope atomic
    const unsigned prev = atom_add_acq_rel_gpu(a.counter, 1u);
    if (prev == gridDim.x - 1) {
      *a.counter = 0u;
      st_release_sys(a.arrive, flag_value(a.value, a.base));
    }
  }
}

// Deferred stream-K fix-up + residual + RMSNorm, one CTA per row (see resid_norm_launch), one
// thread per 8-feature vector (h <= 8 * 640; longer rows loop).  Per vector the fp32 partial
// slices of its tile are summed in slice order, the bf16 residual added in fp32 and the sum
// rounded once to bf16 (x_out, the residual stream); the norm statistics use the rounded
// x_out, exactly as rmsnorm_kernel on a stored x_out.  The slice loads of a vector are issued
// together (unrolled, predicated): the kernel is bound by their L2 round trips otherwise.
// Deferred stream-K fix-up + residual + RMSNorm (see resid_norm_launch): the rows are walked by
// a grid of at most one CTA per SM (fits beside the next kernel's early-launched PDL CTAs); one
// thread per 8-feature vector.  When every thread holds one vector (h <= 8 x blockDim) the
// slices, residual and gain of a row are all loaded in ONE round trip and x stays in registers
// for the scaling pass; the norm statistics use the rounded x_out, exactly as rmsnorm_kernel
// would on a stored x_out.  Longer rows take the looped path (re-reads its own x_out).
template <int NS, int MAXT>
__global__ void __launch_bounds__(MAXT, 1) resid_norm_kernel(
    const PartialSrc ps, const bf16* __restrict__ resid, int ldr, bf16* xout, int ldx,
    const bf16* __restrict__ g, float eps, bf16* __restrict__ u, int ldu, int h, int rows,
    int late_trigger, unsigned long long* post) {
  if (!late_trigger) pdl_trigger();
  pdl_wait();
  if (post && blockIdx.x == 0 && threadIdx.x == 0) {
    // WaS slot release (kernels/ring.cu): the predecessor — the last reader of the slot's
    // weights — has completed, so the fetch stream may refill the slot
    __threadfence();
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(post) : "memory");
  }
  const int nvec = h / 8;
  const size_t slice = (size_t)ps.M * ps.N;
  const bool one = nvec <= (int)blockDim.x;
  __shared__ float red[32];
  auto block_sum = [&](float v) {
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
      float t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0f;
      t = warp_sum(t);
      if (threadIdx.x == 0) red[0] = t;
    }
    __syncthreads();
    const float tot = red[0];
    __syncthreads();   // red is reused by the next row
    return tot;
  };
  for (int row = blockIdx.x; row < rows; row += gridDim.x) {
    const float* wrow = ps.ws + (size_t)row * ps.N;
    if (one) {
      const int k = threadIdx.x, n = k * 8;
      uint4 x = make_uint4(0u, 0u, 0u, 0u), gw = x;
      if (k < nvec) {
        gw = *reinterpret_cast<const uint4*>(g + n);
        const uint4 rr = *reinterpret_cast<const uint4*>(resid + (size_t)row * ldr + n);
        x = fix_vector<NS>(ps, wrow + n, slice, ps.nseg[partial_tile(ps, row, n)], rr);
        *reinterpret_cast<uint4*>(xout + (size_t)row * ldx + n) = x;
      }
      const float r = rsqrtf(block_sum(k < nvec ? sumsq8(x) : 0.0f) / (float)h + eps);
      if (k < nvec) *reinterpret_cast<uint4*>(u + (size_t)row * ldu + n) = scale8(x, gw, r);
    } else {
      float ss = 0.0f;
      for (int k = threadIdx.x; k < nvec; k += blockDim.x) {
        const int n = k * 8;
        const uint4 rr = *reinterpret_cast<const uint4*>(resid + (size_t)row * ldr + n);
        const uint4 x = fix_vector<NS>(ps, wrow + n, slice, ps.nseg[partial_tile(ps, row, n)], rr);
        *reinterpret_cast<uint4*>(xout + (size_t)row * ldx + n) = x;
        ss += sumsq8(x);
      }
      const float r = rsqrtf(block_sum(ss) / (float)h + eps);
      for (int k = threadIdx.x; k < nvec; k += blockDim.x) {
        const int n = k * 8;
        *reinterpret_cast<uint4*>(u + (size_t)row * ldu + n) =
            scale8(*reinterpret_cast<const uint4*>(xout + (size_t)row * ldx + n),
                   *reinterpret_cast<const uint4*>(g + n), r);
      }
    }
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

cudaError_t cas_send_norm_launch(const CasSendArgs& a, cudaStream_t s) {
  if (a.rows <= 0) return cudaSuccess;
  if ((a.h & 7) || !a.counter || !a.arrive || a.wait.n > 16) return cudaErrorInvalidValue;
  return launch_pdl(cas_send_norm_kernel, dim3(std::min(a.rows, 148)), dim3(kNormThreads), 0, s, a);
}

cudaError_t resid_norm_launch(const PartialSrc& ps, const bf16* resid, int ldr, bf16* xout, int ldx,
                              const bf16* g, float eps, bf16* u, int ldu, int rows, int h,
                              cudaStream_t s, unsigned long long* post) {
  if (rows <= 0) return cudaSuccess;
  if (h % 8 || ps.ws == nullptr || ps.N != h || rows > ps.M) return cudaErrorInvalidValue;
  const int threads = std::min(1024, (h / 8 + 31) / 32 * 32);
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  // SIDP_FIX_GRID: 0 = one CTA per row; else <= 1 per SM walking rows (default: measured M2
  // 29.22 vs 29.36 ms/step over 3 A/B pairs once qkv_post ran in one wave; r1 had it 0.1 ms slower)
  static const int grid_mode = getenv("SIDP_FIX_GRID") ? atoi(getenv("SIDP_FIX_GRID")) : 1;
  static const int late = getenv("SIDP_FIX_LATE_TRIGGER") ? atoi(getenv("SIDP_FIX_LATE_TRIGGER")) : 0;
  const int grid = grid_mode ? std::min(rows, sms) : rows;
  // slices loaded in one round trip: up to 8 per vector (640-thread rows, 96 registers) when the
  // producer split tiles into more than 4 segments (the fused MLP's down units); else 4
  int max_seg = 0;
  const int tiles = ps.m_tiles * ps.f_tiles;
  for (int t = 0; t < tiles && t < kPartialMaxTiles; ++t) max_seg = std::max(max_seg, (int)ps.nseg[t]);
  static const int env_ns = getenv("SIDP_FIX_NS") ? atoi(getenv("SIDP_FIX_NS")) : 0;
  const bool wide = env_ns ? env_ns == 8 : max_seg > 4;
  if (wide && threads <= 640)
    return launch_pdl(resid_norm_kernel<8, 640>, dim3(grid), dim3(threads), 0, s, ps, resid, ldr,
                      xout, ldx, g, eps, u, ldu, h, rows, late, post);
  return launch_pdl(resid_norm_kernel<kFixSeg, 1024>, dim3(grid), dim3(threads), 0, s, ps, resid,
                    ldr, xout, ldx, g, eps, u, ldu, h, rows, late, post);
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
  if (cudaFuncGetAttributes(&fa, cas_send_norm_kernel) != cudaSuccess) e = cudaGetLastError();
  if (cudaFuncGetAttributes(&fa, embed_kernel) != cudaSuccess) e = cudaGetLastError();
  if (cudaFuncGetAttributes(&fa, resid_norm_kernel<8, 640>) != cudaSuccess) e = cudaGetLastError();
  if (cudaFuncGetAttributes(&fa, resid_norm_kernel<kFixSeg, 1024>) != cudaSuccess) e = cudaGetLastError();
  if (cudaFuncGetAttributes(&fa, argmax_finalize_kernel) != cudaSuccess) e = cudaGetLastError();
  if (cudaFuncGetAttributes(&fa, argmax_reset_kernel) != cudaSuccess) e = cudaGetLastError();
  return e;
}

}  // namespace sidp
