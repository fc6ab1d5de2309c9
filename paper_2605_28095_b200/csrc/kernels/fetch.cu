// fetch.cu — K1 remote-weight fetch and the CaS signalling kernels.
//
// WaS fetch ("non-owner issues non-blocking device-to-device copies from
// r(l)'s HBM into its local cache"): a verbatim copy of one packed pooled layer from the
// owner's arena (a peer VA imported over CUDA IPC, NVLink/NVSwitch) into a local slot.
// SM-issued, coalesced 16-byte loads with 8 loads in flight per thread before the stores
// (L1::no_allocate: streamed once), on a bounded number of CTAs so the concurrently
// running GEMMs keep the rest of the SMs.
#include <algorithm>

#include "../common.cuh"
#include "../kernels.h"

namespace sidp {

namespace {

__device__ __forceinline__ uint4 ld_nc_v4(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st_na_v4(uint4* p, const uint4& v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// ns_per_iter > 0 paces the copy: iteration `it` (U x grid x T x 16 B) starts no earlier than
// it x ns_per_iter after the CTA's start (NVLink-rate emulation on one GPU).
template <int T, int U>
__global__ void __launch_bounds__(T) fetch_kernel(uint4* __restrict__ dst,
                                                  const uint4* __restrict__ src, size_t nvec,
                                                  uint64_t ns_per_iter) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t t0 = ns_per_iter ? globaltimer_ns() : 0;
  uint64_t it = 0;
  for (; i + (U - 1) * stride < nvec; i += U * stride, ++it) {
    if (ns_per_iter)
      while (globaltimer_ns() - t0 < it * ns_per_iter) __nanosleep(200);
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ld_nc_v4(src + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) st_na_v4(dst + i + u * stride, v[u]);
  }
  for (; i < nvec; i += stride) st_na_v4(dst + i, ld_nc_v4(src + i));
}

// Pacing of a copy-engine fetch (NVLink-rate emulation): chunk 0 stamps the start time,
// chunk i waits until offset_ns after it.
__global__ void pace_kernel(unsigned long long* t0, int first, uint64_t offset_ns) {
  if (first) {
    *reinterpret_cast<volatile unsigned long long*>(t0) = globaltimer_ns();
    return;
  }
  const unsigned long long start = *reinterpret_cast<volatile unsigned long long*>(t0);
  while (globaltimer_ns() - start < offset_ns) __nanosleep(500);
}

__global__ void delay_kernel(uint64_t ns) {
  const uint64_t t0 = globaltimer_ns();
  while (globaltimer_ns() - t0 < ns) {
  }
}

// Post a flag after all prior work of this stream (kernel boundary orders the data).
__global__ void signal_kernel(uint64_t* flag, uint64_t value, const uint64_t* base) {
  // the stream's earlier kernels completed: their stores performed
  st_release_sys(flag, flag_value(value, base));
}

__global__ void base_add_kernel(uint64_t* base, uint64_t delta) { *base += delta; }

// Wait until every flag >= value (system-scope acquire); bounded by timeout_ns, after
// which *err is set and the kernel returns (surfaced as SIDP_ETIMEOUT by the host).
__global__ void wait_kernel(const FlagSet flags, uint64_t value, uint64_t timeout_ns, int* err,
                            const uint64_t* base) {
  value = flag_value(value, base);
  const int i = threadIdx.x;
  if (i < flags.n) {
    const uint64_t t0 = globaltimer_ns();
    while (ld_acquire_sys(flags.p[i]) < value) {
      if (globaltimer_ns() - t0 > timeout_ns) {
        *reinterpret_cast<volatile int*>(err) = 1;   // mapped host word (read without a sync)
        __threadfence_system();
        break;
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
}

__global__ void copy_rows_kernel(uint8_t* dst, int ldd, const uint8_t* src, int lds, int rows,
                                 int row_bytes) {
  const int nvec = row_bytes / 16;
  for (int r = blockIdx.y; r < rows; r += gridDim.y) {
    const uint4* s = reinterpret_cast<const uint4*>(src + (size_t)r * lds);
    uint4* d = reinterpret_cast<uint4*>(dst + (size_t)r * ldd);
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < nvec; v += gridDim.x * blockDim.x)
      d[v] = s[v];
  }
}

// every CTA waits for the flags (thread 0, acquire), then copies its rows
__global__ void wait_copy_kernel(const FlagWait w, uint8_t* dst, int ldd, const uint8_t* src,
                                 int lds, int rows, int row_bytes) {
  if (threadIdx.x == 0) flags_wait(w.p, w.n, w.value, w.timeout_ns, w.err, w.base);
  __syncthreads();
  const int nvec = row_bytes / 16;
  for (int r = blockIdx.y; r < rows; r += gridDim.y) {
    const uint4* s = reinterpret_cast<const uint4*>(src + (size_t)r * lds);
    uint4* d = reinterpret_cast<uint4*>(dst + (size_t)r * ldd);
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < nvec; v += gridDim.x * blockDim.x)
      d[v] = __ldcg(s + v);
  }
}

}  // namespace

cudaError_t wait_copy_launch(const FlagWait& w, void* dst, int ldd, const void* src, int lds,
                             int rows, int row_bytes, cudaStream_t s) {
  if (rows <= 0 || row_bytes <= 0) return cudaSuccess;
  if (row_bytes % 16 || w.n > 16) return cudaErrorInvalidValue;
  dim3 grid((row_bytes / 16 + 255) / 256, rows < 1024 ? rows : 1024);
  wait_copy_kernel<<<grid, 256, 0, s>>>(w, reinterpret_cast<uint8_t*>(dst), ldd,
                                        reinterpret_cast<const uint8_t*>(src), lds, rows, row_bytes);
  return cudaGetLastError();
}

cudaError_t fetch_launch(void* dst, const void* src, size_t bytes, int ctas, cudaStream_t s,
                         float pace_gbps) {
  if (bytes == 0) return cudaSuccess;
  if ((bytes & 15) || (reinterpret_cast<uintptr_t>(dst) & 15) ||
      (reinterpret_cast<uintptr_t>(src) & 15))
    return cudaErrorInvalidValue;
  if (ctas <= 0) ctas = 32;
  // threads x loads in flight per thread (SIDP_LDG_CFG: 0 = 512 x 8, 1 = 1024 x 8, 2 = 256 x 16,
  // 3 = 1024 x 4) — per-SM copy-rate probes
  static const int cfg = getenv("SIDP_LDG_CFG") ? atoi(getenv("SIDP_LDG_CFG")) : 0;
  const int T = cfg == 1 || cfg == 3 ? 1024 : cfg == 2 ? 256 : 512;
  const int U = cfg == 2 ? 16 : cfg == 3 ? 4 : 8;
  // bytes per iteration of all CTAs / (GB/s == bytes per ns)
  const uint64_t ns_per_iter =
      pace_gbps > 0.0f ? (uint64_t)((double)U * ctas * T * 16 / pace_gbps) : 0;
  uint4* d = reinterpret_cast<uint4*>(dst);
  const uint4* sp = reinterpret_cast<const uint4*>(src);
  if (cfg == 1) fetch_kernel<1024, 8><<<ctas, 1024, 0, s>>>(d, sp, bytes / 16, ns_per_iter);
  else if (cfg == 2) fetch_kernel<256, 16><<<ctas, 256, 0, s>>>(d, sp, bytes / 16, ns_per_iter);
  else if (cfg == 3) fetch_kernel<1024, 4><<<ctas, 1024, 0, s>>>(d, sp, bytes / 16, ns_per_iter);
  else fetch_kernel<512, 8><<<ctas, 512, 0, s>>>(d, sp, bytes / 16, ns_per_iter);
  return cudaGetLastError();
}

cudaError_t pace_launch(unsigned long long* t0, int first, uint64_t offset_ns, cudaStream_t s) {
  pace_kernel<<<1, 32, 0, s>>>(t0, first, offset_ns);
  return cudaGetLastError();
}

cudaError_t delay_launch(uint64_t ns, cudaStream_t s) {
  if (ns == 0) return cudaSuccess;
  delay_kernel<<<1, 32, 0, s>>>(ns);
  return cudaGetLastError();
}

cudaError_t signal_launch(uint64_t* flag, uint64_t value, cudaStream_t s, const uint64_t* base) {
  signal_kernel<<<1, 1, 0, s>>>(flag, value, base);
  return cudaGetLastError();
}

cudaError_t base_add_launch(uint64_t* base, uint64_t delta, cudaStream_t s) {
  base_add_kernel<<<1, 1, 0, s>>>(base, delta);
  return cudaGetLastError();
}

cudaError_t wait_launch(const FlagSet& flags, uint64_t value, uint64_t timeout_ns, int* err,
                        cudaStream_t s, const uint64_t* base) {
  if (flags.n <= 0) return cudaSuccess;
  if (flags.n > 16) return cudaErrorInvalidValue;
  wait_kernel<<<1, 32, 0, s>>>(flags, value, timeout_ns, err, base);
  return cudaGetLastError();
}

cudaError_t copy_rows_launch(void* dst, int ldd, const void* src, int lds, int rows, int row_bytes,
                             cudaStream_t s) {
  if (rows <= 0 || row_bytes <= 0) return cudaSuccess;
  if (row_bytes % 16) return cudaErrorInvalidValue;
  dim3 grid((row_bytes / 16 + 255) / 256, rows < 1024 ? rows : 1024);
  copy_rows_kernel<<<grid, 256, 0, s>>>(reinterpret_cast<uint8_t*>(dst), ldd,
                                        reinterpret_cast<const uint8_t*>(src), lds, rows,
                                        row_bytes);
  return cudaGetLastError();
}

// grid-strided over each job's 16-byte vectors, 4 loads in flight per thread; then each CTA's
// thread 0 counts the CTA in with an acq_rel gpu-scope atomic (after the CTA barrier) and the
// last CTA to arrive publishes the flags with release stores (no fence.sc.sys: ~5 us each)
__global__ void __launch_bounds__(256) xfer_kernel(const XferSet x) {
  const int gt = blockIdx.x * blockDim.x + threadIdx.x, gs = gridDim.x * blockDim.x;
  for (int j = 0; j < x.njobs; ++j) {
    const XferJob& jb = x.job[j];
    const int nvec = jb.row_bytes / 16;
    const long long total = (long long)jb.rows * nvec;
    auto src_of = [&](long long i) {
      const int r = (int)(i / nvec), v = (int)(i % nvec);
      return reinterpret_cast<const uint4*>(reinterpret_cast<const uint8_t*>(jb.src) + (size_t)r * jb.lds) + v;
    };
    auto dst_of = [&](long long i) {
      const int r = (int)(i / nvec), v = (int)(i % nvec);
      return reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(jb.dst) + (size_t)r * jb.ldd) + v;
    };
    long long i = gt;
    for (; i + 3LL * gs < total; i += 4LL * gs) {
      uint4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldcg(src_of(i + u * (long long)gs));
#pragma unroll
      for (int u = 0; u < 4; ++u) *dst_of(i + u * (long long)gs) = v[u];
    }
    for (; i < total; i += gs) *dst_of(i) = __ldcg(src_of(i));
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned prev = atom_add_acq_rel_gpu(x.counter, 1u);
    if (prev == gridDim.x - 1) {
      *x.counter = 0u;
      for (int f = 0; f < x.nflags; ++f) st_release_sys(x.flag[f], x.value);
    }
  }
}

cudaError_t xfer_launch(const XferSet& x, cudaStream_t s) {
  if (x.njobs < 0 || x.njobs > 16 || x.nflags < 0 || x.nflags > 18 || !x.counter)
    return cudaErrorInvalidValue;
  long long vecs = 0;
  for (int j = 0; j < x.njobs; ++j) {
    if (x.job[j].row_bytes % 16) return cudaErrorInvalidValue;
    vecs = std::max<long long>(vecs, (long long)x.job[j].rows * (x.job[j].row_bytes / 16));
  }
  const int grid = (int)std::max<long long>(1, std::min<long long>(148, (vecs + 1023) / 1024));
  xfer_kernel<<<grid, 256, 0, s>>>(x);
  return cudaGetLastError();
}

cudaError_t fetch_preload() {
  cudaFuncAttributes fa;
  cudaError_t e = cudaSuccess;
  if (cudaFuncGetAttributes(&fa, fetch_kernel<512, 8>) != cudaSuccess) e = cudaGetLastError();
  if (cudaFuncGetAttributes(&fa, delay_kernel) != cudaSuccess) e = cudaGetLastError();
  if (cudaFuncGetAttributes(&fa, pace_kernel) != cudaSuccess) e = cudaGetLastError();
  if (cudaFuncGetAttributes(&fa, signal_kernel) != cudaSuccess) e = cudaGetLastError();
  if (cudaFuncGetAttributes(&fa, wait_kernel) != cudaSuccess) e = cudaGetLastError();
  if (cudaFuncGetAttributes(&fa, base_add_kernel) != cudaSuccess) e = cudaGetLastError();
  if (cudaFuncGetAttributes(&fa, copy_rows_kernel) != cudaSuccess) e = cudaGetLastError();
  if (cudaFuncGetAttributes(&fa, xfer_kernel) != cudaSuccess) e = cudaGetLastError();
  if (cudaFuncGetAttributes(&fa, wait_copy_kernel) != cudaSuccess) e = cudaGetLastError();
  return e;
}

}  // namespace sidp
