// mma_probe.cu — measure raw tcgen05.mma throughput on this B200 (standalone; not the product).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2605_28095_b200/csrc tools/mma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "common.cuh"

using namespace sidp;

__device__ __forceinline__ uint32_t ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

template <int CG, int N>
__global__ void __launch_bounds__(128, 1) probe(int iters, int commit_every, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    if (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(256));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(256));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
  }
  tc_fence_before();
  __syncthreads();
  if (CG == 2) {
    asm volatile("barrier.cluster.arrive.release.aligned;");
    asm volatile("barrier.cluster.wait.acquire.aligned;");
  }
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t M = CG == 1 ? 128 : 256;
  const uint32_t idesc = umma_idesc_bf16(M, N);
  const bool leader = CG == 1 || ctarank() == 0;
  unsigned long long t0 = clock64();
  if (warp == 1 && leader && threadIdx.x == 32) {
    const uint32_t a0 = smem_u32(smem), b0 = smem_u32(smem + 16384);
    uint32_t ph = 0;
    for (int i = 0; i < iters; ++i) {
      for (int k = 0; k < 4; ++k) {
        if (CG == 1)
          umma_bf16(tmem, umma_desc_sw128(a0 + k * 32), umma_desc_sw128(b0 + k * 32), idesc, 1);
        else
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                       ::"r"(tmem), "l"(umma_desc_sw128(a0 + k * 32)), "l"(umma_desc_sw128(b0 + k * 32)), "r"(idesc), "r"(1));
      }
      if (commit_every && (i % commit_every) == commit_every - 1) {
        if (CG == 1)
          umma_commit(&bar);
        else
          asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "h"((uint16_t)1));
        if (commit_every == 1 || true) {
          mbar_wait(&bar, ph);
          ph ^= 1;
        }
      }
    }
    if (CG == 1)
      umma_commit(&bar);
    else
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "h"((uint16_t)1));
    mbar_wait(&bar, ph);
    out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (CG == 2) {
    asm volatile("barrier.cluster.arrive.release.aligned;");
    asm volatile("barrier.cluster.wait.acquire.aligned;");
  }
  if (warp == 0) {
    tc_fence_after();
    if (CG == 1)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
  }
}

template <int CG, int N>
void run(const char* name, int commit_every) {
  int iters = 4096;
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  cudaMemset(d, 0, 148 * 8);
  auto k = probe<CG, N>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = 100 * 1024;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CG;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaLaunchKernelEx(&cfg, k, iters, commit_every, d);
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, k, iters, commit_every, d);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  unsigned long long cyc = 0;
  for (int i = 0; i < 148; ++i) cyc = h[i] > cyc ? h[i] : cyc;
  const double macs_per_sm = (double)iters * 4 * (CG == 1 ? 128 : 128) * N * 16;
  const double flops = 2.0 * macs_per_sm * 148;
  printf("%-28s commit/%d: %s  %.3f ms  %.1f TFLOP/s  cycles/mma-per-SM=%.1f  (%.0f MHz eff)\n", name,
         commit_every, cudaGetErrorString(err), ms, flops / ms / 1e9, (double)cyc / (iters * 4),
         (double)cyc / (ms * 1e3));
}

// Ring mode: the GEMM mainloop's MMA side without loads — S stages, each 8 MMAs (two 64-deep
// k-blocks) then a commit to that stage's barrier; stage i waits for the commit of stage i - S.
template <int N, int S, bool MOVE = false>
__global__ void __launch_bounds__(128, 1) ring_probe(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bars[S];
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) mbar_init(&bars[i], 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;");
  asm volatile("barrier.cluster.wait.acquire.aligned;");
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t idesc = umma_idesc_bf16(256, N);
  const bool leader = ctarank() == 0;
  unsigned long long t0 = clock64();
  if (warp == 1 && leader && threadIdx.x == 32) {
    for (int i = 0; i < iters; ++i) {
      const int st = i % S;
      // MOVE: every stage reads its own 50 KB operand buffers (as the GEMM's ring does)
      const uint32_t a0 = smem_u32(smem) + (MOVE ? (uint32_t)(st % 4) * 51200u : 0u);
      const uint32_t b0 = a0 + 32768;
      if (i >= S) mbar_wait(&bars[st], ((i / S) - 1) & 1);
      tc_fence_after();
      for (int j = 0; j < 2; ++j)
        for (int k = 0; k < 4; ++k)
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                       ::"r"(tmem), "l"(umma_desc_sw128(a0 + j * 16384 + k * 32)), "l"(umma_desc_sw128(b0 + j * 16384 + k * 32)), "r"(idesc), "r"(1));
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(smem_u32(&bars[st])), "h"((uint16_t)1));
    }
    for (int i = iters; i < iters + S; ++i) {
      const int st = i % S;
      mbar_wait(&bars[st], ((i / S) - 1) & 1);
    }
    out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;");
  asm volatile("barrier.cluster.wait.acquire.aligned;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

template <int N, int S, bool MOVE = false>
void run_ring(const char* name) {
  unsigned long long* d;
  cudaMalloc(&d, 148 * sizeof(unsigned long long));
  auto k = ring_probe<N, S, MOVE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = 210 * 1024;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const int iters = 2048;
  cudaLaunchKernelEx(&cfg, k, iters, d);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, k, iters, d);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  unsigned long long cyc = 0;
  for (int i = 0; i < 148; ++i) cyc = h[i] > cyc ? h[i] : cyc;
  printf("%-34s %s  %.3f ms  cycles per 8-MMA stage=%.1f (floor %d)\n", name, cudaGetErrorString(err), ms,
         (double)cyc / iters, 8 * 128 * N / 512);
}

int main() {
  run<1, 256>("1-CTA M=128 N=256", 0);
  run<1, 256>("1-CTA M=128 N=256", 1);
  run<2, 256>("2-CTA M=256 N=256", 0);
  run<2, 256>("2-CTA M=256 N=256", 1);
  run<2, 256>("2-CTA M=256 N=256", 4);
  run<2, 128>("2-CTA M=256 N=128", 0);
  run<2, 144>("2-CTA M=256 N=144", 0);
  run<2, 144>("2-CTA M=256 N=144", 2);
  run<2, 144>("2-CTA M=256 N=144", 8);
  run<2, 256>("2-CTA M=256 N=256", 8);
  run_ring<144, 4>("ring N=144 S=4");
  run_ring<144, 2>("ring N=144 S=2");
  run_ring<144, 8>("ring N=144 S=8");
  run_ring<256, 4>("ring N=256 S=4");
  run_ring<144, 4, true>("ring N=144 S=4 moving buffers");
  run<1, 128>("1-CTA M=128 N=128", 0);
  return 0;
}
