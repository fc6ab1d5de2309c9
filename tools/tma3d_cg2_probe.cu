// Probe: 3-D TMA over a k-block-major [K/64][rows][64] matrix, box {64, 128, 2}, issued
// (a) plain by one CTA, (b) with .cta_group::2 from both CTAs of a pair signalling the leader's
// mbarrier.  Checks the bytes landed (standalone experiment).
#include <cstdio>
#include <vector>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>
#include "common.cuh"
using namespace sidp;
typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);
__device__ uint32_t ctarank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ uint32_t mapa(uint32_t a, uint32_t r) { uint32_t o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r)); return o; }

__global__ void plain3d(const __grid_constant__ CUtensorMap tm, unsigned short* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar, 2 * 128 * 128);
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
                 " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(smem)),
                 "l"(reinterpret_cast<uint64_t>(&tm)), "r"(0), "r"(0), "r"(2), "r"(smem_u32(&bar)) : "memory");
  }
  mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < 2 * 128 * 64; i += blockDim.x) out[i] = reinterpret_cast<unsigned short*>(smem)[i];
}

template <int DIMS>
__global__ void __cluster_dims__(2, 1, 1) cg2(const __grid_constant__ CUtensorMap tm, unsigned short* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t rank = ctarank();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x == 0) {
    const uint32_t lbar = mapa(smem_u32(&bar), 0);
    if (rank == 0) mbar_arrive_expect_tx(&bar, 2 * 2 * 128 * 128);
    if (DIMS == 3) {
      asm volatile("cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
                   " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(smem)),
                   "l"(reinterpret_cast<uint64_t>(&tm)), "r"(0), "r"((int)rank * 128), "r"(2), "r"(lbar) : "memory");
    } else {
      for (int j = 0; j < 2; ++j)
        asm volatile("cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
                     " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(smem + j * 16384)),
                     "l"(reinterpret_cast<uint64_t>(&tm)), "r"(0), "r"((2 + j) * 256 + (int)rank * 128), "r"(lbar) : "memory");
    }
  }
  if (rank == 0) mbar_wait(&bar, 0);
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  for (int i = threadIdx.x; i < 2 * 128 * 64; i += blockDim.x) out[rank * 2 * 128 * 64 + i] = reinterpret_cast<unsigned short*>(smem)[i];
}

int main() {
  void* fnp; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)fnp;
  const int rows = 256, K = 512, nkb = K / 64;
  // kb-major: element (n, k) at (k/64 * rows + n) * 64 + k%64; value tags (kb, n, c)
  std::vector<unsigned short> h(rows * K);
  for (int kb = 0; kb < nkb; ++kb) for (int n = 0; n < rows; ++n) for (int c = 0; c < 64; ++c)
    h[((size_t)kb * rows + n) * 64 + c] = (unsigned short)((kb * 4099 + n * 67 + c) & 0xFFFF);
  unsigned short *d, *o; cudaMalloc(&d, h.size() * 2); cudaMalloc(&o, 4 * 128 * 64 * 2);
  cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  CUtensorMap tm3, tm2;
  cuuint64_t dims[3] = {64, (cuuint64_t)rows, (cuuint64_t)nkb};
  cuuint64_t st[2] = {128, (cuuint64_t)rows * 128};
  cuuint32_t box[3] = {64, 128, 2}, es[3] = {1, 1, 1};
  const bool swz = getenv("SWZ") != nullptr;
  CUresult r3 = enc(&tm3, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, d, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cuuint64_t d2[2] = {64, (cuuint64_t)rows * nkb};
  cuuint64_t s2[1] = {128};
  cuuint32_t b2[2] = {64, 128}, e2[2] = {1, 1};
  CUresult r2 = enc(&tm2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, d2, s2, b2, e2, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode: 3d %d 2d %d\n", (int)r3, (int)r2);
  auto check = [&](const char* name, int nct) {
    std::vector<unsigned short> g(nct * 2 * 128 * 64);
    cudaMemcpy(g.data(), o, g.size() * 2, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int rk = 0; rk < nct; ++rk) for (int j = 0; j < 2; ++j) for (int n = 0; n < 128; ++n) for (int c = 0; c < 64; ++c) {
      const int kb = 2 + j, row = rk * 128 + n;
      if (g[((rk * 2 + j) * 128 + n) * 64 + c] != (unsigned short)((kb * 4099 + row * 67 + c) & 0xFFFF)) ++bad;
    }
    printf("%s: bad=%d\n", name, bad);
  };
  cudaFuncSetAttribute(plain3d, cudaFuncAttributeMaxDynamicSharedMemorySize, 80000);
  cudaFuncSetAttribute(cg2<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 80000);
  cudaFuncSetAttribute(cg2<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 80000);
  cudaMemset(o, 0, 4 * 128 * 64 * 2);
  cg2<2><<<2, 128, 70000>>>(tm2, o);
  printf("cg2 2d: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  check("cg2 2d", 2);
  cudaMemset(o, 0, 4 * 128 * 64 * 2);
  plain3d<<<1, 128, 70000>>>(tm3, o);
  printf("plain 3d: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  check("plain 3d", 1);
  cudaMemset(o, 0, 4 * 128 * 64 * 2);
  cg2<3><<<2, 128, 70000>>>(tm3, o);
  printf("cg2 3d: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  check("cg2 3d", 2);
  return 0;
}
