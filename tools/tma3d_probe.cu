// Probe: does a 3-D TMA box over a row-major matrix viewed as {64, rows, K/64} with strides
// {ld, 128 B} (non-monotonic) load correctly?  (standalone experiment)
#include <cstdio>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>
#include "common.cuh"
using namespace sidp;
typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);
__global__ void k3(const __grid_constant__ CUtensorMap tm, unsigned short* out, int swz) {
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
int main() {
  void* fnp; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)fnp;
  const int rows = 256, K = 512;
  std::vector<unsigned short> h(rows * K);
  for (int r = 0; r < rows; ++r) for (int c = 0; c < K; ++c) h[r * K + c] = (unsigned short)((r * 7 + c) & 0xFFFF);
  unsigned short *d, *o; cudaMalloc(&d, h.size() * 2); cudaMalloc(&o, 2 * 128 * 64 * 2);
  cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  for (int swz = 0; swz < 2; ++swz) {
    CUtensorMap tm;
    cuuint64_t dims[3] = {64, (cuuint64_t)rows, (cuuint64_t)K / 64};
    cuuint64_t st[2] = {(cuuint64_t)K * 2, 128};
    cuuint32_t box[3] = {64, 128, 2}, es[3] = {1, 1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, d, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaFuncSetAttribute(k3, cudaFuncAttributeMaxDynamicSharedMemorySize, 80000);
    k3<<<1, 128, 70000>>>(tm, o, swz);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<unsigned short> g(2 * 128 * 64);
    cudaMemcpy(g.data(), o, g.size() * 2, cudaMemcpyDeviceToHost);
    int bad = 0;
    if (!swz) for (int j = 0; j < 2; ++j) for (int r2 = 0; r2 < 128; ++r2) for (int c = 0; c < 64; ++c)
      if (g[(j * 128 + r2) * 64 + c] != h[r2 * K + (2 + j) * 64 + c]) ++bad;
    printf("swizzle=%d encode=%d kernel=%s mismatches(no-swz check)=%d first=%u expect=%u\n", swz, (int)r,
           cudaGetErrorString(e), bad, g[0], h[2 * 64]);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
