// tma_probe.cu — W-streaming bandwidth of TMA boxes from a row-major [N x K] bf16 matrix vs a
// tile-contiguous layout (standalone experiment, not the product).
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>

#include "common.cuh"

using namespace sidp;

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);

template <int DIMS>
__global__ void __launch_bounds__(64, 1) stream_kernel(const __grid_constant__ CUtensorMap tm, int n_tiles,
                                                      int kblocks, int stages) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * 16384);
  uint64_t* empty = full + stages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int it = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x)
      for (int kb = 0; kb < kblocks; ++kb, ++it) {
        const int s = it % stages;
        mbar_wait(&empty[s], ((it / stages) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[s], 16384);
        if (DIMS == 2) {
          tma_load_2d(&tm, &full[s], smem + s * 16384, kb * 64, t * 128);
        } else {
          const int c2 = t * kblocks + kb;
          asm volatile(
              "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(smem + s * 16384)),
              "l"(reinterpret_cast<uint64_t>(&tm)), "r"(0), "r"(0), "r"(c2), "r"(smem_u32(&full[s]))
              : "memory");
        }
      }
  } else if (threadIdx.x == 32) {
    int it = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x)
      for (int kb = 0; kb < kblocks; ++kb, ++it) {
        const int s = it % stages;
        mbar_wait(&full[s], (it / stages) & 1);
        mbar_arrive(&empty[s]);
      }
  }
}

int main() {
  void* fnp;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)fnp;
  const int shapes[][2] = {{51200, 5120}, {5120, 25600}, {5120, 8192}};
  for (auto& sh : shapes) {
    const long N = sh[0], K = sh[1];
    const int copies = 4;
    void* buf;
    const size_t bytes = (size_t)N * K * 2;
    cudaMalloc(&buf, bytes * copies);
    cudaMemset(buf, 1, bytes * copies);
    for (int dims = 2; dims <= 3; ++dims)
      for (int stages : {6, 12}) {
        CUtensorMap tm[copies];
        for (int c = 0; c < copies; ++c) {
          char* base = (char*)buf + c * bytes;
          if (dims == 2) {
            cuuint64_t d[2] = {(cuuint64_t)K, (cuuint64_t)N};
            cuuint64_t st[1] = {(cuuint64_t)K * 2};
            cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
            enc(&tm[c], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, d, st, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
          } else {   // tiled: [N/128 * K/64][128][64]
            cuuint64_t d[3] = {64, 128, (cuuint64_t)(N / 128) * (K / 64)};
            cuuint64_t st[2] = {128, 128 * 128};
            cuuint32_t box[3] = {64, 128, 1}, es[3] = {1, 1, 1};
            enc(&tm[c], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, base, d, st, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
          }
        }
        auto kfn = dims == 2 ? stream_kernel<2> : stream_kernel<3>;
        const int smem = stages * 16384 + 1024;
        cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        kfn<<<148, 64, smem>>>(tm[0], N / 128, K / 64, stages);
        cudaEventRecord(e0);
        const int reps = 8;
        for (int r = 0; r < reps; ++r) kfn<<<148, 64, smem>>>(tm[r % copies], N / 128, K / 64, stages);
        cudaEventRecord(e1);
        cudaError_t err = cudaDeviceSynchronize();
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("N=%ld K=%ld %s stages=%d: %.1f us  %.0f GB/s  (%s)\n", N, K,
               dims == 2 ? "row-major 2D box" : "tile-contiguous", stages, ms / reps * 1e3,
               bytes / (ms / reps * 1e-3) / 1e9, cudaGetErrorString(err));
      }
    cudaFree(buf);
  }
  return 0;
}
