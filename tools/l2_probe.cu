// l2_probe.cu — aggregate L2 -> SM bandwidth with TMA: every CTA streams 2D boxes out of one
// small L2-resident bf16 matrix (standalone experiment, not the product).
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>

#include "common.cuh"

using namespace sidp;

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);

__global__ void __launch_bounds__(64, 1) stream_kernel(const __grid_constant__ CUtensorMap tm, int n_tiles,
                                                      int kblocks, int stages, int reps, int box_bytes) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * box_bytes);
  uint64_t* empty = full + stages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const int total = reps * kblocks;
  if (threadIdx.x == 0) {
    for (int it = 0; it < total; ++it) {
      const int s = it % stages;
      mbar_wait(&empty[s], ((it / stages) & 1) ^ 1);
      mbar_arrive_expect_tx(&full[s], box_bytes);
      const int t = (blockIdx.x + it / kblocks) % n_tiles;
      tma_load_2d(&tm, &full[s], smem + s * box_bytes, (it % kblocks) * 64, t * (box_bytes / 128));
    }
  } else if (threadIdx.x == 32) {
    for (int it = 0; it < total; ++it) {
      const int s = it % stages;
      mbar_wait(&full[s], (it / stages) & 1);
      mbar_arrive(&empty[s]);
    }
  }
}

int main(int argc, char** argv) {
  void* fnp;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)fnp;
  for (long mb : {16L, 2048L}) {
    const long K = 4096, N = mb * 1024 * 1024 / (K * 2);
    void* buf;
    const size_t bytes = (size_t)N * K * 2;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 1, bytes);
    for (int rows : {32, 64, 128, 256}) {
      for (int stages : {3, 6}) {
        CUtensorMap tm;
        cuuint64_t d[2] = {(cuuint64_t)K, (cuuint64_t)N};
        cuuint64_t st[1] = {(cuuint64_t)K * 2};
        cuuint32_t box[2] = {64, (cuuint32_t)rows}, es[2] = {1, 1};
        enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, d, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        const int smem = stages * rows * 128 + 1024;
        cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        const int n_tiles = N / rows, kblocks = K / 64;
        const int reps = mb >= 1024 ? 1 : 8;
        const int box_bytes = rows * 128;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        stream_kernel<<<148, 64, smem>>>(tm, n_tiles, kblocks, stages, reps, box_bytes);
        cudaEventRecord(e0);
        stream_kernel<<<148, 64, smem>>>(tm, n_tiles, kblocks, stages, reps, box_bytes);
        cudaEventRecord(e1);
        cudaError_t err = cudaDeviceSynchronize();
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double moved = 148.0 * reps * kblocks * box_bytes;
        printf("buffer %5ld MB box %3d rows stages %2d: %.1f us  %.0f GB/s into SMs (%s)\n", mb, rows, stages,
               ms * 1e3, moved / (ms * 1e-3) / 1e9, cudaGetErrorString(err));
      }
    }
    cudaFree(buf);
  }
  return 0;
}
