// gemm.cu — tcgen05/TMEM decode GEMM for sm_100a.
//
// Y[m, n] = sum_k X[m, k] W[n, k], bf16 in, fp32 accumulate (north_star: "bf16 weights
// with fp32 accumulation").  Decode shapes have few tokens (M = batch rows) and many
// features, so the kernel is "swap-AB": a 128-row W tile is the UMMA A operand
// (UMMA_M = 128), the token tile is the UMMA N operand (16..256), and the fp32
// accumulator D^T[feature, token] lives in TMEM (lane = feature, column = token).
//
// Warp roles (192 threads, one CTA per SM):
//   warp 0      TMA producer: W tile [128 x 64] + X tile [BM x 64] per stage, 128B swizzle
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2..5  epilogue: tcgen05.ld -> registers -> fused epilogue -> global
// Split-K (for shapes with fewer tiles than SMs): every split writes fp32 partials to a
// workspace; the last-arriving CTA of a tile (atomic counter) sums the partials in split
// order 0..S-1 (deterministic) and runs the epilogue.
#include <algorithm>
#include <cstdio>

#include "../common.cuh"
#include "../kernels.h"

namespace sidp {

namespace {

constexpr int BN = 128;      // features per tile (UMMA_M)
constexpr int BK = 64;       // 64 bf16 = 128 B per row -> SWIZZLE_128B atom
constexpr int kThreads = 192;
constexpr int kSmemBudget = 220 * 1024;

struct KParams {
  int M, N, K;
  int BM;                    // token tile (UMMA_N)
  int stages;
  int splits;
  int kb_per_split;
  int epi;
  void* out; int ldo;
  const bf16* resid; int ldr;
  const bf16* bias;
  float* ws;
  int* counters;
};

__device__ __forceinline__ unsigned long long argmax_key(float v, int n) {
  uint32_t u = __float_as_uint(v);
  u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  return ((unsigned long long)u << 32) | (unsigned long long)(0xFFFFFFFFu - (uint32_t)n);
}

// Epilogue of one 32-column chunk for one thread (feature row `n`, tokens m0..m0+31).
__device__ __forceinline__ void epilogue_chunk(const KParams& p, const float (&v)[32], int n,
                                               int m0, int lane_in_tile, float* xchg,
                                               int epi_tid) {
  const int epi = p.epi;
  if (epi == EPI_SILU_MUL) {
    // rows 0..63 of the tile are gate features, rows 64..127 the matching up features
    const bool is_up = lane_in_tile >= 64;
    const int i = lane_in_tile & 63;
    if (is_up) {
#pragma unroll
      for (int j = 0; j < 32; ++j) xchg[j * 64 + i] = v[j];
    }
    named_bar_sync(1, 128);
    if (!is_up) {
      const int f = (n / BN) * 64 + i;        // output feature
      const int F = p.N / 2;
      bf16* out = reinterpret_cast<bf16*>(p.out);
      if (f < F) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int m = m0 + j;
          if (m < p.M) {
            const float g = v[j], u = xchg[j * 64 + i];
            const float s = g / (1.0f + __expf(-g));
            out[(size_t)m * p.ldo + f] = f_to_bf16(s * u);
          }
        }
      }
    }
    named_bar_sync(1, 128);
    return;
  }
  if (epi == EPI_ARGMAX) {
    unsigned long long* out = reinterpret_cast<unsigned long long*>(p.out);
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      unsigned long long key = (n < p.N) ? argmax_key(v[j], n) : 0ull;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        unsigned long long other = __shfl_xor_sync(0xffffffffu, key, o);
        key = other > key ? other : key;
      }
      const int m = m0 + j;
      if ((threadIdx.x & 31) == 0 && m < p.M) atomicMax(out + m, key);
    }
    return;
  }
  if (n >= p.N) return;
  const float b = p.bias ? bf16_to_f(p.bias[n]) : 0.0f;
  if (epi == EPI_F32) {
    float* out = reinterpret_cast<float*>(p.out);
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int m = m0 + j;
      if (m < p.M) out[(size_t)m * p.ldo + n] = v[j] + b;
    }
  } else if (epi == EPI_BF16) {
    bf16* out = reinterpret_cast<bf16*>(p.out);
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int m = m0 + j;
      if (m < p.M) out[(size_t)m * p.ldo + n] = f_to_bf16(v[j] + b);
    }
  } else {  // EPI_RESID
    bf16* out = reinterpret_cast<bf16*>(p.out);
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int m = m0 + j;
      if (m < p.M) {
        const float r = bf16_to_f(p.resid[(size_t)m * p.ldr + n]);
        out[(size_t)m * p.ldo + n] = f_to_bf16(v[j] + r);
      }
    }
  }
}

__global__ void __launch_bounds__(kThreads, 1)
gemm_tc_kernel(const __grid_constant__ CUtensorMap tm_w, const __grid_constant__ CUtensorMap tm_x,
               const KParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const int stages = p.stages;
  const int BM = p.BM;
  const uint32_t a_bytes = BN * BK * 2;                 // 16 KB
  const uint32_t b_bytes = (uint32_t)BM * BK * 2;
  uint8_t* sA = smem;
  uint8_t* sB = sA + (size_t)stages * a_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + (size_t)stages * b_bytes);
  uint64_t* empty = full + stages;
  uint64_t* tmem_full = empty + stages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);
  int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);
  float* xchg = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(tmem_full) + 64);  // 8 KB

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n_blk = blockIdx.x, m_blk = blockIdx.y, split = blockIdx.z;
  const int nkb = p.K / BK;
  const int kb0 = split * p.kb_per_split;
  const int kb1 = min(nkb, kb0 + p.kb_per_split);
  const int tmem_cols = BM <= 32 ? 32 : (BM <= 64 ? 64 : (BM <= 128 ? 128 : 256));

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_w);
    tma_prefetch_desc(&tm_x);
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      for (int kb = kb0, i = 0; kb < kb1; ++kb, ++i) {
        const int s = i % stages;
        const uint32_t ph = (i / stages) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&full[s], a_bytes + b_bytes);
        tma_load_2d(&tm_w, &full[s], sA + (size_t)s * a_bytes, kb * BK, n_blk * BN);
        tma_load_2d(&tm_x, &full[s], sB + (size_t)s * b_bytes, kb * BK, m_blk * BM);
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = umma_idesc_bf16(BN, BM);
    for (int kb = kb0, i = 0; kb < kb1; ++kb, ++i) {
      const int s = i % stages;
      const uint32_t ph = (i / stages) & 1;
      mbar_wait(&full[s], ph);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t a0 = smem_u32(sA + (size_t)s * a_bytes);
        const uint32_t b0 = smem_u32(sB + (size_t)s * b_bytes);
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) {
          umma_bf16(tmem_base, umma_desc_sw128(a0 + k * 32), umma_desc_sw128(b0 + k * 32), idesc,
                    (i > 0 || k > 0) ? 1u : 0u);
        }
        umma_commit(&empty[s]);
      }
      __syncwarp();
    }
    if (lane == 0) umma_commit(tmem_full);
    __syncwarp();
  } else {
    // ---------------------------------------------------------------- epilogue warps
    const int quarter = warp & 3;                 // TMEM lane quarter this warp may access
    const int lane_in_tile = quarter * 32 + lane;
    const int n = n_blk * BN + lane_in_tile;
    const int epi_tid = (warp - 2) * 32 + lane;
    mbar_wait(tmem_full, 0);
    tc_fence_after();
    const uint32_t t_lane = tmem_base + ((uint32_t)(quarter * 32) << 16);
    const int tile_id = m_blk * gridDim.x + n_blk;
    const size_t tile_elems = (size_t)BN * BM;

    if (p.splits == 1) {
      for (int c = 0; c < BM; c += 32) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(t_lane + c, r);
        tmem_ld_wait();
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
        epilogue_chunk(p, v, n, m_blk * BM + c, lane_in_tile, xchg, epi_tid);
      }
    } else {
      // write this split's partial, then the last CTA of the tile reduces in split order
      float* my = p.ws + ((size_t)tile_id * p.splits + split) * tile_elems;
      for (int c = 0; c < BM; c += 32) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(t_lane + c, r);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) my[(size_t)(c + j) * BN + lane_in_tile] = __uint_as_float(r[j]);
      }
      __threadfence();
      named_bar_sync(1, 128);
      if (epi_tid == 0) {
        const int old = atomicAdd(p.counters + tile_id, 1);
        *last_flag = (old == p.splits - 1);
        if (old == p.splits - 1) p.counters[tile_id] = 0;   // re-arm for the next launch
      }
      named_bar_sync(1, 128);
      if (*last_flag) {
        __threadfence();
        const float* base = p.ws + (size_t)tile_id * p.splits * tile_elems;
        for (int c = 0; c < BM; c += 32) {
          float v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = 0.0f;
          for (int s = 0; s < p.splits; ++s) {
            const float* src = base + (size_t)s * tile_elems + (size_t)c * BN + lane_in_tile;
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] += __ldcg(src + (size_t)j * BN);
          }
          epilogue_chunk(p, v, n, m_blk * BM + c, lane_in_tile, xchg, epi_tid);
        }
      }
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, tmem_cols);
  }
}

// ---------------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

bool make_tmap_2d(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer,
                  uint64_t ld_elems, uint32_t box_inner, uint32_t box_outer) {
  EncodeTiledFn fn = get_encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld_elems * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                  box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int g_num_sms = 0;

}  // namespace

int gemm_pick_splits(int tiles, int nkb, int sms) {
  if (tiles >= sms) return 1;
  int best = 1;
  double best_t = 1e30;
  for (int s = 1; s <= 16; ++s) {
    const int per = (nkb + s - 1) / s;
    if (per < 2 && s > 1) break;
    const int waves = (tiles * s + sms - 1) / sms;
    const double t = waves * (per + 2.0);
    if (t < best_t - 1e-9) {
      best_t = t;
      best = s;
    }
  }
  return best;
}

cudaError_t gemm_launch(const GemmArgs& a, const GemmWorkspace& w, cudaStream_t stream) {
  if (a.M <= 0) return cudaSuccess;
  if (a.K % BK != 0 || a.N <= 0 || a.x == nullptr || a.w == nullptr) return cudaErrorInvalidValue;
  if (a.epi == EPI_SILU_MUL && (a.N % BN) != 0) return cudaErrorInvalidValue;
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(gemm_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kSmemBudget + 1024);
  }
  const int sms = a.max_ctas > 0 ? std::min(a.max_ctas, g_num_sms) : g_num_sms;
  int BM = std::min(256, ((a.M + 15) / 16) * 16);
  if (BM > 32 && BM % 32) BM = ((BM + 31) / 32) * 32;   // epilogue walks 32-column chunks
  if (BM < 32) BM = 32;
  const int m_tiles = (a.M + BM - 1) / BM;
  const int n_tiles = (a.N + BN - 1) / BN;
  const int nkb = a.K / BK;
  int splits = a.k_splits > 0 ? a.k_splits : gemm_pick_splits(n_tiles * m_tiles, nkb, sms);
  splits = std::max(1, std::min(splits, nkb));
  const int kb_per = (nkb + splits - 1) / splits;
  splits = (nkb + kb_per - 1) / kb_per;                   // no empty split
  const size_t tile_elems = (size_t)BN * BM;
  if (splits > 1) {
    if ((size_t)n_tiles * m_tiles * splits * tile_elems * 4 > w.ws_bytes ||
        n_tiles * m_tiles > w.n_counters)
      return cudaErrorMemoryAllocation;
  }
  const size_t stage_bytes = (size_t)BN * BK * 2 + (size_t)BM * BK * 2;
  const size_t extra = 2048 + 64 * 32 * 4 + 64;            // barriers + epilogue exchange
  int stages = (int)std::min<size_t>(8, (kSmemBudget - extra) / stage_bytes);
  stages = std::max(2, std::min(stages, std::max(2, kb_per)));

  CUtensorMap tw, tx;
  if (!make_tmap_2d(&tw, a.w, a.K, a.N, a.ldw, BK, BN)) return cudaErrorInvalidValue;
  if (!make_tmap_2d(&tx, a.x, a.K, a.M, a.ldx, BK, BM)) return cudaErrorInvalidValue;

  KParams p;
  p.M = a.M; p.N = a.N; p.K = a.K; p.BM = BM; p.stages = stages; p.splits = splits;
  p.kb_per_split = kb_per; p.epi = a.epi; p.out = a.out; p.ldo = a.ldo; p.resid = a.resid;
  p.ldr = a.ldr; p.bias = a.bias; p.ws = w.ws; p.counters = w.counters;
  const size_t smem = stages * stage_bytes + extra + 1024;
  dim3 grid(n_tiles, m_tiles, splits);
  gemm_tc_kernel<<<grid, kThreads, smem, stream>>>(tw, tx, p);
  return cudaGetLastError();
}

}  // namespace sidp
