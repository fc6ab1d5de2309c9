// gemm.cu — tcgen05/TMEM decode GEMM for sm_100a.
//
// Y[m, n] = sum_k X[m, k] W[n, k], bf16 in, fp32 accumulate (north_star: "bf16 weights with
// fp32 accumulation").  Decode shapes have few tokens (M = batch rows) and many features, so the
// kernel is swap-AB: W rows are the UMMA "M" operand, tokens the UMMA "N" operand.
//
// Design (B200-first):
//  * CTA pairs (cluster 2, tcgen05.mma.cta_group::2): a pair owns a 256-feature tile; each CTA
//    TMA-loads its 128 W rows and half of the token tile, the leader issues one M=256 UMMA over
//    both CTAs' shared memory, each CTA's TMEM holds its 128 features x all tokens.  This halves
//    the per-SM token-tile (L2) traffic and runs the tensor core at the 2-SM rate.
//  * Persistent: grid = (#SMs / 2) pairs walking a static list of (feature tile, token tile,
//    k-split) units; two TMEM accumulators so the epilogue of unit i overlaps the mainloop of
//    unit i+1.
//  * Warp roles (192 threads / CTA): warp 0 TMA producer, warp 1 TMEM allocator + MMA issuer
//    (leader CTA), warps 2-5 epilogue (tcgen05.ld -> smem transpose -> 16-byte coalesced stores).
//  * Epilogue kind is a template parameter (one compact kernel per kind).
//  * Split-K for shapes with few feature tiles: fp32 partials to a workspace; the last-arriving
//    split of a tile half sums the partials in split order 0..S-1 (deterministic) and runs the
//    epilogue.
#include <algorithm>
#include <map>
#include <tuple>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../common.cuh"
#include "../kernels.h"

namespace sidp {

namespace {

constexpr int BK = 64;          // 64 bf16 = 128 B rows -> SWIZZLE_128B atom
constexpr int WROWS = 128;      // W rows per CTA (UMMA M = 256 per pair)
constexpr int kThreads = 192;
constexpr int kSmemBudget = 224 * 1024;
constexpr int SROW = 132;       // padded fp32 staging row (32 tokens x 128 features)

struct KParams {
  int M, N, K;
  int BNT;                      // token tile (UMMA N), multiple of 32, <= 256
  int stages;
  int m_tiles, n_pairs, tiles;
  int streamk;                  // 1: k-block ranges split evenly over clusters; 0: whole tiles
  long long total_kb;           // tiles * nks (work in k-steps)
  int kps, nks;                 // k-blocks (64 deep) per pipeline stage; k-steps per tile
  int clusters;                 // concurrent CTA pairs (fixed per launch configuration)
  int sk;                       // pairs sharing the stream-K region (<= clusters; hybrid tails of
                                // few k-steps go to the first sk pairs only)
  void* out; int ldo;
  const bf16* resid; int ldr;
  const bf16* bias;
  float* ws;
  int* counters;
  int a3d, b3d;                 // operand map is k-block-major 3-D: one TMA box per stage
  int dp_tiles;                 // hybrid: tiles [0, dp_tiles) whole, round-robin; stream-K after
  int compact;                  // stream-K partials in per-cluster tile buffers (see part_tile)
  int partial_all;              // EPI_PARTIAL: every unit writes its fp32 partial slice
  int w_evict;                  // weight TMA loads carry an L2 evict-first policy
  int debug;                    // perf experiments only: 1 = skip MMA, 2 = skip TMA; SW EPI_QKV:
                                // 4 = no stores, 8 = no RoPE loads, 16 = no slice loads, 32 = no gains
  unsigned long long* trace;    // perf experiments only: per-k-block timestamps of cluster 0
  QkvEpi qkv;                   // EPI_QKV destination
  int qkv_cnt_off;              // SW EPI_QKV: first of this launch's split-tile arrival counters
  FlagWait wait;                // CaS owner: activation loads wait for the arrival flags
  RowScatter scatter;           // CaS owner: output rows straight into the requesters' buffers
  PostFlags post;               // CaS owner: done + served, posted by this launch's last CTA
};

// After every thread of this CTA finished its stores: the last CTA of the grid posts the flags
// (gpu-scope election, cumulative sys-scope releases; see atom_add_acq_rel_gpu).
SIDP_DEV void post_after_grid(const PostFlags& f) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned total = gridDim.x * gridDim.y * gridDim.z;
    const unsigned prev = atom_add_acq_rel_gpu(f.counter, 1u);
    if (prev == total - 1) {
      *f.counter = 0u;
      const uint64_t v = flag_value(f.value, f.base);
      for (int i = 0; i < f.n; ++i) st_release_sys(f.flag[i], v);
    }
  }
}

// Base of output row m (elements of size ES): out + m * ldo, or the requester's receive buffer
// holding fused row m (CaS scatter; rows of one requester are contiguous in both).
template <typename T>
SIDP_DEV T* out_row(const KParams& p, int m) {
  if (p.scatter.n == 0) return reinterpret_cast<T*>(p.out) + (size_t)m * p.ldo;
  int q = 0;
  while (q + 1 < p.scatter.n && m >= p.scatter.row0[q + 1]) ++q;
  return reinterpret_cast<T*>(p.scatter.base[q]) + (size_t)(m - p.scatter.row0[q]) * p.ldo;
}

// ---- cluster / 2-SM helpers ------------------------------------------------------
SIDP_DEV uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
SIDP_DEV void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
SIDP_DEV uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
SIDP_DEV void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
SIDP_DEV void tma_load_2d_2sm(const CUtensorMap* m, uint32_t leader_bar, void* smem_dst, int c0,
                              int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(leader_bar)
      : "memory");
}
// same, with an L2 cache policy (createpolicy): weights are streamed exactly once per step,
// so they are loaded evict-first and the small re-read tensors (activations, partial slices)
// keep their L2 lines
SIDP_DEV void tma_load_2d_2sm_hint(const CUtensorMap* m, uint32_t leader_bar, void* smem_dst, int c0,
                                   int c1, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(leader_bar), "l"(policy)
      : "memory");
}
SIDP_DEV uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
SIDP_DEV void tma_load_3d_2sm(const CUtensorMap* m, uint32_t leader_bar, void* smem_dst, int c0,
                              int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(leader_bar)
      : "memory");
}
SIDP_DEV void umma2_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                         uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
SIDP_DEV void umma2_commit_mc(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
SIDP_DEV void tmem_alloc2(uint32_t* smem_dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(smem_dst)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
SIDP_DEV void tmem_dealloc2(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}

// ---- work decomposition ---------------------------------------------------------
// Stream-K: the tiles*nkb k-blocks (tile-major, tokens fastest within a feature tile so W
// tiles are re-read from L2 across token tiles) are split into `clusters` equal contiguous
// ranges; cluster c owns [b_c, b_{c+1}), b_c = floor(c * total / C).  A range crossing tile
// boundaries yields several units; a tile covered by one unit is finished in the GEMM
// epilogue, otherwise each covering unit writes its fp32 partial to slice `seg` and
// gemm_reduce_kernel sums slices 0..nseg-1 in order (deterministic: depends only on shapes
// and C).  Whole-tile mode (fused argmax) walks tiles round-robin.
SIDP_DEV int cluster_of_kb(long long g, long long total, int C) {
  return (int)(((g + 1) * (long long)C + total - 1) / total) - 1;
}
__host__ __device__ inline long long range_begin(int c, long long total, int C) {
  return (long long)c * total / C;
}

struct Unit {
  int ft, mt, kb0, kb1, seg, nseg;
  int slot;   // 0: the unit starts this cluster's stream-K range, 1: it ends it
};

struct UnitIter {
  long long g, g0, end;   // stream-K cursor (k-steps of tiles >= dp_tiles)
  int u;                  // whole-tile cursor
  SIDP_DEV void init(const KParams& p, int cluster) {
    if (cluster < p.sk) {
      g0 = g = range_begin(cluster, p.total_kb, p.sk);
      end = range_begin(cluster + 1, p.total_kb, p.sk);
    } else {
      g0 = g = end = 0;   // no stream-K work for this pair
    }
    u = cluster;
  }
  SIDP_DEV bool next(const KParams& p, int cluster, Unit& x) {
    const int nkb = p.nks;   // k-steps per tile
    int t;
    x.slot = 0;
    if (p.streamk && u < p.dp_tiles) {   // hybrid: the whole-tile waves first
      t = u;
      u += p.clusters;
      x.kb0 = 0;
      x.kb1 = nkb;
      x.seg = 0;
      x.nseg = 1;
    } else if (p.streamk) {
      if (g >= end) return false;
      const int tl = (int)(g / nkb);            // tile within the stream-K region
      const long long tile_end = (long long)(tl + 1) * nkb;
      const long long seg_end = end < tile_end ? end : tile_end;
      x.kb0 = (int)(g - (long long)tl * nkb);
      x.kb1 = x.kb0 + (int)(seg_end - g);
      const int first = cluster_of_kb((long long)tl * nkb, p.total_kb, p.sk);
      const int last = cluster_of_kb(tile_end - 1, p.total_kb, p.sk);
      x.seg = cluster - first;
      x.nseg = last - first + 1;
      x.slot = g == g0 ? 0 : 1;
      t = p.dp_tiles + tl;
      g = seg_end;
    } else {
      if (u >= p.tiles) return false;
      t = u;
      u += p.clusters;
      x.kb0 = 0;
      x.kb1 = nkb;
      x.seg = 0;
      x.nseg = 1;
    }
    x.mt = t % p.m_tiles;
    x.ft = t / p.m_tiles;
    return true;
  }
};

// Sequential (unit, k-block) cursor — drives the W L2 prefetch ahead of the TMA ring.
struct KbCursor {
  UnitIter ui;
  Unit x;
  int kb;
  bool valid;
  SIDP_DEV void init(const KParams& p, int cluster) {
    ui.init(p, cluster);
    valid = ui.next(p, cluster, x);
    kb = valid ? x.kb0 : 0;
  }
  SIDP_DEV void advance(const KParams& p, int cluster) {
    if (!valid) return;
    if (++kb >= x.kb1) {
      valid = ui.next(p, cluster, x);
      if (valid) kb = x.kb0;
    }
  }
};

SIDP_DEV unsigned long long argmax_key(float v, int n) {
  uint32_t u = __float_as_uint(v);
  u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  return ((unsigned long long)u << 32) | (unsigned long long)(0xFFFFFFFFu - (uint32_t)n);
}

SIDP_DEV void unpack_bf16x8(const uint4& raw, float (&f)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}
SIDP_DEV uint4 pack_bf16x8(const float (&f)[8]) {
  uint4 r;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&r);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  return r;
}

// Store phase: sm holds fp32 [32 tokens][SROW] (features 0..127 of this CTA's W rows).
// m0 = first token of the chunk, n0 = first feature (W row) of this CTA, pt = packed tile id.
template <int EPI>
SIDP_DEV void store_phase(const KParams& p, const float* sm, int m0, int n0, int pt, int tid) {
  if constexpr (EPI == EPI_F32) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int v = tid + 128 * i, j = v >> 5, f = (v & 31) * 4;
      const int m = m0 + j, n = n0 + f;
      if (m < p.M && n < p.N) {
        float4 x = *reinterpret_cast<const float4*>(sm + j * SROW + f);
        if (p.bias) {
          const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(p.bias + n);
          const float2 b0 = __bfloat1622float2(b2[0]), b1 = __bfloat1622float2(b2[1]);
          x.x += b0.x; x.y += b0.y; x.z += b1.x; x.w += b1.y;
        }
        *reinterpret_cast<float4*>(out_row<float>(p, m) + n) = x;
      }
    }
  } else if constexpr (EPI == EPI_BF16 || EPI == EPI_RESID) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int v = tid + 128 * i, j = v >> 4, f = (v & 15) * 8;
      const int m = m0 + j, n = n0 + f;
      if (m < p.M && n < p.N) {
        float x[8];
        const float4 a = *reinterpret_cast<const float4*>(sm + j * SROW + f);
        const float4 b = *reinterpret_cast<const float4*>(sm + j * SROW + f + 4);
        x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w; x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
        float y[8];
        if constexpr (EPI == EPI_RESID) {
          unpack_bf16x8(*reinterpret_cast<const uint4*>(p.resid + (size_t)m * p.ldr + n), y);
        } else {
          if (p.bias) {
            unpack_bf16x8(*reinterpret_cast<const uint4*>(p.bias + n), y);
          } else {
#pragma unroll
            for (int q = 0; q < 8; ++q) y[q] = 0.0f;
          }
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) x[q] += y[q];
        *reinterpret_cast<uint4*>(out_row<bf16>(p, m) + n) = pack_bf16x8(x);
      }
    }
  } else if constexpr (EPI == EPI_SILU_MUL) {
    // this CTA's 128 W rows = 8 groups [gate 8 | up 8] of packed tile pt -> outputs pt*64 .. +64
    bf16* out = reinterpret_cast<bf16*>(p.out);
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int v = tid + 128 * i, j = v >> 3, f = (v & 7) * 8;
      const int m = m0 + j;
      const int of = pt * 64 + f;
      if (m < p.M && of < p.N / 2) {
        float x[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float g = sm[j * SROW + 2 * f + q], u = sm[j * SROW + 2 * f + 8 + q];
          x[q] = g / (1.0f + __expf(-g)) * u;
        }
        *reinterpret_cast<uint4*>(out + (size_t)m * p.ldo + of) = pack_bf16x8(x);
      }
    }
  } else if constexpr (EPI == EPI_QKV) {
    // warp w handles tokens w*8 .. w*8+7; lane l holds features 4l..4l+3 of the 128-row tile,
    // which lies entirely in the q, k or v region (q_dim, kv_dim multiples of 128)
    const QkvEpi& e = p.qkv;
    const int w = tid >> 5, lane = tid & 31;
    const int hd = e.hd, half = hd / 2;
    const int qd = e.nq * hd, kvd = e.nkv * hd;
    const int region = n0 < qd ? 0 : (n0 < qd + kvd ? 1 : 2);
    const int f = lane * 4;                          // feature within tile
    const int nabs = n0 + f;
    const int lane_span = hd / 4;                    // lanes per head (32 or 16)
    float bias4[4] = {0.f, 0.f, 0.f, 0.f};
    if (p.bias) {
      const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(p.bias + nabs);
      const float2 t0 = __bfloat1622float2(b2[0]), t1 = __bfloat1622float2(b2[1]);
      bias4[0] = t0.x; bias4[1] = t0.y; bias4[2] = t1.x; bias4[3] = t1.y;
    }
    const bf16* gain = region == 0 ? e.gq : (region == 1 ? e.gk : nullptr);
    const int d = (n0 - (region == 0 ? 0 : (region == 1 ? qd : qd + kvd)) + f) % hd;  // dim in head
    const int head = (n0 - (region == 0 ? 0 : (region == 1 ? qd : qd + kvd)) + f) / hd;
    float g4[4] = {1.f, 1.f, 1.f, 1.f};
    if (gain) {
#pragma unroll
      for (int q = 0; q < 4; ++q) g4[q] = bf16_to_f(gain[d + q]);
    }
    // positions of this warp's 8 tokens (one load per lane, broadcast by shuffles) and the
    // RoPE table entries of 4 tokens at a time issued before use: no dependent global loads
    // inside the per-token loop
    int mypos = 0;
    if (lane < 8 && m0 + w * 8 + lane < p.M) mypos = e.pos[m0 + w * 8 + lane];
    const bool lo = d < half;
    const int rd = lo ? d : d - half;
#pragma unroll
    for (int grp = 0; grp < 2; ++grp) {
      float2 cs[4][4];
      int posv[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        posv[t] = __shfl_sync(0xffffffffu, mypos, grp * 4 + t);
        if (region < 2) {
          const float2* row = e.rope + (size_t)posv[t] * half + rd;
#pragma unroll
          for (int q = 0; q < 4; ++q) cs[t][q] = row[q];
        }
      }
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int j = w * 8 + grp * 4 + t, m = m0 + j;
        const float4 v4 = *reinterpret_cast<const float4*>(sm + j * SROW + f);
        float x[4] = {v4.x + bias4[0], v4.y + bias4[1], v4.z + bias4[2], v4.w + bias4[3]};
        if (region < 2) {
          if (gain) {   // per-head RMSNorm over hd dims (Qwen3 qk_norm)
            float ss = x[0] * x[0] + x[1] * x[1] + x[2] * x[2] + x[3] * x[3];
            for (int o = lane_span / 2; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
            const float r = rsqrtf(ss / (float)hd + e.eps);
#pragma unroll
            for (int q = 0; q < 4; ++q) x[q] = x[q] * r * g4[q];
          }
          // rotate-half RoPE: partner of dim d is d +- hd/2, held by lane ^ (hd/8)
          float y[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) y[q] = __shfl_xor_sync(0xffffffffu, x[q], hd / 8);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            x[q] = lo ? x[q] * cs[t][q].x - y[q] * cs[t][q].y : x[q] * cs[t][q].x + y[q] * cs[t][q].y;
        }
        if (m < p.M) {
          __nv_bfloat162 o0 = __floats2bfloat162_rn(x[0], x[1]), o1 = __floats2bfloat162_rn(x[2], x[3]);
          uint2 pk;
          pk.x = *reinterpret_cast<uint32_t*>(&o0);
          pk.y = *reinterpret_cast<uint32_t*>(&o1);
          bf16* dst;
          if (region == 0) {
            dst = e.q + ((size_t)m * e.nq + head) * hd + d;
          } else {
            bf16* cache = region == 1 ? e.kc : e.vc;
            dst = cache + kv_off(e.bt, e.bt_stride, e.nkv, e.smax, hd, m, head, posv[t]) + d;
          }
          *reinterpret_cast<uint2*>(dst) = pk;
        }
      }
    }
  } else if constexpr (EPI == EPI_ARGMAX) {  // warp w reduces tokens w*8 .. w*8+7 over the 128 features
    unsigned long long* out = reinterpret_cast<unsigned long long*>(p.out);
    const int w = tid >> 5, lane = tid & 31;
    for (int jj = 0; jj < 8; ++jj) {
      const int j = w * 8 + jj, m = m0 + j;
      unsigned long long key = 0ull;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int n = n0 + lane * 4 + q;
        if (n < p.N) {
          const unsigned long long k2 = argmax_key(sm[j * SROW + lane * 4 + q], n);
          key = k2 > key ? k2 : key;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long other = __shfl_xor_sync(0xffffffffu, key, o);
        key = other > key ? other : key;
      }
      if (lane == 0 && m < p.M && key) atomicMax(out + m, key);
    }
  }
}

// Token-major (SW) epilogue: this thread holds fp32 accumulators of token m, features
// n0..n0+31; nlim = min(N, end of this feature tile) (N and the tile width are multiples of 8,
// so 8-feature groups are all in or all out — columns past the tile belong to the next tile).
template <int EPI>
SIDP_DEV void store_row(const KParams& p, const uint32_t (&r)[32], int m, int n0, int nlim,
                        unsigned long long& best) {
  if constexpr (EPI == EPI_F32) {
    float* out = out_row<float>(p, m);
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      const int n = n0 + 4 * g;
      if (n < nlim) {
        float4 v = make_float4(__uint_as_float(r[4 * g]), __uint_as_float(r[4 * g + 1]),
                               __uint_as_float(r[4 * g + 2]), __uint_as_float(r[4 * g + 3]));
        if (p.bias) {
          const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(p.bias + n);
          const float2 b0 = __bfloat1622float2(b2[0]), b1 = __bfloat1622float2(b2[1]);
          v.x += b0.x; v.y += b0.y; v.z += b1.x; v.w += b1.y;
        }
        *reinterpret_cast<float4*>(out + n) = v;
      }
    }
  } else if constexpr (EPI == EPI_BF16 || EPI == EPI_RESID) {
    bf16* out = out_row<bf16>(p, m);
    uint4 addv[4];
#pragma unroll
    for (int g = 0; g < 4; ++g) {   // issue the residual / bias loads first
      const int n = n0 + 8 * g;
      addv[g] = make_uint4(0u, 0u, 0u, 0u);
      if (n < nlim) {
        if constexpr (EPI == EPI_RESID) addv[g] = *reinterpret_cast<const uint4*>(p.resid + (size_t)m * p.ldr + n);
        else if (p.bias) addv[g] = *reinterpret_cast<const uint4*>(p.bias + n);
      }
    }
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      const int n = n0 + 8 * g;
      if (n < nlim) {
        float y[8], x[8];
        unpack_bf16x8(addv[g], y);
#pragma unroll
        for (int q = 0; q < 8; ++q) x[q] = __uint_as_float(r[8 * g + q]) + y[q];
        *reinterpret_cast<uint4*>(out + n) = pack_bf16x8(x);
      }
    }
  } else if constexpr (EPI == EPI_SILU_MUL) {
    // columns [16h, 16h+16) = one [gate 8 | up 8] group -> outputs (n0 + 16h) / 2 .. +8
    bf16* out = reinterpret_cast<bf16*>(p.out) + (size_t)m * p.ldo;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int n = n0 + 16 * h;
      if (n < nlim) {
        float x[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float g = __uint_as_float(r[16 * h + q]), u = __uint_as_float(r[16 * h + 8 + q]);
          x[q] = g / (1.0f + __expf(-g)) * u;
        }
        *reinterpret_cast<uint4*>(out + n / 2) = pack_bf16x8(x);
      }
    }
  } else if constexpr (EPI == EPI_ARGMAX) {
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      if (n0 + q < nlim) {
        const unsigned long long k2 = argmax_key(__uint_as_float(r[q]), n0 + q);
        best = k2 > best ? k2 : best;
      }
    }
  }
}

// 32 fp32 values -> 32 bf16 at dst (64 contiguous bytes, 16-byte stores)
SIDP_DEV void store_bf16x32(bf16* dst, const float (&v)[32]) {
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    float t[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) t[q] = v[8 * g + q];
    reinterpret_cast<uint4*>(dst)[g] = pack_bf16x8(t);
  }
}
SIDP_DEV void add_bias32(const bf16* bias, int n, float (&v)[32]) {
  if (!bias) return;
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    float t[8];
    unpack_bf16x8(*reinterpret_cast<const uint4*>(bias + n + 8 * g), t);
#pragma unroll
    for (int q = 0; q < 8; ++q) v[8 * g + q] += t[q];
  }
}

// Token-major fused QKV epilogue (SW EPI_QKV): this thread's token m, the
// tile's features [fbase, nlim) are whole heads whose fp32 accumulators sit in this thread's
// TMEM lane at columns tl + (f - fbase).  Per head, the arithmetic of qkv_post_kernel: + bias,
// per-head RMSNorm (Qwen3 qk_norm: x * r * g), rotate-half RoPE from the fp32 (cos, sin) table
// at pos, bf16 -> q [m][head] or the KV cache row pos (the KV cache is local).
// The whole head lies in this thread: the norm needs no reduction and the RoPE partner d + hd/2
// is the same thread's chunk c + hd/64.  TMEM reads are warp-collective: every lane runs every
// read; only global loads / stores are predicated on `valid`.  sg = the qk-norm gains staged in
// shared memory ([0, hd) q, [hd, 2 hd) k) — global gain loads inside the per-head chain cost
// ~12 us per launch (measured, tools/qkv_bench.py), the RoPE rows are issued ahead of the TMEM
// reads they are combined with.
SIDP_DEV void qkv_sw_row(const KParams& p, int m, bool valid, int pos, int fbase, int nlim,
                         uint32_t tl, const float* sg) {
  const QkvEpi& e = p.qkv;
  const int hd = e.hd, hc = hd / 64;                 // chunk pairs (x1 chunk c, x2 chunk c + hc)
  auto get = [&](int c, float (&v)[32]) {
    uint32_t r[32];
    tmem_ld_32x32b_x32(tl + c * 32, r);
    tmem_ld_wait();
#pragma unroll
    for (int q = 0; q < 32; ++q) v[q] = __uint_as_float(r[q]);
  };
  for (int f0 = fbase; f0 < nlim; f0 += hd) {
    const int head = f0 / hd;
    const int region = head < e.nq ? 0 : (head < e.nq + e.nkv ? 1 : 2);
    const int c0 = (f0 - fbase) / 32;
    bf16* dst;
    if (region == 0) {
      dst = e.q + ((size_t)m * e.nq + head) * hd;
    } else {
      const int g = head - e.nq - (region == 2 ? e.nkv : 0);
      dst = (region == 1 ? e.kc : e.vc) + (valid ? kv_off(e.bt, e.bt_stride, e.nkv, e.smax, hd, m, g, pos) : 0);
    }
    const bool st = valid && !(p.debug & 4);
    if (region == 2) {
      for (int c = 0; c < 2 * hc; ++c) {
        float v[32];
        get(c0 + c, v);
        add_bias32(p.bias, f0 + 32 * c, v);
        if (st) store_bf16x32(dst + 32 * c, v);
      }
      continue;
    }
    const bool has_gain = !(p.debug & 32) && (region == 0 ? e.gq : e.gk) != nullptr;
    const float* gs = sg + (region == 0 ? 0 : hd);
    for (int c = 0; c < hc; ++c) {
      // (cos, sin) of dims 32c .. 32c + 31: requested before the norm pass / TMEM reads
      float4 cs[16];
      const float4* rp = reinterpret_cast<const float4*>(e.rope + (size_t)pos * (hd / 2) + 32 * c);
#pragma unroll
      for (int q2 = 0; q2 < 16; ++q2)
        cs[q2] = (valid && !(p.debug & 8)) ? __ldg(rp + q2) : make_float4(1.f, 0.f, 1.f, 0.f);
      float r = 1.0f;
      if (has_gain) {   // RMSNorm statistic over the whole head (recomputed per chunk pair: TMEM is cheap)
        float ss = 0.0f;
        for (int cc = 0; cc < 2 * hc; ++cc) {
          float v[32];
          get(c0 + cc, v);
          add_bias32(p.bias, f0 + 32 * cc, v);
#pragma unroll
          for (int q = 0; q < 32; ++q) ss += v[q] * v[q];
        }
        r = rsqrtf(ss / (float)hd + e.eps);
      }
      float a[32], b[32];
      get(c0 + c, a);
      get(c0 + c + hc, b);
      add_bias32(p.bias, f0 + 32 * c, a);
      add_bias32(p.bias, f0 + hd / 2 + 32 * c, b);
      if (has_gain) {
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          a[q] = a[q] * r * gs[32 * c + q];
          b[q] = b[q] * r * gs[hd / 2 + 32 * c + q];
        }
      }
#pragma unroll
      for (int q2 = 0; q2 < 16; ++q2) {   // (cos, sin) of dims 2 q2, 2 q2 + 1
        const float4 t = cs[q2];
        const float a0 = a[2 * q2], b0 = b[2 * q2], a1 = a[2 * q2 + 1], b1 = b[2 * q2 + 1];
        a[2 * q2] = a0 * t.x - b0 * t.y;
        b[2 * q2] = b0 * t.x + a0 * t.y;
        a[2 * q2 + 1] = a1 * t.z - b1 * t.w;
        b[2 * q2 + 1] = b1 * t.z + a1 * t.w;
      }
      if (st) {
        store_bf16x32(dst + 32 * c, a);
        store_bf16x32(dst + hd / 2 + 32 * c, b);
      }
    }
  }
}

// perf experiment timeline: per CTA, slot k of TL(k) = globaltimer at a kernel milestone
#define SIDP_TL(k) \
  do { if (p.trace && blockIdx.x < 512) p.trace[6 * 4096 + blockIdx.x * 8 + (k)] = globaltimer_ns(); } while (0)

// SW = false: A = W (128 rows per CTA, 256-feature pair tile), B = tokens (BNT per pair).
// SW = true (token-major, large batches): A = X (128 tokens per CTA, 256-token pair tile),
//   B = W (BNT features per pair, any multiple of 32), so the feature tile can be sized to give
//   every CTA pair work without splitting K; TMEM lanes are tokens, columns features, and the
//   epilogue writes each thread's token row straight from registers.  The mainloop is the same
//   code: the host passes the X map as tm_w and the W map as tm_x.
template <int EPI, int KPS, bool SW>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
gemm2_kernel(const __grid_constant__ CUtensorMap tm_w, const __grid_constant__ CUtensorMap tm_x,
             const KParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const int stages = p.stages, BNT = p.BNT, HALF = p.BNT / 2;
  constexpr int kps = KPS;
  const uint32_t a_sub = WROWS * BK * 2, b_sub = (uint32_t)HALF * BK * 2;   // one 64-deep k-block
  const uint32_t a_bytes = kps * a_sub;                 // stage = kps k-blocks
  const uint32_t b_bytes = kps * b_sub;
  uint8_t* sA = smem;
  uint8_t* sB = sA + (size_t)stages * a_bytes;
  float* stg = reinterpret_cast<float*>(sB + (size_t)stages * b_bytes);   // [32][SROW]
  uint64_t* full = reinterpret_cast<uint64_t*>(stg + 32 * SROW);
  uint64_t* empty = full + stages;
  uint64_t* tfull = empty + stages;                      // [2]
  uint64_t* tempty = tfull + 2;                          // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int cluster = blockIdx.x >> 1, n_clusters = gridDim.x >> 1;
  const int ACCS = (BNT + 31) / 32 * 32;                 // TMEM columns per accumulator
  const uint32_t tmem_cols = ACCS <= 16 ? 32 : (ACCS <= 32 ? 64 : (ACCS <= 64 ? 128 : (ACCS <= 128 ? 256 : 512)));

  if (threadIdx.x == 0) {
    SIDP_TL(0);
    tma_prefetch_desc(&tm_w);
    tma_prefetch_desc(&tm_x);
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);          // leader's arrive + expect_tx(bytes of both CTAs)
      mbar_init(&empty[s], 1);         // MMA commit (multicast to both CTAs)
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 8);        // 4 epilogue warps x 2 CTAs (leader's copy is used)
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc2(tmem_slot, tmem_cols);
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // prologue done: let the next kernel of the chain launch, then wait for our inputs
  pdl_trigger();
  if (threadIdx.x != 0) pdl_wait();   // the producer waits after issuing its weight prefetch
  if (threadIdx.x == 0) SIDP_TL(1);

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    if (lane == 0) {
      // Only the leader arrives on a stage's full barrier (expecting both CTAs' bytes); the
      // peer's TMA completes its transaction bytes on the leader's barrier directly.
      const uint32_t stage_tx = 2 * (a_bytes + b_bytes);
      const uint64_t wpol = policy_evict_first();
      // issue one operand of ring iteration (unit x, k-step kb) into stage s
      auto load_a = [&](const Unit& x, int kb, int s, uint32_t lbar) {
        const int arow = x.ft * 2 * WROWS + rank * WROWS;
        if (p.a3d) {
          tma_load_3d_2sm(&tm_w, lbar, sA + (size_t)s * a_bytes, 0, arow, kb * KPS);
        } else {
#pragma unroll
          for (int j = 0; j < KPS; ++j) {
            if (!SW && p.w_evict)
              tma_load_2d_2sm_hint(&tm_w, lbar, sA + (size_t)s * a_bytes + j * a_sub, (kb * KPS + j) * BK, arow, wpol);
            else
              tma_load_2d_2sm(&tm_w, lbar, sA + (size_t)s * a_bytes + j * a_sub, (kb * KPS + j) * BK, arow);
          }
        }
      };
      auto load_b = [&](const Unit& x, int kb, int s, uint32_t lbar) {
        const int brow = x.mt * BNT + rank * HALF;
        if (p.b3d) {
          tma_load_3d_2sm(&tm_x, lbar, sB + (size_t)s * b_bytes, 0, brow, kb * KPS);
        } else {
#pragma unroll
          for (int j = 0; j < KPS; ++j) {
            if (SW && p.w_evict)
              tma_load_2d_2sm_hint(&tm_x, lbar, sB + (size_t)s * b_bytes + j * b_sub, (kb * KPS + j) * BK, brow, wpol);
            else
              tma_load_2d_2sm(&tm_x, lbar, sB + (size_t)s * b_bytes + j * b_sub, (kb * KPS + j) * BK, brow);
          }
        }
      };
      // Weights never depend on the preceding kernel of the chain (they are resident, or were
      // fetched before the layer's first kernel could start), so the first ring stages' weight
      // tiles are requested before griddepcontrol.wait: their HBM latency overlaps the
      // predecessor's tail.  Activations (the other operand) are loaded after the wait.
      KbCursor cur;
      cur.init(p, cluster);
      int npre = 0;
      {
        KbCursor pre = cur;
        for (; npre < stages && pre.valid; ++npre, pre.advance(p, cluster)) {
          const uint32_t lbar = mapa_shared(smem_u32(&full[npre]), 0);
          if (leader) mbar_arrive_expect_tx(&full[npre], stage_tx);
          if (SW) load_b(pre.x, pre.kb, npre, lbar);
          else load_a(pre.x, pre.kb, npre, lbar);
        }
      }
      pdl_wait();
      if (p.wait.n) flags_wait(p.wait.p, p.wait.n, p.wait.value, p.wait.timeout_ns, p.wait.err, p.wait.base);
      for (int it = 0; cur.valid; cur.advance(p, cluster), ++it) {
        const int s = it % stages;
        const uint32_t ph = (it / stages) & 1;
        const uint32_t lbar = mapa_shared(smem_u32(&full[s]), 0);
        if (it >= npre) {
          if (p.trace && cluster == 0 && it < 4096) p.trace[rank * 4096 + it] = globaltimer_ns();
          mbar_wait(&empty[s], ph ^ 1);
          if (p.trace && cluster == 0 && it < 4096) p.trace[(2 + rank) * 4096 + it] = globaltimer_ns();
          if (p.debug & 2) {   // perf experiment: MMA-only (stale stage data, no loads)
            if (leader) mbar_arrive(&full[s]);
            continue;
          }
          if (leader) mbar_arrive_expect_tx(&full[s], stage_tx);
          load_a(cur.x, cur.kb, s, lbar);
          load_b(cur.x, cur.kb, s, lbar);
        } else if (SW) {
          load_a(cur.x, cur.kb, s, lbar);
        } else {
          load_b(cur.x, cur.kb, s, lbar);
        }
        if (p.trace && cluster == 0 && it < 4096 && rank == 0) p.trace[5 * 4096 + it] = globaltimer_ns();
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader only)
    if (leader) {
      const uint32_t idesc = umma_idesc_bf16(2 * WROWS, BNT);
      int it = 0, un = 0;
      UnitIter ui;
      ui.init(p, cluster);
      Unit x;
      while (ui.next(p, cluster, x)) {
        const int acc = un & 1;
        const uint32_t aph = (un >> 1) & 1;
        ++un;
        mbar_wait(&tempty[acc], aph ^ 1);
        tc_fence_after();
        const uint32_t dcol = tmem_base + acc * ACCS;
        for (int kb = x.kb0; kb < x.kb1; ++kb, ++it) {
          const int s = it % stages;
          const uint32_t ph = (it / stages) & 1;
          mbar_wait(&full[s], ph);
          if (lane == 0 && it == 0) SIDP_TL(2);
          if (p.trace && cluster == 0 && it < 4096 && lane == 0) p.trace[4 * 4096 + it] = globaltimer_ns();
          tc_fence_after();
          if (lane == 0 && (p.debug & 1)) {
            mbar_arrive(&empty[s]);
            mbar_arrive_cluster(mapa_shared(smem_u32(&empty[s]), 1));
          } else if (lane == 0) {
            const uint32_t a0 = smem_u32(sA + (size_t)s * a_bytes);
            const uint32_t b0 = smem_u32(sB + (size_t)s * b_bytes);
#pragma unroll
            for (int j = 0; j < KPS; ++j) {
#pragma unroll
              for (int k = 0; k < BK / 16; ++k)
                umma2_bf16(dcol, umma_desc_sw128(a0 + j * a_sub + k * 32),
                           umma_desc_sw128(b0 + j * b_sub + k * 32), idesc,
                           (kb > x.kb0 || j > 0 || k > 0) ? 1u : 0u);
            }
            umma2_commit_mc(&empty[s]);
          }
          __syncwarp();
        }
        if (lane == 0) umma2_commit_mc(&tfull[acc]);
        __syncwarp();
      }
      if (lane == 0) SIDP_TL(3);
    }
  } else {
    // ------------------------------------------------------------ epilogue (both CTAs)
    const int quarter = warp & 3;                       // TMEM lane quarter of this warp
    const int row = quarter * 32 + lane;                // TMEM lane (W row, or token if SW)
    const int tid = (warp - 2) * 32 + lane;             // 0..127
    if constexpr (SW) {
      if constexpr (EPI == EPI_QKV) {   // qk-norm gains -> shared memory (stg is unused when SW)
        const int hd = p.qkv.hd;
        for (int i = tid; i < 2 * hd; i += 128) {
          const bf16* g = i < hd ? p.qkv.gq : p.qkv.gk;
          stg[i] = g ? bf16_to_f(g[i < hd ? i : i - hd]) : 1.0f;
        }
        named_bar_sync(1, 128);
      }
      int un = 0;
      UnitIter ui;
      ui.init(p, cluster);
      Unit x;
      while (ui.next(p, cluster, x)) {
        const int acc = un & 1;
        const uint32_t aph = (un >> 1) & 1;
        ++un;
        const int m = x.ft * 2 * WROWS + rank * WROWS + row;   // this thread's token
        const int fbase = x.mt * BNT;                           // first feature of the tile
        const int nlim = min(p.N, fbase + BNT);
        const int nch = (nlim - fbase + 31) / 32;
        int pos_m = 0;   // EPI_QKV: the new token's position, loaded before the accumulator wait
        if constexpr (EPI == EPI_QKV) pos_m = m < p.M ? p.qkv.pos[m] : 0;
        mbar_wait(&tfull[acc], aph);
        tc_fence_after();
        const uint32_t tl = tmem_base + acc * ACCS + ((uint32_t)(quarter * 32) << 16);
        if constexpr (EPI == EPI_QKV) {
          const bool valid = m < p.M;
          const float* sg = stg;   // qk-norm gains, staged at the epilogue's start
          if (x.nseg == 1) {   // whole dot products in TMEM: the fused epilogue reads them there
            qkv_sw_row(p, m, valid, pos_m, fbase, nlim, tl, sg);
          } else {
            // stream-K segment of a split tile: fp32 partial -> ws[seg][m][features]; the last
            // of the tile half's nseg segments to arrive folds the other slices into its TMEM
            // accumulator in slice order (deterministic: its own slice equals its TMEM values)
            // and runs the fused epilogue from TMEM
            float* dst = p.ws + (size_t)x.seg * p.M * p.N + (size_t)m * p.N;
            for (int c = 0; c < nch; ++c) {
              uint32_t r[32];
              tmem_ld_32x32b_x32(tl + c * 32, r);
              tmem_ld_wait();
              if (valid) {
#pragma unroll
                for (int g = 0; g < 8; ++g)
                  __stcg(reinterpret_cast<float4*>(dst + fbase + c * 32 + 4 * g),
                         make_float4(__uint_as_float(r[4 * g]), __uint_as_float(r[4 * g + 1]),
                                     __uint_as_float(r[4 * g + 2]), __uint_as_float(r[4 * g + 3])));
              }
            }
            // arrival: the CTA's slice stores, then one thread's gpu-scope fence + counter add
            // (the cooperative-groups grid-barrier pattern: bar.sync orders the other threads'
            // stores before thread 0's cumulative fence)
            named_bar_sync(1, 128);
            if (tid == 0) {
              int* cnt = p.counters + p.qkv_cnt_off + 2 * (x.ft * p.m_tiles + x.mt) + rank;
              __threadfence();
              const int prev = atomicAdd(cnt, 1);
              __threadfence();
              *last_flag = prev == x.nseg - 1;
              if (prev == x.nseg - 1) *cnt = 0;   // zero between launches
            }
            named_bar_sync(1, 128);
            const bool last = *last_flag;
            named_bar_sync(1, 128);   // last_flag is rewritten by the next split unit
            if (last) {
              const float* src = p.ws + (size_t)m * p.N + fbase;
              const size_t slice = (size_t)p.M * p.N;
              for (int c = 0; c < nch; c += 2) {   // two 32-column chunks per slice round trip
                float v[64];
#pragma unroll
                for (int q = 0; q < 64; ++q) v[q] = 0.0f;
                for (int s = 0; s < x.nseg; ++s) {
                  if (s == x.seg) {
                    uint32_t r0[32], r1[32];
                    tmem_ld_32x32b_x32(tl + c * 32, r0);
                    tmem_ld_32x32b_x32(tl + c * 32 + 32, r1);
                    tmem_ld_wait();
#pragma unroll
                    for (int q = 0; q < 32; ++q) {
                      v[q] += __uint_as_float(r0[q]);
                      v[32 + q] += __uint_as_float(r1[q]);
                    }
                  } else if (valid && !(p.debug & 16)) {
                    const float4* s4 = reinterpret_cast<const float4*>(src + s * slice + 32 * c);
                    float4 t[16];
#pragma unroll
                    for (int g = 0; g < 16; ++g) t[g] = __ldcg(s4 + g);
#pragma unroll
                    for (int g = 0; g < 16; ++g) {
                      v[4 * g] += t[g].x; v[4 * g + 1] += t[g].y; v[4 * g + 2] += t[g].z; v[4 * g + 3] += t[g].w;
                    }
                  }
                }
                uint32_t w0[32], w1[32];
#pragma unroll
                for (int q = 0; q < 32; ++q) {
                  w0[q] = __float_as_uint(v[q]);
                  w1[q] = __float_as_uint(v[32 + q]);
                }
                tmem_st_32x32b_x32(tl + c * 32, w0);
                tmem_st_32x32b_x32(tl + c * 32 + 32, w1);
              }
              tmem_st_wait();
              qkv_sw_row(p, m, valid, pos_m, fbase, nlim, tl, sg);
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[acc]), 0));
          continue;
        }
        unsigned long long best = 0ull;
        for (int c = 0; c < nch; ++c) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(tl + c * 32, r);
          tmem_ld_wait();
          if (c == nch - 1) {   // last TMEM read of this accumulator: hand it back early
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[acc]), 0));
          }
          const int n0 = fbase + c * 32;
          if (m < p.M) {
            if (x.nseg > 1 || p.partial_all) {
              // k-range partial of this token row -> ws[seg][m][n0 .. n0+31], straight from
              // registers (TMEM lanes are tokens: 128 contiguous bytes per thread)
              float* dst = p.ws + (size_t)x.seg * p.M * p.N + (size_t)m * p.N;
#pragma unroll
              for (int g = 0; g < 8; ++g) {
                const int n = n0 + 4 * g;
                if (n < nlim)
                  __stcg(reinterpret_cast<float4*>(dst + n),
                         make_float4(__uint_as_float(r[4 * g]), __uint_as_float(r[4 * g + 1]),
                                     __uint_as_float(r[4 * g + 2]), __uint_as_float(r[4 * g + 3])));
              }
            } else {
              store_row<EPI>(p, r, m, n0, nlim, best);
            }
          }
        }
        if (nch <= 0) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[acc]), 0));
        }
        if constexpr (EPI == EPI_ARGMAX) {
          if (m < p.M && best) atomicMax(reinterpret_cast<unsigned long long*>(p.out) + m, best);
        }
      }
    } else {
      int un = 0;
      UnitIter ui;
      ui.init(p, cluster);
      Unit x;
      while (ui.next(p, cluster, x)) {
        const int acc = un & 1;
        const uint32_t aph = (un >> 1) & 1;
        ++un;
        const int n0 = x.ft * 2 * WROWS + rank * WROWS;
        const int pt = x.ft * 2 + rank;
        const int mbase = x.mt * BNT;
        const int nchunks = min(BNT, ((p.M - mbase + 31) / 32) * 32) / 32;
        // partial of a split tile: a full [M][N] slice per segment, or (compact) this cluster's
        // tile buffer [BNT tokens][256 features] of its first / last stream-K unit
        float* part = p.compact ? p.ws + ((size_t)cluster * 2 + x.slot) * (size_t)(2 * WROWS) * BNT
                                : p.ws + (size_t)x.seg * p.M * p.N;
        mbar_wait(&tfull[acc], aph);
        tc_fence_after();
        const uint32_t tl = tmem_base + acc * ACCS + ((uint32_t)(quarter * 32) << 16);
        for (int c = 0; c < nchunks; ++c) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(tl + c * 32, r);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) stg[j * SROW + row] = __uint_as_float(r[j]);
          if (c == nchunks - 1) {   // last TMEM read of this accumulator: hand it back early
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[acc]), 0));
          }
          named_bar_sync(1, 128);
          if (x.nseg == 1 && !p.partial_all) {
            store_phase<EPI>(p, stg, mbase + c * 32, n0, pt, tid);
          } else {
            // partial of this k-range -> ws[seg][m][n] (token-major, coalesced 16-byte stores)
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int v = tid + 128 * i, j = v >> 5, f = (v & 31) * 4;
              const int m = mbase + c * 32 + j, n = n0 + f;
              if (m < p.M && n < p.N) {
                float* dst = p.compact ? part + (size_t)(c * 32 + j) * (2 * WROWS) + rank * WROWS + f
                                       : part + (size_t)m * p.N + n;
                __stcg(reinterpret_cast<float4*>(dst), *reinterpret_cast<const float4*>(stg + j * SROW + f));
              }
            }
          }
          named_bar_sync(1, 128);
        }
        if (nchunks == 0) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[acc]), 0));
        }
      }
    }
    if (tid == 0) SIDP_TL(4);
  }
  if (warp == 2 && lane == 0) SIDP_TL(5);
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc2(tmem_base, tmem_cols);
  }
  if (threadIdx.x == 0) SIDP_TL(6);
  if (p.post.n) post_after_grid(p.post);
}

// Stream-K fix-up over all SMs: for tiles covered by several k-range segments, each thread sums
// 8 consecutive outputs of one token row across the segment slices in order 0..nseg-1
// (deterministic), then applies EPI.  Tiles finished inside the GEMM are skipped.
template <int EPI>
SIDP_DEV void reduce_body(const KParams& p) {
  // blockIdx.y = cluster boundary c (1..C-1); the tile containing b_c strictly inside is fixed
  // up by the block row of the first boundary that splits it.
  const long long nkb = p.nks;
  const int c = blockIdx.y + 1;
  const long long bc = range_begin(c, p.total_kb, p.sk);
  const int tl = (int)(bc / nkb);                             // tile within the stream-K region
  if (bc % nkb == 0) return;                                  // boundary on a tile edge
  if (c > 1 && range_begin(c - 1, p.total_kb, p.sk) > (long long)tl * nkb) return;
  const int first = cluster_of_kb((long long)tl * nkb, p.total_kb, p.sk);
  const int nseg = cluster_of_kb((long long)(tl + 1) * nkb - 1, p.total_kb, p.sk) - first + 1;
  const int t = p.dp_tiles + tl;
  const int mt = t % p.m_tiles, ft = t / p.m_tiles;
  const int m0 = mt * p.BNT, rows = min(p.BNT, p.M - m0);
  const int tile_out = EPI == EPI_SILU_MUL ? 2 * WROWS / 2 : 2 * WROWS;   // outputs per row
  const int out0 = EPI == EPI_SILU_MUL ? ft * WROWS : ft * 2 * WROWS;
  const int n_out = EPI == EPI_SILU_MUL ? p.N / 2 : p.N;
  const int vec_per_row = tile_out / 8;
  const size_t slice = (size_t)p.M * p.N;
  // compact slot of segment s: 0 when its cluster's range starts inside this tile — every
  // s > 0 — else 1 (the first cluster's range began in an earlier tile and ends here)
  const int slot0 = p.compact && range_begin(first, p.total_kb, p.sk) < (long long)tl * nkb ? 1 : 0;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < rows * vec_per_row;
       idx += gridDim.x * blockDim.x) {
    const int m = m0 + idx / vec_per_row;
    const int f = out0 + (idx % vec_per_row) * 8;
    if (f >= n_out) continue;
    float a[8], b[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] = b[q] = 0.0f;
    int na = f, nb = 0;
    if constexpr (EPI == EPI_SILU_MUL) {
      na = 2 * f;                       // gate rows of 16-row group f/8 (f multiple of 8)
      nb = na + 8;                      // matching up rows
    }
    const float* base = p.ws + (size_t)m * p.N;
#pragma unroll 4
    for (int s = 0; s < nseg; ++s) {
      // segment s = cluster first + s: its full slice, or (compact) its tile buffer — slot 0
      // when its stream-K range starts inside this tile, else 1 (the range ends here)
      const float* src = base + s * slice;
      if (p.compact) {
        const int cs = first + s;
        const int slot = s == 0 ? slot0 : 0;
        src = p.ws + ((size_t)cs * 2 + slot) * (size_t)(2 * WROWS) * p.BNT +
              (size_t)(m - m0) * (2 * WROWS) - (size_t)ft * 2 * WROWS;
      }
      const float4 x0 = __ldcg(reinterpret_cast<const float4*>(src + na));
      const float4 x1 = __ldcg(reinterpret_cast<const float4*>(src + na + 4));
      a[0] += x0.x; a[1] += x0.y; a[2] += x0.z; a[3] += x0.w;
      a[4] += x1.x; a[5] += x1.y; a[6] += x1.z; a[7] += x1.w;
      if constexpr (EPI == EPI_SILU_MUL) {
        const float4 y0 = __ldcg(reinterpret_cast<const float4*>(src + nb));
        const float4 y1 = __ldcg(reinterpret_cast<const float4*>(src + nb + 4));
        b[0] += y0.x; b[1] += y0.y; b[2] += y0.z; b[3] += y0.w;
        b[4] += y1.x; b[5] += y1.y; b[6] += y1.z; b[7] += y1.w;
      }
    }
    if constexpr (EPI == EPI_F32) {
      if (p.bias) {
        float y[8];
        unpack_bf16x8(*reinterpret_cast<const uint4*>(p.bias + f), y);
#pragma unroll
        for (int q = 0; q < 8; ++q) a[q] += y[q];
      }
      float* out = out_row<float>(p, m) + f;
      *reinterpret_cast<float4*>(out) = make_float4(a[0], a[1], a[2], a[3]);
      *reinterpret_cast<float4*>(out + 4) = make_float4(a[4], a[5], a[6], a[7]);
    } else if constexpr (EPI == EPI_BF16 || EPI == EPI_RESID) {
      float y[8];
      if constexpr (EPI == EPI_RESID) {
        unpack_bf16x8(*reinterpret_cast<const uint4*>(p.resid + (size_t)m * p.ldr + f), y);
      } else if (p.bias) {
        unpack_bf16x8(*reinterpret_cast<const uint4*>(p.bias + f), y);
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) y[q] = 0.0f;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) a[q] += y[q];
      *reinterpret_cast<uint4*>(out_row<bf16>(p, m) + f) = pack_bf16x8(a);
    } else if constexpr (EPI == EPI_SILU_MUL) {
#pragma unroll
      for (int q = 0; q < 8; ++q) a[q] = a[q] / (1.0f + __expf(-a[q])) * b[q];
      *reinterpret_cast<uint4*>(reinterpret_cast<bf16*>(p.out) + (size_t)m * p.ldo + f) =
          pack_bf16x8(a);
    }
  }
}

template <int EPI>
__global__ void __launch_bounds__(256) gemm_reduce_kernel(const KParams p) {
  pdl_trigger();
  pdl_wait();
  reduce_body<EPI>(p);
  if (p.post.n) post_after_grid(p.post);
}

// ---------------------------------------------------------------- fused MLP (gate/up -> down)
// One persistent launch runs the layer's gate/up GEMM (whole 256-feature tiles, SiLU*mul epilogue
// -> act) and its down GEMM (k-range units, fp32 partial slices summed later by resid_norm).
// Down k-step k reads act features [128k, 128k+128), produced by gate/up tile k: the TMA
// producer waits on that tile's completion counter (both CTAs of its pair add 1 after their
// stores) before loading the act k-block, so down work fills the CTA pairs that the last,
// partial gate/up wave leaves idle (200 tiles on 74 pairs: 22 pairs idle for a whole tile
// time) instead of waiting for a kernel boundary.  The unit lists are host-built by list
// scheduling (mlp_schedule).  All co-dependent CTAs are of this grid, which depends on nothing
// launched after it: the PDL trigger is issued at exit, so no successor can take SM resources
// from a not-yet-resident CTA of this grid.
struct MlpParams {
  int M, N1, K1, N2, K2;         // gate/up [N1 = 2I][K1 = h]; down [N2 = h][K2 = I]
  int BNT, stages, MT;           // MT token tiles of BNT rows
  const int4* units;             // {phase | seg << 8 | mt << 16, tile, kb0, kb1}; pair c: [uoff[c], uoff[c+1])
  const int* uoff;
  bf16* act; int ldact;          // [M][I]
  float* ws;                     // down partials [seg][M][N2]
  int* flags;                    // [N1 / 256][MT] gate/up tile completion counters (0 between launches)
  unsigned int* done;            // CTA exit counter (the last CTA resets the flags)
  int n_flags;
};

SIDP_DEV int ld_acquire_gpu_s32(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
mlp2_kernel(const __grid_constant__ CUtensorMap tm_w1, const __grid_constant__ CUtensorMap tm_x1,
            const __grid_constant__ CUtensorMap tm_w2, const __grid_constant__ CUtensorMap tm_x2,
            const MlpParams p) {
  constexpr int KPS = 2;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const int stages = p.stages, BNT = p.BNT, HALF = p.BNT / 2;
  const uint32_t a_sub = WROWS * BK * 2, b_sub = (uint32_t)HALF * BK * 2;
  const uint32_t a_bytes = KPS * a_sub, b_bytes = KPS * b_sub;
  uint8_t* sA = smem;
  uint8_t* sB = sA + (size_t)stages * a_bytes;
  float* stg = reinterpret_cast<float*>(sB + (size_t)stages * b_bytes);   // [32][SROW]
  uint64_t* full = reinterpret_cast<uint64_t*>(stg + 32 * SROW);
  uint64_t* empty = full + stages;
  uint64_t* tfull = empty + stages;                      // [2]
  uint64_t* tempty = tfull + 2;                          // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int cluster = blockIdx.x >> 1;
  const int ACCS = (BNT + 31) / 32 * 32;
  const uint32_t tmem_cols = ACCS <= 32 ? 64 : (ACCS <= 64 ? 128 : (ACCS <= 128 ? 256 : 512));
  const int u0 = p.uoff[cluster], u1 = p.uoff[cluster + 1];

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tm_w1);
    tma_prefetch_desc(&tm_x1);
    tma_prefetch_desc(&tm_w2);
    tma_prefetch_desc(&tm_x2);
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 8);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc2(tmem_slot, tmem_cols);
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x != 0) pdl_wait();

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    if (lane == 0) {
      const uint32_t stage_tx = 2 * (a_bytes + b_bytes);
      const uint64_t wpol = policy_evict_first();
      auto issue = [&](const int4 un, int kb, int s, bool pre) {
        const int phase = un.x & 0xff, mt = (un.x >> 16) & 0xffff;
        const uint32_t lbar = mapa_shared(smem_u32(&full[s]), 0);
        const CUtensorMap* tw = phase ? &tm_w2 : &tm_w1;
        const CUtensorMap* tx = phase ? &tm_x2 : &tm_x1;
        const int arow = un.y * 2 * WROWS + rank * WROWS;
#pragma unroll
        for (int j = 0; j < KPS; ++j)
          tma_load_2d_2sm_hint(tw, lbar, sA + (size_t)s * a_bytes + j * a_sub, (kb * KPS + j) * BK, arow, wpol);
        if (pre) return;
        if (phase) {   // act k-block kb is gate/up tile (kb, mt)'s output: wait until both CTAs stored it
          while (ld_acquire_gpu_s32(p.flags + kb * p.MT + mt) < 2) __nanosleep(64);
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
#pragma unroll
        for (int j = 0; j < KPS; ++j)
          tma_load_2d_2sm(tx, lbar, sB + (size_t)s * b_bytes + j * b_sub, (kb * KPS + j) * BK,
                          mt * BNT + rank * HALF);
      };
      // the first stages' weight tiles before griddepcontrol.wait (weights are resident)
      int npre = 0;
      {
        int ui = u0, kb = ui < u1 ? p.units[ui].z : 0;
        for (; npre < stages && ui < u1; ++npre) {
          if (leader) mbar_arrive_expect_tx(&full[npre], stage_tx);
          issue(p.units[ui], kb, npre, true);
          if (++kb >= p.units[ui].w && ++ui < u1) kb = p.units[ui].z;
        }
      }
      pdl_wait();
      int it = 0;
      for (int ui = u0; ui < u1; ++ui) {
        const int4 un = p.units[ui];
        for (int kb = un.z; kb < un.w; ++kb, ++it) {
          const int s = it % stages;
          const uint32_t ph = (it / stages) & 1;
          if (it >= npre) {
            mbar_wait(&empty[s], ph ^ 1);
            if (leader) mbar_arrive_expect_tx(&full[s], stage_tx);
            issue(un, kb, s, false);
          } else {   // weight half already in flight: the activation half now
            const int phase = un.x & 0xff, mt = (un.x >> 16) & 0xffff;
            const uint32_t lbar = mapa_shared(smem_u32(&full[s]), 0);
            const CUtensorMap* tx = phase ? &tm_x2 : &tm_x1;
            if (phase) {
              while (ld_acquire_gpu_s32(p.flags + kb * p.MT + mt) < 2) __nanosleep(64);
              asm volatile("fence.proxy.async.global;" ::: "memory");
            }
#pragma unroll
            for (int j = 0; j < KPS; ++j)
              tma_load_2d_2sm(tx, lbar, sB + (size_t)s * b_bytes + j * b_sub, (kb * KPS + j) * BK,
                              mt * BNT + rank * HALF);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader only)
    if (leader) {
      const uint32_t idesc = umma_idesc_bf16(2 * WROWS, BNT);
      int it = 0, un_i = 0;
      for (int ui = u0; ui < u1; ++ui, ++un_i) {
        const int4 un = p.units[ui];
        const int acc = un_i & 1;
        const uint32_t aph = (un_i >> 1) & 1;
        mbar_wait(&tempty[acc], aph ^ 1);
        tc_fence_after();
        const uint32_t dcol = tmem_base + acc * ACCS;
        for (int kb = un.z; kb < un.w; ++kb, ++it) {
          const int s = it % stages;
          const uint32_t ph = (it / stages) & 1;
          mbar_wait(&full[s], ph);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t a0 = smem_u32(sA + (size_t)s * a_bytes);
            const uint32_t b0 = smem_u32(sB + (size_t)s * b_bytes);
#pragma unroll
            for (int j = 0; j < KPS; ++j) {
#pragma unroll
              for (int k = 0; k < BK / 16; ++k)
                umma2_bf16(dcol, umma_desc_sw128(a0 + j * a_sub + k * 32),
                           umma_desc_sw128(b0 + j * b_sub + k * 32), idesc,
                           (kb > un.z || j > 0 || k > 0) ? 1u : 0u);
            }
            umma2_commit_mc(&empty[s]);
          }
          __syncwarp();
        }
        if (lane == 0) umma2_commit_mc(&tfull[acc]);
        __syncwarp();
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (both CTAs)
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const int tid = (warp - 2) * 32 + lane;
    KParams kp{};   // the SiLU*mul store of store_phase
    kp.M = p.M; kp.N = p.N1; kp.out = p.act; kp.ldo = p.ldact;
    int un_i = 0;
    for (int ui = u0; ui < u1; ++ui, ++un_i) {
      const int4 un = p.units[ui];
      const int phase = un.x & 0xff, seg = (un.x >> 8) & 0xff, mt = (un.x >> 16) & 0xffff;
      const int mbase = mt * BNT;
      const int nchunks = min(BNT, ((p.M - mbase + 31) / 32) * 32) / 32;
      const int acc = un_i & 1;
      const uint32_t aph = (un_i >> 1) & 1;
      const int n0 = un.y * 2 * WROWS + rank * WROWS;
      const int pt = un.y * 2 + rank;
      float* part = p.ws + (size_t)seg * p.M * p.N2;
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      const uint32_t tl = tmem_base + acc * ACCS + ((uint32_t)(quarter * 32) << 16);
      for (int c = 0; c < nchunks; ++c) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(tl + c * 32, r);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) stg[j * SROW + row] = __uint_as_float(r[j]);
        if (c == nchunks - 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[acc]), 0));
        }
        named_bar_sync(1, 128);
        if (phase == 0) {
          store_phase<EPI_SILU_MUL>(kp, stg, mbase + c * 32, n0, pt, tid);
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int v = tid + 128 * i, j = v >> 5, f = (v & 31) * 4;
            const int m = mbase + c * 32 + j, n = n0 + f;
            if (m < p.M && n < p.N2)
              __stcg(reinterpret_cast<float4*>(part + (size_t)m * p.N2 + n),
                     *reinterpret_cast<const float4*>(stg + j * SROW + f));
          }
        }
        named_bar_sync(1, 128);
      }
      if (phase == 0) {   // this CTA's half of gate/up tile un.y is stored: publish it
        __threadfence();
        named_bar_sync(1, 128);
        if (tid == 0) atomicAdd(p.flags + un.y * p.MT + mt, 1);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc2(tmem_base, tmem_cols);
  }
  if (threadIdx.x == 0) {   // the last CTA out resets the tile counters for the next launch
    __threadfence();
    if (atomicAdd(p.done, 1u) == gridDim.x - 1) {
      for (int i = 0; i < p.n_flags; ++i) p.flags[i] = 0;
      *p.done = 0u;
      __threadfence();
    }
  }
  pdl_trigger();
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

// Row-major [rows x K] bf16 viewed as {64 (k in block), rows, K/64 (k-block)} with strides
// {ld, 128 B}: a box {64, box_rows, kps} lands as kps canonical SW128 K-major tiles back to back.
bool make_tmap_3d(CUtensorMap* m, const void* base, uint64_t K, uint64_t rows, uint64_t ld_elems,
                  uint32_t box_rows, uint32_t kps) {
  EncodeTiledFn fn = get_encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {64, rows, K / 64};
  cuuint64_t strides[2] = {ld_elems * 2, 128};
  cuuint32_t box[3] = {64, box_rows, kps};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
                  box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// k-block-major [K/64][rows][64] bf16 (each 64-wide k-block slab of all rows contiguous):
// {64, rows, K/64} with strides {128 B, rows * 128 B}; a box {64, box_rows, kps} lands as kps
// canonical SW128 K-major tiles back to back.
bool make_tmap_kbmajor(CUtensorMap* m, const void* base, uint64_t K, uint64_t rows,
                       uint32_t box_rows, uint32_t kps) {
  EncodeTiledFn fn = get_encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {64, rows, K / 64};
  cuuint64_t strides[2] = {128, rows * 128};
  cuuint32_t box[3] = {64, box_rows, kps};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
                  box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
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
thread_local int g_last_launches = 0;

// the token-major variant exists for every epilogue
template <int EPI>
constexpr bool kHasSw = true;

// EPI_PARTIAL launch geometry (shared by gemm_launch and gemm_partial_ok): W-major, token tile =
// M rounded up to 32 (<= 256), partials staged through shared memory into coalesced rows.
// SIDP_GEMM_PART_SW_MIN_M = m > 0 switches to token-major from m tokens up (feature tile 256,
// each thread stores its token row's partial straight from registers) — measured slower on
// the M2 O / down shapes (O 48.7 vs 35 us live), so off by default.
struct PartialPlan {
  bool sw;
  int BNT, m_tiles, n_pairs, tiles, clusters, nkb, kps;
  long long total;
  int max_seg;
};
PartialPlan plan_partial(int M, int N, int K, int pair_slots) {
  static int env_sw_min = getenv("SIDP_GEMM_PART_SW_MIN_M") ? atoi(getenv("SIDP_GEMM_PART_SW_MIN_M")) : 0;
  static int env_bnf = getenv("SIDP_GEMM_PART_BNF") ? atoi(getenv("SIDP_GEMM_PART_BNF")) : 256;
  PartialPlan q{};
  const int nkb_blocks = K / BK;
  q.kps = nkb_blocks % 2 == 0 ? 2 : 1;
  q.nkb = nkb_blocks / q.kps;
  q.sw = env_sw_min > 0 && M >= env_sw_min;
  if (q.sw) {
    q.BNT = (env_bnf >= 32 && env_bnf <= 256 && env_bnf % 32 == 0) ? env_bnf : 256;
    q.m_tiles = (N + q.BNT - 1) / q.BNT;
    q.n_pairs = (M + 2 * WROWS - 1) / (2 * WROWS);
  } else {
    q.BNT = std::max(32, std::min(256, ((M + 31) / 32) * 32));
    q.m_tiles = (M + q.BNT - 1) / q.BNT;
    q.n_pairs = (N + 2 * WROWS - 1) / (2 * WROWS);
  }
  q.tiles = q.n_pairs * q.m_tiles;
  q.clusters = pair_slots;
  q.total = (long long)q.tiles * q.nkb;
  long long per = q.total / q.clusters;
  if (per < 2) {
    q.clusters = (int)std::max<long long>(1, q.total / 2);
    per = q.total / q.clusters;
  }
  q.max_seg = (int)((q.nkb + per - 1) / std::max<long long>(per, 1)) + 1;
  return q;
}

// Token-major fused-QKV geometry (SW EPI_QKV): feature tiles of whole heads (BNF = hd, or
// SIDP_QKV_BNF), 256-token pair tiles, stream-K over every CTA pair (the head-aligned tile
// count rarely divides the pair count: 80 heads of Qwen3 / Llama on 74 pairs); split tiles go
// through fp32 slices [seg][M][N] and an in-kernel last-arriver fix-up.
struct QkvSwPlan {
  bool ok;
  int BNT, m_tiles, n_pairs, tiles, clusters, nkb, max_seg;
  long long total;
};
constexpr int kQkvCntOff = 1 << 15;   // counters [kQkvCntOff, +2 tiles): split-tile arrivals
QkvSwPlan plan_qkv_sw(int M, int N, int K, int hd, int pair_slots, size_t ws_bytes, int n_counters) {
  static int env_min = getenv("SIDP_QKV_SW_MIN_M") ? atoi(getenv("SIDP_QKV_SW_MIN_M")) : 128;
  static int env_bnf = getenv("SIDP_QKV_BNF") ? atoi(getenv("SIDP_QKV_BNF")) : 0;
  QkvSwPlan q{};
  if (env_min <= 0 || M < env_min || (hd != 64 && hd != 128) || N % hd || K % BK) return q;
  const int nkb_blocks = K / BK;
  const int kps = nkb_blocks % 2 == 0 ? 2 : 1;
  q.nkb = nkb_blocks / kps;
  q.BNT = (env_bnf > 0 && env_bnf % hd == 0 && env_bnf <= 256) ? env_bnf : hd;
  q.m_tiles = N / q.BNT;
  q.n_pairs = (M + 2 * WROWS - 1) / (2 * WROWS);
  q.tiles = q.m_tiles * q.n_pairs;
  q.clusters = pair_slots;
  q.total = (long long)q.tiles * q.nkb;
  long long per = q.total / q.clusters;
  if (per < 2) {
    q.clusters = (int)std::max<long long>(1, q.total / 2);
    per = q.total / q.clusters;
  }
  q.max_seg = (int)((q.nkb + per - 1) / std::max<long long>(per, 1)) + 1;
  q.ok = (size_t)q.max_seg * M * N * 4 <= ws_bytes && kQkvCntOff + 2 * q.tiles <= n_counters;
  return q;
}

template <int EPI>
void set_attr() {
  cudaFuncSetAttribute(gemm2_kernel<EPI, 1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       kSmemBudget + 1024);
  cudaFuncSetAttribute(gemm2_kernel<EPI, 2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       kSmemBudget + 1024);
  if constexpr (kHasSw<EPI>) {
    cudaFuncSetAttribute(gemm2_kernel<EPI, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kSmemBudget + 1024);
    cudaFuncSetAttribute(gemm2_kernel<EPI, 2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kSmemBudget + 1024);
  }
}

template <int EPI>
cudaError_t launch_gemm2(int kps, bool sw, dim3 grid, size_t smem, cudaStream_t st,
                         const CUtensorMap& tw, const CUtensorMap& tx, const KParams& p) {
  if constexpr (kHasSw<EPI>) {
    if (sw) {
      if (kps == 2) return launch_pdl(gemm2_kernel<EPI, 2, true>, grid, dim3(kThreads), smem, st, tw, tx, p);
      return launch_pdl(gemm2_kernel<EPI, 1, true>, grid, dim3(kThreads), smem, st, tw, tx, p);
    }
  }
  if (sw) return cudaErrorInvalidValue;
  if (kps == 2) return launch_pdl(gemm2_kernel<EPI, 2, false>, grid, dim3(kThreads), smem, st, tw, tx, p);
  return launch_pdl(gemm2_kernel<EPI, 1, false>, grid, dim3(kThreads), smem, st, tw, tx, p);
}

}  // namespace

int gemm_pick_splits(int tiles, int nkb, int slots) {
  // tiles = pair-units without split; slots = concurrent pairs.  Cost ~ waves x (k-blocks + c).
  if (tiles >= slots) return 1;
  int best = 1;
  double best_t = 1e30;
  for (int s = 1; s <= 16; ++s) {
    const int per = (nkb + s - 1) / s;
    if (per < 4 && s > 1) break;
    const int waves = (tiles * s + slots - 1) / slots;
    const double t = waves * (per + 6.0) + (s > 1 ? 2.0 : 0.0);
    if (t < best_t - 1e-9) {
      best_t = t;
      best = s;
    }
  }
  return best;
}

int gemm_last_launch_count() { return g_last_launches; }

static int device_sms() {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return g_num_sms;
}

// SMs the compute kernels size their grids for (see kernels.h set_compute_sms): the device's
// count, or fewer while a WaS fetch kernel holds dedicated SMs.  Even, so CTA pairs fill it.
static thread_local int g_sm_budget = 0;
void set_compute_sms(int n) { g_sm_budget = n; }
int get_compute_sms_budget() { return g_sm_budget; }
int compute_sms() {
  static const int env = getenv("SIDP_SM_BUDGET") ? atoi(getenv("SIDP_SM_BUDGET")) : 0;
  int n = device_sms();
  const int b = g_sm_budget > 0 ? g_sm_budget : env;
  if (b > 0 && b < n) n = std::max(2, b & ~1);
  return n;
}
static int num_sms() { return compute_sms(); }

bool gemm_partial_ok(int M, int N, int K, size_t ws_bytes) {
  static int env = getenv("SIDP_GEMM_PARTIAL") ? atoi(getenv("SIDP_GEMM_PARTIAL")) : 1;
  if (!env || M <= 0 || N <= 0 || K % BK != 0 || N % 8 != 0) return false;
  const int pair_slots = std::max(1, num_sms() / 2);
  const long long wm_tiles = (long long)((N + 2 * WROWS - 1) / (2 * WROWS)) * ((M + 255) / 256);
  // Whole tiles that fill the machine need no split and no fix-up, unless their last wave
  // leaves most pairs idle (tile-quantisation efficiency below SIDP_GEMM_PARTIAL_EFF, default
  // 0.6) with too little tail work for gemm_launch's hybrid stream-K tail (the same test as
  // there): e.g. O at M = 1024, 80 tiles on 74 pairs, 125 -> 76 us per layer.
  static double env_eff = getenv("SIDP_GEMM_PARTIAL_EFF") ? atof(getenv("SIDP_GEMM_PARTIAL_EFF")) : 0.6;
  if (wm_tiles >= pair_slots) {
    const long long waves = (wm_tiles + pair_slots - 1) / pair_slots;
    const long long rem = wm_tiles % pair_slots;
    const int nkb_blocks = K / BK;
    const int nkb = nkb_blocks % 2 == 0 ? nkb_blocks / 2 : nkb_blocks;
    const double eff = (double)wm_tiles / (double)(waves * pair_slots);
    if (!(rem != 0 && eff < env_eff && rem * nkb < 12LL * pair_slots)) return false;
  }
  const PartialPlan q = plan_partial(M, N, K, pair_slots);
  return q.tiles <= kPartialMaxTiles && q.max_seg <= 255 && (size_t)q.max_seg * M * N * 4 <= ws_bytes;
}

cudaError_t gemm_launch(const GemmArgs& a, const GemmWorkspace& w, cudaStream_t stream) {
  g_last_launches = 0;
  if (a.M <= 0) return cudaSuccess;
  if (a.K % BK != 0 || a.N <= 0 || a.N % 8 != 0 || a.x == nullptr || a.w == nullptr)
    return cudaErrorInvalidValue;
  if (a.epi == EPI_SILU_MUL && (a.N % 16) != 0) return cudaErrorInvalidValue;
  static unsigned long long attrs = 0;
  if (first_on_device(attrs)) {
    num_sms();
    set_attr<EPI_PARTIAL>();
    set_attr<EPI_F32>();
    set_attr<EPI_BF16>();
    set_attr<EPI_RESID>();
    set_attr<EPI_SILU_MUL>();
    set_attr<EPI_ARGMAX>();
    set_attr<EPI_QKV>();
  }
  static int env_bnt = getenv("SIDP_GEMM_BNT") ? atoi(getenv("SIDP_GEMM_BNT")) : 256;
  static int env_stages = getenv("SIDP_GEMM_STAGES") ? atoi(getenv("SIDP_GEMM_STAGES")) : 12;
  // token-major (SW) orientation from this many tokens up (0 = never); X-tile overhead in
  // equivalent W rows for the feature-tile choice
  static int env_sw_min = getenv("SIDP_GEMM_SW_MIN_M") ? atoi(getenv("SIDP_GEMM_SW_MIN_M")) : 128;
  static int env_sw_c0 = getenv("SIDP_GEMM_SW_C0") ? atoi(getenv("SIDP_GEMM_SW_C0")) : 64;
  static int env_sw_bnf = getenv("SIDP_GEMM_SW_BNF") ? atoi(getenv("SIDP_GEMM_SW_BNF")) : 0;
  const int sms = a.max_ctas > 0 ? std::min(a.max_ctas, num_sms()) : num_sms();
  const int pair_slots = std::max(1, sms / 2);
  const int nkb_blocks = a.K / BK;
  static int env_kps = getenv("SIDP_GEMM_KPS") ? atoi(getenv("SIDP_GEMM_KPS")) : 2;
  const int kps = (env_kps == 2 && nkb_blocks % 2 == 0) ? 2 : 1;
  const int nkb = nkb_blocks / kps;   // k-steps per tile (the unit of stream-K work)
  if (a.epi == EPI_QKV && (!a.qkv || (a.qkv->hd != 64 && a.qkv->hd != 128))) return cudaErrorInvalidValue;
  // SW pays where whole 256-feature tiles would leave CTA pairs idle but are too many for
  // stream-K (e.g. QKV: 40 tiles on 74 pairs): the token tile is re-read per feature tile
  // (256/BNF x the W traffic from L2), so shapes that already fill the machine stay W-major.
  // SIDP_GEMM_SW = 0 never, 1 auto (default), 2 whenever M >= SIDP_GEMM_SW_MIN_M.
  static int env_sw = getenv("SIDP_GEMM_SW") ? atoi(getenv("SIDP_GEMM_SW")) : 1;
  const int wm_tiles = ((a.N + 2 * WROWS - 1) / (2 * WROWS)) *
                       ((a.M + std::min(256, env_bnt) - 1) / std::min(256, env_bnt));
  const bool underfilled = 2 * wm_tiles > pair_slots && wm_tiles < pair_slots;
  // Badly quantised whole W-major tiles whose tail is too small for the hybrid stream-K tail
  // below (e.g. QKV at M = 512: 80 tiles on 74 pairs, ~2 waves for 1.08 waves of work): SW
  // when its own rounds x (BNF + c0) cost is clearly lower (144 tiles of 144 features: 65.7 ->
  // 60.1 us).
  bool quantised = false;
  if (wm_tiles > pair_slots && a.epi != EPI_ARGMAX && a.epi != EPI_PARTIAL) {
    const int waves = (wm_tiles + pair_slots - 1) / pair_slots;
    const int rem = wm_tiles % pair_slots;
    const double eff = (double)wm_tiles / ((double)waves * pair_slots);
    if (rem != 0 && eff < 0.6 && (long long)rem * nkb < 12LL * pair_slots) {
      const int tok_pairs = (a.M + 2 * WROWS - 1) / (2 * WROWS);
      double best_c = 1e30;
      for (int bnf = 256; bnf >= 32; bnf -= 16) {
        const long long t = (long long)tok_pairs * ((a.N + bnf - 1) / bnf);
        best_c = std::min(best_c, (double)((t + pair_slots - 1) / pair_slots) * (bnf + env_sw_c0));
      }
      quantised = best_c < 0.85 * waves * (256 + env_sw_c0);
    }
  }
  bool sw = a.k_splits < 0 ? a.epi != EPI_QKV
                                  : (env_sw > 0 && env_sw_min > 0 && a.M >= env_sw_min &&
                                     a.epi != EPI_QKV && a.k_splits <= 1 &&
                                     (env_sw == 2 || underfilled || quantised));
  int BNT, m_tiles, n_pairs;
  if (sw) {
    // feature tile BNF (UMMA N, multiple of 16) minimising rounds x (BNF + c0): whole tiles
    // on every pair without splitting K (cost ~ W rows + the re-read token tile per tile)
    const int tok_pairs = (a.M + 2 * WROWS - 1) / (2 * WROWS);
    int best = 256;
    double best_c = 1e30;
    // BNF multiple of 16 (UMMA N for M = 256); each CTA supplies BNF/2 B rows, whole 8-row
    // SW128 core-matrix groups.  (BNF = 80 once gave wrong results: the epilogue's last
    // 32-column chunk stored past the tile end into the next tile; it now stops at nlim.)
    for (int bnf = 256; bnf >= 32; bnf -= 16) {
      const long long t = (long long)tok_pairs * ((a.N + bnf - 1) / bnf);
      const double c = (double)((t + pair_slots - 1) / pair_slots) * (bnf + env_sw_c0);
      if (c < best_c - 1e-9) { best_c = c; best = bnf; }
    }
    if (env_sw_bnf >= 32 && env_sw_bnf <= 256 && env_sw_bnf % 16 == 0) best = env_sw_bnf;
    BNT = best;
    m_tiles = (a.N + BNT - 1) / BNT;   // feature tiles (fastest)
    n_pairs = tok_pairs;               // token-pair tiles
  } else {
    BNT = ((a.M + 31) / 32) * 32;
    BNT = std::max(32, std::min(env_bnt, BNT));
    m_tiles = (a.M + BNT - 1) / BNT;
    n_pairs = (a.N + 2 * WROWS - 1) / (2 * WROWS);
  }
  QkvSwPlan qs{};
  if (a.epi == EPI_QKV && a.k_splits != 1 && a.k_splits >= 0 && !a.wait && !a.scatter) {
    qs = plan_qkv_sw(a.M, a.N, a.K, a.qkv->hd, pair_slots, w.ws_bytes, w.n_counters);
    if (qs.ok) {
      sw = true;
      BNT = qs.BNT; m_tiles = qs.m_tiles; n_pairs = qs.n_pairs;
    }
  }
  int tiles = n_pairs * m_tiles;
  // stream-K over all pairs unless the epilogue needs whole dot products (fused argmax) or the
  // caller pins whole tiles (k_splits == 1); max segments per tile bounds the workspace
  int clusters = pair_slots;
  // whole tiles balance well once every pair has >= 1 tile (measured: qkv 40 tiles, gate/up
  // 200 tiles faster whole); stream-K pays off for heavily underfilled shapes (O, down: 20)
  // whole-row epilogues (argmax over a tile, per-head qk-norm/RoPE) need whole dot products
  // (Stream-K for badly quantised larger tile counts — e.g. down at M = 1024: 80 tiles on 74
  // pairs, 2 waves, 282 us vs cuBLAS 192 — measured slower still: 258-295 us at M = 1024 and
  // 431 vs 301 us at M = 1536, so those shapes keep whole tiles.)
  // SIDP_GEMM_SMALL_M_STREAMK = m > 0: underfilled tile counts at M <= m go stream-K too (tiny
  // token tiles are pure weight streaming); default off (measured on the CaS owner)
  static const int env_small = getenv("SIDP_GEMM_SMALL_M_STREAMK") ? atoi(getenv("SIDP_GEMM_SMALL_M_STREAMK")) : 0;
  int streamk = (!sw && a.epi != EPI_ARGMAX && a.epi != EPI_QKV && a.k_splits != 1 &&
                 (a.k_splits > 1 || 2 * tiles <= clusters ||
                  (env_small > 0 && a.M <= env_small && tiles < clusters))) ? 1 : 0;
  if (streamk) {
    const long long total = (long long)tiles * nkb;
    const long long per = total / clusters;
    if (per < 2) clusters = (int)std::max<long long>(1, total / 2);   // tiny problems
    const int max_seg = (int)((nkb + per - 1) / std::max<long long>(per, 1)) + 1;
    if ((size_t)max_seg * a.M * a.N * 4 > w.ws_bytes) streamk = 0;
  }
  // Hybrid data-parallel + stream-K tail: when whole tiles leave the last wave mostly idle
  // (e.g. down at M = 1024: 80 tiles on 74 pairs = 1 full wave + 6 tiles that take a whole
  // wave's time), the full waves stay whole and only the remaining tiles' k-steps are split
  // over every pair; their partials go to per-cluster tile buffers (compact: 2 per cluster),
  // summed by gemm_reduce_kernel in cluster order.
  int dp_tiles = 0, compact = 0, sk = 0;
  static int env_hybrid = getenv("SIDP_GEMM_HYBRID") ? atoi(getenv("SIDP_GEMM_HYBRID")) : 1;
  if (!streamk && env_hybrid && !sw && a.epi != EPI_ARGMAX && a.epi != EPI_QKV && a.epi != EPI_PARTIAL &&
      a.k_splits != 1 && tiles > pair_slots) {
    const int rem = tiles % pair_slots;
    const int waves = (tiles + pair_slots - 1) / pair_slots;
    const double eff = (double)tiles / ((double)waves * pair_slots);
    const size_t need = (size_t)pair_slots * 2 * (2 * WROWS) * BNT * 4;
    // measured (tools/gemm_bench.py): pays for down at M = 1024 (80 tiles: 282 -> 200 us, the
    // tail is 6 tiles of 200 k-steps, ~16 per pair); loses when the tail per pair is a few
    // k-steps (QKV M = 512: 62 -> 67 us, each pair's 256 KB partial costs more than its work) or
    // when the last wave is mostly full (gate/up M = 256: 200 tiles, 121 -> 126 us; M = 1536
    // down 301 -> 319 us: split k-ranges of one feature tile no longer share W lines in L2)
    // (r2) up to a quantisation efficiency of 0.8, and a tail too short to give every pair
    // >= 12 k-steps goes to the first rem x nkb / 12 pairs only: Llama-70B on the 124 WaS compute
    // SMs (62 pairs), down at M = 1024 (128 tiles, eff 0.69) 470 -> 372 us, at M = 1536 631 ->
    // 540; Qwen3 down at M = 1024 283 -> 229 us, O 109 -> 96 (tools/gemm_bench.py)
    static const double env_heff = getenv("SIDP_GEMM_HYBRID_EFF") ? atof(getenv("SIDP_GEMM_HYBRID_EFF")) : 0.8;
    static const int env_hsmall = getenv("SIDP_GEMM_HYBRID_SMALL_TAIL") ? atoi(getenv("SIDP_GEMM_HYBRID_SMALL_TAIL")) : 1;
    const long long tail = (long long)rem * nkb;
    if (rem != 0 && eff < env_heff && need <= w.ws_bytes &&
        (tail >= 12LL * pair_slots || (env_hsmall && tail >= 24))) {
      dp_tiles = tiles - rem;
      streamk = 1;
      compact = 1;
      clusters = pair_slots;
      sk = (int)std::min<long long>(pair_slots, tail / 12);
    }
  }
  if (qs.ok) {
    streamk = 1; dp_tiles = 0; compact = 0;
    clusters = qs.clusters;
  }
  const bool part = a.epi == EPI_PARTIAL;
  if (part) {
    const PartialPlan q = plan_partial(a.M, a.N, a.K, pair_slots);
    if ((size_t)q.max_seg * a.M * a.N * 4 > w.ws_bytes || q.kps != kps) return cudaErrorInvalidValue;
    sw = q.sw; BNT = q.BNT; m_tiles = q.m_tiles; n_pairs = q.n_pairs;
    tiles = q.tiles; clusters = q.clusters; streamk = 1;
    if (a.partial_out) {
      PartialSrc& o = *a.partial_out;
      o.ws = w.ws; o.M = a.M; o.N = a.N; o.sw = sw ? 1 : 0;
      o.tile_m = sw ? 2 * WROWS : BNT; o.tile_f = sw ? BNT : 2 * WROWS;
      o.m_tiles = sw ? n_pairs : m_tiles; o.f_tiles = sw ? m_tiles : n_pairs;
      o.nks = nkb; o.clusters = clusters; o.total_kb = q.total;
      if (tiles > kPartialMaxTiles) return cudaErrorInvalidValue;
      for (int t = 0; t < tiles; ++t)
        o.nseg[t] = (unsigned char)(partial_cluster_of((long long)(t + 1) * nkb - 1, q.total, clusters) -
                                    partial_cluster_of((long long)t * nkb, q.total, clusters) + 1);
    }
  }
  if (!streamk) clusters = std::min(tiles, pair_slots);
  const size_t stage_bytes = kps * ((size_t)WROWS * BK * 2 + (size_t)(BNT / 2) * BK * 2);
  const size_t extra = 32 * SROW * 4 + 512;
  int stages = (int)std::min<size_t>(env_stages, (kSmemBudget - extra) / stage_bytes);
  stages = std::max(2, stages);

  CUtensorMap tw, tx;   // A operand map (128 rows per CTA), B operand map (BNT/2 rows per CTA)
  const bool wkb = a.w_kbmajor != 0;   // W stored k-block-major [K/64][N][64]
  int a3d = 0, b3d = 0;
  if (sw) {
    if (a.x_kbmajor) {
      if (!make_tmap_kbmajor(&tw, a.x, a.K, a.M, WROWS, kps)) return cudaErrorInvalidValue;
      a3d = 1;
    } else if (!make_tmap_2d(&tw, a.x, a.K, a.M, a.ldx, BK, WROWS)) {
      return cudaErrorInvalidValue;
    }
    if (wkb) {
      if (!make_tmap_kbmajor(&tx, a.w, a.K, a.N, BNT / 2, kps)) return cudaErrorInvalidValue;
      b3d = 1;
    } else if (!make_tmap_2d(&tx, a.w, a.K, a.N, a.ldw, BK, BNT / 2)) {
      return cudaErrorInvalidValue;
    }
  } else {
    if (wkb) {
      if (!make_tmap_kbmajor(&tw, a.w, a.K, a.N, WROWS, kps)) return cudaErrorInvalidValue;
      a3d = 1;
    } else if (!make_tmap_2d(&tw, a.w, a.K, a.N, a.ldw, BK, WROWS)) {
      return cudaErrorInvalidValue;
    }
    if (a.x_kbmajor) {
      if (!make_tmap_kbmajor(&tx, a.x, a.K, a.M, BNT / 2, kps)) return cudaErrorInvalidValue;
      b3d = 1;
    } else if (!make_tmap_2d(&tx, a.x, a.K, a.M, a.ldx, BK, BNT / 2)) {
      return cudaErrorInvalidValue;
    }
  }

  KParams p{};
  p.M = a.M; p.N = a.N; p.K = a.K; p.BNT = BNT; p.stages = stages;
  p.m_tiles = m_tiles; p.n_pairs = n_pairs; p.tiles = tiles; p.streamk = streamk;
  p.total_kb = (long long)(tiles - dp_tiles) * nkb; p.clusters = clusters; p.kps = kps; p.nks = nkb;
  p.sk = sk > 0 ? sk : clusters;
  p.dp_tiles = dp_tiles; p.compact = compact;
  p.out = a.out; p.ldo = a.ldo; p.resid = a.resid; p.ldr = a.ldr; p.bias = a.bias;
  p.ws = w.ws; p.counters = w.counters;
  p.a3d = a3d; p.b3d = b3d;
  p.partial_all = part ? 1 : 0;
  static int env_evict = getenv("SIDP_GEMM_W_EVICT") ? atoi(getenv("SIDP_GEMM_W_EVICT")) : 1;
  // evict-first only when every weight tile is read by one unit (one token tile): with
  // several token tiles the other units re-read the same W tile from L2
  p.w_evict = env_evict && (sw ? n_pairs == 1 : m_tiles == 1);
  if (a.qkv) p.qkv = *a.qkv;
  p.qkv_cnt_off = kQkvCntOff;
  if (a.wait) p.wait = *a.wait;
  const PostFlags* post = a.post && a.post->n > 0 ? a.post : nullptr;
  if (a.scatter) {
    if (a.epi != EPI_F32 && a.epi != EPI_BF16 && a.epi != EPI_RESID) return cudaErrorInvalidValue;
    p.scatter = *a.scatter;
  }
  static int env_debug = getenv("SIDP_GEMM_DEBUG") ? atoi(getenv("SIDP_GEMM_DEBUG")) : 0;
  p.debug = env_debug;
  static int env_trace = getenv("SIDP_GEMM_TRACE") ? atoi(getenv("SIDP_GEMM_TRACE")) : 0;
  static unsigned long long* trace_buf = nullptr;
  p.trace = nullptr;
  if (env_trace) {
    if (!trace_buf) cudaMallocManaged(&trace_buf, (6 * 4096 + 512 * 8) * 8);
    cudaMemset(trace_buf, 0, (6 * 4096 + 512 * 8) * 8);
    p.trace = trace_buf;
  }
  const size_t smem = stages * stage_bytes + extra + 1024;
  dim3 grid(2 * clusters);
  const bool reduce_follows = streamk && !part && a.epi != EPI_QKV;
  if (post && !reduce_follows) p.post = *post;   // this launch is the last: it posts
  cudaError_t e0 = cudaSuccess, e1 = cudaSuccess;
  switch (a.epi) {
    case EPI_F32: e0 = launch_gemm2<EPI_F32>(kps, sw, grid, smem, stream, tw, tx, p); break;
    case EPI_BF16: e0 = launch_gemm2<EPI_BF16>(kps, sw, grid, smem, stream, tw, tx, p); break;
    case EPI_RESID: e0 = launch_gemm2<EPI_RESID>(kps, sw, grid, smem, stream, tw, tx, p); break;
    case EPI_SILU_MUL: e0 = launch_gemm2<EPI_SILU_MUL>(kps, sw, grid, smem, stream, tw, tx, p); break;
    case EPI_ARGMAX: e0 = launch_gemm2<EPI_ARGMAX>(kps, sw, grid, smem, stream, tw, tx, p); break;
    case EPI_QKV: e0 = launch_gemm2<EPI_QKV>(kps, sw, grid, smem, stream, tw, tx, p); break;
    case EPI_PARTIAL: e0 = launch_gemm2<EPI_PARTIAL>(kps, sw, grid, smem, stream, tw, tx, p); break;
    default: return cudaErrorInvalidValue;
  }
  g_last_launches = 1;
  if (env_trace) {   // perf experiment: dump per-k-block timing of cluster 0
    cudaStreamSynchronize(stream);
    int n = 0;
    while (n < 4096 && trace_buf[4 * 4096 + n]) ++n;
    double sw = 0, tl = 0, gap = 0, iss = 0, loop = 0;
    for (int i = 0; i < n; ++i) {
      iss += (double)(trace_buf[5 * 4096 + i] - trace_buf[2 * 4096 + i]);     // TMA issue cost
      if (i) loop += (double)(trace_buf[i] - trace_buf[i - 1]);
      sw += (double)(trace_buf[2 * 4096 + i] - trace_buf[i]);           // producer wait on empty
      tl += (double)(trace_buf[4 * 4096 + i] - trace_buf[2 * 4096 + i]); // issue -> full (TMA lat)
      if (i) gap += (double)(trace_buf[4 * 4096 + i] - trace_buf[4 * 4096 + i - 1]);
    }
    if (n > 1)
      fprintf(stderr, "[gemm trace] M=%d N=%d K=%d stages=%d kb=%d: producer empty-wait %.0f ns, "
              "issue->full %.0f ns, full-to-full %.0f ns per kb, TMA issue %.0f ns, producer loop %.0f ns, span %.1f us\n", a.M, a.N, a.K,
              stages, n, sw / n, tl / n, gap / (n - 1), iss / n, loop / (n - 1),
              (trace_buf[4 * 4096 + n - 1] - trace_buf[2 * 4096]) / 1e3);
    // per-CTA milestones relative to the earliest CTA entry: min / median / max (us)
    const int nb = std::min<int>(grid.x, 512);
    unsigned long long t0 = ~0ull;
    for (int b = 0; b < nb; ++b) t0 = std::min(t0, trace_buf[6 * 4096 + b * 8]);
    const char* names[7] = {"entry", "pdl", "1st-full", "mma-done", "epi-done", "tail-done", "exit"};
    for (int k = 0; k < 7; ++k) {
      std::vector<double> v;
      for (int b = 0; b < nb; ++b) {
        const unsigned long long t = trace_buf[6 * 4096 + b * 8 + k];
        if (t) v.push_back((t - t0) / 1e3);
      }
      if (v.empty()) continue;
      std::sort(v.begin(), v.end());
      fprintf(stderr, "[gemm trace]   %-9s n=%3zu min %6.2f med %6.2f max %6.2f us\n", names[k],
              v.size(), v.front(), v[v.size() / 2], v.back());
    }
  }
  if (e0 != cudaSuccess || !streamk || part || a.epi == EPI_QKV) return e0;
  g_last_launches = 2;
  if (post) p.post = *post;   // the fix-up is the last launch: it posts
  dim3 rgrid((BNT * (2 * WROWS / 8) + 255) / 256, std::max(1, p.sk - 1));
  switch (a.epi) {
    case EPI_F32: e1 = launch_pdl(gemm_reduce_kernel<EPI_F32>, rgrid, dim3(256), 0, stream, p); break;
    case EPI_BF16: e1 = launch_pdl(gemm_reduce_kernel<EPI_BF16>, rgrid, dim3(256), 0, stream, p); break;
    case EPI_RESID: e1 = launch_pdl(gemm_reduce_kernel<EPI_RESID>, rgrid, dim3(256), 0, stream, p); break;
    case EPI_SILU_MUL: e1 = launch_pdl(gemm_reduce_kernel<EPI_SILU_MUL>, rgrid, dim3(256), 0, stream, p); break;
    default: return cudaErrorInvalidValue;
  }
  return e1;
}

// ---- fused MLP host side ------------------------------------------------------------
namespace {
struct MlpSched {
  int4* d_units = nullptr;
  int* d_uoff = nullptr;
  std::vector<int> nseg;   // per down tile
  int max_seg = 0;
};
struct MlpKey {   // the unit tables live on the device that was current when they were built
  int dev, max_seg, h, I, C;
  bool operator<(const MlpKey& o) const {
    return std::tie(dev, max_seg, h, I, C) < std::tie(o.dev, o.max_seg, o.h, o.I, o.C);
  }
};

// List scheduling of the two GEMMs' units over C CTA pairs with unit cost = k-steps: gate/up
// tiles round-robin (whole tiles, the SiLU epilogue needs complete sums); then the down tiles'
// k-range chunks in k-major order, each to the earliest-free pair, starting no earlier than the
// gate/up tile producing its first act k-block (a down k-step k depends on gate/up tile k).
}  // namespace

// host-only planning half of build_mlp_sched (exposed for the CPU test of the schedule).
// MT token tiles of 256 rows: gate/up units (g, mt) round-robin, token tile by token tile; the
// down chunks (t, mt, k-range) mt-major then k-major; unit = {phase | seg << 8 | mt << 16, tile,
// kb0, kb1}; nseg is indexed by the W-major tile t * MT + mt.
void plan_mlp_units(int G, int nks1, int D, int nks2, int C, int max_seg, int MT,
                    std::vector<int4>& flat, std::vector<int>& off, std::vector<int>& nseg) {
  std::vector<std::vector<int4>> lists(C);
  std::vector<double> F(C, 0.0), done((size_t)G * MT, 0.0);
  for (int mt = 0; mt < MT; ++mt)
    for (int g = 0; g < G; ++g) {
      const int c = (mt * G + g) % C;
      lists[c].push_back(make_int4(0 | (mt << 16), g, 0, nks1));
      F[c] += nks1;
      done[(size_t)g * MT + mt] = F[c];
    }
  const int nch = std::max(1, std::min(max_seg, nks2));
  const int q = (nks2 + nch - 1) / nch;
  nseg.assign((size_t)D * MT, 0);
  for (int mt = 0; mt < MT; ++mt)
    for (int k0 = 0; k0 < nks2; k0 += q) {
      const int k1 = std::min(nks2, k0 + q);
      for (int t = 0; t < D; ++t) {
        int c = 0;
        for (int i = 1; i < C; ++i)
          if (F[i] < F[c]) c = i;
        const double start = std::max(F[c], done[(size_t)k0 * MT + mt]);
        F[c] = std::max(start + (k1 - k0), done[(size_t)(k1 - 1) * MT + mt] + 1.0);
        int& ns = nseg[(size_t)t * MT + mt];
        lists[c].push_back(make_int4(1 | (ns << 8) | (mt << 16), t, k0, k1));
        ns++;
      }
    }
  flat.clear();
  off.assign(1, 0);
  for (int c = 0; c < C; ++c) {
    flat.insert(flat.end(), lists[c].begin(), lists[c].end());
    off.push_back((int)flat.size());
  }
}

namespace {
MlpSched build_mlp_sched(int G, int nks1, int D, int nks2, int C, int max_seg, int MT) {
  MlpSched sc;
  std::vector<int4> flat;
  std::vector<int> off;
  plan_mlp_units(G, nks1, D, nks2, C, max_seg, MT, flat, off, sc.nseg);
  for (int v : sc.nseg) sc.max_seg = std::max(sc.max_seg, v);
  cudaMalloc(&sc.d_units, flat.size() * sizeof(int4));
  cudaMalloc(&sc.d_uoff, off.size() * sizeof(int));
  cudaMemcpy(sc.d_units, flat.data(), flat.size() * sizeof(int4), cudaMemcpyHostToDevice);
  cudaMemcpy(sc.d_uoff, off.data(), off.size() * sizeof(int), cudaMemcpyHostToDevice);
  return sc;
}
}  // namespace

constexpr int kMlpMaxTokenTiles = 2;   // M <= 512

// The schedule depends on the shapes and the token-tile count, not on M itself (segments are
// sized for MT x 256 rows): built once per (h, I, MT) — mlp_prepare runs it at allocation
// time, outside any CUDA-graph capture.
const MlpSched* mlp_sched(int h, int I, int MT, size_t ws_bytes) {
  static std::map<MlpKey, MlpSched> cache;
  const int C = std::max(1, num_sms() / 2);
  static int env_seg = getenv("SIDP_MLP_SEGS") ? atoi(getenv("SIDP_MLP_SEGS")) : 8;
  const int max_seg =
      (int)std::min<size_t>(std::max(1, env_seg), ws_bytes / ((size_t)MT * 256 * h * 4));
  int dev = 0;
  cudaGetDevice(&dev);
  const MlpKey key{dev, max_seg * 16 + MT, h, I, C};
  auto it = cache.find(key);
  if (it == cache.end()) {
    it = cache.emplace(key, build_mlp_sched(I / 128, h / (BK * 2), (h + 255) / 256, I / (BK * 2), C,
                                            max_seg, MT)).first;
  }
  return &it->second;
}

void mlp_prepare(int h, int I, size_t ws_bytes) {
  if (h > 0 && I > 0 && h % 256 == 0 && I % 128 == 0)
    for (int mt = 1; mt <= kMlpMaxTokenTiles; ++mt) mlp_sched(h, I, mt, ws_bytes);
}

bool gemm_qkv_sw_ok(int M, int N, int K, int hd, size_t ws_bytes, int n_counters) {
  return plan_qkv_sw(M, N, K, hd, std::max(1, compute_sms() / 2), ws_bytes, n_counters).ok;
}

bool mlp_fused_ok(int M, int h, int I, size_t ws_bytes, int n_counters, int max_tt) {
  static int env = getenv("SIDP_MLP_FUSED") ? atoi(getenv("SIDP_MLP_FUSED")) : 1;
  // Policy default: one token tile.  At M = 512 (2 tiles) the fused launch is ~5% faster than
  // gate/up + down, but resid_norm then reads up to 8 fp32 slices of 512 rows instead of one
  // bf16 row block, which cancels it (53.2 vs 53.1 ms/step, B=512).
  static int env_mt = getenv("SIDP_MLP_MAX_TT") ? atoi(getenv("SIDP_MLP_MAX_TT")) : 1;
  if (max_tt <= 0) max_tt = env_mt;
  const int MT = (M + 255) / 256;
  if (!env || M <= 0 || MT > std::min(max_tt, kMlpMaxTokenTiles) || h % 256 || I % 128 || h % BK ||
      I % BK)
    return false;
  const int G = I / 128;                 // gate/up pair tiles = act k-steps of the down GEMM
  if (n_counters < G * MT + 1) return false;
  if ((h + 255) / 256 * MT > kPartialMaxTiles) return false;
  return (size_t)2 * MT * 256 * h * 4 <= ws_bytes;   // at least 2 down segments fit
}

cudaError_t mlp_launch(const MlpArgs& a, const GemmWorkspace& w, cudaStream_t stream) {
  g_last_launches = 0;
  if (!mlp_fused_ok(a.M, a.h, a.I, w.ws_bytes, w.n_counters, kMlpMaxTokenTiles))
    return cudaErrorInvalidValue;
  static unsigned long long attr = 0;
  if (first_on_device(attr))
    cudaFuncSetAttribute(mlp2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget + 1024);
  const int C = std::max(1, num_sms() / 2);
  const int G = a.I / 128, nks1 = a.h / (BK * 2), D = (a.h + 255) / 256, nks2 = a.I / (BK * 2);
  const int MT = (a.M + 255) / 256;
  const int BNT = MT > 1 ? 256 : std::max(32, ((a.M + 31) / 32) * 32);
  const MlpSched* scp = mlp_sched(a.h, a.I, MT, w.ws_bytes);
  if (!scp || !scp->d_units) return cudaErrorMemoryAllocation;
  const MlpSched& sc = *scp;
  CUtensorMap tw1, tx1, tw2, tx2;
  if (!make_tmap_2d(&tw1, a.wgu, a.h, 2 * (uint64_t)a.I, a.h, BK, WROWS) ||
      !make_tmap_2d(&tx1, a.u, a.h, a.M, a.ldu, BK, BNT / 2) ||
      !make_tmap_2d(&tw2, a.wd, a.I, a.h, a.I, BK, WROWS) ||
      !make_tmap_2d(&tx2, a.act, a.I, a.M, a.ldact, BK, BNT / 2))
    return cudaErrorInvalidValue;
  MlpParams p{};
  p.M = a.M; p.N1 = 2 * a.I; p.K1 = a.h; p.N2 = a.h; p.K2 = a.I;
  p.BNT = BNT; p.MT = MT;
  const size_t stage_bytes = 2 * ((size_t)WROWS * BK * 2 + (size_t)(BNT / 2) * BK * 2);
  const size_t extra = 32 * SROW * 4 + 512;
  static int env_stages = getenv("SIDP_GEMM_STAGES") ? atoi(getenv("SIDP_GEMM_STAGES")) : 12;
  p.stages = std::max(2, (int)std::min<size_t>(env_stages, (kSmemBudget - extra) / stage_bytes));
  p.units = sc.d_units; p.uoff = sc.d_uoff;
  p.act = a.act; p.ldact = a.ldact; p.ws = w.ws;
  p.flags = w.counters; p.done = reinterpret_cast<unsigned int*>(w.counters + G * MT);
  p.n_flags = G * MT;
  const size_t smem = p.stages * stage_bytes + extra + 1024;
  cudaError_t e = launch_pdl(mlp2_kernel, dim3(2 * C), dim3(kThreads), smem, stream, tw1, tx1, tw2, tx2, p);
  if (e != cudaSuccess) return e;
  g_last_launches = 1;
  if (a.partial_out) {
    PartialSrc& o = *a.partial_out;
    o = PartialSrc{};
    o.ws = w.ws; o.M = a.M; o.N = a.h; o.sw = 0;
    o.tile_m = BNT; o.tile_f = 2 * WROWS; o.m_tiles = MT; o.f_tiles = D;
    if (D * MT > kPartialMaxTiles) return cudaErrorInvalidValue;
    for (int t = 0; t < D * MT; ++t) o.nseg[t] = (unsigned char)sc.nseg[t];
  }
  return cudaSuccess;
}

// Force-load every kernel of this file (CUDA lazy loading would otherwise load a module on
// first launch, which waits for the device to idle — a deadlock while another virtual rank's
// flag-wait kernel spins; see runtime sidp_alloc).
cudaError_t gemm_preload() {
  cudaFuncAttributes fa;
  cudaError_t e = cudaSuccess;
#define SIDP_PRELOAD(k) if (cudaFuncGetAttributes(&fa, k) != cudaSuccess) e = cudaGetLastError();
  SIDP_PRELOAD((gemm2_kernel<EPI_F32, 1, false>)) SIDP_PRELOAD((gemm2_kernel<EPI_F32, 2, false>))
  SIDP_PRELOAD((gemm2_kernel<EPI_F32, 1, true>)) SIDP_PRELOAD((gemm2_kernel<EPI_F32, 2, true>))
  SIDP_PRELOAD((gemm2_kernel<EPI_BF16, 1, false>)) SIDP_PRELOAD((gemm2_kernel<EPI_BF16, 2, false>))
  SIDP_PRELOAD((gemm2_kernel<EPI_BF16, 1, true>)) SIDP_PRELOAD((gemm2_kernel<EPI_BF16, 2, true>))
  SIDP_PRELOAD((gemm2_kernel<EPI_RESID, 1, false>)) SIDP_PRELOAD((gemm2_kernel<EPI_RESID, 2, false>))
  SIDP_PRELOAD((gemm2_kernel<EPI_RESID, 1, true>)) SIDP_PRELOAD((gemm2_kernel<EPI_RESID, 2, true>))
  SIDP_PRELOAD((gemm2_kernel<EPI_SILU_MUL, 1, false>)) SIDP_PRELOAD((gemm2_kernel<EPI_SILU_MUL, 2, false>))
  SIDP_PRELOAD((gemm2_kernel<EPI_SILU_MUL, 1, true>)) SIDP_PRELOAD((gemm2_kernel<EPI_SILU_MUL, 2, true>))
  SIDP_PRELOAD((gemm2_kernel<EPI_ARGMAX, 1, false>)) SIDP_PRELOAD((gemm2_kernel<EPI_ARGMAX, 2, false>))
  SIDP_PRELOAD((gemm2_kernel<EPI_ARGMAX, 1, true>)) SIDP_PRELOAD((gemm2_kernel<EPI_ARGMAX, 2, true>))
  SIDP_PRELOAD((gemm2_kernel<EPI_QKV, 1, false>)) SIDP_PRELOAD((gemm2_kernel<EPI_QKV, 2, false>))
  SIDP_PRELOAD((gemm2_kernel<EPI_QKV, 1, true>)) SIDP_PRELOAD((gemm2_kernel<EPI_QKV, 2, true>))
  SIDP_PRELOAD((gemm2_kernel<EPI_PARTIAL, 1, false>)) SIDP_PRELOAD((gemm2_kernel<EPI_PARTIAL, 2, false>))
  SIDP_PRELOAD((gemm2_kernel<EPI_PARTIAL, 1, true>)) SIDP_PRELOAD((gemm2_kernel<EPI_PARTIAL, 2, true>))
    SIDP_PRELOAD((mlp2_kernel))
  SIDP_PRELOAD((gemm_reduce_kernel<EPI_F32>)) SIDP_PRELOAD((gemm_reduce_kernel<EPI_BF16>))
  SIDP_PRELOAD((gemm_reduce_kernel<EPI_RESID>)) SIDP_PRELOAD((gemm_reduce_kernel<EPI_SILU_MUL>))
#undef SIDP_PRELOAD
  // the >48 KB shared-memory attributes, for the current device (sidp_alloc calls this)
  set_attr<EPI_PARTIAL>();
  set_attr<EPI_F32>();
  set_attr<EPI_BF16>();
  set_attr<EPI_RESID>();
  set_attr<EPI_SILU_MUL>();
  set_attr<EPI_ARGMAX>();
  set_attr<EPI_QKV>();
  if (cudaFuncSetAttribute(mlp2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           kSmemBudget + 1024) != cudaSuccess)
    e = cudaGetLastError();
  return e;
}

}  // namespace sidp
