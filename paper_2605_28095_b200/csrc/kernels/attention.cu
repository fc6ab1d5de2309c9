// attention.cu — QKV post-processing and GQA decode attention.
//
// qkv_post: per token, per head: optional per-head RMSNorm (Qwen3 qk_norm), rotate-half RoPE
// from an fp64-built (cos, sin) table, q -> bf16, k/v appended to the local KV cache at pos_b.
// The KV cache is local and never pooled.
//
// decode attention: HBM-bound (4096 B of K/V per context token per layer).
// The batch's 16-token K/V chunks are split into equal contiguous ranges, one per CTA (one
// (sequence, kv head) pair per CTA for uniform contexts; pairs split into pieces for small
// batches / long or ragged contexts, see attn_kernel).  4 warps per CTA; each warp streams
// chunks through a 3-stage cp.async ring in XOR-swizzled shared memory and runs the G query
// heads of the group (padded to 16 rows) through mma.sync m16n8k16 bf16 tensor-core tiles for
// S = q K^T and O += P V, with an fp32 online softmax (exp2 domain).  Warps and pieces are
// merged with the usual (max, sum) rescaling.  Measured on the M2 shape (B=256, 1025-token
// contexts, 16 layers): 3 stages (96 KB, 2 CTAs/SM by registers) 181 us vs 2 stages 188 us
// (forcing 3 CTAs/SM with 2 stages spills: 197 us) and 4 stages 214 us; a single wave of
// persistent CTAs over pieces loses to one pair per CTA (per-piece prologue/merge cost).
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "../common.cuh"
#include "../kernels.h"

namespace sidp {

namespace {

// ---------------------------------------------------------------- qkv post
// heads per warp: 5 x 8 warps = 40 heads per CTA, two CTAs per token for nq + 2 nkv = 80
constexpr int kQkvHeadsPerWarp = 5;
// lane l holds dims [E*l, E*l+E) of the first half and the same dims + hd/2 (its RoPE
// partners), E = hd/64: every load and store is one E-wide vector per lane
template <int HD, int HPW>
__global__ void __launch_bounds__(256, 4) qkv_post_kernel(QkvPostArgs a) {
  pdl_trigger();
  pdl_wait();
  constexpr int half = HD / 2, E = HD / 64;
  // grid (B, ceil(nh / (8 HPW))): each warp owns HPW (token, head) vectors and issues all their
  // loads before any arithmetic (one warp per head left ~0.5 KB in flight per warp: at B = 1024
  // the kernel ran at ~0.9 TB/s, latency-bound)
  const int b = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nh = a.nq + 2 * a.nkv;
  if (a.wait.n) {   // CaS: the owner's returned qkv rows have landed (done flag)
    if (threadIdx.x == 0) flags_wait(a.wait.p, a.wait.n, a.wait.value, a.wait.timeout_ns, a.wait.err, a.wait.base);
    __syncthreads();
  }
  const size_t ldqkv = a.ldqkv > 0 ? (size_t)a.ldqkv : (size_t)nh * HD;
  const int pos = a.pos[b];
  const int i0 = E * lane;
  float cs[E][2];
  {
    const float* rp = reinterpret_cast<const float*>(a.rope + (size_t)pos * half + i0);
    if constexpr (E == 2) {
      const float4 t = *reinterpret_cast<const float4*>(rp);
      cs[0][0] = t.x; cs[0][1] = t.y; cs[1][0] = t.z; cs[1][1] = t.w;
    } else {
      const float2 t = *reinterpret_cast<const float2*>(rp);
      cs[0][0] = t.x; cs[0][1] = t.y;
    }
  }
  const size_t slice = (size_t)a.part.M * a.part.N;
  float x1[HPW][E], x2[HPW][E];
#pragma unroll
  for (int hh = 0; hh < HPW; ++hh) {
#pragma unroll
    for (int e = 0; e < E; ++e) x1[hh][e] = x2[hh][e] = 0.0f;
  }
  auto load = [&](const float* src, float (&y1)[E], float (&y2)[E]) {
    if constexpr (E == 2) {
      const float2 u = __ldcg(reinterpret_cast<const float2*>(src + i0));
      const float2 w = __ldcg(reinterpret_cast<const float2*>(src + i0 + half));
      y1[0] += u.x; y1[1] += u.y; y2[0] += w.x; y2[1] += w.y;
    } else {
      y1[0] += __ldcg(src + i0);
      y2[0] += __ldcg(src + i0 + half);
    }
  };
  // phase 1: loads (summing partial slices in slice order when QKV left stream-K partials)
#pragma unroll
  for (int hh = 0; hh < HPW; ++hh) {
    const int head = (blockIdx.y * HPW + hh) * 8 + warp;
    if (head >= nh) continue;
    if (a.part.ws) {
      // deferred stream-K fix-up: a head lies inside one 256-feature tile (hd divides 256),
      // so its partial slices are summed in slice order, then the bias is added
      const int n = head * HD;
      const int nseg = a.part.nseg[partial_tile(a.part, b, n)];
      const float* src = a.part.ws + (size_t)b * a.part.N + n;
#pragma unroll
      for (int sgi = 0; sgi < 4; ++sgi)   // issued together (predicated), summed in order
        if (sgi < nseg) load(src + sgi * slice, x1[hh], x2[hh]);
      for (int sgi = 4; sgi < nseg; ++sgi) load(src + sgi * slice, x1[hh], x2[hh]);
      if (a.bias) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          x1[hh][e] += bf16_to_f(a.bias[n + i0 + e]);
          x2[hh][e] += bf16_to_f(a.bias[n + i0 + e + half]);
        }
      }
    } else {
      load(a.qkv + (size_t)b * ldqkv + (size_t)head * HD, x1[hh], x2[hh]);
    }
  }
  // phase 2: qk-norm, RoPE, stores
#pragma unroll
  for (int hh = 0; hh < HPW; ++hh) {
    const int head = (blockIdx.y * HPW + hh) * 8 + warp;
    if (head >= nh) continue;
    const bool is_v = head >= a.nq + a.nkv;
    const bool is_q = head < a.nq;
    if (!is_v) {
      const bf16* gain = is_q ? a.gq : a.gk;
      if (gain) {
        float ss = 0.0f;
#pragma unroll
        for (int e = 0; e < E; ++e) ss += x1[hh][e] * x1[hh][e] + x2[hh][e] * x2[hh][e];
        ss = warp_sum(ss);
        const float r = rsqrtf(ss / (float)HD + a.eps);
#pragma unroll
        for (int e = 0; e < E; ++e) {
          x1[hh][e] = x1[hh][e] * r * bf16_to_f(gain[i0 + e]);
          x2[hh][e] = x2[hh][e] * r * bf16_to_f(gain[i0 + e + half]);
        }
      }
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const float y1 = x1[hh][e] * cs[e][0] - x2[hh][e] * cs[e][1];
        const float y2 = x2[hh][e] * cs[e][0] + x1[hh][e] * cs[e][1];
        x1[hh][e] = y1;
        x2[hh][e] = y2;
      }
    }
    bf16* dst;
    if (is_q) {
      dst = a.q + ((size_t)b * a.nq + head) * HD;
    } else {
      const int g = is_v ? head - a.nq - a.nkv : head - a.nq;
      bf16* cache = is_v ? a.vc : a.kc;
      dst = cache + kv_off(a.bt, a.bt_stride, a.nkv, a.smax, HD, b, g, pos);
    }
    if constexpr (E == 2) {
      *reinterpret_cast<__nv_bfloat162*>(dst + i0) = __floats2bfloat162_rn(x1[hh][0], x1[hh][1]);
      *reinterpret_cast<__nv_bfloat162*>(dst + i0 + half) = __floats2bfloat162_rn(x2[hh][0], x2[hh][1]);
    } else {
      dst[i0] = f_to_bf16(x1[hh][0]);
      dst[i0 + half] = f_to_bf16(x2[hh][0]);
    }
  }
}

// ---------------------------------------------------------------- attention helpers
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem)
               : "memory");
}
// K/V are streamed once per step: evict-first keeps L2 for the small re-read tensors
__device__ __forceinline__ void cp_async16_ef(void* smem, const void* gmem, uint64_t pol) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(smem_u32(smem)),
               "l"(gmem), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                        uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                          uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void mma_bf16(float (&d)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

struct AttnParams {
  const bf16* q;
  const bf16* kc;
  const bf16* vc;
  const int32_t* pos;
  bf16* o;
  size_t ldo;                // row stride of o per sequence (elements)
  float* ws;                 // [C][2 sides][16 rows][HD + 2] partials of split (b, g) pairs
  int* cnt;                  // [B * nkv] arrival counters of split pairs (zero between launches)
  int B, nq, nkv, smax;
  const int32_t* bt; int bt_stride;   // paged KV (16-token blocks == kChunk), null: contiguous
  int pair_mode;             // grid == B * nkv: one whole (b, g) pair per CTA
  int kv_evict;              // K/V loads carry an L2 evict-first policy
  int pre_wait;              // pair mode: first ring chunks requested before the PDL wait
  float scale_log2;
};

constexpr int kChunk = 16;
constexpr int kWarps = 4;

// One 16-token K/V chunk of a (sequence, kv head) pair for one warp: S = Q K^T (mma.sync),
// masked online softmax in the exp2 domain (rows gid and gid + 8), O += P V.
template <int HD>
__device__ __forceinline__ void attn_chunk(const uint32_t (&qa)[HD / 16][4], uint32_t skb,
                                           uint32_t svb, int t0, int n_tok, float scale_log2,
                                           float (&o)[HD / 8][4], float (&mrow)[2],
                                           float (&lrow)[2], int lane) {
  const int tq = lane & 3;
  // S = Q K^T for 16 tokens (two n-tiles of 8)
  float sc[2][4];
#pragma unroll
  for (int j = 0; j < 2; ++j) sc[j][0] = sc[j][1] = sc[j][2] = sc[j][3] = 0.0f;
#pragma unroll
  for (int kk = 0; kk < HD / 16; ++kk) {
    const int mat = lane >> 3, r = lane & 7;
    const int tok = (mat >> 1) * 8 + r;
    const int cc = kk * 2 + (mat & 1);
    uint32_t b0, b1, b2, b3;
    ldsm_x4(skb + (tok * HD + ((cc ^ (tok & 7)) * 8)) * 2, b0, b1, b2, b3);
    mma_bf16(sc[0], qa[kk], b0, b1);
    mma_bf16(sc[1], qa[kk], b2, b3);
  }
  // mask + online softmax (rows gid and gid+8)
  float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int tok = t0 + j * 8 + 2 * tq + (e & 1);
      sc[j][e] = tok < n_tok ? sc[j][e] * scale_log2 : -INFINITY;
      mx[e >> 1] = fmaxf(mx[e >> 1], sc[j][e]);
    }
  float alpha[2], muse[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    mx[h] = fmaxf(mx[h], __shfl_xor_sync(0xffffffffu, mx[h], 1));
    mx[h] = fmaxf(mx[h], __shfl_xor_sync(0xffffffffu, mx[h], 2));
    const float mnew = fmaxf(mrow[h], mx[h]);
    muse[h] = mnew == -INFINITY ? 0.0f : mnew;
    alpha[h] = exp2f(mrow[h] - muse[h]);
    mrow[h] = mnew;
    lrow[h] *= alpha[h];
  }
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      sc[j][e] = exp2f(sc[j][e] - muse[e >> 1]);
      lrow[e >> 1] += sc[j][e];
    }
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) {
    o[i][0] *= alpha[0];
    o[i][1] *= alpha[0];
    o[i][2] *= alpha[1];
    o[i][3] *= alpha[1];
  }
  uint32_t pa[4];
  pa[0] = pack_bf16(sc[0][0], sc[0][1]);
  pa[1] = pack_bf16(sc[0][2], sc[0][3]);
  pa[2] = pack_bf16(sc[1][0], sc[1][1]);
  pa[3] = pack_bf16(sc[1][2], sc[1][3]);
  // O += P V
#pragma unroll
  for (int dn = 0; dn < HD / 8; dn += 2) {
    const int mat = lane >> 3, r = lane & 7;
    const int tok = (mat & 1) * 8 + r;
    const int cc = dn + (mat >> 1);
    uint32_t b0, b1, b2, b3;
    ldsm_x4_t(svb + (tok * HD + ((cc ^ (tok & 7)) * 8)) * 2, b0, b1, b2, b3);
    mma_bf16(o[dn], pa, b0, b1);
    mma_bf16(o[dn + 1], pa, b2, b3);
  }
}

__device__ __forceinline__ uint32_t movmatrix_trans(uint32_t x) {
  uint32_t y;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}

// One 16-token chunk for a group of exactly 8 query heads, transposed: S^T = K Q^T (m16n8k16 with
// the 16 tokens as rows, K as the A operand, the 8 heads as the n = 8 columns) and O^T += V^T P^T
// (V^T as A through ldmatrix.trans, P^T as B through movmatrix.trans of S^T's fragments).  The
// padded form (Q as A, 16 rows of which 8 are real heads) spends half its MMAs and exp2s on
// padding; here every MMA row and every exp2 is a real (token, head).  Per thread: heads 2tq,
// 2tq+1 (their running max / sum), tokens gid and gid + 8 of the chunk.
template <int HD>
__device__ __forceinline__ void attn_chunk8(const uint32_t (&qb)[HD / 16][2], uint32_t skb,
                                            uint32_t svb, int t0, int n_tok, float scale_log2,
                                            float (&ot)[HD / 16][4], float (&mh)[2],
                                            float (&lh)[2], int lane) {
  const int gid = lane >> 2;
  const int mat = lane >> 3, r = lane & 7;
  float sc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
  for (int kk = 0; kk < HD / 16; ++kk) {
    const int tok = (mat & 1) * 8 + r, cc = kk * 2 + (mat >> 1);
    uint32_t a[4];
    ldsm_x4(skb + (tok * HD + ((cc ^ (tok & 7)) * 8)) * 2, a[0], a[1], a[2], a[3]);
    mma_bf16(sc, a, qb[kk][0], qb[kk][1]);
  }
  // mask, per-head online softmax (exp2 domain); a head's 16 tokens live in the 8 lanes of
  // its tq column x 2 rows
  float mx[2];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int tok = t0 + gid + (e >> 1) * 8;
    sc[e] = tok < n_tok ? sc[e] * scale_log2 : -INFINITY;
  }
  mx[0] = fmaxf(sc[0], sc[2]);
  mx[1] = fmaxf(sc[1], sc[3]);
  float alpha[2], muse[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    mx[h] = fmaxf(mx[h], __shfl_xor_sync(0xffffffffu, mx[h], 4));
    mx[h] = fmaxf(mx[h], __shfl_xor_sync(0xffffffffu, mx[h], 8));
    mx[h] = fmaxf(mx[h], __shfl_xor_sync(0xffffffffu, mx[h], 16));
    const float mnew = fmaxf(mh[h], mx[h]);
    muse[h] = mnew == -INFINITY ? 0.0f : mnew;
    alpha[h] = exp2f(mh[h] - muse[h]);
    mh[h] = mnew;
    lh[h] *= alpha[h];
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    sc[e] = exp2f(sc[e] - muse[e & 1]);
    lh[e & 1] += sc[e];
  }
#pragma unroll
  for (int mt = 0; mt < HD / 16; ++mt) {
    ot[mt][0] *= alpha[0];
    ot[mt][1] *= alpha[1];
    ot[mt][2] *= alpha[0];
    ot[mt][3] *= alpha[1];
  }
  const uint32_t b0 = movmatrix_trans(pack_bf16(sc[0], sc[1]));   // P^T, tokens 0-7
  const uint32_t b1 = movmatrix_trans(pack_bf16(sc[2], sc[3]));   // P^T, tokens 8-15
#pragma unroll
  for (int mt = 0; mt < HD / 16; ++mt) {
    const int tok = (mat >> 1) * 8 + r, cc = mt * 2 + (mat & 1);
    uint32_t a[4];
    ldsm_x4_t(svb + (tok * HD + ((cc ^ (tok & 7)) * 8)) * 2, a[0], a[1], a[2], a[3]);
    mma_bf16(ot[mt], a, b0, b1);
  }
}

// CTA owning global chunk index c when W chunks are split into C ranges [floor(iW/C), ...)
__device__ __forceinline__ int cta_of_chunk(long long c, long long W, int C) {
  return (int)(((c + 1) * (long long)C + W - 1) / W) - 1;
}
__device__ __forceinline__ long long chunk_begin(int i, long long W, int C) {
  return (long long)i * W / C;
}

// Work decomposition: the (sequence b, kv head g) pairs, b-major, each hold
// ceil((pos_b + 1) / 16) 16-token chunks; the W chunks of the whole batch are split into
// gridDim.x equal contiguous ranges, one per resident CTA (a single wave: no tail, and ragged
// context lengths balance by construction).  A CTA walks the pairs its range touches; a pair
// covered by one CTA is finished in place, a pair split over several CTAs ("pieces") has each
// piece write its (max, sum, O) partial, and the last piece to arrive merges all pieces in
// piece order (deterministic) and writes o.  Inside a piece the 4 warps take chunks round
// robin through a 2-stage cp.async ring and merge through shared memory.
// T8: a group of exactly 8 query heads in the transposed form (attn_chunk8); the per-warp
// state is stored to the same [warp][head][HD] merge layout, so the merges are shared.
template <int HD, int ST, bool T8 = false>
__global__ void __launch_bounds__(128) attn_kernel(const AttnParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int CPR = HD / 8;                         // 16-byte chunks per row
  constexpr int TILE = kChunk * HD;                   // elements per K (or V) chunk
  constexpr size_t kRingBytes = (size_t)kWarps * ST * 2 * TILE * 2;   // ST-stage ring per warp
  pdl_trigger();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // Pair mode: the first ST-1 ring chunks of this warp hold only context tokens written by
  // earlier steps (never by the preceding qkv_post, which appends token pos_b), so they are
  // requested before griddepcontrol.wait and stream while qkv_post finishes.  pos_b read here
  // may be one step stale (pos_b - 1): only tokens below it are touched, all complete, and the
  // chunk ids do not depend on pos_b.  SIDP_ATTN_PRE=0 disables.
  bool pre = false;
  if (p.pair_mode && p.pre_wait) {
    const int b0 = blockIdx.x / p.nkv, g0 = blockIdx.x % p.nkv;
    const int pos_pre = p.pos[b0];
    if ((warp + (ST - 2) * kWarps + 1) * kChunk <= pos_pre) {
      const size_t pair_off0 = p.bt ? 0 : ((size_t)b0 * p.nkv + g0) * p.smax * HD;
      const bf16* kb0 = p.kc + pair_off0;   // + the chunk's first token below
      const bf16* vb0 = p.vc + pair_off0;
      bf16* wb = reinterpret_cast<bf16*>(smem) + (size_t)warp * ST * 2 * TILE;
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
#pragma unroll
      for (int j = 0; j < ST - 1; ++j) {
        const int t0 = (warp + j * kWarps) * kChunk;
        const size_t co = p.bt ? kv_off(p.bt, p.bt_stride, p.nkv, p.smax, HD, b0, g0, t0) : (size_t)t0 * HD;
        bf16* sk = wb + j * 2 * TILE;
        bf16* sv = sk + TILE;
#pragma unroll
        for (int it = 0; it < (kChunk * CPR) / 32; ++it) {
          const int e = it * 32 + lane;
          const int row = e / CPR, cc = e % CPR;
          const int sw = (cc ^ (row & 7));
          if (p.kv_evict) {
            cp_async16_ef(sk + row * HD + sw * 8, kb0 + co + (size_t)row * HD + cc * 8, pol);
            cp_async16_ef(sv + row * HD + sw * 8, vb0 + co + (size_t)row * HD + cc * 8, pol);
          } else {
            cp_async16(sk + row * HD + sw * 8, kb0 + co + (size_t)row * HD + cc * 8);
            cp_async16(sv + row * HD + sw * 8, vb0 + co + (size_t)row * HD + cc * 8);
          }
        }
        cp_async_commit();
      }
      pre = true;
    }
  }
  pdl_wait();
  const int gid = lane >> 2, tq = lane & 3;
  const int G = p.nq / p.nkv;
  const int C = gridDim.x, cta = blockIdx.x;
  int* cum = reinterpret_cast<int*>(smem + kRingBytes);   // [B + 1] chunk prefix sums
  __shared__ int s_last;

  // ---- pair mode (grid = B * nkv pairs): CTA i is pair i, no prefix sums needed
  // ---- otherwise: prefix sums of per-sequence chunk counts (block scan, 128 threads)
  if (!p.pair_mode) {
    const int per = (p.B + 127) / 128;
    const int e0 = threadIdx.x * per, e1 = min(p.B, e0 + per);
    int local = 0;
    for (int e = e0; e < e1; ++e) local += (p.pos[e] + kChunk) / kChunk;
    int incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    __shared__ int wsum[kWarps];
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    int off = 0;
    for (int w = 0; w < warp; ++w) off += wsum[w];
    int run = off + incl - local;
    if (threadIdx.x == 0) cum[0] = 0;
    for (int e = e0; e < e1; ++e) {
      run += (p.pos[e] + kChunk) / kChunk;
      cum[e + 1] = run;
    }
    __syncthreads();
  }
  const long long W = p.pair_mode ? 1 : (long long)p.nkv * cum[p.B];
  const long long c0 = p.pair_mode ? 0 : chunk_begin(cta, W, C);
  const long long c1 = p.pair_mode ? 1 : chunk_begin(cta + 1, W, C);
  if (c0 >= c1) return;
  // sequence holding c0: largest b with nkv * cum[b] <= c0
  int b = 0;
  if (!p.pair_mode) {
    int lo = 0, hi = p.B - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if ((long long)p.nkv * cum[mid] <= c0) lo = mid; else hi = mid - 1;
    }
    b = lo;
  }
  bf16* wring = reinterpret_cast<bf16*>(smem);
  long long c = c0;
  while (c < c1) {
    int g, chb, lo, hi, side;
    long long pstart, pend;
    if (p.pair_mode) {
      b = cta / p.nkv;
      g = cta % p.nkv;
      chb = (p.pos[b] + kChunk) / kChunk;
      lo = 0; hi = chb; side = 0; pstart = 0; pend = chb;
      c = c1;
    } else {
      chb = cum[b + 1] - cum[b];
      const long long base_b = (long long)p.nkv * cum[b];
      if (c >= base_b + (long long)p.nkv * chb) { ++b; continue; }
      g = (int)((c - base_b) / chb);
      pstart = base_b + (long long)g * chb;
      pend = pstart + chb;
      lo = (int)(c - pstart);
      hi = (int)(min(c1, pend) - pstart);
      side = c == c0 ? 0 : 1;
      c = pstart + hi;
    }

    // ------------------------------------------------ one piece: chunks [lo, hi) of (b, g)
    const int n_tok = p.pos[b] + 1;
    bf16* wbuf = wring + (size_t)warp * ST * 2 * TILE;   // [stage][K|V]
    // contiguous: the pair's base once, chunk offsets t0 * HD; paged: per-chunk block lookups
    const size_t pair_off = p.bt ? 0 : ((size_t)b * p.nkv + g) * p.smax * HD;
    const bf16* kbase = p.kc + pair_off;
    const bf16* vbase = p.vc + pair_off;
    uint32_t qa[T8 ? 1 : HD / 16][4];
    uint32_t qb8[T8 ? HD / 16 : 1][2];
    if constexpr (T8) {   // B = Q^T: (dims 2tq.., head gid), (dims 2tq + 8.., head gid)
      const bf16* qr = p.q + ((size_t)b * p.nq + (size_t)g * 8 + gid) * HD + 2 * tq;
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) {
        qb8[kk][0] = *reinterpret_cast<const uint32_t*>(qr + kk * 16);
        qb8[kk][1] = *reinterpret_cast<const uint32_t*>(qr + kk * 16 + 8);
      }
    } else {
      const bf16* qb = p.q + ((size_t)b * p.nq + (size_t)g * G) * HD;
      const int r0 = gid, r1 = gid + 8;
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) {
        const int cc = kk * 16 + 2 * tq;
        qa[kk][0] = r0 < G ? *reinterpret_cast<const uint32_t*>(qb + r0 * HD + cc) : 0u;
        qa[kk][1] = r1 < G ? *reinterpret_cast<const uint32_t*>(qb + r1 * HD + cc) : 0u;
        qa[kk][2] = r0 < G ? *reinterpret_cast<const uint32_t*>(qb + r0 * HD + cc + 8) : 0u;
        qa[kk][3] = r1 < G ? *reinterpret_cast<const uint32_t*>(qb + r1 * HD + cc + 8) : 0u;
      }
    }
    // padded form: o = O[16 rows][HD] fragments; transposed form: O^T[HD][8 heads] fragments
    constexpr int NO = T8 ? HD / 16 : HD / 8;
    float o[NO][4];
#pragma unroll
    for (int i = 0; i < NO; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.0f;
    float mrow[2] = {-INFINITY, -INFINITY};
    float lrow[2] = {0.0f, 0.0f};

    uint64_t kvpol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(kvpol));
    auto load_chunk = [&](int stage, int ch) {
      const int t0 = ch * kChunk;
      // the chunk's 16 tokens are contiguous in both layouts (a paged block is one chunk)
      const size_t co = p.bt ? kv_off(p.bt, p.bt_stride, p.nkv, p.smax, HD, b, g, t0) : (size_t)t0 * HD;
      bf16* sk = wbuf + stage * 2 * TILE;
      bf16* sv = sk + TILE;
#pragma unroll
      for (int it = 0; it < (kChunk * CPR) / 32; ++it) {
        const int e = it * 32 + lane;
        const int row = e / CPR, cc = e % CPR;
        const int t = min(t0 + row, n_tok - 1);
        const int sw = (cc ^ (row & 7));
        if (p.kv_evict) {
          cp_async16_ef(sk + row * HD + sw * 8, kbase + co + (size_t)(t - t0) * HD + cc * 8, kvpol);
          cp_async16_ef(sv + row * HD + sw * 8, vbase + co + (size_t)(t - t0) * HD + cc * 8, kvpol);
        } else {
          cp_async16(sk + row * HD + sw * 8, kbase + co + (size_t)(t - t0) * HD + cc * 8);
          cp_async16(sv + row * HD + sw * 8, vbase + co + (size_t)(t - t0) * HD + cc * 8);
        }
      }
    };

    // ST-1 chunks in flight per warp ahead of the one being consumed (already requested
    // before the PDL wait when pre)
    if (!pre) {
#pragma unroll
      for (int j = 0; j < ST - 1; ++j) {
        if (lo + warp + j * kWarps < hi) load_chunk(j, lo + warp + j * kWarps);
        cp_async_commit();
      }
    }
    int it = 0;
    for (int ch = lo + warp; ch < hi; ch += kWarps, ++it) {
      const int cn = ch + (ST - 1) * kWarps;
      if (cn < hi) load_chunk((it + ST - 1) % ST, cn);
      cp_async_commit();
      cp_async_wait<ST - 1>();
      __syncwarp();
      const bf16* sk = wbuf + (it % ST) * 2 * TILE;
      const bf16* sv = sk + TILE;
      const uint32_t skb = smem_u32(sk), svb = smem_u32(sv);
      const int t0 = ch * kChunk;

      if constexpr (T8)
        attn_chunk8<HD>(qb8, skb, svb, t0, n_tok, p.scale_log2, o, mrow, lrow, lane);
      else
        attn_chunk<HD>(qa, skb, svb, t0, n_tok, p.scale_log2, o, mrow, lrow, lane);
      __syncwarp();
    }
    cp_async_wait<0>();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if constexpr (T8) {   // a head's sum is spread over the 8 gid lanes of its tq column
        lrow[h] += __shfl_xor_sync(0xffffffffu, lrow[h], 4);
        lrow[h] += __shfl_xor_sync(0xffffffffu, lrow[h], 8);
        lrow[h] += __shfl_xor_sync(0xffffffffu, lrow[h], 16);
      } else {
        lrow[h] += __shfl_xor_sync(0xffffffffu, lrow[h], 1);
        lrow[h] += __shfl_xor_sync(0xffffffffu, lrow[h], 2);
      }
    }
    __syncthreads();
    // ---- merge the 4 warps through shared memory (reuses the K/V ring)
    float* sm_o = reinterpret_cast<float*>(smem);                 // [warp][16][HD]
    float* sm_m = sm_o + kWarps * 16 * HD;                        // [warp][16]
    float* sm_l = sm_m + kWarps * 16;
    if constexpr (T8) {
      // O^T fragment: dim = mt * 16 + gid (+ 8), head = 2 tq (+ 1); heads 8-15 are never read
#pragma unroll
      for (int mt = 0; mt < HD / 16; ++mt)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int head = 2 * tq + (e & 1), dim = mt * 16 + gid + 8 * (e >> 1);
          sm_o[(warp * 16 + head) * HD + dim] = o[mt][e];
        }
      if (gid == 0) {
        sm_m[warp * 16 + 2 * tq] = mrow[0];
        sm_m[warp * 16 + 2 * tq + 1] = mrow[1];
        sm_l[warp * 16 + 2 * tq] = lrow[0];
        sm_l[warp * 16 + 2 * tq + 1] = lrow[1];
      }
    } else {
#pragma unroll
      for (int dn = 0; dn < HD / 8; ++dn)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int row = gid + 8 * (e >> 1), col = dn * 8 + 2 * tq + (e & 1);
          sm_o[(warp * 16 + row) * HD + col] = o[dn][e];
        }
      if (tq == 0) {
        sm_m[warp * 16 + gid] = mrow[0];
        sm_m[warp * 16 + gid + 8] = mrow[1];
        sm_l[warp * 16 + gid] = lrow[0];
        sm_l[warp * 16 + gid + 8] = lrow[1];
      }
    }
    __syncthreads();
    const bool whole = lo == 0 && hi == chb;
    float* part = p.ws + (size_t)(cta * 2 + side) * 16 * (HD + 2);
    for (int idx = threadIdx.x; idx < G * HD; idx += blockDim.x) {
      const int row = idx / HD, col = idx % HD;
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) M = fmaxf(M, sm_m[w * 16 + row]);
      float L = 0.0f, O = 0.0f;
      if (M != -INFINITY) {
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
          const float mw = sm_m[w * 16 + row];
          const float f = mw == -INFINITY ? 0.0f : exp2f(mw - M);
          L += f * sm_l[w * 16 + row];
          O += f * sm_o[(w * 16 + row) * HD + col];
        }
      }
      if (whole) {
        p.o[(size_t)b * p.ldo + (size_t)(g * G + row) * HD + col] = f_to_bf16(L > 0.0f ? O / L : 0.0f);
      } else {
        float* pr = part + (size_t)row * (HD + 2);
        __stcg(pr + 2 + col, O);
        if (col == 0) {
          __stcg(pr, M);
          __stcg(pr + 1, L);
        }
      }
    }
    if (!whole) {
      // publish this piece; the last of the pair's pieces merges them all (piece order)
      const int first = cta_of_chunk(pstart, W, C), last = cta_of_chunk(pend - 1, W, C);
      const int npieces = last - first + 1;
      int* counter = p.cnt + (size_t)b * p.nkv + g;
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) s_last = atomicAdd(counter, 1) == npieces - 1;
      __syncthreads();
      if (s_last) {
        __threadfence();
        // Merge the pieces in order, 64 at a time with online rescaling: each batch's
        // (max, sum) pairs are staged in shared memory (one round trip), then every thread
        // folds its (row, col) outputs over the batch with 4 pieces' loads in flight.
        float* sm_f = sm_o;                           // [64][16] batch scale factors
        float* sm_lk = sm_f + 64 * 16;                // [64][16] batch sums
        float* sm_M = sm_lk + 64 * 16;                // [16] running max
        float* sm_L = sm_M + 16;                      // [16] running sum
        float* sm_s = sm_L + 16;                      // [16] rescale of the running output
        constexpr int kPer = (16 * HD + 127) / 128;   // outputs per thread (G <= 16)
        float acc[kPer];
#pragma unroll
        for (int u = 0; u < kPer; ++u) acc[u] = 0.0f;
        if (threadIdx.x < 16) {
          sm_M[threadIdx.x] = -INFINITY;
          sm_L[threadIdx.x] = 0.0f;
        }
        for (int kb0 = 0; kb0 < npieces; kb0 += 64) {
          const int nb = min(64, npieces - kb0);
          __syncthreads();
          for (int e = threadIdx.x; e < nb * G; e += blockDim.x) {
            const int k = e / G, row = e % G, j = first + kb0 + k;
            const int sd = chunk_begin(j, W, C) >= pstart ? 0 : 1;
            const float* pr = p.ws + ((size_t)(j * 2 + sd) * 16 + row) * (HD + 2);
            sm_f[k * 16 + row] = __ldcg(pr);
            sm_lk[k * 16 + row] = __ldcg(pr + 1);
          }
          __syncthreads();
          if (threadIdx.x < G) {
            const int row = threadIdx.x;
            const float Mold = sm_M[row];
            float M = Mold;
            for (int k = 0; k < nb; ++k) M = fmaxf(M, sm_f[k * 16 + row]);
            const float so = (Mold == -INFINITY) ? 0.0f : exp2f(Mold - M);
            float L = sm_L[row] * so;
            for (int k = 0; k < nb; ++k) {
              const float mk = sm_f[k * 16 + row];
              const float f = mk == -INFINITY ? 0.0f : exp2f(mk - M);
              sm_f[k * 16 + row] = f;
              L += f * sm_lk[k * 16 + row];
            }
            sm_M[row] = M;
            sm_L[row] = L;
            sm_s[row] = so;
          }
          __syncthreads();
#pragma unroll
          for (int u = 0; u < kPer; ++u) {
            const int row = (threadIdx.x + 128 * u) / HD;
            if (row < G) acc[u] *= sm_s[row];
          }
          for (int k0 = 0; k0 < nb; k0 += 4) {
            float v[4][kPer];
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const int k = k0 + kk, j = first + kb0 + k;
              const int sd = chunk_begin(j, W, C) >= pstart ? 0 : 1;
#pragma unroll
              for (int u = 0; u < kPer; ++u) {
                const int idx = threadIdx.x + 128 * u, row = idx / HD, col = idx % HD;
                v[kk][u] = (k < nb && row < G)
                               ? __ldcg(p.ws + ((size_t)(j * 2 + sd) * 16 + row) * (HD + 2) + 2 + col)
                               : 0.0f;
              }
            }
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              if (k0 + kk < nb) {
#pragma unroll
                for (int u = 0; u < kPer; ++u) {
                  const int row = (threadIdx.x + 128 * u) / HD;
                  if (row < G) acc[u] += sm_f[(k0 + kk) * 16 + row] * v[kk][u];
                }
              }
            }
          }
        }
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
          const int idx = threadIdx.x + 128 * u, row = idx / HD, col = idx % HD;
          if (row < G) {
            const float L = sm_L[row];
            p.o[(size_t)b * p.ldo + (size_t)(g * G + row) * HD + col] = f_to_bf16(L > 0.0f ? acc[u] / L : 0.0f);
          }
        }
        if (threadIdx.x == 0) *counter = 0;   // every piece has arrived: reset for the next launch
      }
    }
    __syncthreads();   // the next piece's loads reuse the merge buffers
  }
}

// Warp-per-pair decode attention for many SHORT pairs: each warp owns whole (sequence, kv
// head) pairs (strided over the grid's warps), streams the pair's chunks through its own
// ST-stage ring and normalises and stores o itself — no cross-warp merge, no CTA barrier, so
// one warp's per-pair prologue (q load, first chunks) overlaps the other warps' streaming.
template <int HD, int ST>
__global__ void __launch_bounds__(128) attn_warp_kernel(const AttnParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int CPR = HD / 8;
  constexpr int TILE = kChunk * HD;
  pdl_trigger();
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tq = lane & 3;
  const int G = p.nq / p.nkv;
  const int pairs = p.B * p.nkv;
  bf16* wbuf = reinterpret_cast<bf16*>(smem) + (size_t)warp * ST * 2 * TILE;
  uint64_t kvpol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(kvpol));
  for (int pr = blockIdx.x * kWarps + warp; pr < pairs; pr += gridDim.x * kWarps) {
    const int b = pr / p.nkv, g = pr % p.nkv;
    const int n_tok = p.pos[b] + 1;
    const int chb = (p.pos[b] + kChunk) / kChunk;
    // contiguous: the pair's base once, chunk offsets t0 * HD; paged: per-chunk block lookups
    const size_t pair_off = p.bt ? 0 : ((size_t)b * p.nkv + g) * p.smax * HD;
    const bf16* kbase = p.kc + pair_off;
    const bf16* vbase = p.vc + pair_off;
    auto load_chunk = [&](int stage, int ch) {
      const int t0 = ch * kChunk;
      // the chunk's 16 tokens are contiguous in both layouts (a paged block is one chunk)
      const size_t co = p.bt ? kv_off(p.bt, p.bt_stride, p.nkv, p.smax, HD, b, g, t0) : (size_t)t0 * HD;
      bf16* sk = wbuf + stage * 2 * TILE;
      bf16* sv = sk + TILE;
#pragma unroll
      for (int it = 0; it < (kChunk * CPR) / 32; ++it) {
        const int e = it * 32 + lane;
        const int row = e / CPR, cc = e % CPR;
        const int t = min(t0 + row, n_tok - 1);
        const int sw = (cc ^ (row & 7));
        if (p.kv_evict) {
          cp_async16_ef(sk + row * HD + sw * 8, kbase + co + (size_t)(t - t0) * HD + cc * 8, kvpol);
          cp_async16_ef(sv + row * HD + sw * 8, vbase + co + (size_t)(t - t0) * HD + cc * 8, kvpol);
        } else {
          cp_async16(sk + row * HD + sw * 8, kbase + co + (size_t)(t - t0) * HD + cc * 8);
          cp_async16(sv + row * HD + sw * 8, vbase + co + (size_t)(t - t0) * HD + cc * 8);
        }
      }
    };
#pragma unroll
    for (int j = 0; j < ST - 1; ++j) {
      if (j < chb) load_chunk(j, j);
      cp_async_commit();
    }
    uint32_t qa[HD / 16][4];
    {
      const bf16* qb = p.q + ((size_t)b * p.nq + (size_t)g * G) * HD;
      const int r0 = gid, r1 = gid + 8;
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) {
        const int cc = kk * 16 + 2 * tq;
        qa[kk][0] = r0 < G ? *reinterpret_cast<const uint32_t*>(qb + r0 * HD + cc) : 0u;
        qa[kk][1] = r1 < G ? *reinterpret_cast<const uint32_t*>(qb + r1 * HD + cc) : 0u;
        qa[kk][2] = r0 < G ? *reinterpret_cast<const uint32_t*>(qb + r0 * HD + cc + 8) : 0u;
        qa[kk][3] = r1 < G ? *reinterpret_cast<const uint32_t*>(qb + r1 * HD + cc + 8) : 0u;
      }
    }
    float o[HD / 8][4];
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.0f;
    float mrow[2] = {-INFINITY, -INFINITY};
    float lrow[2] = {0.0f, 0.0f};
    for (int ch = 0; ch < chb; ++ch) {
      const int cn = ch + ST - 1;
      if (cn < chb) load_chunk(cn % ST, cn);
      cp_async_commit();
      cp_async_wait<ST - 1>();
      __syncwarp();
      const bf16* sk = wbuf + (ch % ST) * 2 * TILE;
      attn_chunk<HD>(qa, smem_u32(sk), smem_u32(sk + TILE), ch * kChunk, n_tok, p.scale_log2, o,
                     mrow, lrow, lane);
      __syncwarp();
    }
    cp_async_wait<0>();
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      lrow[h] += __shfl_xor_sync(0xffffffffu, lrow[h], 1);
      lrow[h] += __shfl_xor_sync(0xffffffffu, lrow[h], 2);
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int row = gid + 8 * h;
      if (row < G) {
        const float L = lrow[h];
        bf16* dst = p.o + (size_t)b * p.ldo + (size_t)(g * G + row) * HD + 2 * tq;
#pragma unroll
        for (int dn = 0; dn < HD / 8; ++dn)
          *reinterpret_cast<__nv_bfloat162*>(dst + dn * 8) =
              __floats2bfloat162_rn(L > 0.0f ? o[dn][2 * h] / L : 0.0f,
                                    L > 0.0f ? o[dn][2 * h + 1] / L : 0.0f);
      }
    }
  }
}

// attn_warp_kernel for G = 8 (Qwen3-32B, Llama-3.1-70B, Qwen2.5-72B: 64 / 8 heads) with the
// transposed chunk math above; same partition, ring and loads.
template <int HD, int ST>
__global__ void __launch_bounds__(128) attn_warp8_kernel(const AttnParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int CPR = HD / 8;
  constexpr int TILE = kChunk * HD;
  pdl_trigger();
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tq = lane & 3;
  const int pairs = p.B * p.nkv;
  bf16* wbuf = reinterpret_cast<bf16*>(smem) + (size_t)warp * ST * 2 * TILE;
  uint64_t kvpol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(kvpol));
  for (int pr = blockIdx.x * kWarps + warp; pr < pairs; pr += gridDim.x * kWarps) {
    const int b = pr / p.nkv, g = pr % p.nkv;
    const int n_tok = p.pos[b] + 1;
    const int chb = (p.pos[b] + kChunk) / kChunk;
    const size_t pair_off = p.bt ? 0 : ((size_t)b * p.nkv + g) * p.smax * HD;
    const bf16* kbase = p.kc + pair_off;
    const bf16* vbase = p.vc + pair_off;
    auto load_chunk = [&](int stage, int ch) {
      const int t0 = ch * kChunk;
      const size_t co = p.bt ? kv_off(p.bt, p.bt_stride, p.nkv, p.smax, HD, b, g, t0) : (size_t)t0 * HD;
      bf16* sk = wbuf + stage * 2 * TILE;
      bf16* sv = sk + TILE;
#pragma unroll
      for (int it = 0; it < (kChunk * CPR) / 32; ++it) {
        const int e = it * 32 + lane;
        const int row = e / CPR, cc = e % CPR;
        const int t = min(t0 + row, n_tok - 1);
        const int sw = (cc ^ (row & 7));
        if (p.kv_evict) {
          cp_async16_ef(sk + row * HD + sw * 8, kbase + co + (size_t)(t - t0) * HD + cc * 8, kvpol);
          cp_async16_ef(sv + row * HD + sw * 8, vbase + co + (size_t)(t - t0) * HD + cc * 8, kvpol);
        } else {
          cp_async16(sk + row * HD + sw * 8, kbase + co + (size_t)(t - t0) * HD + cc * 8);
          cp_async16(sv + row * HD + sw * 8, vbase + co + (size_t)(t - t0) * HD + cc * 8);
        }
      }
    };
#pragma unroll
    for (int j = 0; j < ST - 1; ++j) {
      if (j < chb) load_chunk(j, j);
      cp_async_commit();
    }
    uint32_t qb[HD / 16][2];   // B = Q^T: (dims 2tq.., head gid) and (dims 2tq + 8.., head gid)
    {
      const bf16* qr = p.q + ((size_t)b * p.nq + (size_t)g * 8 + gid) * HD + 2 * tq;
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) {
        qb[kk][0] = *reinterpret_cast<const uint32_t*>(qr + kk * 16);
        qb[kk][1] = *reinterpret_cast<const uint32_t*>(qr + kk * 16 + 8);
      }
    }
    float ot[HD / 16][4];
#pragma unroll
    for (int i = 0; i < HD / 16; ++i) ot[i][0] = ot[i][1] = ot[i][2] = ot[i][3] = 0.0f;
    float mh[2] = {-INFINITY, -INFINITY};
    float lh[2] = {0.0f, 0.0f};
    for (int ch = 0; ch < chb; ++ch) {
      const int cn = ch + ST - 1;
      if (cn < chb) load_chunk(cn % ST, cn);
      cp_async_commit();
      cp_async_wait<ST - 1>();
      __syncwarp();
      const bf16* sk = wbuf + (ch % ST) * 2 * TILE;
      attn_chunk8<HD>(qb, smem_u32(sk), smem_u32(sk + TILE), ch * kChunk, n_tok, p.scale_log2,
                      ot, mh, lh, lane);
      __syncwarp();
    }
    cp_async_wait<0>();
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      lh[h] += __shfl_xor_sync(0xffffffffu, lh[h], 4);
      lh[h] += __shfl_xor_sync(0xffffffffu, lh[h], 8);
      lh[h] += __shfl_xor_sync(0xffffffffu, lh[h], 16);
    }
    // o[b][g * 8 + head][dim] = O^T[dim][head] / L[head]
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float L = lh[h];
      bf16* dst = p.o + (size_t)b * p.ldo + (size_t)(g * 8 + 2 * tq + h) * HD + gid;
#pragma unroll
      for (int mt = 0; mt < HD / 16; ++mt) {
        dst[mt * 16] = f_to_bf16(L > 0.0f ? ot[mt][h] / L : 0.0f);
        dst[mt * 16 + 8] = f_to_bf16(L > 0.0f ? ot[mt][2 + h] / L : 0.0f);
      }
    }
  }
}

int g_sms = 0;
thread_local int g_attn_launches = 0;

}  // namespace

cudaError_t qkv_post_launch(const QkvPostArgs& a, cudaStream_t s) {
  if (a.B <= 0) return cudaSuccess;
  if (a.hd != 64 && a.hd != 128) return cudaErrorInvalidValue;
  const int nh = a.nq + 2 * a.nkv;
  constexpr int HPW = kQkvHeadsPerWarp;
  const dim3 grid(a.B, (nh + 8 * HPW - 1) / (8 * HPW));
  if (a.hd == 128) return launch_pdl(qkv_post_kernel<128, HPW>, grid, dim3(256), 0, s, a);
  return launch_pdl(qkv_post_kernel<64, HPW>, grid, dim3(256), 0, s, a);
}

int attention_last_launch_count() { return g_attn_launches; }

template <int HD, int ST>
cudaError_t attn_launch_t(const AttnArgs& a, cudaStream_t s) {
  const size_t ring = (size_t)kWarps * ST * 2 * kChunk * HD * 2;
  const size_t smem = ring + (((size_t)a.B + 1) * 4 + 15) / 16 * 16;
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  static unsigned long long attr = 0, attr8 = 0;
  if (first_on_device(attr))
    cudaFuncSetAttribute(attn_kernel<HD, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  if (first_on_device(attr8))
    cudaFuncSetAttribute(attn_kernel<HD, ST, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  // groups of 8 query heads: the transposed chunk math (SIDP_ATTN_SWAP=0: the padded form)
  static const int env_swap = getenv("SIDP_ATTN_SWAP") ? atoi(getenv("SIDP_ATTN_SWAP")) : 1;
  const bool swap8 = env_swap && a.nq == 8 * a.nkv;
  // one wave of resident CTAs; fewer when the batch has little work (>= 8 chunks per CTA at
  // the host's context bound, so each warp streams at least two chunks)
  int per_sm = 0;
  if (swap8)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, attn_kernel<HD, ST, true>, 128, smem);
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, attn_kernel<HD, ST>, 128, smem);
  per_sm = std::max(1, per_sm);
  const int max_tok = (a.max_tokens > 0 && a.max_tokens < a.smax) ? a.max_tokens : a.smax;
  const long long w_max = (long long)a.B * a.nkv * ((max_tok + kChunk - 1) / kChunk);
  // Enough (b, g) pairs: one CTA per pair's worth of chunks (uniform contexts -> one pair per
  // CTA, no pieces); few pairs (small batch, long context): one wave of CTAs splitting the
  // pairs into pieces (split-KV) with >= 8 chunks per CTA at the host's context bound.
  const long long pairs = (long long)a.B * a.nkv;
  const long long slots = (long long)compute_sms() * per_sm;
  // Many pairs of < 64 chunks each at the context bound: one wave of CTAs walking contiguous
  // chunk ranges instead of one CTA per pair (the per-CTA launch, prologue and warp merge
  // dominated).  Measured per layer, pair mode vs one wave: B = 1024 / S_ctx = 256 (17 chunks)
  // 414 vs 307 us; B = 768 / 512 430 vs 323; B = 512 / 768 389 vs 293; B = 256 / 1024
  // (65 chunks) 194-197 vs 190-191, step equal; B = 128 / 2048 177 vs 190; B = 64 / 4096
  // 170 vs 185 (long pairs keep pair mode); B = 1536 / 32 326 vs 254-260.
  const long long chunks_per_pair = (max_tok + kChunk - 1) / kChunk;
  // Fewer pairs than CTA slots (the CaS tail, small batches): each pair split into k equal pieces,
  // k = 128 / pairs but >= 32 chunks per piece, so a CTA never straddles two pairs and the
  // last-arriver merge folds at most k pieces.  Measured (bench, 8 layers; was one wave of
  // w_max / 8 CTAs): B = 1 / S_ctx 4096 48.9 -> 25.1 us (k = 8), B = 4 / 4096 39.4 -> 28.7
  // (k = 4), B = 16 / 1024 33.0 -> 20.6 and B = 16 / 4096 62.3 -> 49.4 (k = 1: no pieces).
  long long cl;
  if (pairs >= slots) {
    cl = chunks_per_pair >= 64 ? pairs : slots;
  } else {
    static const long long env_tgt = getenv("SIDP_ATTN_SPLIT_TARGET") ? atoll(getenv("SIDP_ATTN_SPLIT_TARGET")) : 128;
    static const long long env_minch = getenv("SIDP_ATTN_SPLIT_MINCH") ? atoll(getenv("SIDP_ATTN_SPLIT_MINCH")) : 32;
    const long long k = std::max<long long>(1, std::min<long long>(std::max<long long>(1, env_tgt / pairs),
                                                                   chunks_per_pair / env_minch));
    cl = std::min(slots, pairs * k);
  }
  // Many pairs of < SIDP_ATTN_WARP_CH (default 128) chunks: warp-per-pair kernel, one wave
  // (B = 1024 / S_ctx = 256: 301 -> 185 us; 768 / 512: 322 -> 277; 512 / 768: 290 -> 259;
  // M2, 65 chunks: step 29.52-29.63 -> 29.29-29.34 ms; B = 128 / 2048 equal)
  static const int env_warp_ch = getenv("SIDP_ATTN_WARP_CH") ? atoi(getenv("SIDP_ATTN_WARP_CH")) : 128;
  if (pairs >= slots && chunks_per_pair < env_warp_ch) {
    static unsigned long long wattr = 0;
    if (first_on_device(wattr))
      cudaFuncSetAttribute(attn_warp_kernel<HD, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           200 * 1024);
    int wper = 0;
    if (swap8)
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&wper, attn_warp8_kernel<HD, ST>, 128, ring);
    else
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&wper, attn_warp_kernel<HD, ST>, 128, ring);
    const long long wslots = (long long)compute_sms() * std::max(1, wper);
    const int wctas = (int)std::min<long long>(wslots, (pairs + kWarps - 1) / kWarps);
    AttnParams p{};
    p.q = a.q; p.kc = a.kc; p.vc = a.vc; p.pos = a.pos; p.o = a.o; p.ldo = a.ldo > 0 ? (size_t)a.ldo : (size_t)a.nq * a.hd; p.ws = a.ws; p.cnt = a.cnt;
    p.B = a.B; p.nq = a.nq; p.nkv = a.nkv; p.smax = a.smax; p.bt = a.bt; p.bt_stride = a.bt_stride;
    static const int env_evict_w = getenv("SIDP_ATTN_EVICT") ? atoi(getenv("SIDP_ATTN_EVICT")) : 1;
    p.kv_evict = env_evict_w;
    p.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)HD));
    if (swap8)
      return launch_pdl(attn_warp8_kernel<HD, ST>, dim3(wctas), dim3(128), ring, s, p);
    return launch_pdl(attn_warp_kernel<HD, ST>, dim3(wctas), dim3(128), ring, s, p);
  }
  int ctas = (int)cl;
  static const int env_ctas = getenv("SIDP_ATTN_CTAS") ? atoi(getenv("SIDP_ATTN_CTAS")) : 0;
  if (env_ctas > 0) ctas = env_ctas;   // perf experiments
  if ((size_t)ctas * 2 * 16 * (HD + 2) * 4 > a.ws_bytes)
    ctas = (int)(a.ws_bytes / ((size_t)2 * 16 * (HD + 2) * 4));
  if (ctas < 1) return cudaErrorInvalidValue;
  AttnParams p;
  p.q = a.q; p.kc = a.kc; p.vc = a.vc; p.pos = a.pos; p.o = a.o; p.ldo = a.ldo > 0 ? (size_t)a.ldo : (size_t)a.nq * a.hd; p.ws = a.ws; p.cnt = a.cnt;
  p.B = a.B; p.nq = a.nq; p.nkv = a.nkv; p.smax = a.smax; p.bt = a.bt; p.bt_stride = a.bt_stride;
  static const int env_evict = getenv("SIDP_ATTN_EVICT") ? atoi(getenv("SIDP_ATTN_EVICT")) : 1;
  p.kv_evict = env_evict;
  static const int env_pre = getenv("SIDP_ATTN_PRE") ? atoi(getenv("SIDP_ATTN_PRE")) : 1;
  p.pre_wait = env_pre;
  p.pair_mode = (long long)ctas == pairs ? 1 : 0;
  p.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)HD));
  if (swap8) return launch_pdl(attn_kernel<HD, ST, true>, dim3(ctas), dim3(128), smem, s, p);
  return launch_pdl(attn_kernel<HD, ST>, dim3(ctas), dim3(128), smem, s, p);
}

cudaError_t attention_launch(const AttnArgs& a, cudaStream_t s) {
  if (a.B <= 0) return cudaSuccess;
  if ((a.hd != 64 && a.hd != 128) || a.nq % a.nkv || a.nq / a.nkv > 16 || !a.cnt ||
      a.n_cnt < a.B * a.nkv)
    return cudaErrorInvalidValue;
  if (!g_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  // SIDP_ATTN_STAGES = 2 selects the 2-stage rings (3, the default, measured fastest: M2 29.05 vs
  // 29.72 ms with the transposed kernels).  The 4-stage instantiations are no longer selectable:
  // they raised cudaErrorIllegalInstruction on sm_100a in r2 (not investigated; r1 had measured
  // them slower, 214 vs 181 us).
  static const int stages = getenv("SIDP_ATTN_STAGES") ? atoi(getenv("SIDP_ATTN_STAGES")) : 3;
  g_attn_launches = 1;
  if (a.hd == 128) {
    if (stages == 2) return attn_launch_t<128, 2>(a, s);
    return attn_launch_t<128, 3>(a, s);
  }
  if (stages == 2) return attn_launch_t<64, 2>(a, s);
  return attn_launch_t<64, 3>(a, s);
}

cudaError_t attention_preload() {
  cudaFuncAttributes fa;
  cudaError_t e = cudaSuccess;
  if (cudaFuncGetAttributes(&fa, qkv_post_kernel<128, kQkvHeadsPerWarp>) != cudaSuccess) e = cudaGetLastError();
  if (cudaFuncGetAttributes(&fa, qkv_post_kernel<64, kQkvHeadsPerWarp>) != cudaSuccess) e = cudaGetLastError();
  // every kernel the launcher can pick — including the warp-per-pair kernels, which CaS steps
  // select from B * n_kv >= one wave of pairs: a module loaded lazily at its first launch waits
  // for the device to idle, a deadlock while another rank's flag wait spins — and the
  // >48 KB shared-memory attribute, set here for this device (sidp_alloc calls this)
#define SIDP_PRELOAD_ATTN(hd, st)                                                                \
  if (cudaFuncGetAttributes(&fa, attn_kernel<hd, st>) != cudaSuccess) e = cudaGetLastError();    \
  if (cudaFuncGetAttributes(&fa, attn_kernel<hd, st, true>) != cudaSuccess) e = cudaGetLastError(); \
  if (cudaFuncSetAttribute(attn_kernel<hd, st, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                           200 * 1024) != cudaSuccess) e = cudaGetLastError();                     \
  if (cudaFuncGetAttributes(&fa, attn_warp_kernel<hd, st>) != cudaSuccess) e = cudaGetLastError(); \
  if (cudaFuncGetAttributes(&fa, attn_warp8_kernel<hd, st>) != cudaSuccess) e = cudaGetLastError(); \
  if (cudaFuncSetAttribute(attn_warp8_kernel<hd, st>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                           200 * 1024) != cudaSuccess) e = cudaGetLastError();                     \
  if (cudaFuncSetAttribute(attn_kernel<hd, st>, cudaFuncAttributeMaxDynamicSharedMemorySize,      \
                           200 * 1024) != cudaSuccess) e = cudaGetLastError();                     \
  if (cudaFuncSetAttribute(attn_warp_kernel<hd, st>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                           200 * 1024) != cudaSuccess) e = cudaGetLastError();
  SIDP_PRELOAD_ATTN(128, 2) SIDP_PRELOAD_ATTN(128, 3)
  SIDP_PRELOAD_ATTN(64, 2) SIDP_PRELOAD_ATTN(64, 3)
#undef SIDP_PRELOAD_ATTN
  return e;
}

}  // namespace sidp
