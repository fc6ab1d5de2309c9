// attention.cu — QKV post-processing and GQA decode attention.
//
// qkv_post: per token, per head: optional per-head RMSNorm (Qwen3 qk_norm), rotate-half RoPE
// from an fp64-built (cos, sin) table, q -> bf16, k/v appended to the local KV cache at pos_b.
// The KV cache is local and never pooled.
//
// decode attention: HBM-bound (4096 B of K/V per context token per layer).
// One CTA per (kv head, sequence, split), 4 warps; each warp streams 16-token K/V chunks
// through a 2-stage cp.async ring in XOR-swizzled shared memory and runs the G query heads
// of the group (padded to 16 rows) through mma.sync m16n8k16 bf16 tensor-core tiles for
// S = q K^T and O += P V, with an fp32 online softmax (exp2 domain).  Warps and splits are
// merged with the usual (max, sum) rescaling.
#include <cmath>

#include "../common.cuh"
#include "../kernels.h"

namespace sidp {

namespace {

// ---------------------------------------------------------------- qkv post
// lane l holds dims [E*l, E*l+E) of the first half and the same dims + hd/2 (its RoPE
// partners), E = hd/64: every load and store is one E-wide vector per lane
template <int HD>
__global__ void __launch_bounds__(256) qkv_post_kernel(QkvPostArgs a) {
  pdl_trigger();
  pdl_wait();
  constexpr int half = HD / 2, E = HD / 64;
  // grid (B, ceil(nh / 8)): one warp per (token, head) so every load is issued up front
  const int b = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nh = a.nq + 2 * a.nkv;
  const int nwarps = (blockDim.x >> 5) * gridDim.y;
  const int head0 = blockIdx.y * (blockDim.x >> 5) + warp;
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
  for (int head = head0; head < nh; head += nwarps) {
    const float* src = a.qkv + ((size_t)b * nh + head) * HD;
    const bool is_v = head >= a.nq + a.nkv;
    const bool is_q = head < a.nq;
    float x1[E], x2[E];
    if constexpr (E == 2) {
      const float2 u = *reinterpret_cast<const float2*>(src + i0);
      const float2 w = *reinterpret_cast<const float2*>(src + i0 + half);
      x1[0] = u.x; x1[1] = u.y; x2[0] = w.x; x2[1] = w.y;
    } else {
      x1[0] = src[i0];
      x2[0] = src[i0 + half];
    }
    if (!is_v) {
      const bf16* gain = is_q ? a.gq : a.gk;
      if (gain) {
        float ss = 0.0f;
#pragma unroll
        for (int e = 0; e < E; ++e) ss += x1[e] * x1[e] + x2[e] * x2[e];
        ss = warp_sum(ss);
        const float r = rsqrtf(ss / (float)HD + a.eps);
#pragma unroll
        for (int e = 0; e < E; ++e) {
          x1[e] = x1[e] * r * bf16_to_f(gain[i0 + e]);
          x2[e] = x2[e] * r * bf16_to_f(gain[i0 + e + half]);
        }
      }
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const float y1 = x1[e] * cs[e][0] - x2[e] * cs[e][1];
        const float y2 = x2[e] * cs[e][0] + x1[e] * cs[e][1];
        x1[e] = y1;
        x2[e] = y2;
      }
    }
    bf16* dst;
    if (is_q) {
      dst = a.q + ((size_t)b * a.nq + head) * HD;
    } else {
      const int g = is_v ? head - a.nq - a.nkv : head - a.nq;
      bf16* cache = is_v ? a.vc : a.kc;
      dst = cache + (((size_t)b * a.nkv + g) * a.smax + pos) * HD;
    }
    if constexpr (E == 2) {
      *reinterpret_cast<__nv_bfloat162*>(dst + i0) = __floats2bfloat162_rn(x1[0], x1[1]);
      *reinterpret_cast<__nv_bfloat162*>(dst + i0 + half) = __floats2bfloat162_rn(x2[0], x2[1]);
    } else {
      dst[i0] = f_to_bf16(x1[0]);
      dst[i0 + half] = f_to_bf16(x2[0]);
    }
  }
}

// ---------------------------------------------------------------- attention helpers
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem)
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
  float* ws;
  int nq, nkv, smax, splits, tok_per_split;
  float scale_log2;
};

constexpr int kChunk = 16;
constexpr int kWarps = 4;

template <int HD>
__global__ void __launch_bounds__(128) attn_kernel(const AttnParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int CPR = HD / 8;                         // 16-byte chunks per row
  constexpr int TILE = kChunk * HD;                   // elements per K (or V) chunk
  pdl_trigger();
  pdl_wait();
  const int g = blockIdx.x, b = blockIdx.y, split = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tq = lane & 3;
  const int G = p.nq / p.nkv;
  const int n_tok = p.pos[b] + 1;
  const int t_begin = split * p.tok_per_split;
  const int t_end = min(n_tok, t_begin + p.tok_per_split);
  const int nchunks = t_end > t_begin ? (t_end - t_begin + kChunk - 1) / kChunk : 0;

  bf16* wbuf = reinterpret_cast<bf16*>(smem) + (size_t)warp * 4 * TILE;   // [stage][K|V]
  const bf16* kbase = p.kc + ((size_t)b * p.nkv + g) * p.smax * HD;
  const bf16* vbase = p.vc + ((size_t)b * p.nkv + g) * p.smax * HD;

  // Q fragments (rows = heads of the group, padded to 16)
  uint32_t qa[HD / 16][4];
  {
    const bf16* qb = p.q + ((size_t)b * p.nq + (size_t)g * G) * HD;
    const int r0 = gid, r1 = gid + 8;
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
      const int c = kk * 16 + 2 * tq;
      qa[kk][0] = r0 < G ? *reinterpret_cast<const uint32_t*>(qb + r0 * HD + c) : 0u;
      qa[kk][1] = r1 < G ? *reinterpret_cast<const uint32_t*>(qb + r1 * HD + c) : 0u;
      qa[kk][2] = r0 < G ? *reinterpret_cast<const uint32_t*>(qb + r0 * HD + c + 8) : 0u;
      qa[kk][3] = r1 < G ? *reinterpret_cast<const uint32_t*>(qb + r1 * HD + c + 8) : 0u;
    }
  }

  float o[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.0f;
  float mrow[2] = {-INFINITY, -INFINITY};
  float lrow[2] = {0.0f, 0.0f};

  auto load_chunk = [&](int stage, int c) {
    const int t0 = t_begin + c * kChunk;
    bf16* sk = wbuf + stage * 2 * TILE;
    bf16* sv = sk + TILE;
#pragma unroll
    for (int it = 0; it < (kChunk * CPR) / 32; ++it) {
      const int e = it * 32 + lane;
      const int row = e / CPR, cc = e % CPR;
      const int t = min(t0 + row, n_tok - 1);
      const int sw = (cc ^ (row & 7));
      cp_async16(sk + row * HD + sw * 8, kbase + (size_t)t * HD + cc * 8);
      cp_async16(sv + row * HD + sw * 8, vbase + (size_t)t * HD + cc * 8);
    }
  };

  if (warp < nchunks) load_chunk(0, warp);
  cp_async_commit();
  int it = 0;
  for (int c = warp; c < nchunks; c += kWarps, ++it) {
    const int cn = c + kWarps;
    if (cn < nchunks) load_chunk((it + 1) & 1, cn);
    cp_async_commit();
    cp_async_wait<1>();
    __syncwarp();
    const bf16* sk = wbuf + (it & 1) * 2 * TILE;
    const bf16* sv = sk + TILE;
    const uint32_t skb = smem_u32(sk), svb = smem_u32(sv);
    const int t0 = t_begin + c * kChunk;

    // S = Q K^T for 16 tokens (two n-tiles of 8)
    float s[2][4];
#pragma unroll
    for (int j = 0; j < 2; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.0f;
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
      const int mat = lane >> 3, r = lane & 7;
      const int tok = (mat >> 1) * 8 + r;
      const int cc = kk * 2 + (mat & 1);
      uint32_t b0, b1, b2, b3;
      ldsm_x4(skb + (tok * HD + ((cc ^ (tok & 7)) * 8)) * 2, b0, b1, b2, b3);
      mma_bf16(s[0], qa[kk], b0, b1);
      mma_bf16(s[1], qa[kk], b2, b3);
    }
    // mask + online softmax (rows gid and gid+8)
    float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int tok = t0 + j * 8 + 2 * tq + (e & 1);
        s[j][e] = tok < t_end ? s[j][e] * p.scale_log2 : -INFINITY;
        mx[e >> 1] = fmaxf(mx[e >> 1], s[j][e]);
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
        s[j][e] = exp2f(s[j][e] - muse[e >> 1]);
        lrow[e >> 1] += s[j][e];
      }
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) {
      o[i][0] *= alpha[0];
      o[i][1] *= alpha[0];
      o[i][2] *= alpha[1];
      o[i][3] *= alpha[1];
    }
    uint32_t pa[4];
    pa[0] = pack_bf16(s[0][0], s[0][1]);
    pa[1] = pack_bf16(s[0][2], s[0][3]);
    pa[2] = pack_bf16(s[1][0], s[1][1]);
    pa[3] = pack_bf16(s[1][2], s[1][3]);
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
    __syncwarp();
  }
  cp_async_wait<0>();
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    lrow[h] += __shfl_xor_sync(0xffffffffu, lrow[h], 1);
    lrow[h] += __shfl_xor_sync(0xffffffffu, lrow[h], 2);
  }
  __syncthreads();
  // ---- merge the 4 warps through shared memory
  float* sm_o = reinterpret_cast<float*>(smem);                 // [warp][16][HD]
  float* sm_m = sm_o + kWarps * 16 * HD;                        // [warp][16]
  float* sm_l = sm_m + kWarps * 16;
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
  __syncthreads();
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
    const int head = g * G + row;
    if (p.splits == 1) {
      p.o[((size_t)b * p.nq + head) * HD + col] = f_to_bf16(L > 0.0f ? O / L : 0.0f);
    } else {
      float* part = p.ws + (((size_t)b * p.nq + head) * p.splits + split) * (HD + 2);
      part[2 + col] = O;
      if (col == 0) {
        part[0] = M;
        part[1] = L;
      }
    }
  }
}

template <int HD>
__global__ void attn_combine_kernel(const float* ws, bf16* o, int nq, int splits) {
  pdl_trigger();
  pdl_wait();
  const int bh = blockIdx.x;   // b * nq + head
  const float* part = ws + (size_t)bh * splits * (HD + 2);
  float M = -INFINITY;
  for (int s = 0; s < splits; ++s) M = fmaxf(M, part[s * (HD + 2)]);
  for (int col = threadIdx.x; col < HD; col += blockDim.x) {
    float L = 0.0f, O = 0.0f;
    if (M != -INFINITY) {
      for (int s = 0; s < splits; ++s) {
        const float ms = part[s * (HD + 2)];
        const float f = ms == -INFINITY ? 0.0f : exp2f(ms - M);
        L += f * part[s * (HD + 2) + 1];
        O += f * part[s * (HD + 2) + 2 + col];
      }
    }
    o[(size_t)bh * HD + col] = f_to_bf16(L > 0.0f ? O / L : 0.0f);
  }
}

int g_sms = 0;
thread_local int g_attn_launches = 0;

}  // namespace

cudaError_t qkv_post_launch(const QkvPostArgs& a, cudaStream_t s) {
  if (a.B <= 0) return cudaSuccess;
  if (a.hd != 64 && a.hd != 128) return cudaErrorInvalidValue;
  const int nh = a.nq + 2 * a.nkv;
  if (a.hd == 128) return launch_pdl(qkv_post_kernel<128>, dim3(a.B, (nh + 7) / 8), dim3(256), 0, s, a);
  return launch_pdl(qkv_post_kernel<64>, dim3(a.B, (nh + 7) / 8), dim3(256), 0, s, a);
}

int attention_last_launch_count() { return g_attn_launches; }

cudaError_t attention_launch(const AttnArgs& a, cudaStream_t s) {
  if (a.B <= 0) return cudaSuccess;
  if ((a.hd != 64 && a.hd != 128) || a.nq % a.nkv || a.nq / a.nkv > 16) return cudaErrorInvalidValue;
  if (!g_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(attn_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaFuncSetAttribute(attn_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  }
  // split the context so the grid covers the SMs ~2x when B * n_kv is small
  const int max_tok = (a.max_tokens > 0 && a.max_tokens < a.smax) ? a.max_tokens : a.smax;
  const int base = a.B * a.nkv;
  int splits = 1;
  const int target = 2 * g_sms * 3;
  if (base < target) splits = (target + base - 1) / base;
  const int max_splits = (max_tok + 255) / 256;
  if (splits > max_splits) splits = max_splits;
  if (splits < 1) splits = 1;
  int tok_per = (max_tok + splits - 1) / splits;
  tok_per = ((tok_per + 63) / 64) * 64;
  splits = (max_tok + tok_per - 1) / tok_per;
  if (splits > 1 && (size_t)a.B * a.nq * splits * (a.hd + 2) * 4 > a.ws_bytes) {
    splits = 1;
    tok_per = max_tok;
  }
  AttnParams p;
  p.q = a.q; p.kc = a.kc; p.vc = a.vc; p.pos = a.pos; p.o = a.o; p.ws = a.ws;
  p.nq = a.nq; p.nkv = a.nkv; p.smax = a.smax; p.splits = splits; p.tok_per_split = tok_per;
  p.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)a.hd));
  dim3 grid(a.nkv, a.B, splits);
  const size_t smem = (size_t)kWarps * 4 * kChunk * a.hd * 2;
  cudaError_t e = a.hd == 128 ? launch_pdl(attn_kernel<128>, grid, dim3(128), smem, s, p)
                              : launch_pdl(attn_kernel<64>, grid, dim3(128), smem, s, p);
  g_attn_launches = 1;
  if (e != cudaSuccess || splits == 1) return e;
  g_attn_launches = 2;
  const float* wsc = a.ws;
  bf16* oc = a.o;
  const int nq = a.nq;
  return a.hd == 128 ? launch_pdl(attn_combine_kernel<128>, dim3(a.B * a.nq), dim3(128), 0, s, wsc, oc, nq, splits)
                     : launch_pdl(attn_combine_kernel<64>, dim3(a.B * a.nq), dim3(64), 0, s, wsc, oc, nq, splits);
}

cudaError_t attention_preload() {
  cudaFuncAttributes fa;
  cudaError_t e = cudaSuccess;
  if (cudaFuncGetAttributes(&fa, qkv_post_kernel<128>) != cudaSuccess) e = cudaGetLastError();
  if (cudaFuncGetAttributes(&fa, qkv_post_kernel<64>) != cudaSuccess) e = cudaGetLastError();
  if (cudaFuncGetAttributes(&fa, attn_kernel<128>) != cudaSuccess) e = cudaGetLastError();
  if (cudaFuncGetAttributes(&fa, attn_kernel<64>) != cudaSuccess) e = cudaGetLastError();
  if (cudaFuncGetAttributes(&fa, attn_combine_kernel<128>) != cudaSuccess) e = cudaGetLastError();
  if (cudaFuncGetAttributes(&fa, attn_combine_kernel<64>) != cudaSuccess) e = cudaGetLastError();
  return e;
}

}  // namespace sidp
