// fixup.cuh — device helpers of the deferred stream-K fix-up (summing fp32 k-range slices in
// slice order + the bf16 residual, RMSNorm statistics and scaling), shared by resid_norm_kernel
// (kernels/norm.cu) and the fused MLP kernel's fix-up tail (kernels/gemm.cu).
#pragma once
#include "common.cuh"
#include "kernels.h"

namespace sidp {

SIDP_DEV float2 bf16x2_to_f2(uint32_t w) {
  __nv_bfloat162 h;
  memcpy(&h, &w, 4);
  return __bfloat1622float2(h);
}
SIDP_DEV uint32_t f2_to_bf16x2(float a, float b) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  uint32_t w;
  memcpy(&w, &h, 4);
  return w;
}

constexpr int kFixSeg = 4;
// one 8-feature vector of the deferred fix-up: fp32 slices summed in slice order (slices past
// nseg add +0), + the bf16 residual, rounded once; the loads of a vector are issued together
template <int NS = kFixSeg>
SIDP_DEV uint4 fix_vector(const PartialSrc& ps, const float* src, size_t slice,
                                            int nseg, uint4 rr) {
  float4 lo[NS], hi[NS];
#pragma unroll
  for (int q = 0; q < NS; ++q) {
    lo[q] = hi[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (q < nseg) {
      lo[q] = __ldcg(reinterpret_cast<const float4*>(src + q * slice));
      hi[q] = __ldcg(reinterpret_cast<const float4*>(src + q * slice + 4));
    }
  }
  float4 al = make_float4(0.f, 0.f, 0.f, 0.f), ah = al;
#pragma unroll
  for (int q = 0; q < NS; ++q) {
    al.x += lo[q].x; al.y += lo[q].y; al.z += lo[q].z; al.w += lo[q].w;
    ah.x += hi[q].x; ah.y += hi[q].y; ah.z += hi[q].z; ah.w += hi[q].w;
  }
  for (int q = NS; q < nseg; ++q) {
    const float4 x0 = __ldcg(reinterpret_cast<const float4*>(src + q * slice));
    const float4 x1 = __ldcg(reinterpret_cast<const float4*>(src + q * slice + 4));
    al.x += x0.x; al.y += x0.y; al.z += x0.z; al.w += x0.w;
    ah.x += x1.x; ah.y += x1.y; ah.z += x1.z; ah.w += x1.w;
  }
  const float2 r0 = bf16x2_to_f2(rr.x), r1 = bf16x2_to_f2(rr.y), r2 = bf16x2_to_f2(rr.z),
               r3 = bf16x2_to_f2(rr.w);
  return make_uint4(f2_to_bf16x2(al.x + r0.x, al.y + r0.y), f2_to_bf16x2(al.z + r1.x, al.w + r1.y),
                    f2_to_bf16x2(ah.x + r2.x, ah.y + r2.y), f2_to_bf16x2(ah.z + r3.x, ah.w + r3.y));
}
SIDP_DEV float sumsq8(uint4 v) {
  const float2 o0 = bf16x2_to_f2(v.x), o1 = bf16x2_to_f2(v.y), o2 = bf16x2_to_f2(v.z),
               o3 = bf16x2_to_f2(v.w);
  return o0.x * o0.x + o0.y * o0.y + o1.x * o1.x + o1.y * o1.y + o2.x * o2.x + o2.y * o2.y +
         o3.x * o3.x + o3.y * o3.y;
}
SIDP_DEV uint4 scale8(uint4 v, uint4 gw, float r) {
  uint4 o;
  uint32_t* ow = reinterpret_cast<uint32_t*>(&o);
  const uint32_t vw[4] = {v.x, v.y, v.z, v.w}, gg[4] = {gw.x, gw.y, gw.z, gw.w};
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float2 x = bf16x2_to_f2(vw[q]), gf = bf16x2_to_f2(gg[q]);
    ow[q] = f2_to_bf16x2(x.x * r * gf.x, x.y * r * gf.y);
  }
  return o;
}


}  // namespace sidp
