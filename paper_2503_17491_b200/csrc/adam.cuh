// Adam over the packed raw gradient (n x 12: centers 3 | raw_t_alpha 3 | raw_t_beta 3 |
// log_scales 2 | logit_opacity 1) with per-group learning rates, bias correction and the
// log-scale clamp of refine (mapping.py:367-379, 495-496).  Shared by k_adam / k_adam_dev
// (loss.cu) and the Adam epilogue of k_finalize (blend.cu), so both give the same bits.
#pragma once
#include "common.cuh"

namespace ss {

struct AdamK {
  float* p[5];
  float lr[5];
  float b1, b2, eps, b1c, b2c, lo, hi;
};

// one splat: gradient row gg (12 values), moments rows m, v (float4 x 3 each), in place
__device__ __forceinline__ void adam_row(int i, const AdamK& a, float ib1c, float ib2c, const float (&gg)[12],
                                         float* __restrict__ m, float* __restrict__ v) {
  float4* m4 = reinterpret_cast<float4*>(m) + 3 * (size_t)i;
  float4* v4 = reinterpret_cast<float4*>(v) + 3 * (size_t)i;
  float mm[12], vv[12];
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    const float4 b4 = m4[q], c4 = v4[q];
    mm[4 * q] = b4.x; mm[4 * q + 1] = b4.y; mm[4 * q + 2] = b4.z; mm[4 * q + 3] = b4.w;
    vv[4 * q] = c4.x; vv[4 * q + 1] = c4.y; vv[4 * q + 2] = c4.z; vv[4 * q + 3] = c4.w;
  }
  constexpr int grp_of[12] = {0, 0, 0, 1, 1, 1, 2, 2, 2, 3, 3, 4};
  constexpr int off_of[12] = {0, 1, 2, 0, 1, 2, 0, 1, 2, 0, 1, 0};
  constexpr int width[5] = {3, 3, 3, 2, 1};
#pragma unroll
  for (int c = 0; c < 12; ++c) {
    const int grp = grp_of[c];
    mm[c] = a.b1 * mm[c] + (1.f - a.b1) * gg[c];
    vv[c] = a.b2 * vv[c] + (1.f - a.b2) * gg[c] * gg[c];
    const float upd = a.lr[grp] * (mm[c] * ib1c) / (sqrtf(vv[c] * ib2c) + a.eps);
    float* pp = a.p[grp] + (size_t)i * width[grp] + off_of[c];
    float x = *pp - upd;
    if (grp == 3) x = fminf(fmaxf(x, a.lo), a.hi);
    *pp = x;
  }
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    m4[q] = make_float4(mm[4 * q], mm[4 * q + 1], mm[4 * q + 2], mm[4 * q + 3]);
    v4[q] = make_float4(vv[4 * q], vv[4 * q + 1], vv[4 * q + 2], vv[4 * q + 3]);
  }
}

// One thread per splat: its 12 gradient values as three float4 rows (one thread per
// (splat, component) measured 40 us for 200 k splats: five scattered parameter arrays per
// warp instruction).
__device__ __forceinline__ void adam_splat(int i, const AdamK& a, float ib1c, float ib2c,
                                           const float* __restrict__ g, float* __restrict__ m,
                                           float* __restrict__ v) {
  const float4* g4 = reinterpret_cast<const float4*>(g) + 3 * (size_t)i;
  float gg[12];
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    const float4 a4 = g4[q];
    gg[4 * q] = a4.x; gg[4 * q + 1] = a4.y; gg[4 * q + 2] = a4.z; gg[4 * q + 3] = a4.w;
  }
  adam_row(i, a, ib1c, ib2c, gg, m, v);
}

}  // namespace ss
