// Fused mapping loss: pixel gradients + loss parts for one keyframe
// (pkg/src/splatscan/mapping.py:128-196, range/opacity/normal terms; the
// per-splat scale hinge stays on the host, mapping.py:166-178).
#include "common.cuh"

namespace ss {

__global__ void k_mapping_loss(int P, const float* __restrict__ D, const float* __restrict__ N,
                               const float* __restrict__ O, const float* __restrict__ kf_range,
                               const uint8_t* __restrict__ kf_valid, const float* __restrict__ kf_normal,
                               const uint8_t* __restrict__ kf_nvalid, double w_opacity, double w_normal,
                               double range_floor, float* __restrict__ dD, float* __restrict__ dN,
                               float* __restrict__ dO, double* __restrict__ parts) {
  double ld = 0.0, lo = 0.0, ln = 0.0;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < P; p += gridDim.x * blockDim.x) {
    bool M = kf_valid[p] != 0;
    float gd = 0.f, go = 0.f, gn0 = 0.f, gn1 = 0.f, gn2 = 0.f;
    if (M) {
      double kr = kf_range[p];
      double w = 1.0 / fmax(kr, range_floor);
      double diff = (double)D[p] - kr;
      ld += w * fabs(diff);
      gd = (float)(diff > 0 ? w : (diff < 0 ? -w : 0.0));
      if (w_opacity != 0.0) {
        double o = O[p];
        double cl = fmax(o, 1e-6);
        lo += -log(cl);
        if (o > 1e-6) go = (float)(w_opacity * (-1.0 / cl));
      }
      if (kf_nvalid[p]) {
        double n0 = kf_normal[3 * p], n1 = kf_normal[3 * p + 1], n2 = kf_normal[3 * p + 2];
        ln += 1.0 - ((double)N[3 * p] * n0 + (double)N[3 * p + 1] * n1 + (double)N[3 * p + 2] * n2);
        gn0 = (float)(-w_normal * n0);
        gn1 = (float)(-w_normal * n1);
        gn2 = (float)(-w_normal * n2);
      }
    }
    dD[p] = gd;
    dO[p] = go;
    dN[3 * p] = gn0;
    dN[3 * p + 1] = gn1;
    dN[3 * p + 2] = gn2;
  }
  for (int off = 16; off > 0; off >>= 1) {
    ld += __shfl_xor_sync(0xffffffffu, ld, off);
    lo += __shfl_xor_sync(0xffffffffu, lo, off);
    ln += __shfl_xor_sync(0xffffffffu, ln, off);
  }
  __shared__ double red[3][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (lane == 0) {
    red[0][warp] = ld;
    red[1][warp] = lo;
    red[2][warp] = ln;
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += red[threadIdx.x][w];
    atomicAdd(&parts[threadIdx.x], s);
  }
}

}  // namespace ss
