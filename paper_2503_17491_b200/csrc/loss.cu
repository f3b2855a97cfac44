// Fused mapping loss: pixel gradients + loss parts for one keyframe
// (pkg/src/splatscan/mapping.py:128-196, range/opacity/normal terms; the
// per-splat scale hinge stays on the host, mapping.py:166-178).
#include "adam.cuh"
#include "common.cuh"

namespace ss {

__global__ void k_mapping_loss(int P, const float* __restrict__ D, const float* __restrict__ N,
                               const float* __restrict__ O, const float* __restrict__ kf_range,
                               const uint8_t* __restrict__ kf_valid, const float* __restrict__ kf_normal,
                               const uint8_t* __restrict__ kf_nvalid, double w_opacity, double w_normal,
                               double range_floor, float* __restrict__ dD, float* __restrict__ dN,
                               float* __restrict__ dO, double* __restrict__ parts) {
  pdl_wait();
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

namespace ss {

// Scale hinge (mapping.py:166-178): gradient w_scale on the larger axis of
// splats whose larger scale exceeds `cap` (first axis on ties, np.argmax),
// and the loss sum into loss[0].
__global__ void k_scale_loss(int n, const float* __restrict__ log_scales, double cap, double w_scale,
                             float* __restrict__ d_scales, double* __restrict__ loss) {
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  double l = 0.0;
  if (i < n) {
    const double s0 = exp((double)log_scales[2 * i]), s1 = exp((double)log_scales[2 * i + 1]);
    const double mx = fmax(s0, s1);
    const double over = mx - cap;
    float g0 = 0.f, g1 = 0.f;
    if (over > 0.0) {
      l = over;
      if (s0 >= s1)
        g0 = (float)w_scale;
      else
        g1 = (float)w_scale;
    }
    d_scales[2 * i] = g0;
    d_scales[2 * i + 1] = g1;
  }
  for (int off = 16; off > 0; off >>= 1) l += __shfl_xor_sync(0xffffffffu, l, off);
  if ((threadIdx.x & 31) == 0 && l != 0.0) atomicAdd(loss, l);
}

// Adam (AdamK, adam_splat): adam.cuh (shared with the finalize's fused epilogue).
__global__ void __launch_bounds__(256) k_adam(int n, AdamK a, const float* __restrict__ g, float* __restrict__ m,
                                              float* __restrict__ v) {
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) adam_splat(i, a, 1.f / a.b1c, 1.f / a.b2c, g, m, v);
}

// Device-resident step counter for CUDA-graph replays of the refine step:
// t += 1 and the bias corrections 1 - beta^t (what the host computes for ss_adam_step).
__global__ void k_adam_tick(int* __restrict__ t_dev, double b1, double b2, float* __restrict__ bias) {
  pdl_wait();
  const int t = *t_dev + 1;
  *t_dev = t;
  bias[0] = (float)(1.0 - pow(b1, (double)t));
  bias[1] = (float)(1.0 - pow(b2, (double)t));
}

__global__ void __launch_bounds__(256) k_adam_dev(int n, AdamK a, const float* __restrict__ bias,
                                                  const float* __restrict__ g, float* __restrict__ m,
                                                  float* __restrict__ v) {
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) adam_splat(i, a, 1.f / bias[0], 1.f / bias[1], g, m, v);
}

// history[it] = the 4 loss parts of this step; it += 1 (graph-replayed refine).
__global__ void k_store_parts(const double* __restrict__ parts, double* __restrict__ hist, int* __restrict__ it,
                              int cap) {
  pdl_wait();
  const int i = *it;
  if (i < cap)
    for (int q = 0; q < 4; ++q) hist[4 * i + q] = parts[q];
  *it = i + 1;
}

}  // namespace ss
