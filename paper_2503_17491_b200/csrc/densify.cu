// Map growth on the device, after the reference's
// mapping.py:202-311 and add_keyframe (:412-438):
//   k_spawn_weights    _range_gradient_weights (:202-239): central / one-sided
//                      range differences over valid neighbours (azimuth wraps
//                      on full-circle cameras), magnitude hypot(gx, gy)
//   k_densify_mask     densify_mask (:306-311): valid & (opacity <= t_o | |D - D_kf| >= t_r)
//   k_spawn            spawn_splats (:283-303): back-projected surface points,
//                      keyframe normal (or facing the sensor), completed
//                      tangent frame, pixel-footprint scales, initial opacity
//   k_prune_flags + k_compact_*   SplatModel.prune / _Adam.prune: stable
//                      compaction of every per-splat array
// The weighted draw without replacement (numpy Generator.choice) stays on
// the host with the reference's own RNG call: the device supplies its
// float64 weights and consumes the drawn pixel indices.
#include "common.cuh"

namespace ss {

__global__ void k_spawn_weights(int W, int H, int wrap, const double* __restrict__ D, const uint8_t* __restrict__ V,
                                double* __restrict__ out) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= W * H) return;
  const int r = p / W, c = p % W;
  if (!V[p]) {
    out[p] = 0.0;
    return;
  }
  double g[2];
  for (int axis = 0; axis < 2; ++axis) {  // 0: columns (azimuth), 1: rows
    int ip, im;                           // +1 and -1 neighbours, -1 when absent
    if (axis == 0) {
      ip = c + 1 < W ? p + 1 : (wrap ? p + 1 - W : -1);
      im = c > 0 ? p - 1 : (wrap ? p - 1 + W : -1);
    } else {
      ip = r + 1 < H ? p + W : -1;
      im = r > 0 ? p - W : -1;
    }
    const bool pv = ip >= 0 && V[ip], mv = im >= 0 && V[im];
    double v = 0.0;
    if (pv && mv)
      v = 0.5 * (D[ip] - D[im]);
    else if (pv)
      v = D[ip] - D[p];
    else if (mv)
      v = D[p] - D[im];
    g[axis] = v;
  }
  out[p] = hypot(g[0], g[1]);
}

__global__ void k_densify_mask(int P, const double* __restrict__ kf_range, const uint8_t* __restrict__ kf_valid,
                               const float* __restrict__ D, const float* __restrict__ O, double t_opacity,
                               double t_range, uint8_t* __restrict__ mask) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const bool thin = (double)O[p] <= t_opacity;
  const bool wrong = fabs((double)D[p] - kf_range[p]) >= t_range;
  mask[p] = kf_valid[p] && (thin || wrong);
}

struct SpawnK {
  int W;
  double fx, fy, cx, cy, off_u, off_v;
  double R[9], t[3];
  double gain, floor_, opacity;
};

__global__ void k_spawn(int m, const long long* __restrict__ pix, SpawnK k, const double* __restrict__ range,
                        const double* __restrict__ normal, const uint8_t* __restrict__ nvalid,
                        float* __restrict__ centers, float* __restrict__ ta_out, float* __restrict__ tb_out,
                        float* __restrict__ log_scales, float* __restrict__ logit) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const long long p = pix[i];
  const int r = (int)(p / k.W), c = (int)(p % k.W);
  const double u = (double)c + k.off_u, v = (double)r + k.off_v;  // sample_grid (geometry.py:176-180)
  const double az = (u - k.cx) / k.fx, el = (v - k.cy) / k.fy;
  const double d = range[p];
  const double ce = cos(el);
  const double ps[3] = {d * (ce * cos(az)), d * (ce * sin(az)), d * sin(el)};
  const double np_ = sqrt(ps[0] * ps[0] + ps[1] * ps[1] + ps[2] * ps[2]);
  double n[3];
  for (int q = 0; q < 3; ++q) n[q] = nvalid[p] ? normal[3 * p + q] : -(ps[q] / np_);
  const double nn = sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]);
  for (int q = 0; q < 3; ++q) n[q] /= nn;
  double cw[3], nw[3];
  for (int q = 0; q < 3; ++q) {
    cw[q] = k.R[3 * q] * ps[0] + k.R[3 * q + 1] * ps[1] + k.R[3 * q + 2] * ps[2] + k.t[q];
    nw[q] = k.R[3 * q] * n[0] + k.R[3 * q + 1] * n[1] + k.R[3 * q + 2] * n[2];
  }
  // _complete_frames (mapping.py:242-251)
  const double ref[3] = {fabs(nw[2]) > 0.9 ? 1.0 : 0.0, 0.0, fabs(nw[2]) > 0.9 ? 0.0 : 1.0};
  double a[3] = {nw[1] * ref[2] - nw[2] * ref[1], nw[2] * ref[0] - nw[0] * ref[2], nw[0] * ref[1] - nw[1] * ref[0]};
  const double na = sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2]);
  for (int q = 0; q < 3; ++q) a[q] /= na;
  const double b[3] = {nw[1] * a[2] - nw[2] * a[1], nw[2] * a[0] - nw[0] * a[2], nw[0] * a[1] - nw[1] * a[0]};
  for (int q = 0; q < 3; ++q) {
    centers[3 * i + q] = (float)cw[q];
    ta_out[3 * i + q] = (float)a[q];
    tb_out[3 * i + q] = (float)b[q];
  }
  const double s0 = fmax(k.gain * d * (1.0 / fabs(k.fx)), k.floor_);
  const double s1 = fmax(k.gain * d * (1.0 / fabs(k.fy)), k.floor_);
  log_scales[2 * i] = (float)log(s0);
  log_scales[2 * i + 1] = (float)log(s1);
  logit[i] = (float)(log(k.opacity) - log1p(-k.opacity));  // splats.py:53-55
}

// keep = sigmoid(logit) >= prune_opacity (SplatModel.opacities, splats.py:44-50, 221-223)
__global__ void k_prune_flags(int n, const float* __restrict__ logit, double prune_opacity,
                              uint32_t* __restrict__ keep, uint32_t* __restrict__ block_sum) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t kf = 0;
  if (i < n) {
    const double x = logit[i];
    double o;
    if (x >= 0) {
      o = 1.0 / (1.0 + exp(-x));
    } else {
      const double e = exp(x);
      o = e / (1.0 + e);
    }
    kf = o >= prune_opacity;
    keep[i] = kf;
  }
  const uint32_t b = __ballot_sync(0xffffffffu, kf);
  __shared__ uint32_t ws[8];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = __popc(b);
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t s = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += ws[w];
    block_sum[blockIdx.x] = s;
  }
}

// Stable compaction of rows (width floats each) with keep[i] set, block offsets
// from the exclusive scan of the per-block counts.
__global__ void k_compact_f32(int n, int width, const uint32_t* __restrict__ keep,
                              const uint32_t* __restrict__ block_off, const float* __restrict__ src,
                              float* __restrict__ dst) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t kf = i < n ? keep[i] : 0u;
  const uint32_t b = __ballot_sync(0xffffffffu, kf);
  __shared__ uint32_t ws[8];
  if (lane == 0) ws[warp] = __popc(b);
  __syncthreads();
  uint32_t off = block_off[blockIdx.x];
  for (int w = 0; w < warp; ++w) off += ws[w];
  off += __popc(b & ((1u << lane) - 1u));
  if (kf)
    for (int q = 0; q < width; ++q) dst[(size_t)off * width + q] = src[(size_t)i * width + q];
}

}  // namespace ss
