// K5 photometric (range-warp) registration on the device.
//
// Reference behaviour (pkg/src/splatscan/):
//   registration.py:170-213   sample_model: confident rendered pixels, range
//                             jumps removed, back-projected to the world
//   geometry.py:252-268       build_range_image: scatter-min of scan ranges
//   registration.py:277-313   _bilinear_range (no seam wrap, spread gate)
//   registration.py:316-362   _photo_system: residuals, median trim, Jacobian
//   registration.py:219-228   Huber weights / value
//   registration.py:470-477   H, b accumulation
// Everything per anchor is float64 (M ~ 4e4 anchors: latency-bound, not
// FLOP-bound); the median of |r| is an exact radix select on the float64
// bit patterns; the 6x6 system and objective are float64 block reductions.
#include "common.cuh"

namespace ss {

struct RegCam {
  int W, H;
  double fx, fy, cx, cy, off_u, off_v;
};

// ---- anchors (sample_model) ---------------------------------------------------
// depth = range / max(opacity, 1e-12) where opacity > vis and range > 0.
__global__ void k_anchor_depth(int P, const float* __restrict__ D, const float* __restrict__ O, double vis,
                               double* __restrict__ depth, uint8_t* __restrict__ m) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const double o = O[p], d = D[p];
  const bool ok = o > vis && d > 0.0;
  m[p] = ok;
  depth[p] = ok ? d / fmax(o, 1e-12) : 0.0;
}

// _jump_mask: a confident pixel whose depth differs by more than `gate` from
// a confident 4-neighbour is dropped (rows never wrap; columns wrap when the
// camera closes the circle).  keep[p] = m & !bad; block sums for compaction.
__global__ void k_anchor_keep(int W, int H, int wrap, double gate, const double* __restrict__ depth,
                              const uint8_t* __restrict__ m, uint8_t* __restrict__ keep,
                              uint32_t* __restrict__ block_sum) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t k = 0;
  if (p < W * H && m[p]) {
    const int r = p / W, c = p % W;
    const double d = depth[p];
    bool bad = false;
    if (r > 0 && m[p - W] && fabs(d - depth[p - W]) > gate) bad = true;
    if (r + 1 < H && m[p + W] && fabs(d - depth[p + W]) > gate) bad = true;
    int cl = c - 1, cr = c + 1;
    if (wrap) {
      cl = (cl + W) % W;
      cr = cr % W;
    }
    if (cl >= 0 && m[r * W + cl] && fabs(d - depth[r * W + cl]) > gate) bad = true;
    if (cr < W && m[r * W + cr] && fabs(d - depth[r * W + cr]) > gate) bad = true;
    k = !bad;
  }
  if (p < W * H) keep[p] = (uint8_t)k;
  for (int off = 16; off > 0; off >>= 1) k += __shfl_xor_sync(0xffffffffu, k, off);
  __shared__ uint32_t ws[8];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = k;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t s = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += ws[w];
    block_sum[blockIdx.x] = s;
  }
}

// Compact kept pixels in row-major order, keep every `thin`-th one
// (X_w = model_pts[::thin], registration.py:430), back-project and map to
// the world with the render pose.
__global__ void k_anchor_emit(int W, int H, RegCam cam, PoseK pose, int thin, const double* __restrict__ depth,
                              const uint8_t* __restrict__ keep, const uint32_t* __restrict__ block_off,
                              double* __restrict__ X, int cap, int* __restrict__ count) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t k = (p < W * H) ? keep[p] : 0u;
  const uint32_t bal = __ballot_sync(0xffffffffu, k);
  __shared__ uint32_t ws[8];
  if (lane == 0) ws[warp] = __popc(bal);
  __syncthreads();
  uint32_t wex = 0, tot = 0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
    if (w < warp) wex += ws[w];
    tot += ws[w];
  }
  const uint32_t idx = block_off[blockIdx.x] + wex + __popc(bal & ((1u << lane) - 1u));
  if (p == W * H - 1 || (blockIdx.x + 1) * blockDim.x >= W * H) {
    if (threadIdx.x == 0) {
      const uint32_t all = block_off[blockIdx.x] + tot;
      count[0] = (int)all;                        // kept pixels (model_pts)
      count[1] = (int)((all + thin - 1) / thin);  // anchors after thinning
    }
  }
  if (!k || (idx % thin) != 0) return;
  const int a = idx / thin;
  if (a >= cap) return;
  const int r = p / W, c = p % W;
  const double u = (double)c + cam.off_u, v = (double)r + cam.off_v;
  const double az = (u - cam.cx) / cam.fx, el = (v - cam.cy) / cam.fy;
  double sa, ca, se, ce;
  sincos(az, &sa, &ca);
  sincos(el, &se, &ce);
  const double d = depth[p];
  const double pc[3] = {d * (ce * ca), d * (ce * sa), d * se};
  for (int q = 0; q < 3; ++q)
    X[3 * a + q] = pose.R[3 * q] * pc[0] + pose.R[3 * q + 1] * pc[1] + pose.R[3 * q + 2] * pc[2] + pose.t[q];
}

__global__ void k_excl_scan_small(int n, uint32_t* __restrict__ v) {
  __shared__ uint32_t part[1024];
  const int tid = threadIdx.x;
  const int per = (n + 1023) / 1024;
  const int b = tid * per, e = min(b + per, n);
  uint32_t s = 0;
  for (int i = b; i < e; ++i) s += v[i];
  part[tid] = s;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {
    const uint32_t x = tid >= off ? part[tid - off] : 0u;
    __syncthreads();
    part[tid] += x;
    __syncthreads();
  }
  uint32_t run = part[tid] - s;
  for (int i = b; i < e; ++i) {
    const uint32_t c = v[i];
    v[i] = run;
    run += c;
  }
}

// ---- scan range image (build_range_image) -------------------------------------
__global__ void k_fill_u64(int n, unsigned long long* __restrict__ p, unsigned long long v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

__global__ void k_range_scatter(const double* __restrict__ pts, int N, RegCam cam,
                                unsigned long long* __restrict__ img) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const double x = pts[3 * i], y = pts[3 * i + 1], z = pts[3 * i + 2];
  const double r = sqrt(x_add(x_add(x_mul(x, x), x_mul(y, y)), x_mul(z, z)));
  if (!(r > 1e-9)) return;
  const double az = atan2(y, x), el = atan2(z, hypot(x, y));
  const double u = x_add(x_mul(cam.fx, az), cam.cx), v = x_add(x_mul(cam.fy, el), cam.cy);
  const double cu = floor(x_add(u, 0.5)), cv = floor(x_add(v, 0.5));  // half-up (geometry.py:136-145)
  if (!(cu >= 0.0 && cu < cam.W && cv >= 0.0 && cv < cam.H)) return;
  atomicMin(&img[(size_t)cv * cam.W + (size_t)cu], (unsigned long long)__double_as_longlong(r));
}

__global__ void k_range_finish(int P, unsigned long long* __restrict__ img, uint8_t* __restrict__ valid) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const unsigned long long b = img[p];
  const bool ok = b != 0x7ff0000000000000ull;  // +inf marks an empty pixel
  valid[p] = ok;
  if (!ok) img[p] = 0ull;  // range 0.0
}

// ---- photometric system (_photo_system) ---------------------------------------
struct PhotoTmp {
  double r, du, dv, q[3];
};

// Residual of anchor i at pose T (registration.py:324-340); false when the
// anchor has no valid bilinear sample.
__device__ __forceinline__ bool photo_resid_one(const double* __restrict__ X, int i, const PoseK& T, const RegCam& cam,
                                                const double* __restrict__ srange,
                                                const uint8_t* __restrict__ svalid, double spread_gate,
                                                PhotoTmp& t) {
  // q = T^-1 X = R^T (X - t)
  double d[3], q[3];
  for (int c = 0; c < 3; ++c) d[c] = X[3 * i + c] - T.t[c];
  for (int c = 0; c < 3; ++c) q[c] = T.R[c] * d[0] + T.R[3 + c] * d[1] + T.R[6 + c] * d[2];
  const double rho2 = q[0] * q[0] + q[1] * q[1];
  const double r2 = rho2 + q[2] * q[2];
  const double az = atan2(q[1], q[0]), el = atan2(q[2], hypot(q[0], q[1]));
  const double u = cam.fx * az + cam.cx - cam.off_u, v = cam.fy * el + cam.cy - cam.off_v;
  const double fi = floor(u), fj = floor(v);
  bool ok = rho2 > 1e-12 && fi >= 0.0 && fi + 1.0 < cam.W && fj >= 0.0 && fj + 1.0 < cam.H;
  if (!ok) return false;
  const int i0 = (int)fi, j0 = (int)fj;
  const double fu = u - fi, fv = v - fj;
  const size_t p00 = (size_t)j0 * cam.W + i0;
  ok = svalid[p00] && svalid[p00 + 1] && svalid[p00 + cam.W] && svalid[p00 + cam.W + 1];
  if (!ok) return false;
  const double d00 = srange[p00], d10 = srange[p00 + 1], d01 = srange[p00 + cam.W], d11 = srange[p00 + cam.W + 1];
  const double hi = fmax(fmax(d00, d10), fmax(d01, d11)), lo = fmin(fmin(d00, d10), fmin(d01, d11));
  ok = hi - lo <= spread_gate;
  const double top = d00 * (1 - fu) + d10 * fu;
  const double bot = d01 * (1 - fu) + d11 * fu;
  const double val = top * (1 - fv) + bot * fv;
  t.r = sqrt(r2) - val;
  t.du = (d10 - d00) * (1 - fv) + (d11 - d01) * fv;
  t.dv = bot - top;
  t.q[0] = q[0];
  t.q[1] = q[1];
  t.q[2] = q[2];
  return ok;
}

// photo_resid_one without branches (out-of-image anchors read pixel 0 and are
// flagged): two calls on independent anchors interleave in the scheduler.
__device__ __forceinline__ bool photo_resid_nb(const double* __restrict__ X, int i, const PoseK& T, const RegCam& cam,
                                               const double* __restrict__ srange,
                                               const uint8_t* __restrict__ svalid, double spread_gate,
                                               PhotoTmp& t) {
  double d[3], q[3];
  for (int c = 0; c < 3; ++c) d[c] = X[3 * i + c] - T.t[c];
  for (int c = 0; c < 3; ++c) q[c] = T.R[c] * d[0] + T.R[3 + c] * d[1] + T.R[6 + c] * d[2];
  const double rho2 = q[0] * q[0] + q[1] * q[1];
  const double r2 = rho2 + q[2] * q[2];
  const double az = atan2(q[1], q[0]), el = atan2(q[2], hypot(q[0], q[1]));
  const double u = cam.fx * az + cam.cx - cam.off_u, v = cam.fy * el + cam.cy - cam.off_v;
  const double fi = floor(u), fj = floor(v);
  const bool in = rho2 > 1e-12 && fi >= 0.0 && fi + 1.0 < cam.W && fj >= 0.0 && fj + 1.0 < cam.H;
  const int i0 = in ? (int)fi : 0, j0 = in ? (int)fj : 0;
  const double fu = u - fi, fv = v - fj;
  const size_t p00 = (size_t)j0 * cam.W + i0;
  const bool val4 = svalid[p00] && svalid[p00 + 1] && svalid[p00 + cam.W] && svalid[p00 + cam.W + 1];
  const double d00 = srange[p00], d10 = srange[p00 + 1], d01 = srange[p00 + cam.W], d11 = srange[p00 + cam.W + 1];
  const double hi = fmax(fmax(d00, d10), fmax(d01, d11)), lo = fmin(fmin(d00, d10), fmin(d01, d11));
  const double top = d00 * (1 - fu) + d10 * fu;
  const double bot = d01 * (1 - fu) + d11 * fu;
  const double val = top * (1 - fv) + bot * fv;
  t.r = sqrt(r2) - val;
  t.du = (d10 - d00) * (1 - fv) + (d11 - d01) * fv;
  t.dv = bot - top;
  t.q[0] = q[0];
  t.q[1] = q[1];
  t.q[2] = q[2];
  return in && val4 && hi - lo <= spread_gate;
}

// Residual of every anchor at pose T; |r| bits for the median of ok anchors.
__global__ void k_photo_resid(const double* __restrict__ X, int M, PoseK T, RegCam cam,
                              const double* __restrict__ srange, const uint8_t* __restrict__ svalid,
                              double spread_gate, PhotoTmp* __restrict__ tmp,
                              unsigned long long* __restrict__ absbits, int* __restrict__ n_ok) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  bool ok = false;
  if (i < M) {
    PhotoTmp t{};
    ok = photo_resid_one(X, i, T, cam, srange, svalid, spread_gate, t);
    if (ok) tmp[i] = t;
    absbits[i] = ok ? (unsigned long long)__double_as_longlong(fabs(t.r)) : ~0ull;
  }
  const unsigned b = __ballot_sync(0xffffffffu, ok);
  if ((threadIdx.x & 31) == 0 && b) atomicAdd(n_ok, __popc(b));
}

// Exact k-th smallest of the ok |r| bit patterns (radix select, 11-bit
// digits, one block); the median of m values: a[m/2] or (a[m/2-1]+a[m/2])/2.
__global__ void __launch_bounds__(1024) k_photo_median(const unsigned long long* __restrict__ bits, int M,
                                                       const int* __restrict__ n_ok, double* __restrict__ median) {
  __shared__ unsigned int hist[2048];
  __shared__ unsigned long long s_prefix;
  __shared__ int s_k;
  const int m = *n_ok;
  if (m == 0) {
    if (threadIdx.x == 0) *median = 0.0;
    return;
  }
  double res[2];
  const int nsel = (m % 2 == 0) ? 2 : 1;
  for (int sel = 0; sel < nsel; ++sel) {
    const int kth = (m % 2 == 0) ? (m / 2 - 1 + sel) : m / 2;
    if (threadIdx.x == 0) {
      s_prefix = 0ull;
      s_k = kth;
    }
    unsigned long long mask = 0ull;
    for (int shift = 53; shift >= 0; shift -= 11) {  // bits 63..0 in 11-bit digits (sign bit always 0)
      for (int i = threadIdx.x; i < 2048; i += blockDim.x) hist[i] = 0u;
      __syncthreads();
      const unsigned long long pref = s_prefix;
      for (int i = threadIdx.x; i < M; i += blockDim.x) {
        const unsigned long long b = bits[i];
        if (b != ~0ull && (b & mask) == pref) atomicAdd(&hist[(b >> shift) & 2047u], 1u);
      }
      __syncthreads();
      {
        // bucket holding the k-th value: block scan of the 2048 bin counts
        const int b0 = 2 * threadIdx.x;
        const unsigned c0 = hist[b0], c1 = hist[b0 + 1];
        unsigned inc = c0 + c1;
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        for (int off = 1; off < 32; off <<= 1) {
          const unsigned y = __shfl_up_sync(0xffffffffu, inc, off);
          if (lane >= off) inc += y;
        }
        __shared__ unsigned wsum[32];
        if (lane == 31) wsum[warp] = inc;
        __syncthreads();
        unsigned wex = 0;
        for (int w = 0; w < warp; ++w) wex += wsum[w];
        const unsigned ex = wex + inc - (c0 + c1);
        const int k = s_k;
        __syncthreads();
        if ((unsigned)k >= ex && (unsigned)k < ex + c0) {
          s_k = k - (int)ex;
          s_prefix = pref | ((unsigned long long)b0 << shift);
        } else if ((unsigned)k >= ex + c0 && (unsigned)k < ex + c0 + c1) {
          s_k = k - (int)(ex + c0);
          s_prefix = pref | ((unsigned long long)(b0 + 1) << shift);
        }
      }
      mask |= 2047ull << shift;
      __syncthreads();
    }
    res[sel] = __longlong_as_double((long long)s_prefix);
    __syncthreads();
  }
  if (threadIdx.x == 0) *median = (nsel == 2) ? (res[0] + res[1]) / 2.0 : res[0];
}

// Trim, Huber-weight and reduce.  out: [0:21] sum w J^T J (upper, row-major),
// [21:27] sum w J r, [27] Huber sum, [28] kept count, [29] sum r^2.
// One kept anchor's contribution (registration.py:342-361, 219-228, 470-477):
// [0:21] w J^T J upper, [21:27] w J r, [27] Huber, [28] count, [29] r^2.
__device__ __forceinline__ void photo_accum_one(const PhotoTmp& t, const RegCam& cam, double thr, double huber,
                                                int objective_only, double (&acc)[30]) {
  const double ar = fabs(t.r);
  if (!(ar <= thr)) return;
  const double x = t.q[0], y = t.q[1], z = t.q[2];
  const double rho2 = x * x + y * y, r2 = rho2 + z * z;
  const double rho = sqrt(rho2), rq = sqrt(r2);
  const double w = ar <= huber ? 1.0 : huber / fmax(ar, 1e-12);
  acc[27] += ar <= huber ? 0.5 * t.r * t.r : huber * (ar - 0.5 * huber);
  acc[28] += 1.0;
  acc[29] += t.r * t.r;
  if (objective_only) return;
  const double dudq[3] = {cam.fx * (-y / rho2), cam.fx * (x / rho2), 0.0};
  const double dvdq[3] = {cam.fy * (-x * z / (r2 * rho)), cam.fy * (-y * z / (r2 * rho)), cam.fy * (rho / r2)};
  const double g[3] = {x / rq - t.du * dudq[0] - t.dv * dvdq[0], y / rq - t.du * dudq[1] - t.dv * dvdq[1],
                       z / rq - t.du * dudq[2] - t.dv * dvdq[2]};
  const double J[6] = {-g[0], -g[1], -g[2], g[1] * z - g[2] * y, g[2] * x - g[0] * z, g[0] * y - g[1] * x};
  int k = 0;
#pragma unroll
  for (int a = 0; a < 6; ++a)
#pragma unroll
    for (int b = a; b < 6; ++b) acc[k++] += w * J[a] * J[b];
#pragma unroll
  for (int a = 0; a < 6; ++a) acc[21 + a] += w * J[a] * t.r;
}

// As above into the registration kernel's 32-slot layout: Huber(huber) in
// slot 30 and Huber(huber_geo) in slot 27.
__device__ __forceinline__ void photo_accum_one(const PhotoTmp& t, const RegCam& cam, double thr, double huber,
                                                double huber_geo, int objective_only, double (&acc)[32]) {
  const double ar = fabs(t.r);
  if (!(ar <= thr)) return;
  const double x = t.q[0], y = t.q[1], z = t.q[2];
  const double rho2 = x * x + y * y, r2 = rho2 + z * z;
  const double rho = sqrt(rho2), rq = sqrt(r2);
  const double w = ar <= huber ? 1.0 : huber / fmax(ar, 1e-12);
  acc[30] += ar <= huber ? 0.5 * t.r * t.r : huber * (ar - 0.5 * huber);
  acc[27] += ar <= huber_geo ? 0.5 * t.r * t.r : huber_geo * (ar - 0.5 * huber_geo);
  acc[28] += 1.0;
  acc[29] += t.r * t.r;
  if (objective_only) return;
  const double dudq[3] = {cam.fx * (-y / rho2), cam.fx * (x / rho2), 0.0};
  const double dvdq[3] = {cam.fy * (-x * z / (r2 * rho)), cam.fy * (-y * z / (r2 * rho)), cam.fy * (rho / r2)};
  const double g[3] = {x / rq - t.du * dudq[0] - t.dv * dvdq[0], y / rq - t.du * dudq[1] - t.dv * dvdq[1],
                       z / rq - t.du * dudq[2] - t.dv * dvdq[2]};
  const double J[6] = {-g[0], -g[1], -g[2], g[1] * z - g[2] * y, g[2] * x - g[0] * z, g[0] * y - g[1] * x};
  int k = 0;
#pragma unroll
  for (int a = 0; a < 6; ++a)
#pragma unroll
    for (int b = a; b < 6; ++b) acc[k++] += w * J[a] * J[b];
#pragma unroll
  for (int a = 0; a < 6; ++a) acc[21 + a] += w * J[a] * t.r;
}

__global__ void __launch_bounds__(256) k_photo_accum(int M, RegCam cam, const PhotoTmp* __restrict__ tmp,
                                                     const unsigned long long* __restrict__ absbits,
                                                     const double* __restrict__ median, double trim_factor,
                                                     double trim_floor, double huber, int objective_only,
                                                     double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  double acc[30];
#pragma unroll
  for (int q = 0; q < 30; ++q) acc[q] = 0.0;
  const double thr = fmax(trim_factor * (*median), trim_floor);
  if (i < M && absbits[i] != ~0ull) photo_accum_one(tmp[i], cam, thr, huber, objective_only, acc);
  __shared__ double red[8][30];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < 30; ++q) {
    double v = acc[q];
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if (lane == 0) red[warp][q] = v;
  }
  __syncthreads();
  if (threadIdx.x < 30) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w][threadIdx.x];
    if (s != 0.0) atomicAdd(&out[threadIdx.x], s);
  }
}

}  // namespace ss
