// Keyframe preparation on the device, after the
// reference's make_keyframe (pkg/src/splatscan/mapping.py:106-114):
//   smooth_range_image    geometry.py:271-287  3x3 median of the valid
//                         ranges (invalid pixels enter as +inf), columns
//                         wrapped for full-circle cameras, rows (and
//                         unwrapped columns) clamped as ndimage's "nearest";
//                         pixels whose median is +inf keep their range
//   range_image_normals   geometry.py:290-338  central differences of the
//                         back-projected ranges, four valid neighbours
//                         (azimuth seam wrapped for full-circle cameras),
//                         unit length, oriented toward the sensor
// (build_range_image is k_range_scatter / k_range_finish in registration.cu.)
// The median is one of the nine inputs, so the smoothed image is bit-exact;
// the normals are float64 in numpy's operation order (no contraction).
#include "common.cuh"

namespace ss {

__device__ __forceinline__ void cswap(double& a, double& b) {
  const double lo = fmin(a, b), hi = fmax(a, b);
  a = lo;
  b = hi;
}

// 5th smallest of 9 (the 19-comparator median network).
__device__ __forceinline__ double median9(double* v) {
  cswap(v[1], v[2]); cswap(v[4], v[5]); cswap(v[7], v[8]);
  cswap(v[0], v[1]); cswap(v[3], v[4]); cswap(v[6], v[7]);
  cswap(v[1], v[2]); cswap(v[4], v[5]); cswap(v[7], v[8]);
  cswap(v[0], v[3]); cswap(v[5], v[8]); cswap(v[4], v[7]);
  cswap(v[3], v[6]); cswap(v[1], v[4]); cswap(v[2], v[5]);
  cswap(v[4], v[7]); cswap(v[4], v[2]); cswap(v[6], v[4]);
  cswap(v[4], v[2]);
  return v[4];
}

__global__ void k_smooth_range(int W, int H, int wrap, const double* __restrict__ range,
                               const uint8_t* __restrict__ valid, double* __restrict__ out) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= W * H) return;
  const int r = p / W, c = p % W;
  double v[9];
  int q = 0;
  for (int dr = -1; dr <= 1; ++dr) {
    const int rr = min(max(r + dr, 0), H - 1);
    for (int dc = -1; dc <= 1; ++dc) {
      int cc = c + dc;
      cc = wrap ? (cc + W) % W : min(max(cc, 0), W - 1);
      const size_t i = (size_t)rr * W + cc;
      v[q++] = valid[i] ? range[i] : __longlong_as_double(0x7ff0000000000000LL);
    }
  }
  const double sm = median9(v);
  out[p] = (valid[p] && isfinite(sm)) ? sm : range[p];
}

// pixel direction of column c / row r (SphericalCamera.pixel_directions, geometry.py:176-185)
__device__ __forceinline__ void pixel_dir(const CamK& k, int c, int r, double d[3]) {
  const double az = ((double)c + k.off_u - k.cx) / k.fx;
  const double el = ((double)r + k.off_v - k.cy) / k.fy;
  const double ce = cos(el);
  d[0] = x_mul(ce, cos(az));
  d[1] = x_mul(ce, sin(az));
  d[2] = sin(el);
}

__global__ void k_range_normals(CamK k, int wrap, const double* __restrict__ range,
                                const uint8_t* __restrict__ valid, double* __restrict__ nrm,
                                uint8_t* __restrict__ ok_out) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  const int W = k.W, H = k.H;
  if (p >= W * H) return;
  const int r = p / W, c = p % W;
  const int cl = wrap ? (c - 1 + W) % W : c - 1, cr = wrap ? (c + 1) % W : c + 1;
  bool ok = valid[p] && r > 0 && r + 1 < H && cl >= 0 && cr < W;
  ok = ok && valid[(size_t)r * W + cl] && valid[(size_t)r * W + cr] && valid[(size_t)(r - 1) * W + c] &&
       valid[(size_t)(r + 1) * W + c];
  double n[3] = {0.0, 0.0, 0.0};
  if (ok) {
    double dl[3], dr_[3], du[3], dd[3], L[3], R[3], U[3], D[3];
    pixel_dir(k, cl, r, dl);
    pixel_dir(k, cr, r, dr_);
    pixel_dir(k, c, r - 1, du);
    pixel_dir(k, c, r + 1, dd);
    const double rl = range[(size_t)r * W + cl], rr = range[(size_t)r * W + cr];
    const double ru = range[(size_t)(r - 1) * W + c], rd = range[(size_t)(r + 1) * W + c];
    for (int q = 0; q < 3; ++q) {
      L[q] = x_mul(rl, dl[q]);
      R[q] = x_mul(rr, dr_[q]);
      U[q] = x_mul(ru, du[q]);
      D[q] = x_mul(rd, dd[q]);
    }
    const double dx[3] = {x_sub(R[0], L[0]), x_sub(R[1], L[1]), x_sub(R[2], L[2])};
    const double dy[3] = {x_sub(D[0], U[0]), x_sub(D[1], U[1]), x_sub(D[2], U[2])};
    // np.cross
    n[0] = x_sub(x_mul(dx[1], dy[2]), x_mul(dx[2], dy[1]));
    n[1] = x_sub(x_mul(dx[2], dy[0]), x_mul(dx[0], dy[2]));
    n[2] = x_sub(x_mul(dx[0], dy[1]), x_mul(dx[1], dy[0]));
    const double norm = sqrt(x_add(x_add(x_mul(n[0], n[0]), x_mul(n[1], n[1])), x_mul(n[2], n[2])));
    ok = norm > 1e-12;
    if (ok) {
      for (int q = 0; q < 3; ++q) n[q] = x_div(n[q], norm);
      double d[3];
      pixel_dir(k, c, r, d);
      const double s = x_add(x_add(x_mul(n[0], d[0]), x_mul(n[1], d[1])), x_mul(n[2], d[2]));
      if (s > 0.0)
        for (int q = 0; q < 3; ++q) n[q] = -n[q];
    } else {
      n[0] = n[1] = n[2] = 0.0;
    }
  }
  nrm[3 * (size_t)p] = n[0];
  nrm[3 * (size_t)p + 1] = n[1];
  nrm[3 * (size_t)p + 2] = n[2];
  ok_out[p] = ok;
}

}  // namespace ss
