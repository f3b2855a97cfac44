// K1 per-splat preprocess and K2 tile binning (duplicate + order).
//
// Reference behaviour (pkg/src/splatscan/):
//   splats.py:112-130,217-231      activation + Gram-Schmidt
//   rasterizer.py:223-241          camera-frame splat arrays
//   rasterizer.py:244-306          cone-bound tile incidence (float64, bit-exact)
//   rasterizer.py:318-339          per-tile lists ordered by (tile, f64 range, index)
//
// Design: the incidence predicate is evaluated exactly as the reference does
// (float64, no contraction) but only on the tiles near the splat's cone
// instead of the dense N x tiles matrix.  Lists are bucketed per tile with
// atomics and each tile's bucket is then sorted in shared memory by the
// 96-bit key (float64 range bits, splat index); tiles longer than the shared
// memory capacity fall back to a global-memory merge sort.
#include "common.cuh"

namespace ss {

struct Incidence {
  double azc, elc, omega, dgam;
  bool alive;
};

__device__ __forceinline__ bool col_hit(const CamK& k, const Incidence& g, int c) {
  double cc, hw;
  tile_col_interval(k, c, cc, hw);
  double d = x_sub(g.azc, cc);
  d = fabs(x_sub(py_mod(x_add(d, SS_PI), 2.0 * SS_PI), SS_PI));
  return d <= x_add(x_add(g.dgam, hw), k.pad_az);
}
__device__ __forceinline__ bool row_hit(const CamK& k, const Incidence& g, int r) {
  double rc, hw;
  tile_row_interval(k, r, rc, hw);
  double d = fabs(x_sub(g.elc, rc));
  return d <= x_add(x_add(g.omega, hw), k.pad_el);
}

// x @ R for a row vector x (numpy matmul of an (N,3) array with R).
__device__ __forceinline__ double rowmat(const double x[3], const double* R, int c) {
  return fma(x[2], R[6 + c], fma(x[1], R[3 + c], x_mul(x[0], R[c])));
}

__global__ void k_preprocess(SplatsK sp, PoseK pose, CamK cam, RasterK rk, SplatRec* __restrict__ rec,
                             SplatRec64* __restrict__ rec64, unsigned long long* __restrict__ key,
                             int4* __restrict__ rect, int* __restrict__ tile_count, int* __restrict__ status) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= sp.n) return;
  int4 empty = make_int4(0, -1, 0, 0);
  // --- Gram-Schmidt (splats.py:112-130), float64
  double a[3], b[3];
  for (int c = 0; c < 3; ++c) {
    a[c] = (double)sp.raw_ta[3 * i + c];
    b[c] = (double)sp.raw_tb[3 * i + c];
  }
  double na = sqrt(x_add(x_add(x_mul(a[0], a[0]), x_mul(a[1], a[1])), x_mul(a[2], a[2])));
  if (na < 1e-12) {
    atomicExch(status, (int)SS_ERR_DEGENERATE);
    rect[i] = empty;
    return;
  }
  double u[3] = {a[0] / na, a[1] / na, a[2] / na};
  double ub = u[0] * b[0] + u[1] * b[1] + u[2] * b[2];
  double w[3] = {b[0] - ub * u[0], b[1] - ub * u[1], b[2] - ub * u[2]};
  double nw = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
  if (nw < 1e-12) {
    atomicExch(status, (int)SS_ERR_DEGENERATE);
    rect[i] = empty;
    return;
  }
  double v[3] = {w[0] / nw, w[1] / nw, w[2] / nw};
  double nn[3] = {u[1] * v[2] - u[2] * v[1], u[2] * v[0] - u[0] * v[2], u[0] * v[1] - u[1] * v[0]};
  double s0 = exp((double)sp.log_scales[2 * i]), s1 = exp((double)sp.log_scales[2 * i + 1]);
  double x = (double)sp.logit_opacity[i], o;
  if (x >= 0) {
    o = 1.0 / (1.0 + exp(-x));
  } else {
    double e = exp(x);
    o = e / (1.0 + e);
  }
  // --- camera-frame arrays (rasterizer.py:223-241)
  double m[3] = {x_sub((double)sp.centers[3 * i], pose.t[0]), x_sub((double)sp.centers[3 * i + 1], pose.t[1]),
                 x_sub((double)sp.centers[3 * i + 2], pose.t[2])};
  double Bc[3], Ba[3], Bb[3], nc[3];
  for (int c = 0; c < 3; ++c) {
    Bc[c] = rowmat(m, pose.R, c);
    Ba[c] = s0 * rowmat(u, pose.R, c);
    Bb[c] = s1 * rowmat(v, pose.R, c);
    nc[c] = rowmat(nn, pose.R, c);
  }
  double range = sqrt(x_add(x_add(x_mul(Bc[0], Bc[0]), x_mul(Bc[1], Bc[1])), x_mul(Bc[2], Bc[2])));

  // --- render records for the blend kernels
  double kq = o / rk.alpha_cutoff;
  float Kp = kq > 1.0 ? (float)(2.0 * log(kq) * (1.0 + 1e-4) + 1e-4) : -1.0f;
  SplatRec r;
  r.r0 = make_float4((float)o, Kp, (float)nc[0], (float)nc[1]);
  r.r1 = make_float4((float)nc[2], 0.f, 0.f, 0.f);
  rec[i] = r;
  SplatRec64 r64;
  r64.v[0] = make_double2(Ba[0], Ba[1]);
  r64.v[1] = make_double2(Ba[2], Bb[0]);
  r64.v[2] = make_double2(Bb[1], Bb[2]);
  r64.v[3] = make_double2(Bc[0], Bc[1]);
  r64.v[4] = make_double2(Bc[2], range);
  rec64[i] = r64;
  key[i] = (unsigned long long)__double_as_longlong(range);

  // --- cone-bound incidence (rasterizer.py:256-305), float64 without contraction
  Incidence g;
  double reach = x_mul(rk.cutoff_sigma, fmax(s0, s1));
  bool near_ = range <= x_add(reach, 1e-12);
  double so = x_div(reach, fmax(range, 1e-12));
  so = fmin(fmax(so, 0.0), 1.0);
  double omega = asin(so);
  g.azc = atan2(Bc[1], Bc[0]);
  g.elc = atan2(Bc[2], hypot(Bc[0], Bc[1]));
  bool pole = x_add(fabs(g.elc), omega) >= (SS_PI / 2 - 1e-9);
  double ce = fmax(cos(g.elc), 1e-12);
  double q = fmin(fmax(x_div(so, ce), 0.0), 1.0);
  double dgam = asin(q);
  if (near_ || pole) dgam = SS_PI;
  if (near_) omega = SS_PI;
  g.omega = omega;
  g.dgam = dgam;
  g.alive = range > 1e-9;
  if (!g.alive) {
    rect[i] = empty;
    return;
  }
  int r_lo = -1, r_hi = -2;
  for (int rr = 0; rr < cam.ty; ++rr) {
    if (row_hit(cam, g, rr)) {
      if (r_lo < 0) r_lo = rr;
      r_hi = rr;
    }
  }
  if (r_lo < 0) {
    rect[i] = empty;
    return;
  }
  int tx = cam.tx;
  int c_start = 0, ncols = 0;
  int h = -1;
  if (dgam < 0.5 * SS_PI) {
    double uu = cam.fx * g.azc + cam.cx - cam.off_u;
    int c0 = (int)floor(uu / cam.T);
    for (int dc = 0; dc < 3 && h < 0; ++dc) {
      int c = c0 + (dc == 0 ? 0 : (dc == 1 ? -1 : 1));
      c = ((c % tx) + tx) % tx;
      if (col_hit(cam, g, c)) h = c;
    }
  }
  if (h >= 0) {
    int lo = h, cnt = 1;
    while (cnt < tx) {
      int c = (lo - 1 + tx) % tx;
      if (!col_hit(cam, g, c)) break;
      lo = c;
      ++cnt;
    }
    int hi = h;
    while (cnt < tx) {
      int c = (hi + 1) % tx;
      if (!col_hit(cam, g, c)) break;
      hi = c;
      ++cnt;
    }
    c_start = lo;
    ncols = cnt;
  } else {
    // wide cone or centre column missed (partial-FoV cameras): scan all
    // columns; the hit set is one circular run.
    int first_miss = -1, nhit = 0;
    for (int c = 0; c < tx; ++c) {
      bool hc = col_hit(cam, g, c);
      nhit += hc;
      if (!hc && first_miss < 0) first_miss = c;
    }
    if (nhit == tx) {
      c_start = 0;
      ncols = tx;
    } else if (nhit > 0) {
      int c = first_miss;
      while (!col_hit(cam, g, c)) c = (c + 1) % tx;
      c_start = c;
      ncols = nhit;
    }
  }
  if (ncols == 0) {
    rect[i] = empty;
    return;
  }
  rect[i] = make_int4(r_lo, r_hi, c_start, ncols);
  for (int rr = r_lo; rr <= r_hi; ++rr) {
    int base = rr * tx;
    for (int j = 0; j < ncols; ++j) {
      int c = c_start + j;
      if (c >= tx) c -= tx;
      atomicAdd(&tile_count[base + c], 1);
    }
  }
}

// Exclusive scans of per-tile pair counts and 32-entry chunk counts; one block.
__global__ void k_scan_tiles(int ntiles, const int* __restrict__ tile_count, int* __restrict__ tile_ptr,
                             int* __restrict__ chunk_ptr, int* __restrict__ cursor, long long* __restrict__ totals) {
  __shared__ long long s_p[1024];
  __shared__ long long s_c[1024];
  int tid = threadIdx.x, nt = blockDim.x;
  int per = (ntiles + nt - 1) / nt;
  int b = tid * per, e = min(b + per, ntiles);
  long long sp = 0, sc = 0;
  for (int t = b; t < e; ++t) {
    int c = tile_count[t];
    sp += c;
    sc += (c + 31) >> 5;
  }
  s_p[tid] = sp;
  s_c[tid] = sc;
  __syncthreads();
  for (int off = 1; off < nt; off <<= 1) {
    long long vp = tid >= off ? s_p[tid - off] : 0;
    long long vc = tid >= off ? s_c[tid - off] : 0;
    __syncthreads();
    s_p[tid] += vp;
    s_c[tid] += vc;
    __syncthreads();
  }
  long long rp = s_p[tid] - sp, rc = s_c[tid] - sc;
  for (int t = b; t < e; ++t) {
    int c = tile_count[t];
    tile_ptr[t] = (int)rp;
    cursor[t] = (int)rp;
    chunk_ptr[t] = (int)rc;
    rp += c;
    rc += (c + 31) >> 5;
  }
  if (tid == nt - 1) {
    tile_ptr[ntiles] = (int)s_p[nt - 1];
    chunk_ptr[ntiles] = (int)s_c[nt - 1];
    totals[0] = s_p[nt - 1];
    totals[1] = s_c[nt - 1];
  }
}

__global__ void k_scatter_pairs(int n, int tx, const int4* __restrict__ rect, int* __restrict__ cursor,
                                int* __restrict__ pairs) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int4 r = rect[i];
  for (int rr = r.x; rr <= r.y; ++rr) {
    int base = rr * tx;
    for (int j = 0; j < r.w; ++j) {
      int c = r.z + j;
      if (c >= tx) c -= tx;
      int pos = atomicAdd(&cursor[base + c], 1);
      pairs[pos] = i;
    }
  }
}

constexpr int kSortMax = 2048;

__device__ __forceinline__ bool key_less(unsigned long long ka, int va, unsigned long long kb, int vb) {
  return ka < kb || (ka == kb && va < vb);
}

// Per-tile bitonic sort by (float64 range bits, splat index) in shared memory.
__global__ void __launch_bounds__(256) k_sort_tiles(const int* __restrict__ tile_ptr, int* __restrict__ pairs,
                                                    const unsigned long long* __restrict__ key,
                                                    int* __restrict__ long_list, int* __restrict__ n_long) {
  __shared__ unsigned long long sk[kSortMax];
  __shared__ int sv[kSortMax];
  int t = blockIdx.x;
  int lo = tile_ptr[t], L = tile_ptr[t + 1] - lo;
  if (L <= 1) return;
  if (L > kSortMax) {
    if (threadIdx.x == 0) long_list[atomicAdd(n_long, 1)] = t;
    return;
  }
  int n = 1;
  while (n < L) n <<= 1;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    if (i < L) {
      int v = pairs[lo + i];
      sv[i] = v;
      sk[i] = key[v];
    } else {
      sv[i] = 0x7fffffff;
      sk[i] = ~0ull;
    }
  }
  __syncthreads();
  for (int k = 2; k <= n; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < (n >> 1); i += blockDim.x) {
        int a = 2 * j * (i / j) + (i % j);
        int b = a + j;
        bool up = (a & k) == 0;
        unsigned long long ka = sk[a], kb = sk[b];
        int va = sv[a], vb = sv[b];
        bool gt = key_less(kb, vb, ka, va);
        if (gt == up) {
          sk[a] = kb;
          sk[b] = ka;
          sv[a] = vb;
          sv[b] = va;
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < L; i += blockDim.x) pairs[lo + i] = sv[i];
}

__device__ int count_less(const int* run, int len, const unsigned long long* key, unsigned long long k, int v) {
  int lo = 0, hi = len;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    int w = run[mid];
    if (key_less(key[w], w, k, v))
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// Fallback for lists longer than kSortMax: bottom-up merge sort in global
// memory, one block per long tile (rare: a few very large or near splats).
__global__ void k_sort_long(const int* __restrict__ tile_ptr, int* __restrict__ pairs, int* __restrict__ tmp,
                            const unsigned long long* __restrict__ key, const int* __restrict__ long_list,
                            const int* __restrict__ n_long) {
  int nl = *n_long;
  for (int idx = blockIdx.x; idx < nl; idx += gridDim.x) {
    int t = long_list[idx];
    int lo = tile_ptr[t], L = tile_ptr[t + 1] - lo;
    int* src = pairs + lo;
    int* dst = tmp + lo;
    for (int w = 1; w < L; w <<= 1) {
      for (int i = threadIdx.x; i < L; i += blockDim.x) {
        int start = (i / (2 * w)) * (2 * w);
        int mid = min(start + w, L), end = min(start + 2 * w, L);
        int v = src[i];
        unsigned long long k = key[v];
        int pos;
        if (i < mid)
          pos = (i - start) + count_less(src + mid, end - mid, key, k, v);
        else
          pos = (i - mid) + count_less(src + start, mid - start, key, k, v);
        dst[start + pos] = v;
      }
      __syncthreads();
      int* s = src;
      src = dst;
      dst = s;
    }
    if (src != pairs + lo) {
      for (int i = threadIdx.x; i < L; i += blockDim.x) pairs[lo + i] = src[i];
    }
    __syncthreads();
  }
}

__global__ void k_widen_i32(int n, const int* __restrict__ in, long long* __restrict__ out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[i];
}

}  // namespace ss
