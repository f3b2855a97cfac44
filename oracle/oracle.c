/*
 * oracle.c -- CPU restatement (float64) of the Splat-LOAM reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product path.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load it.  The product path
 * (paper_2503_17491_b200/) never links, imports or calls anything here.
 *
 * It restates, in plain C with float64 arithmetic, the algorithm of the
 * reference package `splatscan` (reference tree: pkg/src/splatscan/):
 *   camera intrinsics / grid offset / pixel rays   geometry.py:95-109,160-185,60-65
 *   pixel planes (h_x, h_y, ray_ok)                 rasterizer.py:158-175
 *   splat activation + Gram-Schmidt                 splats.py:44-50,112-130,217-231
 *   camera-frame splat arrays                       rasterizer.py:223-241
 *   cone-bound tile incidence                       rasterizer.py:244-306
 *   pair expansion + (tile, range, index) order     rasterizer.py:309-339
 *   per-pair intersection + cutoffs                 rasterizer.py:363-399
 *   transmittance / blend                           rasterizer.py:402-452
 *   analytic backward + world mapping               rasterizer.py:534-701
 *   Gram-Schmidt backward                           splats.py:133-163
 *   raw-parameter chain rule                        mapping.py:479-494
 * Parity of this restatement is pinned against golden vectors produced by
 * the live reference (tests/golden/make_golden.py, tests/test_oracle_golden.py).
 *
 * Evaluation order differs from the reference's chunked numpy code (it is
 * per pixel, front to back); results agree to float64 round-off.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_PI 3.14159265358979323846

typedef struct {
  int width, height;
  double az_min, az_max, el_min, el_max;
} orc_camera;

typedef struct {
  int tile_size;
  double alpha_cutoff, alpha_clamp, min_transmittance, denom_eps, cutoff_sigma, bbox_pad_px;
} orc_raster_cfg;

/* Python-style float modulo (result has the sign of the divisor), as np.mod. */
static double py_mod(double a, double b) {
  double m = fmod(a, b);
  if (m != 0.0 && ((b < 0.0) != (m < 0.0))) m += b;
  return m;
}

typedef struct { double fx, fy, cx, cy, off_u, off_v; } cam_k;

/* geometry.py:95-109 and grid_offset geometry.py:160-174 */
static cam_k cam_intrinsics(const orc_camera* c) {
  cam_k k;
  double fov_h = c->az_max - c->az_min, fov_v = c->el_max - c->el_min;
  k.fx = -(double)(c->width - 1) / fov_h;
  k.fy = -(double)(c->height - 1) / fov_v;
  k.cx = 0.5 * c->width * (1.0 + (c->az_max + c->az_min) / fov_h);
  k.cy = 0.5 * c->height * (1.0 + (c->el_max + c->el_min) / fov_v);
  double first_u = k.fx * c->az_max + k.cx, first_v = k.fy * c->el_max + k.cy;
  k.off_u = py_mod(first_u + 0.5, 1.0) - 0.5;
  k.off_v = py_mod(first_v + 0.5, 1.0) - 0.5;
  return k;
}

void orc_camera_intrinsics(const orc_camera* c, double out6[6]) {
  cam_k k = cam_intrinsics(c);
  out6[0] = k.fx; out6[1] = k.fy; out6[2] = k.cx; out6[3] = k.cy; out6[4] = k.off_u; out6[5] = k.off_v;
}

/* Unit ray of every pixel sample plus the two origin planes
 * (geometry.py:176-185 / rasterizer.py:158-175).  dirs/hx/hy: H*W*3. */
void orc_pixel_planes(const orc_camera* c, double* dirs, double* hx, double* hy, uint8_t* ok) {
  cam_k k = cam_intrinsics(c);
  for (int i = 0; i < c->height; ++i) {
    for (int j = 0; j < c->width; ++j) {
      size_t p = (size_t)i * c->width + j;
      double u = (double)j + k.off_u, v = (double)i + k.off_v;
      double az = (u - k.cx) / k.fx, el = (v - k.cy) / k.fy;
      double ce = cos(el);
      double d0 = ce * cos(az), d1 = ce * sin(az), d2 = sin(el);
      dirs[3 * p] = d0; dirs[3 * p + 1] = d1; dirs[3 * p + 2] = d2;
      /* h_x = (d_y, -d_x, 0) / |.|, h_y = h_x x d */
      double n = sqrt(d1 * d1 + d0 * d0);
      int good = n > 1e-9;
      double s = 1.0 / (n > 1e-9 ? n : 1e-9);
      double x0 = d1 * s, x1 = -d0 * s, x2 = 0.0;
      double y0 = x1 * d2 - x2 * d1, y1 = x2 * d0 - x0 * d2, y2 = x0 * d1 - x1 * d0;
      if (!good) { x0 = x1 = x2 = y0 = y1 = y2 = 0.0; }
      hx[3 * p] = x0; hx[3 * p + 1] = x1; hx[3 * p + 2] = x2;
      hy[3 * p] = y0; hy[3 * p + 1] = y1; hy[3 * p + 2] = y2;
      ok[p] = (uint8_t)good;
    }
  }
}

static double dot3(const double* a, const double* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }

/* Per-splat camera-frame arrays (rasterizer.py:223-241 with splats.py:44-50,112-130).
 * Layout of `arr` (22 doubles per splat):
 *  0 Ba[3] 3 Bb[3] 6 Bc[3] 9 ncam[3] 12 ta_c[3] 15 tb_c[3] 18 opac 19 s_a 20 s_b 21 range
 * Returns -1 when Gram-Schmidt degenerates (splats.py:123-129), else 0. */
int orc_splat_arrays(int n, const double* centers, const double* raw_ta, const double* raw_tb,
                     const double* log_scales, const double* logit_opacity, const double* R,
                     const double* t, double* arr) {
  int bad = 0;
  for (int i = 0; i < n; ++i) {
    const double *a = raw_ta + 3 * i, *b = raw_tb + 3 * i;
    double na = sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2]);
    if (na < 1e-12) { bad = 1; continue; }
    double u[3] = {a[0] / na, a[1] / na, a[2] / na};
    double ub = u[0] * b[0] + u[1] * b[1] + u[2] * b[2];
    double w[3] = {b[0] - ub * u[0], b[1] - ub * u[1], b[2] - ub * u[2]};
    double nw = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
    if (nw < 1e-12) { bad = 1; continue; }
    double v[3] = {w[0] / nw, w[1] / nw, w[2] / nw};
    double nn[3] = {u[1] * v[2] - u[2] * v[1], u[2] * v[0] - u[0] * v[2], u[0] * v[1] - u[1] * v[0]};
    double sa = exp(log_scales[2 * i]), sb = exp(log_scales[2 * i + 1]);
    double x = logit_opacity[i], o;
    if (x >= 0) o = 1.0 / (1.0 + exp(-x));
    else { double e = exp(x); o = e / (1.0 + e); }
    double* r = arr + 22 * (size_t)i;
    double m[3] = {centers[3 * i] - t[0], centers[3 * i + 1] - t[1], centers[3 * i + 2] - t[2]};
    for (int c = 0; c < 3; ++c) {
      /* row-vector times R: x @ R  ->  sum_k x_k R[k][c] */
      /* numpy matmul (OpenBLAS dgemm) accumulates with fused multiply-adds */
      double tac = fma(u[2], R[6 + c], fma(u[1], R[3 + c], u[0] * R[c]));
      double tbc = fma(v[2], R[6 + c], fma(v[1], R[3 + c], v[0] * R[c]));
      double bc = fma(m[2], R[6 + c], fma(m[1], R[3 + c], m[0] * R[c]));
      double nc = fma(nn[2], R[6 + c], fma(nn[1], R[3 + c], nn[0] * R[c]));
      r[0 + c] = sa * tac;
      r[3 + c] = sb * tbc;
      r[6 + c] = bc;
      r[9 + c] = nc;
      r[12 + c] = tac;
      r[15 + c] = tbc;
    }
    r[18] = o; r[19] = sa; r[20] = sb;
    r[21] = sqrt(r[6] * r[6] + r[7] * r[7] + r[8] * r[8]);
  }
  return bad ? -1 : 0;
}

/* Tile incidence by cone bound (rasterizer.py:244-306).  row_hit: n*tiles_y,
 * col_hit: n*tiles_x (uint8). */
void orc_tile_hits(const orc_camera* c, const orc_raster_cfg* cfg, int n, const double* arr,
                   uint8_t* row_hit, uint8_t* col_hit) {
  cam_k k = cam_intrinsics(c);
  int T = cfg->tile_size;
  int tx = (c->width + T - 1) / T, ty = (c->height + T - 1) / T;
  double* cc = (double*)malloc(sizeof(double) * (tx + ty) * 2);
  double *chw = cc + tx, *rc = cc + 2 * tx, *rhw = rc + ty;
  for (int q = 0; q < tx; ++q) {
    int f = q * T, l = (f + T < c->width ? f + T : c->width) - 1;
    double a0 = ((double)f + k.off_u - k.cx) / k.fx, a1 = ((double)l + k.off_u - k.cx) / k.fx;
    cc[q] = 0.5 * (a0 + a1);
    chw[q] = 0.5 * fabs(a0 - a1);
  }
  for (int q = 0; q < ty; ++q) {
    int f = q * T, l = (f + T < c->height ? f + T : c->height) - 1;
    double e0 = ((double)f + k.off_v - k.cy) / k.fy, e1 = ((double)l + k.off_v - k.cy) / k.fy;
    rc[q] = 0.5 * (e0 + e1);
    rhw[q] = 0.5 * fabs(e0 - e1);
  }
  double pad_az = cfg->bbox_pad_px * (1.0 / fabs(k.fx));
  double pad_el = cfg->bbox_pad_px * (1.0 / fabs(k.fy));
#pragma omp parallel for schedule(static)
  for (int i = 0; i < n; ++i) {
    const double* r = arr + 22 * (size_t)i;
    const double* Bc = r + 6;
    double rng = r[21];
    double smax = r[19] > r[20] ? r[19] : r[20];
    if (r[19] != r[19] || r[20] != r[20]) smax = NAN;
    double reach = cfg->cutoff_sigma * smax;
    int near = rng <= reach + 1e-12;
    double so = reach / (rng > 1e-12 ? rng : 1e-12);
    so = so < 0.0 ? 0.0 : (so > 1.0 ? 1.0 : so);
    double omega = asin(so);
    double azc = atan2(Bc[1], Bc[0]);
    double elc = atan2(Bc[2], hypot(Bc[0], Bc[1]));
    int pole = fabs(elc) + omega >= ORC_PI / 2 - 1e-9;
    double ce = cos(elc);
    ce = ce > 1e-12 ? ce : 1e-12;
    double q = so / ce;
    q = q < 0.0 ? 0.0 : (q > 1.0 ? 1.0 : q);
    double dgam = asin(q);
    if (near || pole) dgam = ORC_PI;
    if (near) omega = ORC_PI;
    int alive = rng > 1e-9;
    for (int j = 0; j < tx; ++j) {
      double d = azc - cc[j];
      d = fabs(py_mod(d + ORC_PI, 2.0 * ORC_PI) - ORC_PI);
      col_hit[(size_t)i * tx + j] = (uint8_t)(alive && d <= dgam + chw[j] + pad_az);
    }
    for (int j = 0; j < ty; ++j) {
      double d = fabs(elc - rc[j]);
      row_hit[(size_t)i * ty + j] = (uint8_t)(alive && d <= omega + rhw[j] + pad_el);
    }
  }
  free(cc);
}

typedef struct { int32_t tile; int32_t idx; double key; } pair_t;

static int pair_cmp(const void* pa, const void* pb) {
  const pair_t *a = (const pair_t*)pa, *b = (const pair_t*)pb;
  if (a->tile != b->tile) return a->tile < b->tile ? -1 : 1;
  if (a->key != b->key) return a->key < b->key ? -1 : 1;
  return a->idx < b->idx ? -1 : (a->idx > b->idx);
}

/* Pair count for a binning (call before orc_bin to size pair_splats). */
int64_t orc_count_pairs(int n, int tx, int ty, const uint8_t* row_hit, const uint8_t* col_hit) {
  int64_t total = 0;
  for (int i = 0; i < n; ++i) {
    int64_t nr = 0, nc = 0;
    for (int j = 0; j < ty; ++j) nr += row_hit[(size_t)i * ty + j];
    for (int j = 0; j < tx; ++j) nc += col_hit[(size_t)i * tx + j];
    total += nr * nc;
  }
  return total;
}

/* Ordered per-tile lists: (tile id, float64 range, splat index) order
 * (rasterizer.py:318-339).  tile_ptr: tx*ty+1 int64, pair_splats: count int64. */
void orc_bin(int n, int tx, int ty, const uint8_t* row_hit, const uint8_t* col_hit,
             const double* arr, int64_t* tile_ptr, int64_t* pair_splats) {
  int64_t total = orc_count_pairs(n, tx, ty, row_hit, col_hit);
  pair_t* p = (pair_t*)malloc(sizeof(pair_t) * (total > 0 ? total : 1));
  int64_t w = 0;
  for (int i = 0; i < n; ++i) {
    for (int r = 0; r < ty; ++r) {
      if (!row_hit[(size_t)i * ty + r]) continue;
      for (int c = 0; c < tx; ++c) {
        if (!col_hit[(size_t)i * tx + c]) continue;
        p[w].tile = r * tx + c; p[w].idx = i; p[w].key = arr[22 * (size_t)i + 21];
        ++w;
      }
    }
  }
  qsort(p, (size_t)total, sizeof(pair_t), pair_cmp);
  int ntiles = tx * ty;
  for (int t = 0; t <= ntiles; ++t) tile_ptr[t] = 0;
  for (int64_t q = 0; q < total; ++q) tile_ptr[p[q].tile + 1]++;
  for (int t = 0; t < ntiles; ++t) tile_ptr[t + 1] += tile_ptr[t];
  for (int64_t q = 0; q < total; ++q) pair_splats[q] = p[q].idx;
  free(p);
}

/* Intersection quantities of one pixel/splat pair (rasterizer.py:363-399). */
typedef struct {
  double a1, a2, a4, b1, b2, b4, den, sa, sb, nu[3], d, G, alpha;
  int use, clamped;
} pair_geo;

static void pair_geometry(const double* hx, const double* hy, const double* V, int ray_ok,
                          const double* r, const orc_raster_cfg* cfg, pair_geo* g) {
  const double *Ba = r, *Bb = r + 3, *Bc = r + 6;
  g->a1 = dot3(hx, Ba); g->a2 = dot3(hx, Bb); g->a4 = dot3(hx, Bc);
  g->b1 = dot3(hy, Ba); g->b2 = dot3(hy, Bb); g->b4 = dot3(hy, Bc);
  double den = g->a1 * g->b2 - g->a2 * g->b1;
  int big = fabs(den) >= cfg->denom_eps;
  int ok = big && ray_ok;
  double safe = big ? den : 1.0;
  g->den = safe;
  g->sa = (g->a2 * g->b4 - g->a4 * g->b2) / safe;
  g->sb = (g->a4 * g->b1 - g->a1 * g->b4) / safe;
  for (int c = 0; c < 3; ++c) g->nu[c] = g->sa * Ba[c] + g->sb * Bb[c] + Bc[c];
  ok = ok && dot3(g->nu, V) > 0;
  double d = sqrt(dot3(g->nu, g->nu));
  g->G = exp(-0.5 * (g->sa * g->sa + g->sb * g->sb));
  double araw = r[18] * g->G;
  g->clamped = araw > cfg->alpha_clamp;
  double alpha = araw < cfg->alpha_clamp ? araw : cfg->alpha_clamp;
  g->use = ok && alpha >= cfg->alpha_cutoff;
  g->alpha = g->use ? alpha : 0.0;
  g->d = g->use ? d : 0.0;
}

typedef struct {
  cam_k k;
  double *dirs, *hx, *hy;
  uint8_t* ok;
} plane_tab;

static void planes_alloc(const orc_camera* c, plane_tab* pt) {
  size_t P = (size_t)c->width * c->height;
  pt->dirs = (double*)malloc(sizeof(double) * P * 9);
  pt->hx = pt->dirs + 3 * P; pt->hy = pt->hx + 3 * P;
  pt->ok = (uint8_t*)malloc(P);
  orc_pixel_planes(c, pt->dirs, pt->hx, pt->hy, pt->ok);
}
static void planes_free(plane_tab* pt) { free(pt->dirs); free(pt->ok); }

/* Forward blend of pre-binned lists (rasterizer.py:402-452).
 * Outputs D (H*W), N (H*W*3), O (H*W).  Optional counters (may be NULL):
 * stats[0] += evaluated pairs, stats[1] += pairs passing `use`, stats[2] += contributing.
 * Optional margin (H*W, may be NULL): per pixel, the smallest relative distance
 * of any discrete decision to its threshold (parity protocol):
 * |alpha_raw/cutoff - 1| over evaluated pairs, |alpha_raw/clamp - 1| and
 * |nu.v|/|nu| over pairs passing the cutoff, |T/min_T - 1| over used pairs. */
void orc_forward_lists(const orc_camera* c, const orc_raster_cfg* cfg, const double* arr,
                       const int64_t* tile_ptr, const int64_t* pair_splats, double* D, double* N,
                       double* O, int64_t* stats, double* margin) {
  plane_tab pt; planes_alloc(c, &pt);
  int T = cfg->tile_size, W = c->width, H = c->height;
  int tx = (W + T - 1) / T, ty = (H + T - 1) / T;
  size_t P = (size_t)W * H;
  memset(D, 0, sizeof(double) * P); memset(O, 0, sizeof(double) * P); memset(N, 0, sizeof(double) * 3 * P);
  int64_t s0 = 0, s1 = 0, s2 = 0;
#pragma omp parallel for schedule(dynamic, 4) reduction(+ : s0, s1, s2)
  for (int t = 0; t < tx * ty; ++t) {
    int64_t lo = tile_ptr[t], hi = tile_ptr[t + 1];
    if (lo == hi) continue;
    int r0 = (t / tx) * T, c0 = (t % tx) * T;
    for (int i = r0; i < r0 + T && i < H; ++i) {
      for (int j = c0; j < c0 + T && j < W; ++j) {
        size_t p = (size_t)i * W + j;
        double Tr = 1.0, dacc = 0, oacc = 0, nacc[3] = {0, 0, 0};
        double mg = 1e300;
        for (int64_t q = lo; q < hi; ++q) {
          const double* r = arr + 22 * (size_t)pair_splats[q];
          pair_geo g;
          pair_geometry(pt.hx + 3 * p, pt.hy + 3 * p, pt.dirs + 3 * p, pt.ok[p], r, cfg, &g);
          ++s0;
          if (margin && pt.ok[p]) {
            double araw = r[18] * g.G;
            double m1 = fabs(araw / cfg->alpha_cutoff - 1.0);
            if (m1 < mg) mg = m1;
            if (araw >= cfg->alpha_cutoff) {
              double m2 = fabs(araw / cfg->alpha_clamp - 1.0);
              double nn = sqrt(dot3(g.nu, g.nu));
              double m3 = nn > 0 ? fabs(dot3(g.nu, pt.dirs + 3 * p)) / nn : 0.0;
              if (m2 < mg) mg = m2;
              if (m3 < mg) mg = m3;
            }
            if (g.use) {
              double m4 = fabs(Tr / cfg->min_transmittance - 1.0);
              if (m4 < mg) mg = m4;
            }
          }
          if (g.use) ++s1;
          double w = (Tr >= cfg->min_transmittance) ? g.alpha * Tr : 0.0;
          if (w > 0) ++s2;
          dacc += w * g.d; oacc += w;
          for (int cc = 0; cc < 3; ++cc) nacc[cc] += w * r[9 + cc];
          Tr *= (1.0 - g.alpha);
          if (Tr < cfg->min_transmittance) break; /* all later weights vanish */
        }
        if (margin) margin[p] = mg;
        D[p] = dacc; O[p] = oacc;
        for (int cc = 0; cc < 3; ++cc) N[3 * p + cc] = nacc[cc];
      }
    }
  }
  if (stats) { stats[0] += s0; stats[1] += s1; stats[2] += s2; }
  planes_free(&pt);
}

/* Backward of a pixel-space loss (rasterizer.py:534-701).  Inputs: lists,
 * rendered images, pixel gradients gD (H*W), gN (H*W*3), gO (H*W).
 * Output: 15 doubles per splat in plain space:
 *  0 d_centers[3] 3 d_t_alpha[3] 6 d_t_beta[3] 9 d_normal[3] 12 d_scales[2] 14 d_opacity
 * max_threads bounds the private accumulator copies (13 doubles per splat each). */
void orc_backward_lists(const orc_camera* c, const orc_raster_cfg* cfg, int n, const double* arr,
                        const double* R, const int64_t* tile_ptr, const int64_t* pair_splats,
                        const double* Dt, const double* Nt, const double* Ot, const double* gD,
                        const double* gN, const double* gO, double* out, int max_threads) {
  plane_tab pt; planes_alloc(c, &pt);
  int T = cfg->tile_size, W = c->width, H = c->height;
  int tx = (W + T - 1) / T, ty = (H + T - 1) / T;
  int nthr = 1;
#ifdef _OPENMP
  nthr = omp_get_max_threads();
  if (max_threads > 0 && nthr > max_threads) nthr = max_threads;
#endif
  double* acc = (double*)calloc((size_t)nthr * n * 13, sizeof(double));
#pragma omp parallel for schedule(dynamic, 4) num_threads(nthr)
  for (int t = 0; t < tx * ty; ++t) {
    int tid = 0;
#ifdef _OPENMP
    tid = omp_get_thread_num();
#endif
    double* A = acc + (size_t)tid * n * 13;
    int64_t lo = tile_ptr[t], hi = tile_ptr[t + 1];
    if (lo == hi) continue;
    int r0 = (t / tx) * T, c0 = (t % tx) * T;
    for (int i = r0; i < r0 + T && i < H; ++i) {
      for (int j = c0; j < c0 + T && j < W; ++j) {
        size_t p = (size_t)i * W + j;
        const double *hx = pt.hx + 3 * p, *hy = pt.hy + 3 * p;
        double gd = gD[p], go = gO[p];
        const double* gn = gN + 3 * p;
        double Tr = 1.0, pre_d = 0, pre_o = 0, pre_n[3] = {0, 0, 0};
        for (int64_t q = lo; q < hi; ++q) {
          int64_t s = pair_splats[q];
          const double* r = arr + 22 * (size_t)s;
          const double *Ba = r, *Bb = r + 3, *ncam = r + 9;
          pair_geo g;
          pair_geometry(hx, hy, pt.dirs + 3 * p, pt.ok[p], r, cfg, &g);
          double Tb = Tr;
          double w = (Tb >= cfg->min_transmittance) ? g.alpha * Tb : 0.0;
          Tr *= (1.0 - g.alpha);
          if (w > 0.0) {
            double wd = w * g.d;
            pre_d += wd; pre_o += w;
            double wn[3] = {w * ncam[0], w * ncam[1], w * ncam[2]};
            for (int cc = 0; cc < 3; ++cc) pre_n[cc] += wn[cc];
            /* suffix sums = total minus inclusive prefix */
            double Bd = Dt[p] - pre_d, Bo = Ot[p] - pre_o;
            double Bn[3] = {Nt[3 * p] - pre_n[0], Nt[3 * p + 1] - pre_n[1], Nt[3 * p + 2] - pre_n[2]};
            double om = 1.0 - g.alpha;
            double dal = gd * (g.d * Tb - Bd / om) + go * (Tb - Bo / om);
            for (int cc = 0; cc < 3; ++cc) dal += gn[cc] * (ncam[cc] * Tb - Bn[cc] / om);
            int free_ = !g.clamped;
            double dd = gd * w;
            double dsafe = g.d > 0 ? g.d : 1.0;
            double nuba = dot3(g.nu, Ba), nubb = dot3(g.nu, Bb);
            double dsa = (free_ ? -dal * g.alpha * g.sa : 0.0) + dd * nuba / dsafe;
            double dsb = (free_ ? -dal * g.alpha * g.sb : 0.0) + dd * nubb / dsafe;
            double* Acc = A + (size_t)s * 13;
            if (free_) Acc[12] += dal * g.G;
            double gp1 = dsa / g.den, gp2 = dsb / g.den, gp3 = -(g.sa * dsa + g.sb * dsb) / g.den;
            double ra0 = gp2 * g.a4 - gp3 * g.a2, ra1 = gp3 * g.a1 - gp1 * g.a4, ra2 = gp1 * g.a2 - gp2 * g.a1;
            double rb0 = gp2 * g.b4 - gp3 * g.b2, rb1 = gp3 * g.b1 - gp1 * g.b4, rb2 = gp1 * g.b2 - gp2 * g.b1;
            double sc = dd / dsafe;
            for (int cc = 0; cc < 3; ++cc) {
              Acc[0 + cc] += -rb0 * hx[cc] + ra0 * hy[cc] + sc * g.sa * g.nu[cc];
              Acc[3 + cc] += -rb1 * hx[cc] + ra1 * hy[cc] + sc * g.sb * g.nu[cc];
              Acc[6 + cc] += -rb2 * hx[cc] + ra2 * hy[cc] + sc * g.nu[cc];
              Acc[9 + cc] += w * gn[cc];
            }
          }
          if (Tr < cfg->min_transmittance) break;
        }
      }
    }
  }
  /* reduce private copies, then camera frame -> world frame parameters */
  for (int th = 1; th < nthr; ++th) {
    double* A = acc + (size_t)th * n * 13;
    for (size_t q = 0; q < (size_t)n * 13; ++q) acc[q] += A[q];
  }
  for (int i = 0; i < n; ++i) {
    const double* a = acc + (size_t)i * 13;
    const double* r = arr + 22 * (size_t)i;
    double* o = out + 15 * (size_t)i;
    for (int c3 = 0; c3 < 3; ++c3) {
      /* x @ R.T -> sum_k x_k R[c3][k] (dgemm order) */
      const double* Rr = R + 3 * c3;
      double mba = fma(a[2], Rr[2], fma(a[1], Rr[1], a[0] * Rr[0]));
      double mbb = fma(a[5], Rr[2], fma(a[4], Rr[1], a[3] * Rr[0]));
      double mbc = fma(a[8], Rr[2], fma(a[7], Rr[1], a[6] * Rr[0]));
      double mn = fma(a[11], Rr[2], fma(a[10], Rr[1], a[9] * Rr[0]));
      o[0 + c3] = mbc;
      o[3 + c3] = r[19] * mba;
      o[6 + c3] = r[20] * mbb;
      o[9 + c3] = mn;
    }
    o[12] = dot3(a + 0, r + 12);
    o[13] = dot3(a + 3, r + 15);
    o[14] = a[12];
  }
  free(acc);
  planes_free(&pt);
}

/* Gram-Schmidt backward (splats.py:133-163) and the raw-space chain rule of
 * refine (mapping.py:479-494).  plain: 15 per splat (layout above);
 * d_scales_extra: n*2 extra scale-loss gradient (may be NULL).
 * raw out: 12 per splat: d_centers[3] d_raw_t_alpha[3] d_raw_t_beta[3] d_log_scales[2] d_logit */
void orc_raw_gradients(int n, const double* raw_ta, const double* raw_tb, const double* log_scales,
                       const double* logit_opacity, const double* plain, const double* d_scales_extra,
                       double* raw) {
  for (int i = 0; i < n; ++i) {
    const double *a = raw_ta + 3 * i, *b = raw_tb + 3 * i, *g = plain + 15 * (size_t)i;
    double* o = raw + 12 * (size_t)i;
    double na = sqrt(dot3(a, a));
    double u[3] = {a[0] / na, a[1] / na, a[2] / na};
    double ub = dot3(u, b);
    double w[3] = {b[0] - ub * u[0], b[1] - ub * u[1], b[2] - ub * u[2]};
    double nw = sqrt(dot3(w, w));
    double v[3] = {w[0] / nw, w[1] / nw, w[2] / nw};
    const double *gu0 = g + 3, *gv0 = g + 6, *gn = g + 9;
    double gu[3], gv[3];
    /* n = u x v: fold d(loss)/dn into the columns */
    gu[0] = gu0[0] + (v[1] * gn[2] - v[2] * gn[1]);
    gu[1] = gu0[1] + (v[2] * gn[0] - v[0] * gn[2]);
    gu[2] = gu0[2] + (v[0] * gn[1] - v[1] * gn[0]);
    gv[0] = gv0[0] + (gn[1] * u[2] - gn[2] * u[1]);
    gv[1] = gv0[1] + (gn[2] * u[0] - gn[0] * u[2]);
    gv[2] = gv0[2] + (gn[0] * u[1] - gn[1] * u[0]);
    double vg = dot3(v, gv);
    double q[3] = {(gv[0] - vg * v[0]) / nw, (gv[1] - vg * v[1]) / nw, (gv[2] - vg * v[2]) / nw};
    double qu = dot3(q, u);
    double inner[3];
    for (int c = 0; c < 3; ++c) {
      o[6 + c] = q[c] - qu * u[c];
      inner[c] = gu[c] - ub * q[c] - qu * b[c];
    }
    double ui = dot3(u, inner);
    for (int c = 0; c < 3; ++c) {
      o[3 + c] = (inner[c] - ui * u[c]) / na;
      o[c] = g[c];
    }
    double s0 = exp(log_scales[2 * i]), s1 = exp(log_scales[2 * i + 1]);
    double e0 = d_scales_extra ? d_scales_extra[2 * i] : 0.0, e1 = d_scales_extra ? d_scales_extra[2 * i + 1] : 0.0;
    o[9] = (g[12] + e0) * s0;
    o[10] = (g[13] + e1) * s1;
    double x = logit_opacity[i], op;
    if (x >= 0) op = 1.0 / (1.0 + exp(-x));
    else { double e = exp(x); op = e / (1.0 + e); }
    o[11] = g[14] * op * (1.0 - op);
  }
}

int orc_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
