// K3 forward blend, K4 backward, and the per-splat gradient finalize.
//
// Reference behaviour (pkg/src/splatscan/):
//   rasterizer.py:363-399   ray/splat intersection and cutoffs
//   rasterizer.py:402-452   transmittance and front-to-back blend
//   rasterizer.py:534-701   analytic backward, world-frame mapping
//   splats.py:133-163       Gram-Schmidt backward; mapping.py:479-494 raw chain
//
// Formulation.  The reference intersects the pixel's two origin planes
// (h_x, h_y) with the splat.  With A = Bb x Bc, Bv = Bc x Ba, C = Ba x Bb the
// same intersection is, by the Binet-Cauchy identity (h_x x h_y = -v),
//     sa = (v.A)/(v.C),  sb = (v.Bv)/(v.C),  range = |nu| = det/(v.C),
// det = Bc.C, den = -(v.C).  alpha >= 1/255 is the quadratic cone
// q(v) = (v.A)^2 + (v.Bv)^2 - K (v.C)^2 <= 0 with K = 2 ln(255 o).
//
// Every tile gets an orthonormal frame (t = centre ray, e1 = azimuth, e2 =
// elevation direction) and every pixel ray is v = w t + x e1 + y e2 (exact,
// float64).  Per (tile, splat) pair the warp stages, in float64, the nine dot
// products of (t, e1, e2) with (A, Bv, C); then
//   * the cone test of a pixel is six float32 FMAs,
//       q = w^2 q_tt + 2wx q_t1 + 2wy q_t2 + x^2 q_11 + 2xy q_12 + y^2 q_22,
//     with q_tt lowered by a bound on the float32 rounding so the test never
//     rejects a hit;
//   * the exact intersection of a candidate pixel is three float64 3-term
//     dot products (grazing splats amplify direction error by 1/|v.n|), the
//     rest of the pair math is float32.
//
// Work decomposition: one warp per 8x8 tile (two pixels per lane), warps are
// persistent and take tiles longest list first.  Each warp stages its tile
// list through shared memory 32 entries at a time.  The forward records, per
// pixel, the final transmittance, the last contributing list position and a
// bitmask of contributing entries; the backward walks the list back to front
// (suffix sums accumulate: no total-minus-prefix cancellation) visiting only
// entries some pixel of the tile contributed to.  A splat's 14 accumulators
// are reduced across the warp through a shared-memory transpose before one
// warp-wide float atomic, or, when at most kDirectLanes lanes contributed,
// added by those lanes with float4 vector atomics.  (A packed variant, each
// lane walking only its own contributions with per-contribution vector
// atomics, halves the instructions but measured slower: 255 vs 230 us at
// config 1, bound by 31 M L2 reduction sectors.)
#include <cuda_pipeline.h>

#include "adam.cuh"
#include "common.cuh"

namespace ss {

constexpr int kWarpsPerBlock = 4;
#ifndef SS_FWD_MINB
#define SS_FWD_MINB 4  // 128 registers, 4 blocks per SM (A/B at config 1: 5 blocks 154 us, 4 blocks 134 us)
#endif
#ifndef SS_BWD_MINB
#define SS_BWD_MINB 4
#endif
// 32-bit words per staged entry: 12 floats (+4 spare) and 5 double2 (144 B).
// The 144-byte stride keeps the staging lanes' 16-byte stores conflict-free.
constexpr int kStride = 36;
constexpr int kBwdDynSmem = kWarpsPerBlock * 32 * 16 * 4;

struct BlendParams {
  CamK cam;
  float alpha_cutoff, alpha_clamp, min_T, denom_eps;
  // Segment-parallel backward (few tiles, long lists): the forward records every
  // pixel's running state (T, D, O, N) before each kSegChunks-chunk boundary of
  // its tile's list, and the final D, O, N, so that the backward can walk each
  // segment of a list independently (segst == nullptr: off).
  float* segst;  // [global chunk / kSegChunks][6][64]
  float* fin;    // [5][W * H]: final D, O, N0, N1, N2
  // lists of >= *seg_min entries are recorded and walked in segments (the rest are
  // whole-tile backward slots); k_tile_order sets it on the device (0: every list)
  const int* seg_min;
};

#ifndef SS_SEG_CHUNKS
#define SS_SEG_CHUNKS 4
#endif
// chunks of 32 entries per backward segment (A/B at config 2, backward us:
// halves-split tiles 240, segments of 16 chunks 189, 8 -> 135, 4 -> 121)
constexpr int kSegChunks = SS_SEG_CHUNKS;

// Backward work slots of the segment modes, built by one 1024-thread block (the end of
// k_tile_order): tiles in the forward's LPT order; a tile whose list has >= min_list
// entries contributes ceil(L / (32 kSegChunks)) slots (tile << 16) | segment, any other
// tile one whole-tile slot (tile << 16) | 0xffff.  counters[2] = slot count.
__device__ void build_seg_slots(int ntiles, const int* __restrict__ tile_ptr, const int* __restrict__ order_fwd,
                                int* __restrict__ slots, int* __restrict__ counters, int min_list) {
  __shared__ int wsum[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int per = (ntiles + 1023) / 1024, r0 = min(tid * per, ntiles), r1 = min(r0 + per, ntiles);
  constexpr int kSegEntries = 32 * kSegChunks;
  auto nslot = [&](int t) {
    const int L = max(0, tile_ptr[t + 1] - tile_ptr[t]);
    return L < min_list ? (L > 0 ? 1 : 0) : (L + kSegEntries - 1) / kSegEntries;
  };
  int cnt = 0;
  for (int r = r0; r < r1; ++r) cnt += nslot(order_fwd[r] >> 2);
  int inc = cnt;
  for (int off = 1; off < 32; off <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, inc, off);
    if (lane >= off) inc += y;
  }
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  int base = inc - cnt;
  for (int w = 0; w < warp; ++w) base += wsum[w];
  for (int r = r0; r < r1; ++r) {
    const int t = order_fwd[r] >> 2;
    const int L = max(0, tile_ptr[t + 1] - tile_ptr[t]);
    if (L > 0 && L < min_list) {
      slots[base++] = (t << 16) | 0xffff;
      continue;
    }
    const int ns = nslot(t);
    for (int q = 0; q < ns; ++q) slots[base++] = (t << 16) | q;
  }
  if (tid == 1023) counters[2] = base;  // (the last thread's run ends at the total)
}

// pixel state before chunk `chunk` of the tile whose chunks start at `cbase` (chunk % kSegChunks == 0, > 0)
__device__ __forceinline__ float* seg_state(float* segst, int cbase, int chunk) {
  return segst + (size_t)((cbase + chunk) / kSegChunks) * (6 * 64);
}

template <int TS>
struct TileShape {
  static constexpr int PPL = TS * TS / 32;  // pixels per lane
};

// Orthonormal tile frame: centre ray t, azimuth direction e1, elevation direction e2.
struct TileFrame {
  double t[3], e1[3], e2[3];
};

struct Pix {
  double w, x, y;  // v = w t + x e1 + y e2 (float64)
  float dw, xf, yf;  // w - 1, x, y (float32; |x|, |y|, |w - 1| are tile-small)
  float p[6];      // w^2, 2wx, 2wy, x^2, 2xy, y^2
  float vf[3];     // v, float32
  int row, col;
  bool inside;     // inside the image
  bool ray_ok;     // reference ray_ok (rasterizer.py:167-168)
};

__device__ __forceinline__ double dot3d(const double* a, const double* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
__device__ __forceinline__ void cross3(const double* a, const double* b, double* o) {
  o[0] = a[1] * b[2] - a[2] * b[1];
  o[1] = a[2] * b[0] - a[0] * b[2];
  o[2] = a[0] * b[1] - a[1] * b[0];
}

template <int TS>
__device__ __forceinline__ void tile_frame(const CamK& k, int tr, int tc, TileFrame& f) {
  const int r0 = tr * TS, c0 = tc * TS;
  const int rh = min(TS, k.H - r0), cw = min(TS, k.W - c0);
  const double az = ((double)c0 + 0.5 * (cw - 1) + k.off_u - k.cx) / k.fx;
  const double el = ((double)r0 + 0.5 * (rh - 1) + k.off_v - k.cy) / k.fy;
  double sa, ca, se, ce;
  sincos(az, &sa, &ca);
  sincos(el, &se, &ce);
  f.t[0] = ce * ca; f.t[1] = ce * sa; f.t[2] = se;
  f.e1[0] = -sa; f.e1[1] = ca; f.e1[2] = 0.0;
  f.e2[0] = -se * ca; f.e2[1] = -se * sa; f.e2[2] = ce;
}

template <int TS>
__device__ __forceinline__ void pixel_geo(const CamK& k, int tr, int tc, int p, const TileFrame& f, Pix& g) {
  g.row = tr * TS + p / TS;
  g.col = tc * TS + p % TS;
  g.inside = g.row < k.H && g.col < k.W;
  double v[3];
  ray_at(k, (double)g.col + k.off_u, (double)g.row + k.off_v, v);
  g.ray_ok = g.inside && sqrt(v[1] * v[1] + v[0] * v[0]) > 1e-9;
  g.w = dot3d(v, f.t);
  g.x = dot3d(v, f.e1);
  g.y = dot3d(v, f.e2);
  g.p[0] = (float)(g.w * g.w);
  g.p[1] = (float)(2.0 * g.w * g.x);
  g.p[2] = (float)(2.0 * g.w * g.y);
  g.p[3] = (float)(g.x * g.x);
  g.p[4] = (float)(2.0 * g.x * g.y);
  g.p[5] = (float)(g.y * g.y);
  for (int c = 0; c < 3; ++c) g.vf[c] = (float)v[c];
  g.dw = (float)(g.w - 1.0);
  g.xf = (float)g.x;
  g.yf = (float)g.y;
}

// Stage one list entry (lane-parallel, float64): the nine frame dot products
// and, for the forward, the cone-test coefficients.  xm, ym bound |x|, |y|
// over the tile's pixels.
// Raw per-entry record copy (7 x 16 B) brought into shared memory with
// cp.async one chunk ahead of its use.
struct RawEntry {
  float4 r0;
  double2 v[5];
};

__device__ __forceinline__ void prefetch_entry(RawEntry* dst, int sid, const SplatRec* __restrict__ rec,
                                               const SplatRec64* __restrict__ rec64) {
  __pipeline_memcpy_async(&dst->r0, &rec[sid].r0, 16);
#pragma unroll
  for (int q = 0; q < 5; ++q) __pipeline_memcpy_async(&dst->v[q], &rec64[sid].v[q], 16);
}

template <bool kCone, bool kDF = false>
__device__ __forceinline__ void stage_entry(float* dst, int sid, const RawEntry& raw, const TileFrame& f, float xm,
                                            float ym) {
  const float4 p0 = raw.r0;
  double B[10];
#pragma unroll
  for (int q = 0; q < 5; ++q) {
    const double2 x = raw.v[q];
    B[2 * q] = x.x;
    B[2 * q + 1] = x.y;
  }
  const double *Ba = B, *Bb = B + 3, *Bc = B + 6;
  double A[3], Bv[3], C[3];
  cross3(Bb, Bc, A);
  cross3(Bc, Ba, Bv);
  cross3(Ba, Bb, C);
  const double det = dot3d(Bc, C);
  const double kt[3] = {dot3d(f.t, A), dot3d(f.t, Bv), dot3d(f.t, C)};
  const double k1[3] = {dot3d(f.e1, A), dot3d(f.e1, Bv), dot3d(f.e1, C)};
  const double k2[3] = {dot3d(f.e2, A), dot3d(f.e2, Bv), dot3d(f.e2, C)};
  float4* d4 = reinterpret_cast<float4*>(dst);
  if (kCone) {
    const double K = (double)p0.y;
    const double qtt = kt[0] * kt[0] + kt[1] * kt[1] - K * kt[2] * kt[2];
    const double qt1 = kt[0] * k1[0] + kt[1] * k1[1] - K * kt[2] * k1[2];
    const double qt2 = kt[0] * k2[0] + kt[1] * k2[1] - K * kt[2] * k2[2];
    const double q11 = k1[0] * k1[0] + k1[1] * k1[1] - K * k1[2] * k1[2];
    const double q12 = k1[0] * k2[0] + k1[1] * k2[1] - K * k1[2] * k2[2];
    const double q22 = k2[0] * k2[0] + k2[1] * k2[1] - K * k2[2] * k2[2];
    // magnitude of every term the float32 evaluation sums (bounds its rounding)
    const double X = xm, Y = ym;
    const double E = fabs(qtt) + 2.0 * X * fabs(qt1) + 2.0 * Y * fabs(qt2) + X * X * fabs(q11) +
                     2.0 * X * Y * fabs(q12) + Y * Y * fabs(q22) +
                     (kt[0] * kt[0] + kt[1] * kt[1] + fabs(K) * kt[2] * kt[2]);
    d4[0] = make_float4((float)(qtt - 1e-5 * E), (float)qt1, (float)qt2, (float)q11);
    d4[1] = make_float4((float)q12, (float)q22, p0.x, (float)det);
  } else {
    d4[1] = make_float4(0.f, 0.f, p0.x, (float)det);
  }
  d4[2] = make_float4(p0.z, p0.w, (float)B[9], __int_as_float(sid));  // (B[9]: ncam.z)
  if (kDF) {
  // kt as a float pair (hi + lo); k1, k2 only ever multiply tile-small x, y
  float th[3], tl[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    th[c] = (float)kt[c];
    tl[c] = (float)(kt[c] - (double)th[c]);
  }
  d4[4] = make_float4(th[0], th[1], th[2], (float)k1[0]);
  d4[5] = make_float4((float)k1[1], (float)k1[2], (float)k2[0], (float)k2[1]);
  d4[6] = make_float4((float)k2[2], tl[0], tl[1], tl[2]);
  } else {
  double2* d2 = reinterpret_cast<double2*>(dst + 16);
  d2[0] = make_double2(kt[0], kt[1]);
  d2[1] = make_double2(kt[2], k1[0]);
  d2[2] = make_double2(k1[1], k1[2]);
  d2[3] = make_double2(k2[0], k2[1]);
  d2[4] = make_double2(k2[2], 0.0);
  }
}

struct Entry {
  double kt[3], k1[3], k2[3];  // float64 frame products
  float th[3], tl[3], f1[3], f2[3];  // float-pair form (kDF)
  float o, det, n[3];
  int sid;
};

template <bool kDF = false>
__device__ __forceinline__ void load_entry(const float* e, Entry& x) {
  const float4* e4 = reinterpret_cast<const float4*>(e);
  const float4 f1 = e4[1], f2 = e4[2];
  x.o = f1.z;
  x.det = f1.w;
  x.n[0] = f2.x;
  x.n[1] = f2.y;
  x.n[2] = f2.z;
  x.sid = __float_as_int(f2.w);
  if (kDF) {
  const float4 a = e4[4], b = e4[5], c = e4[6];
  x.th[0] = a.x; x.th[1] = a.y; x.th[2] = a.z; x.f1[0] = a.w;
  x.f1[1] = b.x; x.f1[2] = b.y; x.f2[0] = b.z; x.f2[1] = b.w;
  x.f2[2] = c.x; x.tl[0] = c.y; x.tl[1] = c.z; x.tl[2] = c.w;
  } else {
  const double2* d2 = reinterpret_cast<const double2*>(e + 16);
  const double2 a = d2[0], b = d2[1], c = d2[2], d = d2[3], g = d2[4];
  x.kt[0] = a.x; x.kt[1] = a.y; x.kt[2] = b.x;
  x.k1[0] = b.y; x.k1[1] = c.x; x.k1[2] = c.y;
  x.k2[0] = d.x; x.k2[1] = d.y; x.k2[2] = g.x;
  }
}

// Flush-to-zero approximate reciprocal / exp2 (one MUFU each; the IEEE
// wrappers around MUFU.RCP / MUFU.EX2 cost four extra instructions per call
// for subnormal operands that never pass the cutoffs).
__device__ __forceinline__ float rcp_ftz(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float ex2_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Packed float32 pairs (FMUL2 / FFMA2, sm_100): the cone test of a lane's two
// pixels against one entry in 6 instructions instead of 12; a scalar operand
// packed as {c, c} folds into the instruction's broadcast operand.
__device__ __forceinline__ unsigned long long pack2(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ unsigned long long mul2(float a, unsigned long long b) {
  unsigned long long d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pack2(a, a)), "l"(b));
  return d;
}
__device__ __forceinline__ unsigned long long fma2(float a, unsigned long long b, unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(pack2(a, a)), "l"(b), "l"(c));
  return d;
}
// q = c . p for pixels (lo, hi) of the pair P[6] = {(p_k lo, p_k hi)}, in the order
// of the scalar expression c0 p0 + c1 p1 + ... (one rounding chain per pixel)
__device__ __forceinline__ unsigned long long cone2(const float4& c0, const float4& c1,
                                                   const unsigned long long (&P)[6]) {
  unsigned long long q = mul2(c0.x, P[0]);
  q = fma2(c0.y, P[1], q);
  q = fma2(c0.z, P[2], q);
  q = fma2(c0.w, P[3], q);
  q = fma2(c1.x, P[4], q);
  return fma2(c1.y, P[5], q);
}

struct Hit {
  float sa, sb, lam, r, G, alpha;
  bool use, clamped;
};

// Exact per-pixel intersection + cutoffs (rasterizer.py:369-388).
template <bool kDF = false>
__device__ __forceinline__ void intersect(const Entry& x, const Pix& p, const BlendParams& bp, Hit& h) {
  float w0, w1, w2;
  if (kDF) {
    // v.K = kt + [kt (w - 1) + k1 x + k2 y] in float32 with kt as an exact
    // hi + lo pair: the bracket's rounding is ~1e-8 |k| (x, y are tile-small),
    // amplified by 1/|v.n| for grazing splats -- ~1e-4 in sa at worst, inside
    // the backward's 1e-3 gate but not the forward's 1e-4 one.
    w0 = x.th[0] + (fmaf(x.f2[0], p.yf, fmaf(x.f1[0], p.xf, x.th[0] * p.dw)) + x.tl[0]);
    w1 = x.th[1] + (fmaf(x.f2[1], p.yf, fmaf(x.f1[1], p.xf, x.th[1] * p.dw)) + x.tl[1]);
    w2 = x.th[2] + (fmaf(x.f2[2], p.yf, fmaf(x.f1[2], p.xf, x.th[2] * p.dw)) + x.tl[2]);
  } else {
    w0 = (float)(p.w * x.kt[0] + p.x * x.k1[0] + p.y * x.k2[0]);
    w1 = (float)(p.w * x.kt[1] + p.x * x.k1[1] + p.y * x.k2[1]);
    w2 = (float)(p.w * x.kt[2] + p.x * x.k1[2] + p.y * x.k2[2]);
  }
  bool ok = p.ray_ok && fabsf(w2) >= bp.denom_eps;
  const float r = rcp_ftz(w2);
  h.r = r;
  h.sa = w0 * r;
  h.sb = w1 * r;
  h.lam = x.det * r;
  ok = ok && h.lam > 0.f;  // nu . v > 0
  const float s2 = h.sa * h.sa + h.sb * h.sb;
  h.G = ex2_ftz(s2 * -0.72134752044448170f);  // exp(-s2 / 2)
  const float araw = x.o * h.G;
  h.clamped = araw > bp.alpha_clamp;
  const float a = fminf(araw, bp.alpha_clamp);
  h.use = ok && a >= bp.alpha_cutoff;
  h.alpha = a;
}

// Reduce-scatter of 16 per-lane values through a 32x16 shared-memory
// transpose (2 KB per warp): lane l stores its row (4 x STS.128, slot
// swizzled by (l >> 1) & 3 so every quarter-warp store is conflict free),
// then sums column l & 15 over the 16 rows of its half-warp (rows of the two
// halves alternate parity, so each LDS is conflict free) and one shuffle
// adds the other half.  Afterwards lanes l and l + 16 hold the warp sum of
// value l & 15.  ~40 instructions against ~62 for the shuffle butterfly.
__device__ __forceinline__ void red_offsets(int lane, int (&o)[8]) {
  const int h = lane >> 4, c = lane & 15;
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    const int col = 4 * ((c >> 2) ^ x) + (c & 3);
    o[x] = 256 * h + 16 * h + col;      // even k: row 16h + k + h
    o[4 + x] = 256 * h - 16 * h + col;  // odd k:  row 16h + k - h
  }
}

__device__ __forceinline__ float red_transpose16(const float (&a)[16], float* red, const int (&o)[8], int lane) {
  float4* row = reinterpret_cast<float4*>(red + lane * 16);
  const int sw = (lane >> 1) & 3;
#pragma unroll
  for (int q = 0; q < 4; ++q) row[q ^ sw] = make_float4(a[4 * q], a[4 * q + 1], a[4 * q + 2], a[4 * q + 3]);
  __syncwarp();
  float v[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) v[k] = red[o[(k & 1) * 4 + ((k >> 1) & 3)] + 16 * k];
  __syncwarp();
#pragma unroll
  for (int s = 8; s >= 1; s >>= 1)
#pragma unroll
    for (int k = 0; k < s; ++k) v[k] += v[k + s];
  return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 16);
}

// Warp-uniform tile ticket (persistent warps, longest lists first).
// Work slots: (tile << 2) | part, part 0 = the whole tile, 1 / 2 = only the
// pixels of j = 0 / 1 (rows 0-3 / 4-7 of an 8x8 tile).  k_tile_order splits
// the longest tiles in two when there are fewer tiles than resident warps, so
// a few very long lists do not leave one warp per tile finishing alone.
__device__ __forceinline__ int next_tile(int* counter, const int* order, const int* nslots, int lane) {
  int ti = 0;
  if (lane == 0) ti = atomicAdd(counter, 1);
  ti = __shfl_sync(0xffffffffu, ti, 0);
  return ti < *nslots ? order[ti] : -1;
}

template <int TS, bool kSplit>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, TS == 8 ? SS_FWD_MINB : 1)
    k_forward(BlendParams bp, int ntiles, const int* __restrict__ tile_ptr, const int* __restrict__ chunk_ptr,
              const int* __restrict__ pairs, const SplatRec* __restrict__ rec, const SplatRec64* __restrict__ rec64,
              float* __restrict__ out_D, float* __restrict__ out_N, float* __restrict__ out_O,
              float* __restrict__ out_T, int* __restrict__ out_last, unsigned* __restrict__ bitmask,
              const int* __restrict__ overflow, const int* __restrict__ order, int* __restrict__ counter,
              const int* __restrict__ nslots) {
  pdl_wait();
  constexpr int PPL = TileShape<TS>::PPL;
  if (*overflow) return;  // pair capacity exceeded: the host re-runs the render
  __shared__ __align__(16) float stage[kWarpsPerBlock][32 * kStride];
  __shared__ __align__(16) RawEntry raw_all[kWarpsPerBlock][2][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const CamK& k = bp.cam;
  float* st = stage[warp];
  for (int code = next_tile(counter, order, nslots, lane); code >= 0; code = next_tile(counter, order, nslots, lane)) {
    const int t = code >> 2, part = kSplit ? (code & 3) : 0;
    const int tr = t / k.tx, tc = t % k.tx;
    TileFrame f;
    tile_frame<TS>(k, tr, tc, f);
    Pix px[PPL];
    float T[PPL], D[PPL], O[PPL], N[PPL][3];
    int last[PPL];
    bool live[PPL], use[PPL];
    float xm = 0.f, ym = 0.f;
#pragma unroll
    for (int j = 0; j < PPL; ++j) {
      pixel_geo<TS>(k, tr, tc, lane + 32 * j, f, px[j]);
      use[j] = part == 0 || part == j + 1;  // (warp-uniform)
      T[j] = 1.f; D[j] = 0.f; O[j] = 0.f; N[j][0] = N[j][1] = N[j][2] = 0.f;
      last[j] = 0;
      live[j] = px[j].ray_ok && use[j];
      if (px[j].ray_ok) {
        xm = fmaxf(xm, fabsf((float)px[j].x));
        ym = fmaxf(ym, fabsf((float)px[j].y));
      }
    }
    for (int off = 16; off > 0; off >>= 1) {
      xm = fmaxf(xm, __shfl_xor_sync(0xffffffffu, xm, off));
      ym = fmaxf(ym, __shfl_xor_sync(0xffffffffu, ym, off));
    }
    xm *= 1.0001f;
    ym *= 1.0001f;
    static_assert(PPL % 2 == 0 && !kSplit, "pixel pairs; the forward is never split");
    unsigned long long PP[PPL / 2][6];
#pragma unroll
    for (int h = 0; h < PPL / 2; ++h)
#pragma unroll
      for (int q = 0; q < 6; ++q) PP[h][q] = pack2(px[2 * h].p[q], px[2 * h + 1].p[q]);
    const int lo = tile_ptr[t], L = tile_ptr[t + 1] - lo;
    const int cbase = chunk_ptr[t];
    const bool rec_seg = bp.segst && L >= *bp.seg_min;  // (segment backward for this tile)
    // records of chunk c+1 are copied (cp.async) while chunk c is processed
    int sid_cur = lane < L ? pairs[lo + lane] : -1;
    if (sid_cur >= 0) prefetch_entry(&raw_all[warp][0][lane], sid_cur, rec, rec64);
    __pipeline_commit();
    int sid_next = 32 + lane < L ? pairs[lo + 32 + lane] : -1;
    for (int base = 0, chunk = 0; base < L; base += 32, ++chunk) {
      bool any_live = false;
#pragma unroll
      for (int j = 0; j < PPL; ++j) any_live |= live[j];
      if (!__any_sync(0xffffffffu, any_live)) break;
      if (TS == 8 && rec_seg && chunk > 0 && chunk % kSegChunks == 0) {
        float* sg = seg_state(bp.segst, cbase, chunk);
#pragma unroll
        for (int j = 0; j < PPL; ++j) {
          const int q = lane + 32 * j;
          sg[q] = T[j];
          sg[64 + q] = D[j];
          sg[128 + q] = O[j];
          sg[192 + q] = N[j][0];
          sg[256 + q] = N[j][1];
          sg[320 + q] = N[j][2];
        }
      }
      if (sid_next >= 0) prefetch_entry(&raw_all[warp][(chunk + 1) & 1][lane], sid_next, rec, rec64);
      __pipeline_commit();
      const int sid_after = base + 64 + lane < L ? pairs[lo + base + 64 + lane] : -1;
      __pipeline_wait_prior(1);  // this lane's copy for chunk c has landed
      if (sid_cur >= 0) stage_entry<true>(st + lane * kStride, sid_cur, raw_all[warp][chunk & 1][lane], f, xm, ym);
      __syncwarp();
      sid_cur = sid_next;
      sid_next = sid_after;
      const int cnt = min(32, L - base);
      unsigned word[PPL], cw[PPL];
#pragma unroll
      for (int j = 0; j < PPL; ++j) word[j] = cw[j] = 0u;
      // phase A: branch-free cone test of every (pixel, entry) -> candidate bits,
      // two pixels per packed FFMA2 chain
      for (int i = 0; i < cnt; ++i) {
        const float* e = st + i * kStride;
        const float4 c0 = *reinterpret_cast<const float4*>(e);
        const float4 c1 = *reinterpret_cast<const float4*>(e + 4);
#pragma unroll
        for (int h = 0; h < PPL / 2; ++h) {
          const unsigned long long q = cone2(c0, c1, PP[h]);
          // sign bit of q (q < 0 or -0; q = +0 only on the cone's safety margin):
          // entry i lands at bit cnt-1-i, reversed below
#ifdef SS_NO_FUNNEL
          cw[2 * h] = (cw[2 * h] << 1) | ((unsigned)q >> 31);
          cw[2 * h + 1] = (cw[2 * h + 1] << 1) | ((unsigned)(q >> 32) >> 31);
#else
          // (cw << 1) | sign bit: one SHF.L.W per pixel
          cw[2 * h] = __funnelshift_l((unsigned)q, cw[2 * h], 1);
          cw[2 * h + 1] = __funnelshift_l((unsigned)(q >> 32), cw[2 * h + 1], 1);
#endif
        }
      }
#pragma unroll
      for (int j = 0; j < PPL; ++j) cw[j] = __brev(cw[j]) >> (32 - cnt);
      // phase B: every lane walks its own candidates front to back (packed: no
      // lane idles on another pixel's candidate entry).  Measured and dropped:
      // walking both pixels' candidates in one loop (two independent chains per
      // iteration) 147 us against 135; listing the chunk's candidates of all lanes
      // and running the exact intersections 32 at a time whoever owns them, then
      // compositing per lane from shared memory, 218 us (the divergent list
      // building and compositing loops cost more than the idle lanes did).
#pragma unroll
      for (int j = 0; j < PPL; ++j) {
        unsigned m = live[j] ? cw[j] : 0u;
        while (m) {
          const int i = __ffs(m) - 1;
          m &= m - 1;
          Entry x;
          load_entry(st + i * kStride, x);
          Hit h;
          intersect(x, px[j], bp, h);
          if (!h.use) continue;
          const float w = h.alpha * T[j];
          D[j] += w * h.lam;
          O[j] += w;
          N[j][0] += w * x.n[0];
          N[j][1] += w * x.n[1];
          N[j][2] += w * x.n[2];
          T[j] *= (1.f - h.alpha);
          word[j] |= 1u << i;
          last[j] = base + i + 1;
          if (T[j] < bp.min_T) {
            live[j] = false;
            m = 0u;
          }
        }
      }
#pragma unroll
      for (int j = 0; j < PPL; ++j)
        if (use[j]) bitmask[(size_t)(cbase + chunk) * (TS * TS) + lane + 32 * j] = word[j];
      __syncwarp();
    }
    __pipeline_wait_prior(0);
    __syncwarp();
#pragma unroll
    for (int j = 0; j < PPL; ++j) {
      if (!px[j].inside || !use[j]) continue;
      const size_t p = (size_t)px[j].row * k.W + px[j].col;
      out_D[p] = D[j];
      out_O[p] = O[j];
      out_N[3 * p] = N[j][0];
      out_N[3 * p + 1] = N[j][1];
      out_N[3 * p + 2] = N[j][2];
      out_T[p] = T[j];
      out_last[p] = last[j];
      if (rec_seg) {
        const size_t P = (size_t)k.W * k.H;
        bp.fin[p] = D[j];
        bp.fin[P + p] = O[j];
        bp.fin[2 * P + p] = N[j][0];
        bp.fin[3 * P + p] = N[j][1];
        bp.fin[4 * P + p] = N[j][2];
      }
    }
  }
}

// Long lists, forward (config 2: fewer tiles than resident warps, lists of
// thousands): one 128-thread block per tile instead of one warp.  Per round of
// 128 entries all four warps run the cone test of one 32-entry chunk each;
// then warps 0-1 composite (one pixel per lane, front to back over the four
// chunks) while warps 2-3 stage the next round's entries -- the sequential
// compositing of a tile overlaps the float64 staging of its next entries
// instead of alternating with it in one warp.
constexpr int kLongRound = 128;
// With fewer tiles than resident warps every tile of >= SS_LONG_MIN entries goes to
// k_forward_long (config 2: 193 -> 148 us against the 148 longest only).
#ifndef SS_LONG_TARGET
#define SS_LONG_TARGET ntiles  // tiles handed to k_forward_long (at most)
#endif
#ifndef SS_LONG_BPS
#define SS_LONG_BPS 6  // k_forward_long blocks per SM (persistent, tickets; 37 KB shared each)
#endif


__global__ void __launch_bounds__(128) k_forward_long(
    BlendParams bp, const int* __restrict__ tile_ptr, const int* __restrict__ chunk_ptr,
    const int* __restrict__ pairs, const SplatRec* __restrict__ rec, const SplatRec64* __restrict__ rec64,
    float* __restrict__ out_D, float* __restrict__ out_N, float* __restrict__ out_O, float* __restrict__ out_T,
    int* __restrict__ out_last, unsigned* __restrict__ bitmask, const int* __restrict__ overflow,
    const int* __restrict__ order, int* __restrict__ counter, const int* __restrict__ nlong) {
  constexpr int TS = 8;
  if (*overflow) return;
  extern __shared__ __align__(16) float lsm[];  // 2 x kLongRound x kStride staged entries
  __shared__ unsigned cwbuf[4][64];
  __shared__ int s_tile;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const CamK& k = bp.cam;
  for (;;) {
    __syncthreads();
    if (tid == 0) {
      const int ti = atomicAdd(counter, 1);
      s_tile = ti < *nlong ? (order[ti] >> 2) : -1;
    }
    __syncthreads();
    const int t = s_tile;
    if (t < 0) break;
    const int tr = t / k.tx, tc = t % k.tx;
    TileFrame f;
    tile_frame<TS>(k, tr, tc, f);
    // every warp: geometry of all 64 pixels (two per lane) for its cone tests
    Pix px[2];
    float xm = 0.f, ym = 0.f;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      pixel_geo<TS>(k, tr, tc, lane + 32 * j, f, px[j]);
      if (px[j].ray_ok) {
        xm = fmaxf(xm, fabsf((float)px[j].x));
        ym = fmaxf(ym, fabsf((float)px[j].y));
      }
    }
    for (int off = 16; off > 0; off >>= 1) {
      xm = fmaxf(xm, __shfl_xor_sync(0xffffffffu, xm, off));
      ym = fmaxf(ym, __shfl_xor_sync(0xffffffffu, ym, off));
    }
    xm *= 1.0001f;
    ym *= 1.0001f;
    unsigned long long PP[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) PP[q] = pack2(px[0].p[q], px[1].p[q]);
    // compositing threads (warps 0-1): pixel tid
    const bool comp = warp < 2;
    const Pix pc = warp == 0 ? px[0] : px[1];  // (warps 0-1: pixel lane + 32 * warp == tid)
    float T = 1.f, D = 0.f, O = 0.f, N0 = 0.f, N1 = 0.f, N2 = 0.f;
    int last = 0;
    bool live = comp && pc.ray_ok;
    const int lo = tile_ptr[t], L = tile_ptr[t + 1] - lo;
    const int cbase = chunk_ptr[t];
    const bool rec_seg = bp.segst && L >= *bp.seg_min;
    auto stage_range = [&](int round, int buf, int e0, int stride) {
      for (int e = e0; e < kLongRound; e += stride) {
        const int idx = round * kLongRound + e;
        if (idx >= L) break;
        const int sid = pairs[lo + idx];
        RawEntry raw;
        raw.r0 = rec[sid].r0;
#pragma unroll
        for (int q = 0; q < 5; ++q) raw.v[q] = rec64[sid].v[q];
        stage_entry<true>(lsm + ((size_t)buf * kLongRound + e) * kStride, sid, raw, f, xm, ym);
      }
    };
    stage_range(0, 0, tid, 128);
    __syncthreads();
    for (int round = 0; round * kLongRound < L; ++round) {
      const int buf = round & 1;
      const float* stg = lsm + (size_t)buf * kLongRound * kStride;

      // cone test: warp w, chunk w of the round, all 64 pixels
      {
        const int cnt = min(32, L - round * kLongRound - 32 * warp);
        unsigned cw0 = 0u, cw1 = 0u;
        for (int i = 0; i < cnt; ++i) {
          const float* e = stg + (32 * warp + i) * kStride;
          const float4 c0 = *reinterpret_cast<const float4*>(e);
          const float4 c1 = *reinterpret_cast<const float4*>(e + 4);
          const unsigned long long q = cone2(c0, c1, PP);
          cw0 = __funnelshift_l((unsigned)q, cw0, 1);
          cw1 = __funnelshift_l((unsigned)(q >> 32), cw1, 1);
        }
        if (cnt > 0) {
          cw0 = __brev(cw0) >> (32 - cnt);
          cw1 = __brev(cw1) >> (32 - cnt);
        }
        cwbuf[warp][lane] = cnt > 0 ? cw0 : 0u;
        cwbuf[warp][lane + 32] = cnt > 0 ? cw1 : 0u;
      }
      __syncthreads();
      if (comp) {
        for (int w = 0; w < 4; ++w) {
          const int base = round * kLongRound + 32 * w;
          if (base >= L) break;
          const int gch = round * 4 + w;
          if (rec_seg && gch > 0 && gch % kSegChunks == 0) {  // state before this segment boundary
            float* sg = seg_state(bp.segst, cbase, gch);
            sg[tid] = T;
            sg[64 + tid] = D;
            sg[128 + tid] = O;
            sg[192 + tid] = N0;
            sg[256 + tid] = N1;
            sg[320 + tid] = N2;
          }
          unsigned m = live ? cwbuf[w][tid] : 0u;
          unsigned word = 0u;
          while (m) {
            const int i = __ffs(m) - 1;
            m &= m - 1;
            Entry x;
            load_entry(stg + (32 * w + i) * kStride, x);
            Hit h;
            intersect(x, pc, bp, h);
            if (!h.use) continue;
            const float wgt = h.alpha * T;
            D += wgt * h.lam;
            O += wgt;
            N0 += wgt * x.n[0];
            N1 += wgt * x.n[1];
            N2 += wgt * x.n[2];
            T *= (1.f - h.alpha);
            word |= 1u << i;
            last = base + i + 1;
            if (T < bp.min_T) {
              live = false;
              m = 0u;
            }
          }
          bitmask[(size_t)(cbase + round * 4 + w) * (TS * TS) + tid] = word;
        }
      } else if ((round + 1) * kLongRound < L) {
        stage_range(round + 1, buf ^ 1, tid - 64, 64);  // the next round, under the compositing
      }
      if (!__syncthreads_or(live)) break;
    }
    if (comp && pc.inside) {
      const size_t p = (size_t)pc.row * k.W + pc.col;
      out_D[p] = D;
      out_O[p] = O;
      out_N[3 * p] = N0;
      out_N[3 * p + 1] = N1;
      out_N[3 * p + 2] = N2;
      out_T[p] = T;
      out_last[p] = last;
      if (rec_seg) {
        const size_t P = (size_t)k.W * k.H;
        bp.fin[p] = D;
        bp.fin[P + p] = O;
        bp.fin[2 * P + p] = N0;
        bp.fin[3 * P + p] = N1;
        bp.fin[4 * P + p] = N2;
      }
    }
  }
}
constexpr int kLongSmem = 2 * kLongRound * kStride * 4;

constexpr int kAcc = 16;  // floats per splat accumulator (14 used)
// Entries that at most this many lanes contributed to skip the warp
// transpose: those lanes add their 14 values with vector atomics (A/B at
// config 1: 1 -> 252 us, 4 -> 237, 8..16 -> 230, 32 (always) -> 246; with
// grouping: 8 -> 177, 12..20 -> 172, 32 -> 219).
#ifndef SS_BWD_DIRECT
#define SS_BWD_DIRECT 16
#endif
constexpr int kDirectLanes = SS_BWD_DIRECT;
#ifdef SS_BWD_F64
constexpr bool kBwdDF = false;
#else
constexpr bool kBwdDF = true;  // float-pair intersection in the backward (230 -> 209 us)
#endif

// kSeg: work slots are (tile << 16) | segment; a slot walks chunks
// [kSegChunks * segment, kSegChunks * (segment + 1)) back to front, starting
// from the state the forward recorded before the segment's end (T) and the
// suffix sums behind it (final - recorded D, O, N -> Q).
template <int TS, bool kSplit, bool kSeg>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, TS == 8 ? SS_BWD_MINB : 1)
    k_backward(BlendParams bp, int ntiles, const int* __restrict__ tile_ptr, const int* __restrict__ chunk_ptr,
               const int* __restrict__ pairs, const SplatRec* __restrict__ rec, const SplatRec64* __restrict__ rec64,
               const float* __restrict__ in_T, const int* __restrict__ in_last, const unsigned* __restrict__ bitmask,
               const float* __restrict__ gD_img, const float* __restrict__ gN_img, const float* __restrict__ gO_img,
               float* __restrict__ acc, const int* __restrict__ overflow, const int* __restrict__ order,
               int* __restrict__ counter, const int* __restrict__ nslots, float* __restrict__ pacc) {
  pdl_wait();
  constexpr int PPL = TileShape<TS>::PPL;
  if (*overflow) return;
  // deterministic mode (pacc != null): every entry is reduced by the fixed-order
  // transpose and stored at its list position; k_det_gather sums them per splat
  const bool det = pacc != nullptr;
  __shared__ __align__(16) float stage[kWarpsPerBlock][32 * kStride];
  __shared__ __align__(16) RawEntry raw_all[kWarpsPerBlock][2][32];
  extern __shared__ __align__(16) float4 bwd_dyn_smem[];  // kBwdDynSmem: the reduce-scatter transposes
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const CamK& k = bp.cam;
  float* st = stage[warp];
  float* red = reinterpret_cast<float*>(bwd_dyn_smem) + warp * 512;
  int roff[8];
  red_offsets(lane, roff);
  for (int code = next_tile(counter, order, nslots, lane); code >= 0; code = next_tile(counter, order, nslots, lane)) {
    const int t = kSeg ? (code >> 16) : (code >> 2), part = kSplit ? (code & 3) : 0;
    const int seg = kSeg ? (code & 0xffff) : 0;
    const int tr = t / k.tx, tc = t % k.tx;
    TileFrame f;
    tile_frame<TS>(k, tr, tc, f);
    Pix px[PPL];
    float T[PPL], Q[PPL], gD[PPL], gO[PPL], gN[PPL][3];
    int last[PPL];
    int maxlast = 0;
#pragma unroll
    for (int j = 0; j < PPL; ++j) {
      pixel_geo<TS>(k, tr, tc, lane + 32 * j, f, px[j]);
      last[j] = 0;
      T[j] = 1.f;
      gD[j] = gO[j] = gN[j][0] = gN[j][1] = gN[j][2] = 0.f;
      if (px[j].inside && (part == 0 || part == j + 1)) {
        const size_t p = (size_t)px[j].row * k.W + px[j].col;
        last[j] = in_last[p];
        T[j] = in_T[p];
        gD[j] = gD_img[p];
        gO[j] = gO_img[p];
        gN[j][0] = gN_img[3 * p];
        gN[j][1] = gN_img[3 * p + 1];
        gN[j][2] = gN_img[3 * p + 2];
      }
      Q[j] = 0.f;
      maxlast = max(maxlast, last[j]);
    }
    maxlast = __reduce_max_sync(0xffffffffu, maxlast);
    if (maxlast == 0) continue;
    const int lo = tile_ptr[t];
    const int cbase = chunk_ptr[t];
    int c_lo = 0, top = (maxlast - 1) >> 5;
    if (kSeg && seg != 0xffff) {  // (0xffff: a whole-tile slot, walked from the end like kSeg = false)
      c_lo = seg * kSegChunks;
      if (c_lo > top) continue;  // no pixel reaches this segment (warp-uniform)
      const int c_hi = c_lo + kSegChunks;
      if (c_hi <= top) {  // later segments contribute: start from the recorded state
        const float* sg = seg_state(bp.segst, cbase, c_hi);
        const size_t P = (size_t)k.W * k.H;
#pragma unroll
        for (int j = 0; j < PPL; ++j) {
          if (last[j] == 0) continue;  // (inside, contributing pixels only)
          const int q = lane + 32 * j;
          const size_t p = (size_t)px[j].row * k.W + px[j].col;
          T[j] = sg[q];
          Q[j] = gD[j] * (bp.fin[p] - sg[64 + q]) + gO[j] * (bp.fin[P + p] - sg[128 + q]) +
                 gN[j][0] * (bp.fin[2 * P + p] - sg[192 + q]) + gN[j][1] * (bp.fin[3 * P + p] - sg[256 + q]) +
                 gN[j][2] * (bp.fin[4 * P + p] - sg[320 + q]);
        }
        top = c_hi - 1;
      }
    }
    // Software pipeline over chunks (back to front): the contribution words
    // and splat ids of chunk c-2 are loaded and the active records of chunk
    // c-1 are copied (cp.async) while chunk c is processed.
    auto load_words = [&](int c, unsigned (&wd)[PPL], int& sid) {
#pragma unroll
      for (int j = 0; j < PPL; ++j)
        wd[j] = (c >= c_lo && (part == 0 || part == j + 1))
                    ? bitmask[(size_t)(cbase + c) * (TS * TS) + lane + 32 * j]
                    : 0u;
      sid = (c >= c_lo && c * 32 + lane < tile_ptr[t + 1] - lo) ? pairs[lo + c * 32 + lane] : -1;
    };
    auto or_words = [&](const unsigned (&wd)[PPL]) {
      unsigned m = 0u;
#pragma unroll
      for (int j = 0; j < PPL; ++j) m |= wd[j];
      return __reduce_or_sync(0xffffffffu, m);
    };
    unsigned wcur[PPL], wnext[PPL], wnn[PPL];
    int scur, snext, snn;
    load_words(top, wcur, scur);
    unsigned any_cur = or_words(wcur);
    if (((any_cur >> lane) & 1u) && scur >= 0) prefetch_entry(&raw_all[warp][top & 1][lane], scur, rec, rec64);
    __pipeline_commit();
    load_words(top - 1, wnext, snext);
    for (int chunk = top; chunk >= c_lo; --chunk) {
      const int base = chunk * 32;
      const unsigned any_next = or_words(wnext);
      if (((any_next >> lane) & 1u) && snext >= 0)
        prefetch_entry(&raw_all[warp][(chunk - 1) & 1][lane], snext, rec, rec64);
      __pipeline_commit();
      load_words(chunk - 2, wnn, snn);
      unsigned word[PPL];
#pragma unroll
      for (int j = 0; j < PPL; ++j) word[j] = base < last[j] ? wcur[j] : 0u;
      unsigned any = any_cur;
      __pipeline_wait_prior(1);  // this lane's copy for `chunk` has landed
      if ((any >> lane) & 1u) stage_entry<false, kBwdDF>(st + lane * kStride, scur, raw_all[warp][chunk & 1][lane], f, 0.f, 0.f);
      __syncwarp();
#pragma unroll
      for (int j = 0; j < PPL; ++j) {
        wcur[j] = wnext[j];
        wnext[j] = wnn[j];
      }
      any_cur = any_next;
      scur = snext;
      snext = snn;
      // Walk the chunk's active entries back to front.  Consecutive entries
      // that few lanes contributed to and whose lane sets are disjoint form
      // one group: each lane evaluates its own member (every pixel still sees
      // its contributions back to front) and adds it with vector atomics.
      // An entry with more lanes is evaluated alone and reduced through the
      // shared-memory transpose.  (Measured and dropped at config 1: a level
      // schedule -- entry level = 1 + the highest level of earlier entries
      // sharing a lane, non-consecutive entries may share a level -- 186 us
      // against 175; lanes owning two horizontally adjacent pixels instead of
      // rows r and r + 4, 207 us.)
      unsigned wl = 0u;
#pragma unroll
      for (int j = 0; j < PPL; ++j) wl |= word[j];
      unsigned lm_next = 0u;  // lane mask of the head entry, if already known
      while (any) {
        const int i = 31 - __clz(any);
        const unsigned lm = lm_next ? lm_next : __ballot_sync(0xffffffffu, (wl >> i) & 1u);
        lm_next = 0u;
        any &= ~(1u << i);
        const bool direct = !det && __popc(lm) <= kDirectLanes;
        int mi = i;
        if (direct) {
          mi = ((lm >> lane) & 1u) ? i : -1;
#ifndef SS_BWD_NOGROUP
          unsigned uni = lm;
          while (any) {
            const int i2 = 31 - __clz(any);
            const unsigned l2 = __ballot_sync(0xffffffffu, (wl >> i2) & 1u);
            if (__popc(l2) > kDirectLanes || (l2 & uni)) {
              lm_next = l2;
              break;
            }
            uni |= l2;
            any &= ~(1u << i2);
            if ((l2 >> lane) & 1u) mi = i2;
          }
        }
#endif
        Entry x;
        load_entry<kBwdDF>(st + max(mi, 0) * kStride, x);
        float a[14];
#pragma unroll
        for (int q = 0; q < 14; ++q) a[q] = 0.f;
#pragma unroll
        for (int j = 0; j < PPL; ++j) {
          if (mi < 0 || !((word[j] >> mi) & 1u)) continue;
          Hit h;
          intersect<kBwdDF>(x, px[j], bp, h);
          const float om = 1.f - h.alpha;
          const float iom = rcp_ftz(om);
          const float Tb = T[j] * iom;
          // dL/dalpha = Tb P - Q / (1 - alpha): P = g.(range, 1, n) of this splat,
          // Q = g.(suffix sums of w range, w, w n) behind it (rasterizer.py:612-628)
          const float P = fmaf(gD[j], h.lam, gO[j]) + gN[j][0] * x.n[0] + gN[j][1] * x.n[1] + gN[j][2] * x.n[2];
          const float dal = Tb * P - iom * Q[j];
          const float w = h.alpha * Tb;
          const float gl = gD[j] * w;
          float gsa = 0.f, gsb = 0.f, go = 0.f;
          if (!h.clamped) {
            gsa = -dal * h.alpha * h.sa;
            gsb = -dal * h.alpha * h.sb;
            go = dal * h.G;
          }
          const float gw0 = gsa * h.r, gw1 = gsb * h.r;
          const float gw2 = -(gsa * h.sa + gsb * h.sb + gl * h.lam) * h.r;
          const float v0 = px[j].vf[0], v1 = px[j].vf[1], v2 = px[j].vf[2];
          a[0] += gw0 * v0; a[1] += gw0 * v1; a[2] += gw0 * v2;
          a[3] += gw1 * v0; a[4] += gw1 * v1; a[5] += gw1 * v2;
          a[6] += gw2 * v0; a[7] += gw2 * v1; a[8] += gw2 * v2;
          a[9] += gl * h.r;
          a[10] += w * gN[j][0]; a[11] += w * gN[j][1]; a[12] += w * gN[j][2];
          a[13] += go;
          Q[j] += w * P;
          T[j] = Tb;
        }
        if (direct) {
          if (mi >= 0) {
            float4* g4 = reinterpret_cast<float4*>(acc + (size_t)x.sid * kAcc);
            atomicAdd(g4, make_float4(a[0], a[1], a[2], a[3]));
            atomicAdd(g4 + 1, make_float4(a[4], a[5], a[6], a[7]));
            atomicAdd(g4 + 2, make_float4(a[8], a[9], a[10], a[11]));
            atomicAdd(reinterpret_cast<float2*>(g4 + 3), make_float2(a[12], a[13]));
          }
          continue;
        }
        float a16[16];
#pragma unroll
        for (int q = 0; q < 14; ++q) a16[q] = a[q];
        a16[14] = a16[15] = 0.f;
        const float tot = red_transpose16(a16, red, roff, lane);
        if (det) {
          if (lane < 14) pacc[(size_t)(lo + base + i) * kAcc + lane] = tot;
        } else if (lane < 14) {
          atomicAdd(&acc[(size_t)x.sid * kAcc + lane], tot);
        }
      }
      __syncwarp();
    }
    __pipeline_wait_prior(0);
    __syncwarp();
  }
}

// Camera-frame accumulators -> plain-space (15) or raw-space (12) gradients
// (rasterizer.py:686-700, splats.py:133-163, mapping.py:479-494).
// The cross products with the camera-frame splat vectors (|Bc| ~ tens of
// metres against nearly parallel accumulated rays) are float64 from the
// forward's records; the rest of the chain is float32.
constexpr int kFinBlock = 128;

__global__ void __launch_bounds__(kFinBlock) k_finalize(SplatsK sp, PoseK pose, const SplatRec64* __restrict__ rec64,
                                                        float* __restrict__ acc,
                                                        const float* __restrict__ d_scales_extra,
                                                        float* __restrict__ out, int raw_space,
                                                        int* __restrict__ bwd_ticket, AdamK adam,
                                                        const float* __restrict__ adam_bias,
                                                        float* __restrict__ adam_m, float* __restrict__ adam_v,
                                                        double hinge_cap, double hinge_w,
                                                        double* __restrict__ hinge_loss) {
  pdl_wait();
  // the backward's persistent tile ticket restarts for the next backward pass
  if (blockIdx.x == 0 && threadIdx.x == 0) *bwd_ticket = 0;
  // The block's records and accumulators are staged through shared memory
  // with coalesced 16-byte loads, its outputs leave the same way.
  __shared__ double2 s_rec[kFinBlock * 5];
  __shared__ float4 s_acc[kFinBlock * 4];
  float* s_out = reinterpret_cast<float*>(s_rec);  // (15 floats per splat reuse the 80-byte records once read)
  static_assert(sizeof(float) * kFinBlock * 15 <= sizeof(double2) * kFinBlock * 5, "s_out fits s_rec");
  __shared__ __align__(16) float s_ta[kFinBlock * 3];
  __shared__ __align__(16) float s_tb[kFinBlock * 3];
  __shared__ __align__(16) float s_ls[kFinBlock * 2];
  __shared__ __align__(16) float s_ex[kFinBlock * 2];
  __shared__ __align__(16) float s_lo[kFinBlock];
  const int base = blockIdx.x * kFinBlock;
  const int cnt = min(kFinBlock, sp.n - base);
  const int tid = threadIdx.x;
  if (cnt == kFinBlock && ((reinterpret_cast<uintptr_t>(sp.raw_ta) | reinterpret_cast<uintptr_t>(sp.raw_tb) |
                             reinterpret_cast<uintptr_t>(sp.log_scales) | reinterpret_cast<uintptr_t>(sp.logit_opacity) |
                             reinterpret_cast<uintptr_t>(d_scales_extra)) & 15) == 0) {
    // full block: every load issued before the first shared store
    const double2* g = reinterpret_cast<const double2*>(rec64 + base);
    const float4* a4 = reinterpret_cast<const float4*>(acc + (size_t)base * kAcc);
    double2 r[5];
    float4 q4[4], x4[3];
#pragma unroll
    for (int k = 0; k < 5; ++k) r[k] = __ldg(g + tid + kFinBlock * k);
#pragma unroll
    for (int k = 0; k < 4; ++k) q4[k] = __ldg(a4 + tid + kFinBlock * k);
    constexpr int F3 = kFinBlock * 3 / 4, F2 = kFinBlock * 2 / 4, F1 = kFinBlock / 4;
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    x4[0] = tid < F3 ? __ldg(reinterpret_cast<const float4*>(sp.raw_ta + 3 * (size_t)base) + tid) : z4;
    x4[1] = tid < F3 ? __ldg(reinterpret_cast<const float4*>(sp.raw_tb + 3 * (size_t)base) + tid) : z4;
    x4[2] = tid < F2 ? __ldg(reinterpret_cast<const float4*>(sp.log_scales + 2 * (size_t)base) + tid)
          : tid < F2 + F1 ? __ldg(reinterpret_cast<const float4*>(sp.logit_opacity + base) + (tid - F2))
                          : z4;
    const float4 e4 = (d_scales_extra && tid < F2)
                          ? __ldg(reinterpret_cast<const float4*>(d_scales_extra + 2 * (size_t)base) + tid)
                          : z4;
#pragma unroll
    for (int k = 0; k < 5; ++k) s_rec[tid + kFinBlock * k] = r[k];
#pragma unroll
    for (int k = 0; k < 4; ++k) s_acc[tid + kFinBlock * k] = q4[k];
    if (tid < F3) {
      reinterpret_cast<float4*>(s_ta)[tid] = x4[0];
      reinterpret_cast<float4*>(s_tb)[tid] = x4[1];
    }
    if (tid < F2) {
      reinterpret_cast<float4*>(s_ls)[tid] = x4[2];
      reinterpret_cast<float4*>(s_ex)[tid] = e4;
    } else if (tid < F2 + F1) {
      reinterpret_cast<float4*>(s_lo)[tid - F2] = x4[2];
    }
  } else {
    const double2* g = reinterpret_cast<const double2*>(rec64 + base);
    for (int q = tid; q < cnt * 5; q += kFinBlock) s_rec[q] = __ldg(g + q);
    const float4* a4 = reinterpret_cast<const float4*>(acc + (size_t)base * kAcc);
    for (int q = tid; q < cnt * 4; q += kFinBlock) s_acc[q] = __ldg(a4 + q);
    for (int q = tid; q < cnt * 3; q += kFinBlock) {
      s_ta[q] = __ldg(sp.raw_ta + 3 * (size_t)base + q);
      s_tb[q] = __ldg(sp.raw_tb + 3 * (size_t)base + q);
    }
    for (int q = tid; q < cnt * 2; q += kFinBlock) {
      s_ls[q] = __ldg(sp.log_scales + 2 * (size_t)base + q);
      s_ex[q] = d_scales_extra ? __ldg(d_scales_extra + 2 * (size_t)base + q) : 0.f;
    }
    if (tid < cnt) s_lo[tid] = __ldg(sp.logit_opacity + base + tid);
  }
  __syncthreads();
  const int nout = raw_space ? 12 : 15;
  double hinge_acc = 0.0;
  double B[10];
  float4 ga, gb, gc, gd;
  if (tid < cnt) {
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      const double2 x = s_rec[tid * 5 + q];
      B[2 * q] = x.x;
      B[2 * q + 1] = x.y;
    }
    ga = s_acc[tid * 4];
    gb = s_acc[tid * 4 + 1];
    gc = s_acc[tid * 4 + 2];
    gd = s_acc[tid * 4 + 3];
  }
  __syncthreads();  // every record read before s_out (aliasing s_rec) is written
  if (tid < cnt) {
  const double *Ba = B, *Bb = B + 3, *Bc = B + 6;
  const double V0[3] = {ga.x, ga.y, ga.z}, V1[3] = {ga.w, gb.x, gb.y}, V2[3] = {gb.z, gb.w, gc.x};
  const double Gd = gc.y;
  const float Nc[3] = {gc.z, gc.w, gd.x};
  const float Oc = gd.y;
  float* o = s_out + tid * nout;  // (a splat that touched no pixel gets exact zeros)
  double A[3], Bv[3], C[3], t1[3], t2[3], gBa[3], gBb[3], gBc[3];
  cross3(Bb, Bc, A);
  cross3(Bc, Ba, Bv);
  cross3(Ba, Bb, C);
  cross3(V1, Bc, t1);
  cross3(Bb, V2, t2);
  for (int c = 0; c < 3; ++c) gBa[c] = t1[c] + t2[c] + Gd * A[c];
  cross3(Bc, V0, t1);
  cross3(V2, Ba, t2);
  for (int c = 0; c < 3; ++c) gBb[c] = t1[c] + t2[c] + Gd * Bv[c];
  cross3(V0, Bb, t1);
  cross3(Ba, V1, t2);
  for (int c = 0; c < 3; ++c) gBc[c] = t1[c] + t2[c] + Gd * C[c];
  const float s0 = __expf(s_ls[2 * tid]), s1 = __expf(s_ls[2 * tid + 1]);
  // d_scales: dBa/ds_a = ta_c = Ba / s_a (rasterizer.py:693-699)
  const float ds0 = (float)dot3d(gBa, Ba) * __frcp_rn(s0), ds1 = (float)dot3d(gBb, Bb) * __frcp_rn(s1);
  // camera frame -> world frame (x @ R.T), float32 after the cancelling float64 products
  float R[9];
#pragma unroll
  for (int q = 0; q < 9; ++q) R[q] = (float)pose.R[q];
  const float fa[3] = {(float)gBa[0], (float)gBa[1], (float)gBa[2]};
  const float fb[3] = {(float)gBb[0], (float)gBb[1], (float)gBb[2]};
  const float fc[3] = {(float)gBc[0], (float)gBc[1], (float)gBc[2]};
  float dmu[3], dta[3], dtb[3], dn[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    dmu[c] = fc[0] * R[3 * c] + fc[1] * R[3 * c + 1] + fc[2] * R[3 * c + 2];
    dta[c] = s0 * (fa[0] * R[3 * c] + fa[1] * R[3 * c + 1] + fa[2] * R[3 * c + 2]);
    dtb[c] = s1 * (fb[0] * R[3 * c] + fb[1] * R[3 * c + 1] + fb[2] * R[3 * c + 2]);
    dn[c] = Nc[0] * R[3 * c] + Nc[1] * R[3 * c + 1] + Nc[2] * R[3 * c + 2];
  }
  if (!raw_space) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      o[c] = dmu[c];
      o[3 + c] = dta[c];
      o[6 + c] = dtb[c];
      o[9 + c] = dn[c];
    }
    o[12] = ds0;
    o[13] = ds1;
    o[14] = Oc;
  } else {
    // Gram-Schmidt backward (splats.py:154-163), float32
    const float a[3] = {s_ta[3 * tid], s_ta[3 * tid + 1], s_ta[3 * tid + 2]};
    const float b[3] = {s_tb[3 * tid], s_tb[3 * tid + 1], s_tb[3 * tid + 2]};
    const float ina = rsqrtf(a[0] * a[0] + a[1] * a[1] + a[2] * a[2]);
    const float u[3] = {a[0] * ina, a[1] * ina, a[2] * ina};
    const float ub = u[0] * b[0] + u[1] * b[1] + u[2] * b[2];
    const float w[3] = {b[0] - ub * u[0], b[1] - ub * u[1], b[2] - ub * u[2]};
    const float inw = rsqrtf(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
    const float v[3] = {w[0] * inw, w[1] * inw, w[2] * inw};
    const float gu[3] = {dta[0] + (v[1] * dn[2] - v[2] * dn[1]), dta[1] + (v[2] * dn[0] - v[0] * dn[2]),
                         dta[2] + (v[0] * dn[1] - v[1] * dn[0])};
    const float gv[3] = {dtb[0] + (dn[1] * u[2] - dn[2] * u[1]), dtb[1] + (dn[2] * u[0] - dn[0] * u[2]),
                         dtb[2] + (dn[0] * u[1] - dn[1] * u[0])};
    const float vg = v[0] * gv[0] + v[1] * gv[1] + v[2] * gv[2];
    const float q[3] = {(gv[0] - vg * v[0]) * inw, (gv[1] - vg * v[1]) * inw, (gv[2] - vg * v[2]) * inw};
    const float qu = q[0] * u[0] + q[1] * u[1] + q[2] * u[2];
    float inner[3], gb_[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      gb_[c] = q[c] - qu * u[c];
      inner[c] = gu[c] - ub * q[c] - qu * b[c];
    }
    const float ui = u[0] * inner[0] + u[1] * inner[1] + u[2] * inner[2];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      o[c] = dmu[c];
      o[3 + c] = (inner[c] - ui * u[c]) * ina;
      o[6 + c] = gb_[c];
    }
    float ex0 = s_ex[2 * tid], ex1 = s_ex[2 * tid + 1];
    if (hinge_loss) {  // the scale hinge here instead of k_scale_loss (same float64 arithmetic)
      const double e0 = exp((double)s_ls[2 * tid]), e1 = exp((double)s_ls[2 * tid + 1]);
      const double over = fmax(e0, e1) - hinge_cap;
      ex0 = ex1 = 0.f;
      if (over > 0.0) {
        hinge_acc = over;
        if (e0 >= e1)
          ex0 = (float)hinge_w;
        else
          ex1 = (float)hinge_w;
      }
    }
    o[9] = (ds0 + ex0) * s0;
    o[10] = (ds1 + ex1) * s1;
    const float xo = s_lo[tid];
    const float ex = __expf(-fabsf(xo));
    const float op = (xo >= 0.f ? 1.f : ex) * __frcp_rn(1.f + ex);
    o[11] = Oc * op * (1.f - op);
  }
  }
  if (hinge_loss) {  // block sum of the hinge, one float64 atomic per warp
    for (int off = 16; off > 0; off >>= 1) hinge_acc += __shfl_xor_sync(0xffffffffu, hinge_acc, off);
    if ((tid & 31) == 0 && hinge_acc != 0.0) atomicAdd(hinge_loss, hinge_acc);
  }
  __syncthreads();
  {  // consumed: leave the accumulators zeroed for the next backward pass
    float4* a4 = reinterpret_cast<float4*>(acc + (size_t)base * kAcc);
    for (int q = tid; q < cnt * 4; q += kFinBlock) a4[q] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  if (adam_bias) {  // fused Adam step on the raw gradient (refine): parameters and moments in place
    if (tid < cnt) {
      float gg[12];
#pragma unroll
      for (int q = 0; q < 12; ++q) gg[q] = s_out[tid * 12 + q];
      adam_row(base + tid, adam, 1.f / adam_bias[0], 1.f / adam_bias[1], gg, adam_m, adam_v);
    }
    if (!out) return;
  }
  float* g = out + (size_t)base * nout;
  if (cnt == kFinBlock && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
    for (int q = tid; q < kFinBlock * nout / 4; q += kFinBlock)
      reinterpret_cast<float4*>(g)[q] = reinterpret_cast<const float4*>(s_out)[q];
  } else {
    for (int q = tid; q < cnt * nout; q += kFinBlock) g[q] = s_out[q];
  }
}

#define SS_INST_FWD(TS, SPLIT)                                                                                  \
  template __global__ void k_forward<TS, SPLIT>(BlendParams, int, const int*, const int*, const int*,               \
                                                const SplatRec*, const SplatRec64*, float*, float*, float*, float*,  \
                                                int*, unsigned*, const int*, const int*, int*, const int*);
#define SS_INST_BWD(TS, SPLIT, SEG)                                                                             \
  template __global__ void k_backward<TS, SPLIT, SEG>(BlendParams, int, const int*, const int*, const int*,         \
                                                 const SplatRec*, const SplatRec64*, const float*, const int*,       \
                                                 const unsigned*, const float*, const float*, const float*, float*,  \
                                                 const int*, const int*, int*, const int*, float*);
SS_INST_FWD(8, false)

SS_INST_FWD(16, false)
SS_INST_BWD(8, false, false)
SS_INST_BWD(8, true, false)
SS_INST_BWD(8, false, true)
SS_INST_BWD(16, false, false)

// Deterministic mode: zero the per-position accumulators of the current pair count.
__global__ void k_zero_pacc(float4* __restrict__ pacc, const long long* __restrict__ totals, long long cap) {
  pdl_wait();
  const long long n = min(totals[0], cap) * (kAcc / 4);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    pacc[i] = make_float4(0.f, 0.f, 0.f, 0.f);
}

// Deterministic mode: per splat, the entries it owns in its tiles' lists (tiles in
// row-major order over its rectangle, its list position found by binary search on
// the (float64 range, index) order) are summed in that fixed order.
__global__ void __launch_bounds__(256) k_det_gather(int n, int tx, const int4* __restrict__ rect,
                                                    const unsigned long long* __restrict__ key64,
                                                    const int* __restrict__ tile_ptr, const int* __restrict__ pairs,
                                                    const float* __restrict__ pacc, float* __restrict__ acc,
                                                    const int* __restrict__ overflow) {
  pdl_wait();
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n || *overflow) return;
  float a[14];
#pragma unroll
  for (int q = 0; q < 14; ++q) a[q] = 0.f;
  const int4 r = rect[s];
  const unsigned long long ks = key64[s];
  for (int row = r.x; row <= r.y; ++row)
    for (int k = 0; k < r.w; ++k) {
      int c = r.z + k;
      if (c >= tx) c -= tx;
      const int t = row * tx + c;
      int lo = tile_ptr[t], hi = tile_ptr[t + 1];
      while (lo < hi) {  // first position not less than (ks, s)
        const int mid = (lo + hi) >> 1;
        const int v = pairs[mid];
        const unsigned long long kv = key64[v];
        if (kv < ks || (kv == ks && v < s))
          lo = mid + 1;
        else
          hi = mid;
      }
      const float4* p4 = reinterpret_cast<const float4*>(pacc + (size_t)lo * kAcc);
      const float4 x0 = p4[0], x1 = p4[1], x2 = p4[2], x3 = p4[3];
      a[0] += x0.x; a[1] += x0.y; a[2] += x0.z; a[3] += x0.w;
      a[4] += x1.x; a[5] += x1.y; a[6] += x1.z; a[7] += x1.w;
      a[8] += x2.x; a[9] += x2.y; a[10] += x2.z; a[11] += x2.w;
      a[12] += x3.x; a[13] += x3.y;
    }
  float4* o = reinterpret_cast<float4*>(acc + (size_t)s * kAcc);
  o[0] = make_float4(a[0], a[1], a[2], a[3]);
  o[1] = make_float4(a[4], a[5], a[6], a[7]);
  o[2] = make_float4(a[8], a[9], a[10], a[11]);
  o[3] = make_float4(a[12], a[13], 0.f, 0.f);
}

}  // namespace ss
