// K1 per-splat preprocess and K2 tile binning (duplicate + order).
//
// Reference behaviour (pkg/src/splatscan/):
//   splats.py:112-130,217-231      activation + Gram-Schmidt
//   rasterizer.py:223-241          camera-frame splat arrays
//   rasterizer.py:244-306          cone-bound tile incidence (float64, bit-exact)
//   rasterizer.py:318-339          per-tile lists ordered by (tile, f64 range, index)
//
// Design.  The incidence predicate is evaluated exactly as the reference
// does (float64, no contraction) on the tiles near the splat's cone only.
// Pipeline (no cross-block dependency chains, no global atomics, no host
// synchronisation):
//   1. preprocess: records, tile rectangle, pair count, per-block count sums;
//   2. scan of the block sums; emit every (tile, splat) pair at its offset;
//   3. counting sort of the pairs by tile from per-block shared-memory
//      histograms (order inside a tile is irrelevant, see 4);
//   4. per tile, a shared-memory LSD radix sort by a 16-bit monotone key
//      (float64 range -> float32 rounded down -> relative to the tile's
//      minimum), then runs of equal keys are put in exact (float64 range,
//      splat index) order.  Lists longer than the shared-memory capacity
//      take a global merge-sort fallback with the exact comparator.
// Pair buffers are sized speculatively; an overflow flag is checked by the
// host after the fact (ss_records_check).
#include "common.cuh"

namespace ss {

struct Incidence {
  double azc, elc, omega, dgam;
};

#ifndef SS_SORT_MAX
#define SS_SORT_MAX 2048
#endif
constexpr int kTileSortMax = SS_SORT_MAX;         // entries sorted in shared memory per tile (8 warps)
constexpr int kTileSortBig = 8192;    // long-list variant (32 warps, 98 KB of dynamic shared memory)
constexpr int kTileSortHuge = 16384;  // dense maps: lists up to this in 214 KB (one block per SM)
constexpr int kMaxTieRun = 64;                    // longer runs of equal sort keys: the block's bitonic sort
#ifndef SS_THREAD_TIE
#define SS_THREAD_TIE 5
#endif
#ifndef SS_TIE_STAGE
#define SS_TIE_STAGE 4  // runs at least this long stage their keys in shared memory
#endif
constexpr int kThreadTieRun = SS_THREAD_TIE;                 // runs up to this long: one thread's insertion sort
constexpr int kMaxLongRuns = 128;                 // (more of them per list: merge-sort fallback)

// np.mod(x, 2*pi) for x = d + pi with d a difference of two angles in
// [-pi, pi]: fmod is exact, so the subtraction below is bit-identical.
__device__ __forceinline__ double mod_2pi(double x) {
  const double tp = 2.0 * SS_PI;
  if (x >= 0.0 && x < tp) return x;
  if (x >= tp && x < 2.0 * tp) return x_sub(x, tp);
  return py_mod(x, tp);
}

__device__ __forceinline__ bool col_hit(const CamK& k, const double2* __restrict__ colt, const Incidence& g, int c) {
  const double2 ch = colt[c];
  double d = x_sub(g.azc, ch.x);
  d = fabs(x_sub(mod_2pi(x_add(d, SS_PI)), SS_PI));
  return d <= x_add(x_add(g.dgam, ch.y), k.pad_az);
}
__device__ __forceinline__ bool row_hit(const CamK& k, const double2* __restrict__ rowt, const Incidence& g, int r) {
  const double2 rh = rowt[r];
  const double d = fabs(x_sub(g.elc, rh.x));
  return d <= x_add(x_add(g.omega, rh.y), k.pad_el);
}

// Per-tile-column and -row angular intervals (rasterizer.py:278-294).
// (also clears the forward's status / overflow / ticket words, the pair totals and
// the tile counts: one launch instead of three memsets)
__global__ void k_tile_intervals(CamK k, double2* __restrict__ colt, double2* __restrict__ rowt,
                                 int* __restrict__ misc16, long long* __restrict__ totals2,
                                 int* __restrict__ tile_count, int ntiles) {
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < 16) misc16[i] = 0;
  if (i < 3) totals2[i] = 0;  // pairs, chunks, longest list
  if (i < ntiles) tile_count[i] = 0;
  double c, h;
  if (i < k.tx) {
    tile_col_interval(k, i, c, h);
    colt[i] = make_double2(c, h);
  } else if (i < k.tx + k.ty) {
    tile_row_interval(k, i - k.tx, c, h);
    rowt[i - k.tx] = make_double2(c, h);
  }
}

// x @ R for a row vector x (numpy matmul of an (N,3) array with R uses FMA, OpenBLAS dgemm).
__device__ __forceinline__ double rowmat(const double x[3], const double* R, int c) {
  return fma(x[2], R[6 + c], fma(x[1], R[3 + c], x_mul(x[0], R[c])));
}

__device__ __forceinline__ uint32_t preprocess_one(SplatsK sp, PoseK pose, CamK cam, RasterK rk, const double2* __restrict__ colt,
                                   const double2* __restrict__ rowt, SplatRec* __restrict__ rec,
                                   SplatRec64* __restrict__ rec64, unsigned long long* __restrict__ key64,
                                   uint32_t* __restrict__ key32, int4* __restrict__ rect, int* __restrict__ status,
                                   int i) {
  const int4 empty = make_int4(0, -1, 0, 0);
  key32[i] = 0xffffffffu;
  rect[i] = empty;
  // --- Gram-Schmidt (splats.py:112-130), float64
  double a[3], b[3];
  for (int c = 0; c < 3; ++c) {
    a[c] = (double)sp.raw_ta[3 * i + c];
    b[c] = (double)sp.raw_tb[3 * i + c];
  }
  const double na = sqrt(x_add(x_add(x_mul(a[0], a[0]), x_mul(a[1], a[1])), x_mul(a[2], a[2])));
  if (na < 1e-12) {
    atomicExch(status, (int)SS_ERR_DEGENERATE);
    return 0u;
  }
  const double u[3] = {a[0] / na, a[1] / na, a[2] / na};
  const double ub = u[0] * b[0] + u[1] * b[1] + u[2] * b[2];
  const double w[3] = {b[0] - ub * u[0], b[1] - ub * u[1], b[2] - ub * u[2]};
  const double nw = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
  if (nw < 1e-12) {
    atomicExch(status, (int)SS_ERR_DEGENERATE);
    return 0u;
  }
  const double v[3] = {w[0] / nw, w[1] / nw, w[2] / nw};
  const double nn[3] = {u[1] * v[2] - u[2] * v[1], u[2] * v[0] - u[0] * v[2], u[0] * v[1] - u[1] * v[0]};
  const double s0 = exp((double)sp.log_scales[2 * i]), s1 = exp((double)sp.log_scales[2 * i + 1]);
  const double x = (double)sp.logit_opacity[i];
  double o;
  if (x >= 0) {
    o = 1.0 / (1.0 + exp(-x));
  } else {
    const double e = exp(x);
    o = e / (1.0 + e);
  }
  // --- camera-frame arrays (rasterizer.py:223-241)
  const double m[3] = {x_sub((double)sp.centers[3 * i], pose.t[0]), x_sub((double)sp.centers[3 * i + 1], pose.t[1]),
                       x_sub((double)sp.centers[3 * i + 2], pose.t[2])};
  double Bc[3], Ba[3], Bb[3], nc[3];
  for (int c = 0; c < 3; ++c) {
    Bc[c] = rowmat(m, pose.R, c);
    Ba[c] = s0 * rowmat(u, pose.R, c);
    Bb[c] = s1 * rowmat(v, pose.R, c);
    nc[c] = rowmat(nn, pose.R, c);
  }
  const double range = sqrt(x_add(x_add(x_mul(Bc[0], Bc[0]), x_mul(Bc[1], Bc[1])), x_mul(Bc[2], Bc[2])));

  // --- render records for the blend kernels
  const double kq = o / rk.alpha_cutoff;
  const float Kp = kq > 1.0 ? (float)(2.0 * log(kq) * (1.0 + 1e-4) + 1e-4) : -1.0f;
  SplatRec r;
  r.r0 = make_float4((float)o, Kp, (float)nc[0], (float)nc[1]);
  rec[i] = r;
  SplatRec64 r64;
  r64.v[0] = make_double2(Ba[0], Ba[1]);
  r64.v[1] = make_double2(Ba[2], Bb[0]);
  r64.v[2] = make_double2(Bb[1], Bb[2]);
  r64.v[3] = make_double2(Bc[0], Bc[1]);
  r64.v[4] = make_double2(Bc[2], nc[2]);
  rec64[i] = r64;
  key64[i] = (unsigned long long)__double_as_longlong(range);

  // --- cone-bound incidence (rasterizer.py:256-305), float64 without contraction.
  // (Measured and dropped: deciding every row / column test in float32 first and falling
  // back to float64 only when a margin is under 1e-5 rad -- 0.2 % of the splats at config
  // 1, tile lists still bit-exact -- took 61 us against 52: the float64 transcendentals
  // here are not what bounds this kernel.)
  Incidence g;
  const double reach = x_mul(rk.cutoff_sigma, fmax(s0, s1));
  const bool near_ = range <= x_add(reach, 1e-12);
  double so = x_div(reach, fmax(range, 1e-12));
  so = fmin(fmax(so, 0.0), 1.0);
  double omega = asin(so);
  g.azc = atan2(Bc[1], Bc[0]);
  g.elc = atan2(Bc[2], hypot(Bc[0], Bc[1]));
  const bool pole = x_add(fabs(g.elc), omega) >= (SS_PI / 2 - 1e-9);
  const double ce = fmax(cos(g.elc), 1e-12);
  const double q = fmin(fmax(x_div(so, ce), 0.0), 1.0);
  double dgam = asin(q);
  if (near_ || pole) dgam = SS_PI;
  if (near_) omega = SS_PI;
  g.omega = omega;
  g.dgam = dgam;
  if (!(range > 1e-9)) return 0u;  // not alive (rasterizer.py:303-305)
  // (every row: starting at the splat's own row and extending both ways until a miss,
  // as for the columns below, measured 56 us against 52 at config 1 -- the divergent
  // extension loops cost more than 16 uniform row tests)
  int r_lo = -1, r_hi = -2;
  for (int rr = 0; rr < cam.ty; ++rr) {
    if (row_hit(cam, rowt, g, rr)) {
      if (r_lo < 0) r_lo = rr;
      r_hi = rr;
    }
  }
  if (r_lo < 0) return 0u;
  const int tx = cam.tx;
  int c_start = 0, ncols = 0, h = -1;
  if (dgam < 0.5 * SS_PI) {
    const double uu = cam.fx * g.azc + cam.cx - cam.off_u;
    const int c0 = (int)floor(uu / cam.T);
    for (int dc = 0; dc < 3 && h < 0; ++dc) {
      int c = c0 + (dc == 0 ? 0 : (dc == 1 ? -1 : 1));
      c = ((c % tx) + tx) % tx;  // (c0 may lie anywhere: the only general modulo)
      if (col_hit(cam, colt, g, c)) h = c;
    }
  }
  if (h >= 0) {
    // the hit set is one circular run around h (interval overlap on a circle)
    int lo = h, cnt = 1;
    while (cnt < tx) {  // circular neighbours by compare-and-wrap (no integer division)
      const int c = lo == 0 ? tx - 1 : lo - 1;
      if (!col_hit(cam, colt, g, c)) break;
      lo = c;
      ++cnt;
    }
    int hi = h;
    while (cnt < tx) {
      const int c = hi + 1 == tx ? 0 : hi + 1;
      if (!col_hit(cam, colt, g, c)) break;
      hi = c;
      ++cnt;
    }
    c_start = lo;
    ncols = cnt;
  } else {
    // wide cone or centre column missed (partial field of view): scan all columns
    int first_miss = -1, nhit = 0;
    for (int c = 0; c < tx; ++c) {
      const bool hc = col_hit(cam, colt, g, c);
      nhit += hc;
      if (!hc && first_miss < 0) first_miss = c;
    }
    if (nhit == tx) {
      ncols = tx;
    } else if (nhit > 0) {
      int c = first_miss;
      while (!col_hit(cam, colt, g, c)) c = c + 1 == tx ? 0 : c + 1;
      c_start = c;
      ncols = nhit;
    }
  }
  if (ncols == 0) return 0u;
  rect[i] = make_int4(r_lo, r_hi, c_start, ncols);
  key32[i] = __float_as_uint(__double2float_rd(range));  // monotone in the float64 range
  return (uint32_t)((r_hi - r_lo + 1) * ncols);
}


#ifndef SS_PRE_MINB
#define SS_PRE_MINB 5  // 48 registers (A/B at config 1: 62 -> 53 us)
#endif
__global__ void __launch_bounds__(256, SS_PRE_MINB)
    k_preprocess(SplatsK sp, PoseK pose, CamK cam, RasterK rk, const double2* __restrict__ colt,
                 const double2* __restrict__ rowt, SplatRec* __restrict__ rec, SplatRec64* __restrict__ rec64,
                 unsigned long long* __restrict__ key64, uint32_t* __restrict__ key32, int4* __restrict__ rect,
                 uint32_t* __restrict__ block_sum, int* __restrict__ status) {
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t cnt = 0;
  if (i < sp.n) cnt = preprocess_one(sp, pose, cam, rk, colt, rowt, rec, rec64, key64, key32, rect, status, i);
  // block sum of pair counts (for the emission scan)
  for (int off = 16; off > 0; off >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
  __shared__ uint32_t ws[8];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t s = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += ws[w];
    block_sum[blockIdx.x] = s;
  }
}


// Block-wide (1024 threads) exclusive scan of one 64-bit value per thread by
// warp shuffles (two barriers); *total gets the sum.
__device__ __forceinline__ long long block_exscan_1024(long long v, long long* wsum, long long* total) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  long long inc = v;
  for (int off = 1; off < 32; off <<= 1) {
    const long long y = __shfl_up_sync(0xffffffffu, inc, off);
    if (lane >= off) inc += y;
  }
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const long long w = wsum[lane];
    long long wi = w;
    for (int off = 1; off < 32; off <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, wi, off);
      if (lane >= off) wi += y;
    }
    wsum[lane] = wi - w;
    if (lane == 31) *total = wi;
  }
  __syncthreads();
  return wsum[warp] + inc - v;
}

// Exclusive scan of the per-block pair counts (one block); totals[0] = pairs.
__global__ void __launch_bounds__(1024) k_scan_blocks(int nb, uint32_t* __restrict__ block_sum,
                                                      long long* __restrict__ totals) {
  pdl_wait();
  __shared__ long long wsum[32], tot;
  const int tid = threadIdx.x;
  const int per = (nb + 1023) / 1024;
  const int b = min(tid * per, nb), e = min(b + per, nb);
  uint32_t c[8];
  long long s = 0;
  if (per <= 8) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      c[q] = b + q < e ? block_sum[b + q] : 0u;
      s += c[q];
    }
  } else {
    for (int q = b; q < e; ++q) s += block_sum[q];
  }
  long long run = block_exscan_1024(s, wsum, &tot);
  if (per <= 8) {
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (b + q < e) {
        block_sum[b + q] = (uint32_t)run;
        run += c[q];
      }
  } else {
    for (int q = b; q < e; ++q) {
      const uint32_t cq = block_sum[q];
      block_sum[q] = (uint32_t)run;
      run += cq;
    }
  }
  if (tid == 0) totals[0] = tot;
}

// Emit the pairs of every splat at its offset (index order).  Each warp
// writes the pairs of its 32 splats cooperatively (coalesced), decoding
// (splat, tile) from the warp's inclusive count prefix.  Overflow of the
// speculative capacity sets a flag.
__global__ void __launch_bounds__(256)
    k_emit(int n, const int4* __restrict__ rect, const uint32_t* __restrict__ block_off, int tx, long long cap,
           uint32_t* __restrict__ pair_tile, uint32_t* __restrict__ pair_splat, int* __restrict__ overflow) {
  pdl_wait();
  __shared__ uint32_t ws[8];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int4 r = make_int4(0, -1, 0, 0);
  if (i < n) r = rect[i];
  const uint32_t cnt = (r.y >= r.x) ? (uint32_t)((r.y - r.x + 1) * r.w) : 0u;
  uint32_t inc = cnt;
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, off);
    if (lane >= off) inc += y;
  }
  if (lane == 31) ws[warp] = inc;
  __syncthreads();
  uint32_t wex = 0;
  for (int w = 0; w < warp; ++w) wex += ws[w];
  const uint32_t wtot = __shfl_sync(0xffffffffu, inc, 31);
  const long long off = (long long)block_off[blockIdx.x] + wex;
  if (off + wtot > cap) {
    if (lane == 0 && wtot) atomicExch(overflow, 1);
    return;
  }
  // pair q of this warp belongs to the lane whose inclusive prefix first exceeds q
  for (uint32_t q0 = 0; q0 < wtot; q0 += 32) {
    const uint32_t q = q0 + lane;
    int owner = 0;
    for (int b = 16; b > 0; b >>= 1) {
      const uint32_t v = __shfl_sync(0xffffffffu, inc, owner + b - 1);
      if (v <= q) owner += b;
    }
    const uint32_t ex = __shfl_sync(0xffffffffu, inc - cnt, owner);
    const int4 ro = make_int4(__shfl_sync(0xffffffffu, r.x, owner), 0, __shfl_sync(0xffffffffu, r.z, owner),
                              __shfl_sync(0xffffffffu, r.w, owner));
    if (q < wtot) {
      const uint32_t k = q - ex;
      const int rr = ro.x + (int)(k / (uint32_t)ro.w);
      int c = ro.z + (int)(k % (uint32_t)ro.w);
      if (c >= tx) c -= tx;
      pair_tile[off + q] = (uint32_t)(rr * tx + c);
      pair_splat[off + q] = (uint32_t)(blockIdx.x * blockDim.x + warp * 32 + owner);
    }
  }
}

// Counting sort of the pairs by tile without global atomics:
//   k_tile_hist_blocks  per block of `chunk` pairs, a shared-memory tile
//                       histogram written as row b of a blocks x tiles matrix;
//   k_tile_prefix       per tile, exclusive prefix over blocks + tile totals;
//   k_scan_tiles        tile_ptr and chunk_ptr (32-entry chunks);
//   k_tile_scatter      each block re-reads its pairs and places them with
//                       shared-memory cursors (order inside a tile is
//                       irrelevant: k_tile_sort establishes it).
// pairs per counting-sort block: 16 k when tiles are many (config 1: 37 us, 8 k 40),
// 8 k when they are few (config 2: 29 us, 16 k 34) -- a launch argument `chunk`
constexpr int kPairChunkMany = 16384, kPairChunkFew = 8192;
constexpr int kMaxTiles = 16384;  // shared-memory histogram capacity

__global__ void __launch_bounds__(1024)
    k_tile_hist_blocks(const uint32_t* __restrict__ pair_tile, const long long* __restrict__ totals, long long cap,
                       int ntiles, uint32_t* __restrict__ mat, const int* __restrict__ overflow, int chunk) {
  pdl_wait();
  extern __shared__ uint32_t h[];
  const long long n = min(totals[0], cap);
  const long long b0 = (long long)blockIdx.x * chunk;
  if (b0 >= n && blockIdx.x > 0) return;
  for (int t = threadIdx.x; t < ntiles; t += blockDim.x) h[t] = 0;
  __syncthreads();
  if (!*overflow) {
    const long long e = min(b0 + chunk, n);
    for (long long i = b0 + threadIdx.x; i < e; i += blockDim.x) atomicAdd(&h[pair_tile[i]], 1u);
  }
  __syncthreads();
  for (int t = threadIdx.x; t < ntiles; t += blockDim.x) mat[(size_t)blockIdx.x * ntiles + t] = h[t];
}

// Per tile, exclusive prefix of the block histograms over the pair blocks
// (in place) and the tile totals.  Block = 32 tiles x 32 block-segments.
__global__ void __launch_bounds__(1024) k_tile_prefix(const long long* __restrict__ totals, long long cap, int ntiles,
                                                      uint32_t* __restrict__ mat, int* __restrict__ tile_count,
                                                      int chunk, int nb_fixed) {
  pdl_wait();
  __shared__ uint32_t part[32][33];
  const int tx = threadIdx.x, seg = threadIdx.y;
  const int t = blockIdx.x * 32 + tx;
  const long long n = min(totals[0], cap);
  // (nb_fixed > 0: the direct binning's splat blocks, k_bin_count)
  const int nb = nb_fixed > 0 ? nb_fixed : (int)max(1LL, (n + chunk - 1) / chunk);
  const int per = (nb + 31) / 32;
  const int b0 = min(seg * per, nb), b1 = min(b0 + per, nb);
  uint32_t s = 0;
  if (t < ntiles)
    for (int b = b0; b < b1; ++b) s += mat[(size_t)b * ntiles + t];
  part[seg][tx] = s;
  __syncthreads();
  if (seg == 0) {
    uint32_t run = 0;
    for (int g = 0; g < 32; ++g) {
      const uint32_t c = part[g][tx];
      part[g][tx] = run;
      run += c;
    }
    if (t < ntiles) tile_count[t] = (int)run;
  }
  __syncthreads();
  if (t < ntiles) {
    uint32_t run = part[seg][tx];
    for (int b = b0; b < b1; ++b) {
      const uint32_t c = mat[(size_t)b * ntiles + t];
      mat[(size_t)b * ntiles + t] = run;
      run += c;
    }
  }
}

__global__ void __launch_bounds__(1024) k_scan_tiles(int ntiles, const int* __restrict__ tile_count,
                                                     int* __restrict__ tile_ptr, int* __restrict__ chunk_ptr,
                                                     long long* __restrict__ totals, int* __restrict__ long_list,
                                                     int* __restrict__ n_long, long long cap, int* __restrict__ overflow,
                                                     int set_total) {
  pdl_wait();
  __shared__ long long wsum[32], tot;
  const int tid = threadIdx.x;
  const int per = (ntiles + 1023) / 1024;
  const int b = min(tid * per, ntiles), e = min(b + per, ntiles);
  // pair and chunk counts packed in one 64-bit scan (chunks <= pairs / 32 + tiles < 2^31)
  long long s = 0;
  for (int t = b; t < e; ++t) {
    const int c = tile_count[t];
    s += ((long long)c << 32) + ((c + 31) >> 5);
  }
  const long long ex = block_exscan_1024(s, wsum, &tot);
  long long rp = ex >> 32, rc = ex & 0xffffffffll;
  int cmax = 0;
  for (int t = b; t < e; ++t) {
    const int c = tile_count[t];
    tile_ptr[t] = (int)rp;
    chunk_ptr[t] = (int)rc;
    rp += c;
    rc += (c + 31) >> 5;
    cmax = max(cmax, c);
    if (c > kTileSortMax) long_list[atomicAdd(n_long, 1)] = t;  // k_tile_sort_big, concurrently
  }
  // the longest list (published with the totals: the next render's work layout, see capi.cu)
  cmax = __reduce_max_sync(0xffffffffu, cmax);
  if ((tid & 31) == 0 && cmax > 0) atomicMax(reinterpret_cast<unsigned long long*>(totals + 2), (unsigned long long)cmax);
  if (tid == 0) {
    tile_ptr[ntiles] = (int)(tot >> 32);
    chunk_ptr[ntiles] = (int)(tot & 0xffffffffll);
    totals[1] = tot & 0xffffffffll;
    if (set_total) {  // direct binning: the pair total is first known here
      totals[0] = tot >> 32;
      if ((tot >> 32) > cap) *overflow = 1;
    }
  }
}

// Direct binning (SS_DIRECT_BIN): no (tile, splat) pair list.  k_bin_count builds each
// block's tile histogram straight from the splats' tile rectangles (row b of the blocks x
// tiles matrix, as k_tile_hist_blocks does from the pair list), and k_bin_scatter
// re-expands the rectangles into the tile buckets, staged by tile in shared memory so a
// tile's pairs from one block land as one run (a block with more pairs than the stage
// writes them directly).  Replaces k_scan_blocks + k_emit + k_tile_hist_blocks +
// k_tile_scatter and the pair list's 16 bytes per pair of traffic.
constexpr int kBinSplats = 2048;  // splats per binning block
constexpr int kBinStage = 12288;  // pairs staged in shared memory per block
constexpr uint32_t kBinLane = 8;  // rectangles of up to this many tiles expanded by one lane

__device__ __forceinline__ int rect_tile(int rr, int c, int tx) { return rr * tx + (c >= tx ? c - tx : c); }

// The (tile, splat) pairs of the warp's 32 splats, 32 at a time across the lanes (a splat
// covering many tiles would otherwise hold its lane for its whole rectangle): pair q
// belongs to the lane whose inclusive count prefix first exceeds q.  Warp-uniform call.
template <class F>
__device__ __forceinline__ void warp_pairs(int4 r, int i, int tx, F&& f) {
  const int lane = threadIdx.x & 31;
  const uint32_t all = (r.y >= r.x) ? (uint32_t)((r.y - r.x + 1) * r.w) : 0u;
  // small rectangles (the common case) by their own lane
  if (all <= kBinLane)
    for (int rr = r.x; rr <= r.y; ++rr)
      for (int q = 0; q < r.w; ++q) f(rect_tile(rr, r.z + q, tx), i);
  const uint32_t cnt = all > kBinLane ? all : 0u;
  if (!__any_sync(0xffffffffu, cnt > 0)) return;
  uint32_t inc = cnt;
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, off);
    if (lane >= off) inc += y;
  }
  const uint32_t wtot = __shfl_sync(0xffffffffu, inc, 31);
  for (uint32_t q0 = 0; q0 < wtot; q0 += 32) {
    const uint32_t q = q0 + lane;
    int owner = 0;
    for (int b = 16; b > 0; b >>= 1) {
      const uint32_t v = __shfl_sync(0xffffffffu, inc, owner + b - 1);
      if (v <= q) owner += b;
    }
    const uint32_t ex = __shfl_sync(0xffffffffu, inc - cnt, owner);
    const int rx = __shfl_sync(0xffffffffu, r.x, owner), rz = __shfl_sync(0xffffffffu, r.z, owner);
    const int rw = __shfl_sync(0xffffffffu, r.w, owner), si = __shfl_sync(0xffffffffu, i, owner);
    if (q < wtot) {
      const uint32_t k = q - ex;
      f(rect_tile(rx + (int)(k / (uint32_t)rw), rz + (int)(k % (uint32_t)rw), tx), si);
    }
  }
}

// The block's tile histogram as a 2-D difference array over the tile grid: four shared
// atomics per rectangle (two rectangles when it wraps in azimuth), then row and column
// prefix sums -- a splat covering many tiles costs no more than one covering a few.
__global__ void __launch_bounds__(1024) k_bin_count(int n, const int4* __restrict__ rect, int tx, int ty,
                                                    uint32_t* __restrict__ mat) {
  pdl_wait();
  extern __shared__ int dgrid[];  // (ty + 1) x (tx + 1)
  const int W1 = tx + 1, ncell = (ty + 1) * W1, ntiles = tx * ty;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int q = tid; q < ncell; q += blockDim.x) dgrid[q] = 0;
  __syncthreads();
  auto add_rect = [&](int r0, int r1, int ca, int cb) {  // rows r0..r1, columns ca..cb
    atomicAdd(&dgrid[r0 * W1 + ca], 1);
    atomicAdd(&dgrid[r0 * W1 + cb + 1], -1);
    atomicAdd(&dgrid[(r1 + 1) * W1 + ca], -1);
    atomicAdd(&dgrid[(r1 + 1) * W1 + cb + 1], 1);
  };
  const int i1 = min((blockIdx.x + 1) * kBinSplats, n);
  for (int i = blockIdx.x * kBinSplats + tid; i < i1; i += blockDim.x) {
    const int4 r = rect[i];
    if (r.y < r.x || r.w <= 0) continue;
    const int cend = r.z + r.w - 1;
    if (cend < tx) {
      add_rect(r.x, r.y, r.z, cend);
    } else {
      add_rect(r.x, r.y, r.z, tx - 1);
      add_rect(r.x, r.y, 0, cend - tx);
    }
  }
  __syncthreads();
  // prefix along each row (a warp per row, 32 columns at a time)
  for (int row = warp; row < ty; row += (int)(blockDim.x >> 5)) {
    int carry = 0;
    for (int c0 = 0; c0 < tx; c0 += 32) {
      const int c = c0 + lane;
      int v = c < tx ? dgrid[row * W1 + c] : 0;
      for (int off = 1; off < 32; off <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, v, off);
        if (lane >= off) v += y;
      }
      v += carry;
      if (c < tx) dgrid[row * W1 + c] = v;
      carry = __shfl_sync(0xffffffffu, v, 31);
    }
  }
  __syncthreads();
  // ... then down each column, and out as row b of the blocks x tiles matrix
  for (int c = tid; c < tx; c += blockDim.x) {
    int run = 0;
    for (int row = 0; row < ty; ++row) {
      run += dgrid[row * W1 + c];
      mat[(size_t)blockIdx.x * ntiles + row * tx + c] = (uint32_t)run;
    }
  }
}

__global__ void __launch_bounds__(1024)
    k_bin_scatter(int n, const int4* __restrict__ rect, int tx, int ntiles, const uint32_t* __restrict__ mat, int nbb,
                  const int* __restrict__ tile_ptr, const int* __restrict__ tile_count,
                  uint32_t* __restrict__ bucketed, const int* __restrict__ overflow) {
  pdl_wait();
  extern __shared__ uint32_t sm[];
  uint32_t* lcur = sm;
  uint32_t* gdel = sm + ntiles;
  uint32_t* sspl = sm + 2 * ntiles;
  uint16_t* stile = reinterpret_cast<uint16_t*>(sspl + kBinStage);
  __shared__ long long wsum[32], tot;
  if (*overflow) return;
  const int tid = threadIdx.x;
  const int per = (ntiles + 1023) / 1024;
  const int t0 = min(tid * per, ntiles), t1 = min(t0 + per, ntiles);
  const size_t row = (size_t)blockIdx.x * ntiles, next = row + ntiles;
  const bool last_block = blockIdx.x + 1 >= nbb;
  long long sum = 0;
  for (int t = t0; t < t1; ++t) sum += (last_block ? (uint32_t)tile_count[t] : mat[next + t]) - mat[row + t];
  long long run = block_exscan_1024(sum, wsum, &tot);
  for (int t = t0; t < t1; ++t) {
    const uint32_t c = (last_block ? (uint32_t)tile_count[t] : mat[next + t]) - mat[row + t];
    lcur[t] = (uint32_t)run;
    gdel[t] = (uint32_t)tile_ptr[t] + mat[row + t] - (uint32_t)run;
    run += c;
  }
  __syncthreads();
  const bool staged = tot <= kBinStage;  // (block-uniform)
  const int i1 = min((blockIdx.x + 1) * kBinSplats, n);
  for (int i = blockIdx.x * kBinSplats + tid; i - (tid & 31) < i1; i += 1024) {
    const int4 r = i < i1 ? rect[i] : make_int4(0, -1, 0, 0);
    warp_pairs(r, i, tx, [&](int t, int si) {
      const uint32_t slot = atomicAdd(&lcur[t], 1u);
      if (staged) {
        sspl[slot] = (uint32_t)si;
        stile[slot] = (uint16_t)t;
      } else {
        bucketed[gdel[t] + slot] = (uint32_t)si;
      }
    });
  }
  __syncthreads();
  if (staged)
    for (int q = tid; q < (int)tot; q += 1024) bucketed[gdel[stile[q]] + q] = sspl[q];
}

__global__ void __launch_bounds__(1024)
    k_tile_scatter(const uint32_t* __restrict__ pair_tile, const uint32_t* __restrict__ pair_splat,
                   const long long* __restrict__ totals, long long cap, int ntiles, const uint32_t* __restrict__ mat,
                   const int* __restrict__ tile_ptr, uint32_t* __restrict__ bucketed, const int* __restrict__ overflow,
                   int chunk, const int* __restrict__ tile_count) {
  pdl_wait();
  // The block's pairs are first grouped by tile in shared memory, then written out in that
  // order: every tile's pairs of this block land as one contiguous run (scattered 4-byte
  // stores cost a partial sector each).  Shared memory: per tile the running slot and the
  // global-minus-local offset, the staged ids and tiles.
  extern __shared__ uint32_t sm[];
  uint32_t* lcur = sm;
  uint32_t* gdel = sm + ntiles;
  uint32_t* sspl = sm + 2 * ntiles;
  uint16_t* stile = reinterpret_cast<uint16_t*>(sspl + chunk);
  __shared__ long long wsum[32], tot;
  if (*overflow) return;
  const long long n = min(totals[0], cap);
  const long long b0 = (long long)blockIdx.x * chunk;
  if (b0 >= n) return;
  const int nb = (int)((n + chunk - 1) / chunk);
  const int cnt = (int)(min(b0 + chunk, n) - b0);
  const int tid = threadIdx.x;
  const int per = (ntiles + 1023) / 1024;
  const int t0 = min(tid * per, ntiles), t1 = min(t0 + per, ntiles);
  const size_t row = (size_t)blockIdx.x * ntiles, next = row + ntiles;
  long long sum = 0;
  for (int t = t0; t < t1; ++t)
    sum += (blockIdx.x + 1 < nb ? mat[next + t] : (uint32_t)tile_count[t]) - mat[row + t];
  long long run = block_exscan_1024(sum, wsum, &tot);
  for (int t = t0; t < t1; ++t) {
    const uint32_t c = (blockIdx.x + 1 < nb ? mat[next + t] : (uint32_t)tile_count[t]) - mat[row + t];
    lcur[t] = (uint32_t)run;
    gdel[t] = (uint32_t)tile_ptr[t] + mat[row + t] - (uint32_t)run;
    run += c;
  }
  __syncthreads();
  for (int q = tid; q < cnt; q += 1024) {
    const uint32_t t = pair_tile[b0 + q];
    const uint32_t slot = atomicAdd(&lcur[t], 1u);
    sspl[slot] = pair_splat[b0 + q];
    stile[slot] = (uint16_t)t;
  }
  __syncthreads();
  for (int q = tid; q < cnt; q += 1024) bucketed[gdel[stile[q]] + q] = sspl[q];
}

__device__ __forceinline__ bool key_less(unsigned long long ka, uint32_t va, unsigned long long kb, uint32_t vb) {
  return ka < kb || (ka == kb && va < vb);
}

// Lanes holding the same BITS-bit digit as this lane (0 for an invalid lane): one ballot per
// bit.  (__match_any_sync iterates over the distinct values of the warp; with the ~32
// distinct digits of a sort pass it measured 57.8 -> 44.8 us for k_tile_sort at config 1.)
template <int BITS>
__device__ __forceinline__ uint32_t warp_match(uint32_t d, bool valid) {
  uint32_t m = __ballot_sync(0xffffffffu, valid);
#pragma unroll
  for (int b = 0; b < BITS; ++b) {
    const bool bit = (d >> b) & 1u;
    const uint32_t bb = __ballot_sync(0xffffffffu, bit);
    m &= bit ? bb : ~bb;
  }
  return valid ? m : 0u;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}


struct SortSmem {
  uint16_t* sk[2];  // [MAX] 16-bit keys
  uint32_t* sv[2];  // [MAX] splat ids
  uint16_t* wcnt;   // [NW][256] per-warp digit counts
  uint32_t* dtot;   // [256] digit offsets (and warp partials)
  uint32_t* red;    // [2 * NW] min / max partials
  int* bad;
};

template <int MAX, int NT>
__host__ __device__ constexpr size_t sort_smem_bytes() {
  return 2 * MAX * sizeof(uint16_t) + 2 * MAX * sizeof(uint32_t) + (NT / 32) * 256 * sizeof(uint16_t) +
         256 * sizeof(uint32_t) + 2 * (NT / 32) * sizeof(uint32_t) + 16;
}

template <int MAX, int NT>
__device__ __forceinline__ SortSmem carve_sort_smem(unsigned char* base) {
  SortSmem m;
  unsigned char* p = base;
  m.sv[0] = reinterpret_cast<uint32_t*>(p); p += MAX * 4;
  m.sv[1] = reinterpret_cast<uint32_t*>(p); p += MAX * 4;
  m.dtot = reinterpret_cast<uint32_t*>(p); p += 256 * 4;
  m.red = reinterpret_cast<uint32_t*>(p); p += 2 * (NT / 32) * 4;
  m.bad = reinterpret_cast<int*>(p); p += 16;
  m.sk[0] = reinterpret_cast<uint16_t*>(p); p += MAX * 2;
  m.sk[1] = reinterpret_cast<uint16_t*>(p); p += MAX * 2;
  m.wcnt = reinterpret_cast<uint16_t*>(p);
  return m;
}

// Per-tile ordering in shared memory.  The 32-bit key (float64 range rounded
// down to float32) is reduced to 16 bits relative to the tile's smallest key
// (monotone), sorted by two 8-bit LSD passes with warp multisplit ranking,
// and runs of equal 16-bit keys are then put in exact (float64 range, splat
// index) order by insertion sort.  One block of NT threads per tile, L <= MAX.
// Returns false (nothing written) when a run of equal keys is too long.
template <int MAX, int NT>
__device__ bool sort_tile_smem(const SortSmem& m, uint32_t* __restrict__ pairs, int lo, int L,
                               const uint32_t* __restrict__ key32, const unsigned long long* __restrict__ key64) {
  constexpr int NW = NT / 32, IPL = MAX / NT;
  static_assert(NT >= 64 && 256 % (NT < 256 ? NT : 256) == 0, "digit scan layout");
  // every buffer is shared memory: let the compiler emit LDS/STS, not generic loads
  uint16_t* const sk0 = m.sk[0];
  uint16_t* const sk1 = m.sk[1];
  uint32_t* const sv0 = m.sv[0];
  uint32_t* const sv1 = m.sv[1];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint32_t kmin = 0xffffffffu, kmax = 0u;
  uint32_t kk[IPL];
#pragma unroll
  for (int j = 0; j < IPL; ++j) {
    const int i = tid + NT * j;
    kk[j] = 0;
    if (NT * j >= L) break;
    if (i < L) {
      const uint32_t v = pairs[lo + i];
      kk[j] = key32[v];
      sv0[i] = v;
      kmin = min(kmin, kk[j]);
      kmax = max(kmax, kk[j]);
    }
  }
  for (int off = 16; off > 0; off >>= 1) {
    kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, off));
    kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, off));
  }
  if (lane == 0) {
    m.red[warp] = kmin;
    m.red[NW + warp] = kmax;
  }
  if (tid == 0) {
    m.bad[0] = 0;
    m.bad[1] = 0;  // long equal-key runs listed
    m.bad[2] = 0;  // keys of the short runs staged in shared memory
    m.bad[3] = 0;  // medium runs listed for the warps
  }
  for (int i = tid; i < 256; i += NT) m.dtot[i] = 0;  // first-digit histogram
  __syncthreads();
  for (int w = 0; w < NW; ++w) {
    kmin = min(kmin, m.red[w]);
    kmax = max(kmax, m.red[NW + w]);
  }
  const uint32_t span = kmax - kmin;
  const int shift = span >= 65536u ? (32 - __clz(span)) - 16 : 0;
  // First (low) digit: the order among equal digits is irrelevant -- the second pass is
  // stable and the tie-fix below puts equal 16-bit keys in exact order -- so shared-memory
  // atomics rank the elements (a warp-ballot ranking costs ~70 instructions per 32)
  uint32_t* const hist = m.dtot;
#pragma unroll
  for (int j = 0; j < IPL; ++j) {
    const int i = tid + NT * j;
    if (NT * j >= L) break;
    if (i < L) {
      const uint32_t k16 = (kk[j] - kmin) >> shift;
      sk0[i] = (uint16_t)k16;
      kk[j] = (k16 << 16) | atomicAdd(hist + (k16 & 0xffu), 1u);
    }
  }
  __syncthreads();
  {  // exclusive scan of the 256 digit counts, in place; thread t owns [t*DPT, (t+1)*DPT)
    constexpr int DPT = NT >= 256 ? 1 : 256 / NT;
    const bool act = tid * DPT < 256;  // warp-uniform
    uint32_t sd[DPT], tsum = 0, inc = 0;
    if (act) {
#pragma unroll
      for (int d = 0; d < DPT; ++d) {
        sd[d] = hist[tid * DPT + d];
        tsum += sd[d];
      }
      inc = tsum;
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, off);
        if (lane >= off) inc += y;
      }
      if (lane == 31) m.red[warp] = inc;
    }
    __syncthreads();
    if (act) {
      uint32_t run = inc - tsum;
      for (int w = 0; w < warp; ++w) run += m.red[w];
#pragma unroll
      for (int d = 0; d < DPT; ++d) {
        hist[tid * DPT + d] = run;
        run += sd[d];
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < IPL; ++j) {
    const int i = tid + NT * j;
    if (NT * j >= L) break;
    if (i < L) {
      const uint32_t pos = hist[(kk[j] >> 16) & 0xffu] + (kk[j] & 0xffffu);
      sk1[pos] = (uint16_t)(kk[j] >> 16);
      sv1[pos] = sv0[i];
    }
  }
  __syncthreads();
  const int seg = ((L + NT - 1) / NT) * 32;  // warp w owns [w*seg, (w+1)*seg), lane-striped
  const uint32_t lt = lanemask_lt();
  const uint32_t sspan = span >> shift;
  uint16_t* wc = m.wcnt + warp * 256;
  int cur = 1;
  for (int p = 1; p < 2; ++p) {
    const int sh = 8 * p;
    if (sspan < 256u) break;  // high digit constant
    for (int i = tid; i < NW * 256; i += NT) m.wcnt[i] = 0;
    __syncthreads();
    uint16_t lr[IPL];
    int dg[IPL];
#pragma unroll
    for (int j = 0; j < IPL; ++j) {
      dg[j] = 256;
      if (j * 32 >= seg) break;  // warp-uniform
      const int idx = warp * seg + j * 32 + lane;
      const bool ok = idx < L;
      dg[j] = ok ? (int)(((cur ? sk1 : sk0)[idx] >> sh) & 0xffu) : 256;
      const uint32_t peers = warp_match<8>((uint32_t)dg[j], ok);
      const int leader = 31 - __clz(peers);
      uint16_t before = 0;
      if (dg[j] < 256) before = wc[dg[j]];
      __syncwarp();
      if (lane == leader && dg[j] < 256) wc[dg[j]] = (uint16_t)(before + __popc(peers));
      __syncwarp();
      lr[j] = (uint16_t)(before + __popc(peers & lt));
    }
    __syncthreads();
    // digit offsets: per digit, exclusive over warps (in place) and the block-wide scan of the
    // totals; thread t owns digits [t*DPT, (t+1)*DPT)
    {
      constexpr int DPT = NT >= 256 ? 1 : 256 / NT;
      const bool act = tid * DPT < 256;  // warp-uniform
      uint32_t sd[DPT], tsum = 0, inc = 0;
      if (act) {
#pragma unroll
        for (int d = 0; d < DPT; ++d) {
          const int dig = tid * DPT + d;
          uint32_t sacc = 0;
          for (int w = 0; w < NW; ++w) {
            const uint32_t c = m.wcnt[w * 256 + dig];
            m.wcnt[w * 256 + dig] = (uint16_t)sacc;
            sacc += c;
          }
          sd[d] = sacc;
          tsum += sacc;
        }
        inc = tsum;
        for (int off = 1; off < 32; off <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, inc, off);
          if (lane >= off) inc += y;
        }
        if (lane == 31) m.red[warp] = inc;
      }
      __syncthreads();
      if (act) {
        uint32_t run = inc - tsum;
        for (int w = 0; w < warp; ++w) run += m.red[w];
#pragma unroll
        for (int d = 0; d < DPT; ++d) {
          m.dtot[tid * DPT + d] = run;
          run += sd[d];
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < IPL; ++j) {
      if (j * 32 >= seg) break;
      if (dg[j] < 256) {
        const int idx = warp * seg + j * 32 + lane;
        const uint32_t pos = m.dtot[dg[j]] + wc[dg[j]] + lr[j];
        (cur ? sk0 : sk1)[pos] = (cur ? sk1 : sk0)[idx];
        (cur ? sv0 : sv1)[pos] = (cur ? sv1 : sv0)[idx];
      }
    }
    __syncthreads();
    cur ^= 1;
  }
  // exact (float64, index) order inside runs of equal sort keys: short runs by one
  // thread's insertion sort, longer ones (duplicated splats: maps merged from the same
  // keyframes) listed and then bitonic-sorted by the whole block below
  const uint16_t* K = cur ? sk1 : sk0;
  uint32_t* V = cur ? sv1 : sv0;
  int* runs = reinterpret_cast<int*>(m.dtot);  // (free after the digit passes) [2 * kMaxLongRuns]
  unsigned long long* kbuf = reinterpret_cast<unsigned long long*>(cur ? sv0 : sv1);  // free: MAX / 2 keys
  uint32_t* wruns = reinterpret_cast<uint32_t*>(cur ? sk0 : sk1);  // free: MAX / 4 (start, key offset | n)
  for (int i = tid; i < L; i += NT) {
    const uint16_t k = K[i];
    if (i > 0 && K[i - 1] == k) continue;
    if (i + 1 >= L || K[i + 1] != k) continue;
    int j = i + 1;
    while (j < L && K[j] == k) ++j;
    if (j - i > kMaxTieRun) {
      const int r = atomicAdd(m.bad + 1, 1);
      if (r < kMaxLongRuns) {
        runs[2 * r] = i;
        runs[2 * r + 1] = j;
      } else {
        *m.bad = 1;
      }
      continue;
    }
    // the run's float64 keys first go to a free buffer with independent loads, so the
    // insertion sort compares in shared memory instead of a chain of dependent L2 loads
    const int n = j - i;
    const int off = n >= SS_TIE_STAGE ? atomicAdd(m.bad + 2, n) : MAX;
    if (off + n <= MAX / 2) {
      unsigned long long* kr = kbuf + off;
      int x = 0;
      for (; x + 4 <= n; x += 4) {
        const unsigned long long a0 = key64[V[i + x]], a1 = key64[V[i + x + 1]];
        const unsigned long long a2 = key64[V[i + x + 2]], a3 = key64[V[i + x + 3]];
        kr[x] = a0;
        kr[x + 1] = a1;
        kr[x + 2] = a2;
        kr[x + 3] = a3;
      }
      for (; x < n; ++x) kr[x] = key64[V[i + x]];
      if (n > kThreadTieRun) {  // ranked by a warp after the barrier
        const int q = atomicAdd(m.bad + 3, 1);
        if (q < MAX / 4) {
          wruns[2 * q] = (uint32_t)i;
          wruns[2 * q + 1] = (uint32_t)off | ((uint32_t)n << 24);
          continue;
        }
      }
      uint32_t* Vr = V + i;
      for (int x2 = 1; x2 < n; ++x2) {
        const uint32_t v = Vr[x2];
        const unsigned long long kv = kr[x2];
        int y = x2 - 1;
        while (y >= 0) {
          const uint32_t w = Vr[y];
          const unsigned long long kw = kr[y];
          if (key_less(kw, w, kv, v)) break;
          Vr[y + 1] = w;
          kr[y + 1] = kw;
          --y;
        }
        Vr[y + 1] = v;
        kr[y + 1] = kv;
      }
      continue;
    }
    for (int x = i + 1; x < j; ++x) {
      const uint32_t v = V[x];
      const unsigned long long kv = key64[v];
      int y = x - 1;
      while (y >= i) {
        const uint32_t w = V[y];
        if (key_less(key64[w], w, kv, v)) break;
        V[y + 1] = w;
        --y;
      }
      V[y + 1] = v;
    }
  }
  __syncthreads();
  // medium runs (kThreadTieRun < n <= kMaxTieRun): one warp per run, each element's position is
  // the number of (key, id) pairs of the run below its own, read from the staged keys
  {
    const int nw = min(m.bad[3], MAX / 4);
    for (int q = warp; q < nw; q += NW) {
      const int i = (int)wruns[2 * q];
      const int off = (int)(wruns[2 * q + 1] & 0xffffffu), n = (int)(wruns[2 * q + 1] >> 24);
      const unsigned long long* kr = kbuf + off;
      uint32_t* Vr = V + i;
      const bool h0 = lane < n, h1 = lane + 32 < n;
      const uint32_t v0 = h0 ? Vr[lane] : 0u, v1 = h1 ? Vr[lane + 32] : 0u;
      const unsigned long long k0 = h0 ? kr[lane] : 0ull, k1 = h1 ? kr[lane + 32] : 0ull;
      int r0 = 0, r1 = 0;
      for (int y = 0; y < n; ++y) {
        const unsigned long long ky = kr[y];
        const uint32_t vy = Vr[y];
        r0 += key_less(ky, vy, k0, v0);
        r1 += key_less(ky, vy, k1, v1);
      }
      __syncwarp();
      if (h0) Vr[r0] = v0;
      if (h1) Vr[r1] = v1;
      __syncwarp();
    }
  }
  __syncthreads();
  // long runs: a block bitonic sort by (float64 range bits, id), the bits as two 32-bit
  // halves in buffers the digit passes no longer use, the ids in place; the "flip" form
  // of the network keeps every minimum at the lower index, so the power-of-two padding
  // can stay virtual (+inf, never compared)
  const int nruns = min(m.bad[1], kMaxLongRuns);
  if (nruns > 0 && !*m.bad) {
    uint32_t* khi = cur ? sv0 : sv1;
    uint32_t* klo = reinterpret_cast<uint32_t*>(m.sk[0]);  // sk[0] | sk[1]: MAX x 4 bytes
    for (int r = 0; r < nruns; ++r) {
      const int i0 = runs[2 * r], n = runs[2 * r + 1] - i0;
      uint32_t* Vr = V + i0;
      int P = 1;
      while (P < n) P <<= 1;
      for (int x = tid; x < n; x += NT) {
        const unsigned long long k = key64[Vr[x]];
        khi[x] = (uint32_t)(k >> 32);
        klo[x] = (uint32_t)k;
      }
      __syncthreads();
      auto ce = [&](int x, int y) {  // x < y < n: the smaller (bits, id) to x
        const unsigned long long a = ((unsigned long long)khi[x] << 32) | klo[x];
        const unsigned long long b2 = ((unsigned long long)khi[y] << 32) | klo[y];
        const uint32_t va = Vr[x], vb = Vr[y];
        if (a > b2 || (a == b2 && va > vb)) {
          khi[x] = (uint32_t)(b2 >> 32);
          klo[x] = (uint32_t)b2;
          Vr[x] = vb;
          khi[y] = (uint32_t)(a >> 32);
          klo[y] = (uint32_t)a;
          Vr[y] = va;
        }
      };
      for (int kk = 2; kk <= P; kk <<= 1) {
        for (int x = tid; x < P; x += NT) {  // flip: x against its mirror in the kk-block
          const int y = x ^ (kk - 1);
          if (y > x && y < n) ce(x, y);
        }
        __syncthreads();
        for (int jj = kk >> 2; jj > 0; jj >>= 1) {
          for (int x = tid; x < P; x += NT) {
            const int y = x ^ jj;
            if (y > x && y < n) ce(x, y);
          }
          __syncthreads();
        }
      }
    }
  }
  const bool ok = !*m.bad;
  if (ok)
    for (int i = tid; i < L; i += NT) pairs[lo + i] = V[i];
  __syncthreads();
  return ok;
}

// Regular tiles (L <= kTileSortMax), one 256-thread block per tile; longer
// lists are sorted by k_tile_sort_big on a side stream at the same time.  A
// tile whose shared-memory sort gives up (a long run of equal keys) is merge
// sorted in place by the same block (tmp: scratch of the list's size).
// Block size: 128 threads when tiles are many (short lists: more blocks per SM hide the
// sort's barriers; config 1 63 -> 59 us), 256 when they are few and long (config 2:
// 60 us against 67 with 128).

__device__ void merge_sort_tile(uint32_t* __restrict__ pairs, uint32_t* __restrict__ tmp, int lo, int L,
                                const unsigned long long* __restrict__ key);

template <int NT>
__global__ void __launch_bounds__(NT) k_tile_sort(const int* __restrict__ tile_ptr, uint32_t* __restrict__ pairs,
                                                   uint32_t* __restrict__ tmp, const uint32_t* __restrict__ key32,
                                                   const unsigned long long* __restrict__ key64,
                                                   const int* __restrict__ overflow) {
  pdl_wait();
  __shared__ __align__(16) unsigned char smem[sort_smem_bytes<kTileSortMax, NT>()];
  if (*overflow) return;
  const int t = blockIdx.x;
  const int lo = tile_ptr[t], L = tile_ptr[t + 1] - lo;
  if (L <= 1 || L > kTileSortMax) return;  // (longer lists: k_scan_tiles listed them for the big sort)
  const SortSmem m = carve_sort_smem<kTileSortMax, NT>(smem);
  if (!sort_tile_smem<kTileSortMax, NT>(m, pairs, lo, L, key32, key64)) {
#ifdef SS_DBG_FALLBACK
    if (threadIdx.x == 0) printf("merge-sort fallback: tile %d, list %d\n", t, L);
#endif
    merge_sort_tile(pairs, tmp, lo, L, key64);  // long run of equal keys (block-uniform result)
  }
}

__device__ int count_less(const uint32_t* run, int len, const unsigned long long* key, unsigned long long k,
                          uint32_t v) {
  int lo = 0, hi = len;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    const uint32_t w = run[mid];
    if (key_less(key[w], w, k, v))
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// Fallback for lists longer than kTileSortBig (or with a long run of equal
// sort keys): bottom-up merge sort in global memory by the exact (float64
// range, index) key, by the whole block.
__device__ void merge_sort_tile(uint32_t* __restrict__ pairs, uint32_t* __restrict__ tmp, int lo, int L,
                                const unsigned long long* __restrict__ key) {
  uint32_t* src = pairs + lo;
  uint32_t* dst = tmp + lo;
  for (int w = 1; w < L; w <<= 1) {
    for (int i = threadIdx.x; i < L; i += blockDim.x) {
      const int start = (i / (2 * w)) * (2 * w);
      const int mid = min(start + w, L), end = min(start + 2 * w, L);
      const uint32_t v = src[i];
      const unsigned long long k = key[v];
      int pos;
      if (i < mid)
        pos = (i - start) + count_less(src + mid, end - mid, key, k, v);
      else
        pos = (i - mid) + count_less(src + start, mid - start, key, k, v);
      dst[start + pos] = v;
    }
    __syncthreads();
    uint32_t* s = src;
    src = dst;
    dst = s;
  }
  if (src != pairs + lo)
    for (int i = threadIdx.x; i < L; i += blockDim.x) pairs[lo + i] = src[i];
  __syncthreads();
}

// Tiles k_tile_sort handed over (long_list): lists of up to kTileSortBig
// entries sorted in shared memory by a 1024-thread block, anything else by
// the global merge sort.
// Lists longer than kTileSortMax (listed by k_scan_tiles), sorted on the side stream while
// k_tile_sort sorts the rest: in shared memory up to CAP entries -- kTileSortBig (98 KB),
// or for dense maps (see capi.cu) kTileSortHuge (214 KB: its blocks need an otherwise
// empty SM, so it is not the default) -- longer lists, and lists with more long equal-key
// runs than the shared-memory sort lists, are merge sorted in global memory.  (Config-4b map, 2 M surfels, lists up
// to ~12,800: the merge sort of its 252 lists beyond 8,192 took ~1 ms per render.)
template <int CAP>
__global__ void __launch_bounds__(1024) k_tile_sort_big(const int* __restrict__ tile_ptr, uint32_t* __restrict__ pairs,
                                                        uint32_t* __restrict__ tmp, const uint32_t* __restrict__ key32,
                                                        const unsigned long long* __restrict__ key64,
                                                        const int* __restrict__ long_list,
                                                        const int* __restrict__ n_long) {
  extern __shared__ __align__(16) unsigned char dsmem[];
  const SortSmem m = carve_sort_smem<CAP, 1024>(dsmem);
  const int nl = *n_long;
  for (int r = blockIdx.x; r < nl; r += gridDim.x) {
    const int t = long_list[r];
    const int lo = tile_ptr[t], L = tile_ptr[t + 1] - lo;
    bool ok = false;
    if (L <= CAP) ok = sort_tile_smem<CAP, 1024>(m, pairs, lo, L, key32, key64);
#ifdef SS_DBG_FALLBACK
    if (!ok && threadIdx.x == 0) printf("merge-sort fallback: tile %d, list %d\n", t, L);
#endif
    if (!ok) merge_sort_tile(pairs, tmp, lo, L, key64);
  }
}

// Tile processing order for the blend kernels: longest lists first (the
// kernels fetch tiles dynamically, so this is longest-processing-time-first
// scheduling).  Counting sort on min(L, 4095) / 4, one block.
// Work slots of the blend kernels ((tile << 2) | part, see next_tile in
// blend.cu), longest lists first: order_fwd holds one slot per tile
// (counters[3] = ntiles); for the backward (order_bwd), when there are fewer
// tiles than resident warps (split_target > 0), the split_target longest
// tiles with at least 96 entries become two slots, one per pixel half
// (counters[2] = slot count).  (Splitting the forward measured slower: both
// halves re-stage every entry of the list.)
// long_target > 0: up to long_target of the longest tiles with >= long_min entries go
// to the block-per-tile forward (k_forward_long, tickets counters[4] < counters[5]);
// the warp-per-tile forward starts its tickets after them (counters[0] = nlong).
__device__ void build_seg_slots(int ntiles, const int* __restrict__ tile_ptr, const int* __restrict__ order_fwd,
                                int* __restrict__ slots, int* __restrict__ counters, int min_list);

// (seg_slots != null: also the segment-mode backward slots, with lists of >= seg_min entries
// segmented -- seg_min < 0: automatic, every list when the longest one (totals[2]) exceeds
// twice the pairs per resident blend warp (total pairs / seg_warps), else none -- and the
// threshold to counters[9])
__global__ void __launch_bounds__(1024) k_tile_order(int ntiles, const int* __restrict__ tile_ptr,
                                                     int* __restrict__ order_fwd, int* __restrict__ order,
                                                     int* __restrict__ counters, int split_target,
                                                     int long_target, int long_min, int* __restrict__ seg_slots,
                                                     int seg_min, int seg_warps,
                                                     const long long* __restrict__ totals) {
  __shared__ int hist[1024];
  const int tid = threadIdx.x;
  hist[tid] = 0;
  if (tid < 4) counters[tid] = 0;
  __syncthreads();  // (counters[0] is set to the long-tile count below, after the scan)
  for (int t = tid; t < ntiles; t += 1024) {
    const int L = max(0, tile_ptr[t + 1] - tile_ptr[t]);
    atomicAdd(&hist[1023 - (min(L, 4095) >> 2)], 1);
  }
  __syncthreads();
  // exclusive scan of hist (bucket 0 = longest)
  const int v = hist[tid];
  int inc = v;
  for (int off = 1; off < 32; off <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, inc, off);
    if ((tid & 31) >= off) inc += y;
  }
  __shared__ int wsum[32];
  if ((tid & 31) == 31) wsum[tid >> 5] = inc;
  __syncthreads();
  int wex = 0;
  for (int w = 0; w < (tid >> 5); ++w) wex += wsum[w];
  __syncthreads();
  hist[tid] = wex + inc - v;
  __syncthreads();
  // tiles of >= 96 entries occupy the buckets 0 .. 1023 - 24 (bucket = 1023 - min(L, 4095) / 4)
  __shared__ int s_nsplit;
  if (tid == 0) {
    const int n96 = hist[1023 - 23];  // exclusive prefix: tiles in buckets < 1000, i.e. L >= 96
    s_nsplit = min(split_target, n96);
    // L >= 4 k4 with k4 = ceil(long_min / 4) clamped to [1, 1023]: exclusive prefix hist[1024 - k4]
    const int k4 = min(max((long_min + 3) >> 2, 1), 1023);
    const int n768 = long_min <= 0 ? ntiles : hist[1024 - k4];
    const int nlong = min(long_target, n768);
    counters[0] = nlong;
    counters[4] = 0;
    counters[5] = nlong;
  }
  __syncthreads();
  const int nsplit = s_nsplit;
  for (int t = tid; t < ntiles; t += 1024) {
    const int L = max(0, tile_ptr[t + 1] - tile_ptr[t]);
    const int r = atomicAdd(&hist[1023 - (min(L, 4095) >> 2)], 1);  // LPT rank
    order_fwd[r] = t << 2;
    if (r < nsplit) {
      order[2 * r] = (t << 2) | 1;
      order[2 * r + 1] = (t << 2) | 2;
    } else {
      order[nsplit + r] = t << 2;
    }
  }
  if (tid == 0) {
    counters[2] = ntiles + nsplit;
    counters[3] = ntiles;
  }
  if (seg_slots) {
    int mn = seg_min;
    if (mn < 0) {  // automatic: segments everywhere when the longest list exceeds twice a warp's fair share
      const long long fair = totals[0] / max(seg_warps, 1);
      mn = totals[2] > 2 * fair ? 0 : 0x7fffffff;
    }
    if (tid == 0) counters[9] = mn;
    __syncthreads();  // (order_fwd complete)
    if (mn == 0x7fffffff) {  // whole-tile slots in LPT order
      for (int r = tid; r < ntiles; r += 1024) seg_slots[r] = ((order_fwd[r] >> 2) << 16) | 0xffff;
      if (tid == 0) counters[2] = ntiles;
    } else {
      build_seg_slots(ntiles, tile_ptr, order_fwd, seg_slots, counters, mn);
    }
  }
}

__global__ void k_widen_i32(int n, const int* __restrict__ in, long long* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[i];
}

}  // namespace ss
