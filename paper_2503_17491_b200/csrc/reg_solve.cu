// Device-resident Gauss-Newton / Levenberg loop: the whole register()
// iteration of the reference (registration.py:387-524) -- photometric,
// geometric, joint and sequential modes -- in ONE cooperative kernel, so no
// evaluation round-trips to the host.
//
//   per evaluation (pose P, trim floors, objective-only flag), per residual
//   family of the current phase:
//     geometric: k nearest usable leaf centroids within assoc_gate (brute
//        force over the leaves in shared memory), the leaf whose plane is
//        closest, point-to-plane residual            (_geo_system, :231-274)
//     photometric: residuals of every anchor        (_photo_system, :324-340)
//     exact median of |r| over the valid ones   (np.median, :343): radix
//        select on the float64 bit patterns, 12-bit digits, grid-wide
//        shared-memory histograms merged into global ones (6 passes)
//     trim, Huber weights, 6x6 normal equations (:342-361, :219-228, :470-477)
//        reduced per block, summed by block 0 in block order (deterministic)
//   block 0, one thread, then runs the LM state machine exactly as the
//   reference: solve (H + lam I) delta = -b by LU with partial pivoting
//   (np.linalg.solve / LAPACK dgesv; an exact zero pivot is its LinAlgError),
//   the non-finite check, T_try = T exp(delta) (se3.py:121-150), accept when
//   the trial objective <= obj0 + 1e-12, lam updates, annealed trim floor,
//   convergence on |delta| < tol -- and publishes the next evaluation.
// Phases are separated by grid-wide barriers (cooperative launch, one block
// per SM).  The final SVD re-orthonormalisation stays on the host.
#include <cooperative_groups.h>

#include "registration.cu"

namespace ss {

namespace cg = cooperative_groups;

enum { RM_PHOTO = 0, RM_GEO = 1, RM_JOINT = 2, RM_SEQ = 3 };

struct RegSolveCfg {
  double huber_photo, huber_geo, trim_factor, spread_gate, assoc_gate, floor_photo, floor_geo, tol, damping_init,
      damping_max;
  int max_iters, min_residuals, assoc_k, mode;
};

constexpr int kRsThreads = 256;
constexpr int kRsBins = 4096;  // 12-bit digits
constexpr int kRsPasses = 6;   // bits 63-52, 51-40, 39-28, 27-16, 15-4, 3-0
constexpr int kRsCand = 256;   // a selected bin this small is finished by an exact in-block rank
constexpr int kRsAcc = 32;     // per family: [0:21] H upper, [21:27] b, [27] Huber(huber_geo),
                               // [28] m, [29] sum r^2, [30] Huber(huber_photo)
constexpr int kRsLeafChunk = 256;

enum { RS_EVAL = 0, RS_DONE = 1 };

struct RegSolveState {
  // published evaluation
  double P[12];
  double fg, fp;
  int objective_only, action, eval_geo, eval_photo;
  // LM state (block 0, thread 0)
  double T[12], Ttry[12], H[36], b[6], delta[6];
  double lam, obj0, term_hub[2], term_s[2];
  double last_r2[2];
  int last_m[2], nterms;
  int it_total, converged, status, stage, n_eval, phase, use_geo, use_photo;
  unsigned long long vmin[2][2];
  int ncand[2][2];
  unsigned long long cand[2][2][kRsCand];
};

struct GeoTmp {
  double r, n[3], q[3];
};

__device__ void so3_exp_d(const double* phi, double* R) {
  const double ang = sqrt(phi[0] * phi[0] + phi[1] * phi[1] + phi[2] * phi[2]);
  const double K[9] = {0.0, -phi[2], phi[1], phi[2], 0.0, -phi[0], -phi[1], phi[0], 0.0};
  double K2[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) K2[3 * i + j] = K[3 * i] * K[j] + K[3 * i + 1] * K[3 + j] + K[3 * i + 2] * K[6 + j];
  double a, c;
  if (ang < 1e-8) {
    a = 1.0;
    c = 0.5;
  } else {
    a = sin(ang) / ang;
    c = (1.0 - cos(ang)) / (ang * ang);
  }
  for (int q = 0; q < 9; ++q) R[q] = (q % 4 == 0 ? 1.0 : 0.0) + a * K[q] + c * K2[q];
}

__device__ void left_jacobian_d(const double* phi, double* J) {
  const double ang = sqrt(phi[0] * phi[0] + phi[1] * phi[1] + phi[2] * phi[2]);
  const double K[9] = {0.0, -phi[2], phi[1], phi[2], 0.0, -phi[0], -phi[1], phi[0], 0.0};
  double K2[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) K2[3 * i + j] = K[3 * i] * K[j] + K[3 * i + 1] * K[3 + j] + K[3 * i + 2] * K[6 + j];
  double b, c;
  if (ang < 1e-8) {
    b = 0.5;
    c = 1.0 / 6.0;
  } else {
    const double a2 = ang * ang;
    b = (1.0 - cos(ang)) / a2;
    c = (ang - sin(ang)) / (a2 * ang);
  }
  for (int q = 0; q < 9; ++q) J[q] = (q % 4 == 0 ? 1.0 : 0.0) + b * K[q] + c * K2[q];
}

// T * exp(delta), delta = (rho, phi) (se3.py:121-123, 144-150)
__device__ void retract_d(const double* T, const double* delta, double* out) {
  double Re[9], J[9], te[3];
  so3_exp_d(delta + 3, Re);
  left_jacobian_d(delta + 3, J);
  for (int i = 0; i < 3; ++i) te[i] = J[3 * i] * delta[0] + J[3 * i + 1] * delta[1] + J[3 * i + 2] * delta[2];
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j) out[3 * i + j] = T[3 * i] * Re[j] + T[3 * i + 1] * Re[3 + j] + T[3 * i + 2] * Re[6 + j];
    out[9 + i] = T[3 * i] * te[0] + T[3 * i + 1] * te[1] + T[3 * i + 2] * te[2] + T[9 + i];
  }
}

// Solve A x = y (6x6, row-major) by LU with partial pivoting; false on an
// exact zero pivot (LAPACK dgesv's singular case, numpy's LinAlgError).
__device__ bool solve6(double* A, double* y) {
  for (int k = 0; k < 6; ++k) {
    int p = k;
    double best = fabs(A[6 * k + k]);
    for (int i = k + 1; i < 6; ++i)
      if (fabs(A[6 * i + k]) > best) {
        best = fabs(A[6 * i + k]);
        p = i;
      }
    if (A[6 * p + k] == 0.0) return false;
    if (p != k) {
      for (int j = 0; j < 6; ++j) {
        const double t = A[6 * k + j];
        A[6 * k + j] = A[6 * p + j];
        A[6 * p + j] = t;
      }
      const double t = y[k];
      y[k] = y[p];
      y[p] = t;
    }
    const double inv = 1.0 / A[6 * k + k];
    for (int i = k + 1; i < 6; ++i) {
      const double l = A[6 * i + k] * inv;
      A[6 * i + k] = l;
      for (int j = k + 1; j < 6; ++j) A[6 * i + j] -= l * A[6 * k + j];
      y[i] -= l * y[k];
    }
  }
  for (int k = 5; k >= 0; --k) {
    double s = y[k];
    for (int j = k + 1; j < 6; ++j) s -= A[6 * k + j] * y[j];
    y[k] = s / A[6 * k + k];
  }
  return true;
}

__device__ int rs_phase_mode(const RegSolveCfg& cfg, int phase) {
  if (cfg.mode == RM_SEQ) return phase == 0 ? RM_GEO : RM_JOINT;
  return cfg.mode;
}
__device__ int rs_phase_budget(const RegSolveCfg& cfg, int phase) {
  if (cfg.mode == RM_SEQ) return phase == 0 ? cfg.max_iters / 2 : cfg.max_iters;
  return cfg.max_iters;
}
__device__ int rs_nphases(const RegSolveCfg& cfg) { return cfg.mode == RM_SEQ ? 2 : 1; }

__device__ void rs_begin_iteration(RegSolveState* st, const RegSolveCfg& cfg);

// Start phase `ph` (registration.py:441-450): damping and convergence reset.
__device__ void rs_begin_phase(RegSolveState* st, const RegSolveCfg& cfg, int ph) {
  if (ph >= rs_nphases(cfg)) {
    st->action = RS_DONE;
    return;
  }
  st->phase = ph;
  const int m = rs_phase_mode(cfg, ph);
  st->use_geo = m == RM_GEO || m == RM_JOINT;
  st->use_photo = m == RM_PHOTO || m == RM_JOINT;
  st->lam = cfg.damping_init;
  st->converged = 0;
  rs_begin_iteration(st, cfg);
}

// Next outer iteration of the phase (or the next phase): a full evaluation at T.
__device__ void rs_begin_iteration(RegSolveState* st, const RegSolveCfg& cfg) {
  if (st->it_total >= rs_phase_budget(cfg, st->phase)) {
    rs_begin_phase(st, cfg, st->phase + 1);
    return;
  }
  st->it_total += 1;
  const double anneal = cfg.assoc_gate * pow(0.5, (double)st->it_total);
  st->fg = fmax(cfg.floor_geo, anneal);
  st->fp = fmax(cfg.floor_photo, anneal);
  for (int q = 0; q < 12; ++q) st->P[q] = st->T[q];
  st->objective_only = 0;
  st->eval_geo = st->use_geo;
  st->eval_photo = st->use_photo;
  st->stage = 0;
  st->action = RS_EVAL;
}

// Inner LM loop: next trial pose, or the end of the phase when damping is exhausted.
__device__ void rs_try(RegSolveState* st, const RegSolveCfg& cfg) {
  while (st->lam <= cfg.damping_max) {
    double A[36], y[6];
    for (int q = 0; q < 36; ++q) A[q] = st->H[q] + (q % 7 == 0 ? st->lam : 0.0);
    for (int q = 0; q < 6; ++q) y[q] = -st->b[q];
    bool ok = solve6(A, y);
    for (int q = 0; q < 6 && ok; ++q) ok = isfinite(y[q]);
    if (!ok) {
      st->lam = fmax(st->lam, 1e-8) * 10.0;
      continue;
    }
    for (int q = 0; q < 6; ++q) st->delta[q] = y[q];
    retract_d(st->T, st->delta, st->Ttry);
    for (int q = 0; q < 12; ++q) st->P[q] = st->Ttry[q];
    st->objective_only = 1;
    st->stage = 1;
    st->action = RS_EVAL;
    return;
  }
  rs_begin_phase(st, cfg, st->phase + 1);  // damping exhausted: keep the estimate, end the phase
}

// red: per family (geo, photo) kRsAcc sums of the evaluation just finished.
__device__ void rs_step(RegSolveState* st, const RegSolveCfg& cfg, const double* red) {
  st->n_eval += 1;
  const double* fam[2] = {red, red + kRsAcc};
  const int on[2] = {st->eval_geo, st->eval_photo};
  const double hub_par[2] = {cfg.huber_geo, cfg.huber_photo};
  if (st->stage == 0) {
    for (int q = 0; q < 36; ++q) st->H[q] = 0.0;
    for (int q = 0; q < 6; ++q) st->b[q] = 0.0;
    st->nterms = 0;
    int n_tot = 0;
    double obj0 = 0.0;
    for (int f = 0; f < 2; ++f) {
      const int m = on[f] ? (int)llrint(fam[f][28]) : 0;
      if (m == 0) continue;  // _geo_system / _photo_system returned None
      const double s = 1.0 / m;
      int k = 0;
      for (int a = 0; a < 6; ++a)
        for (int b = a; b < 6; ++b) {
          st->H[6 * a + b] += s * fam[f][k];
          if (b != a) st->H[6 * b + a] += s * fam[f][k];
          ++k;
        }
      for (int a = 0; a < 6; ++a) st->b[a] += s * fam[f][21 + a];
      st->term_hub[st->nterms] = hub_par[f];
      st->term_s[st->nterms] = s;
      st->nterms += 1;
      obj0 += s * fam[f][f == 0 ? 27 : 30];
      st->last_r2[f] = fam[f][29];
      st->last_m[f] = m;
      n_tot += m;
    }
    if (n_tot < cfg.min_residuals) {
      st->status = 1;  // RegistrationError: too few residuals survive association
      st->action = RS_DONE;
      return;
    }
    st->obj0 = obj0;
    rs_try(st, cfg);
    return;
  }
  // trial at Ttry: families that returned a system, paired POSITIONALLY with the
  // frozen terms (registration.py:379-384, 497-504)
  int nt = 0;
  double obj = 0.0;
  for (int f = 0; f < 2; ++f) {
    const int m = on[f] ? (int)llrint(fam[f][28]) : 0;
    if (m == 0) continue;
    if (nt < st->nterms) {
      const double hv = st->term_hub[nt] == cfg.huber_geo ? fam[f][27] : fam[f][30];
      obj += st->term_s[nt] * hv;
    }
    ++nt;
  }
  if (nt > 0 && obj <= st->obj0 + 1e-12) {
    for (int q = 0; q < 12; ++q) st->T[q] = st->Ttry[q];
    st->lam = fmax(st->lam * 0.25, cfg.damping_init);
    const double dn = sqrt(st->delta[0] * st->delta[0] + st->delta[1] * st->delta[1] + st->delta[2] * st->delta[2] +
                           st->delta[3] * st->delta[3] + st->delta[4] * st->delta[4] + st->delta[5] * st->delta[5]);
    if (dn < cfg.tol) {
      st->converged = 1;
      rs_begin_phase(st, cfg, st->phase + 1);
      return;
    }
    rs_begin_iteration(st, cfg);
    return;
  }
  st->lam = fmax(st->lam, 1e-8) * 10.0;
  rs_try(st, cfg);
}

// Block-wide: find the bin of hist[0, nbins) holding rank kk; returns (bin, count before it).
__device__ void rs_find_bin(const unsigned* __restrict__ hist, int nbins, int kk, int* s_bin, int* s_before,
                            unsigned* s_part) {
  constexpr int per = kRsBins / kRsThreads;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  unsigned loc[per];
  unsigned sum = 0;
#pragma unroll
  for (int j = 0; j < per; ++j) {
    const int bin = tid * per + j;
    loc[j] = bin < nbins ? hist[bin] : 0u;
    sum += loc[j];
  }
  unsigned inc = sum;
  for (int off = 1; off < 32; off <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, inc, off);
    if (lane >= off) inc += y;
  }
  if (lane == 31) s_part[warp] = inc;
  __syncthreads();
  unsigned wex = 0;
  for (int w = 0; w < warp; ++w) wex += s_part[w];
  unsigned run = wex + inc - sum;
  if ((unsigned)kk >= run && (unsigned)kk < run + sum) {
#pragma unroll
    for (int j = 0; j < per; ++j) {
      if ((unsigned)kk < run + loc[j]) {
        *s_bin = tid * per + j;
        *s_before = (int)run;
        break;
      }
      run += loc[j];
    }
  }
  __syncthreads();
}

// Huber weight and the two Huber values (deltas huber_geo, huber_photo) of one kept residual
__device__ __forceinline__ double hub_value(double r, double d) {
  const double a = fabs(r);
  return a <= d ? 0.5 * r * r : d * (a - 0.5 * d);
}

// Grid-wide exact median of the valid |r| patterns in bits[0, n) (np.median).
// m: number of valid entries (> 0).  Hc: this evaluation's kRsPasses x kRsBins
// histograms (zeroed); cand / ncand / vmin: this evaluation's scratch.
__device__ double rs_median(cg::grid_group& grid, const unsigned long long* __restrict__ bits, int n, int m,
                            unsigned* __restrict__ Hc, unsigned long long* cand, int* ncand,
                            unsigned long long* vmin, unsigned* sh, unsigned* s_part, int* s_bin, int* s_before,
                            unsigned long long* s_min) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gtid = blockIdx.x * kRsThreads + tid, nthr = gridDim.x * kRsThreads;
  const int k1 = (m % 2 == 0) ? m / 2 - 1 : m / 2;
  unsigned long long prefix = 0ull, mask = 0ull;
  int kk = k1, cnt_eq = 0;
  bool exact = false;
  unsigned long long v2c = ~0ull;
  for (int p = 0; p < kRsPasses; ++p) {
    const int shift = p < 5 ? 52 - 12 * p : 0;
    const int nb = p < 5 ? 12 : 4;
    const unsigned dmask = (1u << nb) - 1u;
    for (int j = tid; j < kRsBins; j += kRsThreads) sh[j] = 0u;
    __syncthreads();
    for (int i = gtid; i < n; i += nthr) {
      const unsigned long long b = bits[i];
      if (b != ~0ull && (b & mask) == prefix) atomicAdd(&sh[(unsigned)(b >> shift) & dmask], 1u);
    }
    __syncthreads();
    unsigned* Hp = Hc + p * kRsBins;
    for (int j = tid; j <= (int)dmask; j += kRsThreads)
      if (sh[j]) atomicAdd(&Hp[j], sh[j]);
    grid.sync();
    rs_find_bin(Hp, (int)dmask + 1, kk, s_bin, s_before, s_part);
    const int bin = *s_bin;
    kk -= *s_before;
    const int cnt_bin = (int)Hp[bin];
    if (p == kRsPasses - 1) cnt_eq = cnt_bin;
    prefix |= (unsigned long long)bin << shift;
    mask |= (unsigned long long)dmask << shift;
    __syncthreads();
    if (p == kRsPasses - 1) {
      exact = true;
      break;
    }
    if (cnt_bin <= kRsCand) {
      // few values share the prefix: gather them and rank them exactly in every block
      for (int i = gtid; i < n; i += nthr) {
        const unsigned long long b = bits[i];
        if (b != ~0ull && (b & mask) == prefix) cand[atomicAdd(ncand, 1)] = b;
      }
      grid.sync();
      unsigned long long* sc = reinterpret_cast<unsigned long long*>(sh);  // kRsCand x 8 B fits
      for (int j = tid; j < cnt_bin; j += kRsThreads) sc[j] = ((volatile unsigned long long*)cand)[j];
      __syncthreads();
      for (int j = tid; j < cnt_bin; j += kRsThreads) {
        const unsigned long long c = sc[j];
        int lt = 0, eqb = 0;
        for (int q = 0; q < cnt_bin; ++q) {
          lt += sc[q] < c;
          eqb += (sc[q] == c) & (q < j);
        }
        const int rank = lt + eqb;  // distinct ranks 0..cnt_bin-1
        if (rank == kk) sh[2 * kRsCand] = (unsigned)j;
        if (rank == kk + 1) sh[2 * kRsCand + 1] = (unsigned)j;
      }
      if (tid == 0 && kk + 1 >= cnt_bin) sh[2 * kRsCand + 1] = 0xffffffffu;
      __syncthreads();
      prefix = sc[sh[2 * kRsCand]];
      const unsigned j2 = sh[2 * kRsCand + 1];
      v2c = j2 == 0xffffffffu ? ~0ull : sc[j2];
      __syncthreads();
      break;
    }
  }
  const double v1 = __longlong_as_double((long long)prefix);
  if (m % 2 != 0) return v1;
  // the next order statistic: v1 again if it repeats, else the smallest larger value
  if (!exact && v2c != ~0ull) return (v1 + __longlong_as_double((long long)v2c)) / 2.0;
  if (exact && k1 + 1 < (k1 - kk) + cnt_eq) return v1;
  unsigned long long mn = ~0ull;
  for (int i = gtid; i < n; i += nthr) {
    const unsigned long long b = bits[i];
    if (b != ~0ull && b > prefix) mn = min(mn, b);
  }
  for (int off = 16; off > 0; off >>= 1) mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, off));
  if (lane == 0) s_min[warp] = mn;
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < kRsThreads / 32; ++w) mn = min(mn, s_min[w]);
    if (mn != ~0ull) atomicMin(vmin, mn);
  }
  grid.sync();
  return (v1 + __longlong_as_double((long long)*((volatile unsigned long long*)vmin))) / 2.0;
}

// Block count of valid entries -> grid total (pcnt: per-block slots).
__device__ int rs_count(cg::grid_group& grid, int okc, int* __restrict__ pcnt, unsigned* s_part, int* s_m) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  okc = __reduce_add_sync(0xffffffffu, okc);
  if (lane == 0) s_part[warp] = (unsigned)okc;
  __syncthreads();
  if (tid == 0) {
    int c = 0;
    for (int w = 0; w < kRsThreads / 32; ++w) c += (int)s_part[w];
    pcnt[blockIdx.x] = c;
  }
  grid.sync();
  if (tid < 32) {
    int c = 0;
    for (int b = lane; b < (int)gridDim.x; b += 32) c += pcnt[b];
    c = __reduce_add_sync(0xffffffffu, c);
    if (lane == 0) *s_m = c;
  }
  __syncthreads();
  return *s_m;
}

struct RsGeo {  // geometric inputs: usable leaves and the (subsampled) scan, sensor frame
  const double* cent;
  const double* nrm;
  int n_leaves;
  const double* scan;
  int n_scan;
};
struct RsPhoto {  // photometric inputs: world anchors and the scan range image
  const double* X;
  int M;
  const double* srange;
  const uint8_t* svalid;
};

__global__ void __launch_bounds__(kRsThreads) k_reg_solve(RsGeo geo, RsPhoto ph, RegCam cam, RegSolveCfg cfg,
                                                         GeoTmp* __restrict__ gtmp, PhotoTmp* __restrict__ ptmp,
                                                         unsigned long long* __restrict__ gbits,
                                                         unsigned long long* __restrict__ pbits,
                                                         unsigned* __restrict__ hist, double* __restrict__ part,
                                                         int* __restrict__ pcnt, RegSolveState* st) {
  cg::grid_group grid = cg::this_grid();
  __shared__ unsigned sh[kRsBins];
  __shared__ double sred[kRsThreads / 32][kRsAcc];
  __shared__ double sfin[2 * kRsAcc];
  __shared__ double s_lc[3 * kRsLeafChunk], s_ln[3 * kRsLeafChunk];
  __shared__ unsigned s_part[kRsThreads / 32];
  __shared__ int s_bin, s_before, s_m;
  __shared__ unsigned long long s_min[kRsThreads / 32];
  const int G = gridDim.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gtid = blockIdx.x * kRsThreads + tid, nthr = G * kRsThreads;
  const int kmax = min(min(cfg.assoc_k, geo.n_leaves), 8);
  if (blockIdx.x == 0 && tid == 0) {
    st->it_total = 0;
    st->status = 0;
    st->n_eval = 0;
    st->last_m[0] = st->last_m[1] = 0;
    st->last_r2[0] = st->last_r2[1] = 0.0;
    for (int a = 0; a < 2; ++a)
      for (int f = 0; f < 2; ++f) {
        st->vmin[a][f] = ~0ull;
        st->ncand[a][f] = 0;
      }
    rs_begin_phase(st, cfg, 0);
  }
  for (int e = 0;; ++e) {
    grid.sync();
    volatile RegSolveState* vs = st;
    if (vs->action == RS_DONE) break;
    PoseK P;
    for (int q = 0; q < 9; ++q) P.R[q] = vs->P[q];
    for (int q = 0; q < 3; ++q) P.t[q] = vs->P[9 + q];
    const double fgeo = vs->fg, fph = vs->fp;
    const int objective_only = vs->objective_only;
    const int fam_on[2] = {vs->eval_geo && geo.n_leaves > 0, vs->eval_photo};
    const int par = e & 1;
    // zero the next evaluation's scratch
    unsigned* Hnext = hist + (size_t)(par ^ 1) * 2 * kRsPasses * kRsBins;
    for (int i = gtid; i < 2 * kRsPasses * kRsBins; i += nthr) Hnext[i] = 0u;
    if (gtid == 0)
      for (int f = 0; f < 2; ++f) {
        st->vmin[par ^ 1][f] = ~0ull;
        st->ncand[par ^ 1][f] = 0;
      }
    double acc[2][kRsAcc];
#pragma unroll
    for (int f = 0; f < 2; ++f)
#pragma unroll
      for (int q = 0; q < kRsAcc; ++q) acc[f][q] = 0.0;
    for (int f = 0; f < 2; ++f) {
      if (!fam_on[f]) continue;  // uniform across the grid
      unsigned* Hc = hist + ((size_t)par * 2 + f) * kRsPasses * kRsBins;
      unsigned long long* bits = f == 0 ? gbits : pbits;
      const int n = f == 0 ? geo.n_scan : ph.M;
      // --- residuals
      int okc = 0;
      if (f == 0) {
        // k nearest usable leaf centroids within the gate, then the leaf whose plane
        // is closest (registration.py:249-265); leaves staged through shared memory
        const int i = gtid;  // one scan point per thread (n_scan <= grid threads, checked by the host)
        double p[3] = {0, 0, 0}, q3[3] = {0, 0, 0};
        if (i < n) {
          for (int c = 0; c < 3; ++c) q3[c] = geo.scan[3 * i + c];
          for (int c = 0; c < 3; ++c)
            p[c] = P.R[3 * c] * q3[0] + P.R[3 * c + 1] * q3[1] + P.R[3 * c + 2] * q3[2] + P.t[c];
        }
        double kd[8];
        int ki[8];
        for (int a = 0; a < 8; ++a) {
          kd[a] = __longlong_as_double(0x7ff0000000000000LL);
          ki[a] = -1;
        }
        for (int c0 = 0; c0 < geo.n_leaves; c0 += kRsLeafChunk) {
          const int cn = min(kRsLeafChunk, geo.n_leaves - c0);
          __syncthreads();
          for (int j = tid; j < 3 * cn; j += kRsThreads) {
            s_lc[j] = geo.cent[3 * c0 + j];
            s_ln[j] = geo.nrm[3 * c0 + j];
          }
          __syncthreads();
          if (i < n)
            for (int j = 0; j < cn; ++j) {
              const double dx = p[0] - s_lc[3 * j], dy = p[1] - s_lc[3 * j + 1], dz = p[2] - s_lc[3 * j + 2];
              const double d2 = dx * dx + dy * dy + dz * dz;
              if (d2 < kd[kmax - 1]) {  // insertion into the sorted k best
                int a = kmax - 1;
                while (a > 0 && kd[a - 1] > d2) {
                  kd[a] = kd[a - 1];
                  ki[a] = ki[a - 1];
                  --a;
                }
                kd[a] = d2;
                ki[a] = c0 + j;
              }
            }
        }
        bool ok = false;
        GeoTmp g{};
        if (i < n) {
          const double gate2 = cfg.assoc_gate * cfg.assoc_gate;
          double best = __longlong_as_double(0x7ff0000000000000LL);
          int bl = -1;
          for (int a = 0; a < kmax; ++a) {
            if (ki[a] < 0 || !(kd[a] < gate2)) continue;  // beyond distance_upper_bound
            const double* nn = geo.nrm + 3 * ki[a];
            const double* cc = geo.cent + 3 * ki[a];
            const double pd = fabs(nn[0] * (p[0] - cc[0]) + nn[1] * (p[1] - cc[1]) + nn[2] * (p[2] - cc[2]));
            if (pd < best) {
              best = pd;
              bl = ki[a];
            }
          }
          ok = ki[0] >= 0 && kd[0] < gate2;
          if (ok) {
            const double* nn = geo.nrm + 3 * bl;
            const double* cc = geo.cent + 3 * bl;
            g.r = (nn[0] * (p[0] - cc[0]) + nn[1] * (p[1] - cc[1])) + nn[2] * (p[2] - cc[2]);
            for (int c = 0; c < 3; ++c) {
              g.n[c] = nn[c];
              g.q[c] = q3[c];
            }
          }
          gtmp[i] = g;
          bits[i] = ok ? (unsigned long long)__double_as_longlong(fabs(g.r)) : ~0ull;
        }
        okc = ok;
      } else {
        for (int i = gtid; i < n; i += nthr) {
          PhotoTmp t{};
          const bool ok = photo_resid_one(ph.X, i, P, cam, ph.srange, ph.svalid, cfg.spread_gate, t);
          ptmp[i] = t;
          bits[i] = ok ? (unsigned long long)__double_as_longlong(fabs(t.r)) : ~0ull;
          okc += ok;
        }
      }
      const int m = rs_count(grid, okc, pcnt, s_part, &s_m);
      if (m == 0) continue;  // the family returns None (uniform)
      const double med = rs_median(grid, bits, n, m, Hc, st->cand[par][f], &st->ncand[par][f], &st->vmin[par][f],
                                   sh, s_part, &s_bin, &s_before, s_min);
      // --- trim, Huber, normal equations
      if (f == 0) {
        const double thr = fmax(cfg.trim_factor * med, fgeo);
        for (int i = gtid; i < n; i += nthr) {
          if (bits[i] == ~0ull) continue;
          const GeoTmp g = gtmp[i];
          const double ar = fabs(g.r);
          if (!(ar <= thr)) continue;
          // J = [n^T R, q x (R^T n)] (registration.py:268-273)
          double nR[3];
          for (int c = 0; c < 3; ++c) nR[c] = g.n[0] * P.R[c] + g.n[1] * P.R[3 + c] + g.n[2] * P.R[6 + c];
          const double J[6] = {nR[0], nR[1], nR[2], g.q[1] * nR[2] - g.q[2] * nR[1], g.q[2] * nR[0] - g.q[0] * nR[2],
                               g.q[0] * nR[1] - g.q[1] * nR[0]};
          const double w = ar <= cfg.huber_geo ? 1.0 : cfg.huber_geo / fmax(ar, 1e-12);
          acc[0][27] += hub_value(g.r, cfg.huber_geo);
          acc[0][30] += hub_value(g.r, cfg.huber_photo);
          acc[0][28] += 1.0;
          acc[0][29] += g.r * g.r;
          if (objective_only) continue;
          int k = 0;
          for (int a = 0; a < 6; ++a)
            for (int b2 = a; b2 < 6; ++b2) acc[0][k++] += w * J[a] * J[b2];
          for (int a = 0; a < 6; ++a) acc[0][21 + a] += w * J[a] * g.r;
        }
      } else {
        const double thr = fmax(cfg.trim_factor * med, fph);
        for (int i = gtid; i < n; i += nthr) {
          if (bits[i] == ~0ull) continue;
          const PhotoTmp& t = ptmp[i];
          double a30[30];
          for (int q = 0; q < 30; ++q) a30[q] = 0.0;
          photo_accum_one(t, cam, thr, cfg.huber_photo, objective_only, a30);
          if (a30[28] == 0.0) continue;
          for (int q = 0; q < 30; ++q) acc[1][q] += a30[q];
          acc[1][30] += a30[27];                       // Huber with huber_photo
          acc[1][27] += hub_value(t.r, cfg.huber_geo);  // ... and with huber_geo (positional pairing)
          acc[1][27] -= a30[27];
        }
      }
    }
    // --- per-block partial sums (families of this evaluation), block 0 reduces them in block order
    for (int f = 0; f < 2; ++f) {
      if (!fam_on[f]) continue;  // (uniform)
#pragma unroll
      for (int q = 0; q < 31; ++q) {
        double v = acc[f][q];
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if (lane == 0) sred[warp][q] = v;
      }
      __syncthreads();
      if (tid < 31) {
        double s = 0.0;
        for (int w = 0; w < kRsThreads / 32; ++w) s += sred[w][tid];
        part[((size_t)blockIdx.x * 2 + f) * kRsAcc + tid] = s;
      }
      __syncthreads();
    }
    grid.sync();
    if (blockIdx.x == 0) {
      for (int f = 0; f < 2; ++f) {
        if (!fam_on[f]) {
          if (tid < kRsAcc) sfin[f * kRsAcc + tid] = 0.0;
          continue;
        }
        const int q = tid & 31, g = tid >> 5;
        double s = 0.0;
        if (q < 31)
          for (int b = g; b < G; b += kRsThreads / 32) s += part[((size_t)b * 2 + f) * kRsAcc + q];
        if (q < 31) sred[g][q] = s;
        __syncthreads();
        if (tid < 31) {
          double t = 0.0;
          for (int w = 0; w < kRsThreads / 32; ++w) t += sred[w][tid];
          sfin[f * kRsAcc + tid] = t;
        }
        __syncthreads();
      }
      if (tid == 0) rs_step(st, cfg, sfin);
    }
  }
}

}  // namespace ss
