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

// -DSS_RS_PROF: block 0 / thread 0 accumulates %globaltimer deltas between
// marks and prints them when the loop ends (tools/reg_stages.sh).
#ifdef SS_RS_PROF
#define RS_MARK(k)                                                                   \
  if (blockIdx.x == 0 && threadIdx.x == 0) {                                         \
    unsigned long long t_;                                                           \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                           \
    rs_prof[k] += t_ - rs_last;                                                      \
    rs_last = t_;                                                                    \
  }
__device__ unsigned long long g_rs_sub[8], g_rs_sub_last;
#define RS_SUB(k)                                                                    \
  if (blockIdx.x == 0 && threadIdx.x == 0) {                                         \
    unsigned long long t_;                                                           \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                           \
    if (k >= 0) g_rs_sub[k < 0 ? 0 : k] += t_ - g_rs_sub_last;                       \
    g_rs_sub_last = t_;                                                              \
  }
#else
#define RS_MARK(k)
#define RS_SUB(k)
#endif

enum { RS_EVAL = 0, RS_DONE = 1 };

// The LM state machine's fields: the published evaluation (the first 20 words,
// read by every block) and the state of block 0 / thread 0, which keeps it in
// shared memory during the launch (the copy in global memory is written back at
// the end; the published words are copied out after every step).
struct RegSolveLM {
  // published evaluation
  double P[12];
  double fg, fp;
  int objective_only, action, eval_geo, eval_photo;
  // a family already evaluated at exactly this pose (the accepted trial before a full
  // evaluation) reuses its residuals, count and median: only the trim floor changed
  int reuse[2], pub_m[2];
  double pub_med[2];
  // the evaluation just finished (block 0, thread 0)
  double lastP[12];
  int last_fam[2], cur_m[2];
  double cur_med[2];
  // LM state (block 0, thread 0)
  double T[12], Ttry[12], H[36], b[6], delta[6];
  double lam, obj0, term_hub[2], term_s[2];
  double last_r2[2];
  int last_m[2], nterms;
  int it_total, converged, status, stage, n_eval, phase, use_geo, use_photo;
};

struct RegSolveState : RegSolveLM {  // + the grid-wide median scratch
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

// Insert (d, id) into a k-best list sorted by (d, id), dropping the last slot.
// Fully unrolled so the list stays in registers.
template <int K>
__device__ __forceinline__ void rs_kbest_insert(double (&kd)[K], int (&ki)[K], double d, int id) {
#pragma unroll
  for (int a = K - 1; a >= 0; --a) {
    const bool before_a = d < kd[a] || (d == kd[a] && id < ki[a]);
    if (a > 0) {
      const bool before_prev = d < kd[a - 1] || (d == kd[a - 1] && id < ki[a - 1]);
      kd[a] = before_prev ? kd[a - 1] : (before_a ? d : kd[a]);
      ki[a] = before_prev ? ki[a - 1] : (before_a ? id : ki[a]);
    } else {
      kd[0] = before_a ? d : kd[0];
      ki[0] = before_a ? id : ki[0];
    }
  }
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

__device__ void rs_begin_iteration(RegSolveLM* st, const RegSolveCfg& cfg);

// Start phase `ph` (registration.py:441-450): damping and convergence reset.
__device__ void rs_begin_phase(RegSolveLM* st, const RegSolveCfg& cfg, int ph) {
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

// Publish-time reuse decision (see RegSolveState::reuse).
__device__ void rs_set_reuse(RegSolveLM* st) {
  bool same = true;
  for (int q = 0; q < 12; ++q)
    same = same && __double_as_longlong(st->P[q]) == __double_as_longlong(st->lastP[q]);
  const int ev[2] = {st->eval_geo, st->eval_photo};
  for (int f = 0; f < 2; ++f) {
    st->reuse[f] = same && ev[f] && st->last_fam[f];
    st->pub_m[f] = st->cur_m[f];
    st->pub_med[f] = st->cur_med[f];
  }
}

// Next outer iteration of the phase (or the next phase): a full evaluation at T.
__device__ void rs_begin_iteration(RegSolveLM* st, const RegSolveCfg& cfg) {
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
  rs_set_reuse(st);
}

// Inner LM loop: next trial pose, or the end of the phase when damping is exhausted.
__device__ void rs_try(RegSolveLM* st, const RegSolveCfg& cfg) {
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
    rs_set_reuse(st);
    return;
  }
  rs_begin_phase(st, cfg, st->phase + 1);  // damping exhausted: keep the estimate, end the phase
}

// red: per family (geo, photo) kRsAcc sums of the evaluation just finished.
__device__ void rs_step(RegSolveLM* st, const RegSolveCfg& cfg, const double* red) {
  st->n_eval += 1;
  for (int q = 0; q < 12; ++q) st->lastP[q] = st->P[q];  // (cur_m / cur_med: written during the evaluation)
  st->last_fam[0] = st->eval_geo;
  st->last_fam[1] = st->eval_photo;
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
// lanes per scan point in the geometric residual loop (the largest power of two <= 32 with
// S n <= grid threads); the point's residual is written by lane 0 of its group
__device__ __forceinline__ int rs_geo_stride(int n, int nthr) {
  int S = 1;
  while (S < 32 && 2 * S * n <= nthr) S *= 2;
  return S;
}

// (*m_io < 0: the count is not known yet -- the first pass then histograms every valid
// pattern on the fixed top digit, bits 62-51, and the count is that histogram's total,
// written back to *m_io: one grid barrier fewer than counting first (rs_count).  With no
// barrier between the residuals and that pass, each pattern is read by the thread that
// wrote it: entry i by thread i * owner_stride + k * nthr (the residual loops' owners).
// A zero count returns 0.)
__device__ double rs_median(cg::grid_group& grid, const unsigned long long* __restrict__ bits, int n, int* m_io,
                            int owner_stride, unsigned long long vlo, unsigned long long vhi, unsigned* __restrict__ Hc,
                            unsigned long long* cand, int* ncand, unsigned long long* vmin, unsigned* sh,
                            unsigned* s_part, int* s_bin, int* s_before, unsigned long long* s_min) {
  // vlo / vhi: smallest / largest valid pattern (rs_count).  The radix passes start at
  // the highest bit in which they differ (12-bit digits downwards).
  int m = *m_io;
  const bool counted = m < 0;
  if (!counted && vlo == vhi) return __longlong_as_double((long long)vlo);  // all equal
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gtid = blockIdx.x * kRsThreads + tid, nthr = gridDim.x * kRsThreads;
  int k1 = counted ? 0 : ((m % 2 == 0) ? m / 2 - 1 : m / 2);
  int top = counted ? 62 : 63 - __clzll(vlo ^ vhi);  // <= 62: valid patterns are non-negative doubles
  unsigned long long mask = ~((2ull << top) - 1ull), prefix = (counted ? 0ull : vlo) & mask;
  int kk = k1, cnt_eq = 0;
  bool exact = false;
  unsigned long long v2c = ~0ull;
  RS_SUB(-1);
  for (int p = 0;; ++p) {
    const int lo = max(top - 11, 0);
    const unsigned dmask = (1u << (top - lo + 1)) - 1u;
    for (int j = tid; j <= (int)dmask; j += kRsThreads) sh[j] = 0u;
    __syncthreads();
    if (p == 0 && counted) {
      const int st = nthr / owner_stride;
      for (int i = gtid % owner_stride == 0 ? gtid / owner_stride : n; i < n; i += st) {
        const unsigned long long b = bits[i];
        if (b != ~0ull) atomicAdd(&sh[(unsigned)(b >> lo) & dmask], 1u);
      }
    } else {
      for (int i = gtid; i < n; i += nthr) {
        const unsigned long long b = bits[i];
        if (b != ~0ull && (b & mask) == prefix) atomicAdd(&sh[(unsigned)(b >> lo) & dmask], 1u);
      }
    }
    __syncthreads();
    unsigned* Hp = Hc + p * kRsBins;  // p < kRsPasses: at most ceil(63 / 12) passes
    for (int j = tid; j <= (int)dmask; j += kRsThreads)
      if (sh[j]) atomicAdd(&Hp[j], sh[j]);
    RS_SUB(0);
    grid.sync();
    RS_SUB(1);
    if (p == 0 && counted) {  // the count: the first histogram's total (every valid pattern)
      unsigned c = 0;
      for (int j = tid; j <= (int)dmask; j += kRsThreads) c += ((volatile unsigned*)Hp)[j];
      c = __reduce_add_sync(0xffffffffu, c);
      if (lane == 0) s_part[warp] = c;
      __syncthreads();
      m = 0;
      for (int w = 0; w < kRsThreads / 32; ++w) m += (int)s_part[w];
      __syncthreads();
      *m_io = m;
      if (m == 0) return 0.0;
      k1 = (m % 2 == 0) ? m / 2 - 1 : m / 2;
      kk = k1;
    }
    rs_find_bin(Hp, (int)dmask + 1, kk, s_bin, s_before, s_part);
    RS_SUB(2);
    const int bin = *s_bin;
    kk -= *s_before;
    const int cnt_bin = (int)Hp[bin];
    prefix |= (unsigned long long)bin << lo;
    mask |= (unsigned long long)dmask << lo;
    __syncthreads();
    if (lo == 0) {
      cnt_eq = cnt_bin;
      exact = true;
      break;
    }
    top = lo - 1;
    if (cnt_bin <= kRsCand) {
      // few values share the prefix: gather them and rank them exactly in every block
      for (int i = gtid; i < n; i += nthr) {
        const unsigned long long b = bits[i];
        if (b != ~0ull && (b & mask) == prefix) cand[atomicAdd(ncand, 1)] = b;
      }
      RS_SUB(3);
      grid.sync();
      RS_SUB(1);
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
      RS_SUB(4);
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
  RS_SUB(5);
  grid.sync();
  RS_SUB(1);
  return (v1 + __longlong_as_double((long long)*((volatile unsigned long long*)vmin))) / 2.0;
}

// Leaf hash grid for the association: cells of edge >= assoc_gate, so every
// leaf within the gate of a point lies in the point's 27-cell neighbourhood
// (and the k nearest within the gate -- the only ones the residual uses -- are
// exactly the k nearest among those).  Cells hash into kRsGridBuckets buckets;
// a bucket's entries carry their cell key so each leaf is seen once.
constexpr int kRsGridBuckets = 4096;
constexpr int kRsCellBias = 1 << 20;  // cell coordinates clamped to [-2^20, 2^20)

struct RsLeafEntry {
  double c[3];
  unsigned long long key;
  int id, pad;
};

__device__ __forceinline__ int rs_cell(double x, double inv_cs) {
  const double f = floor(x * inv_cs);
  return (int)fmin(fmax(f, -(double)kRsCellBias), (double)(kRsCellBias - 1));  // NaN -> lower bound
}
__device__ __forceinline__ unsigned long long rs_cell_key(int ix, int iy, int iz) {
  return ((unsigned long long)(ix + kRsCellBias) << 42) | ((unsigned long long)(iy + kRsCellBias) << 21) |
         (unsigned long long)(iz + kRsCellBias);
}
__device__ __forceinline__ int rs_bucket(unsigned long long k, int mask) {
  k ^= k >> 31;
  k *= 0x7fb5d329728ea185ull;
  k ^= k >> 27;
  k *= 0x81dadef4bc2dd44dull;
  k ^= k >> 33;
  return (int)k & mask;
}
// 1 / cell edge; 0 (one cell) when the gate is not a positive finite number
__host__ __device__ inline double rs_inv_cell(double gate) {
  const double g = gate < 0 ? -gate : gate;
  return (g > 0 && g < 1e300) ? 1.0 / (g * (1.0 + 1e-9)) : 0.0;
}

// One block: counting sort of the leaves into mask + 1 (<= kRsGridBuckets) hash buckets.
__global__ void __launch_bounds__(1024) k_leaf_grid(const double* __restrict__ cent, int nl, double inv_cs, int mask,
                                                    int* __restrict__ bstart, RsLeafEntry* __restrict__ ent,
                                                    int* __restrict__ lbucket) {
  __shared__ int cnt[kRsGridBuckets];
  __shared__ int wsum[32];
  const int tid = threadIdx.x;
  for (int b = tid; b < kRsGridBuckets; b += blockDim.x) cnt[b] = 0;
  __syncthreads();
  for (int l = tid; l < nl; l += blockDim.x) {
    const int b = rs_bucket(rs_cell_key(rs_cell(cent[3 * l], inv_cs), rs_cell(cent[3 * l + 1], inv_cs),
                                        rs_cell(cent[3 * l + 2], inv_cs)), mask);
    lbucket[l] = b;
    atomicAdd(&cnt[b], 1);
  }
  __syncthreads();
  // exclusive scan, 4 buckets per thread (blockDim.x == 1024)
  int v[4], run = 0;
  for (int q = 0; q < 4; ++q) {
    v[q] = run;
    run += cnt[4 * tid + q];
  }
  int incl = run;
  for (int off = 1; off < 32; off <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, off);
    if ((tid & 31) >= off) incl += t;
  }
  if ((tid & 31) == 31) wsum[tid >> 5] = incl;
  __syncthreads();
  if (tid < 32) {
    int w = wsum[tid], wi = w;
    for (int off = 1; off < 32; off <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, wi, off);
      if (tid >= off) wi += t;
    }
    wsum[tid] = wi - w;
  }
  __syncthreads();
  const int base = wsum[tid >> 5] + incl - run;
  __syncthreads();
  for (int q = 0; q < 4; ++q) {
    bstart[4 * tid + q] = base + v[q];
    cnt[4 * tid + q] = base + v[q];  // fill cursor
  }
  if (tid == 0) bstart[kRsGridBuckets] = nl;
  __syncthreads();
  for (int l = tid; l < nl; l += blockDim.x) {
    const int pos = atomicAdd(&cnt[lbucket[l]], 1);  // order inside a bucket is irrelevant
    RsLeafEntry e;
    for (int c = 0; c < 3; ++c) e.c[c] = cent[3 * l + c];
    e.key = rs_cell_key(rs_cell(e.c[0], inv_cs), rs_cell(e.c[1], inv_cs), rs_cell(e.c[2], inv_cs));
    e.id = l;
    e.pad = 0;
    ent[pos] = e;
  }
}

struct RsGeo {  // geometric inputs: usable leaves and the (subsampled) scan, sensor frame
  const double* cent;
  const double* nrm;
  int n_leaves;
  const double* scan;
  int n_scan;
  const int* bstart;  // leaf hash grid (k_leaf_grid): mask + 1 buckets
  const RsLeafEntry* ent;
  double inv_cs;
  int mask;
  int staged;  // the grid fits the dynamic shared memory: copied there once per launch
};

__host__ __device__ inline size_t rs_grid_smem_bytes(int nl, int mask) {
  return ((size_t)(mask + 2) * 4 + 15) / 16 * 16 + (size_t)nl * sizeof(RsLeafEntry);
}

// k nearest leaves (sorted by (d2, leaf index)) of p among the leaves of its
// 27-cell neighbourhood; S consecutive lanes share p, each visiting every S-th
// cell, and merge their lists by butterfly shuffles (all lanes of the warp call
// this).  Results land in kd/ki[0, K), +inf beyond.
template <int K>
__device__ __forceinline__ void rs_knn(const double* p, bool active, int sub, int S, const int* bst,
                                       const RsLeafEntry* ent, int mask, double inv_cs, double (&kd8)[8],
                                       int (&ki8)[8]) {
  double kd[K];
  int ki[K];
#pragma unroll
  for (int a = 0; a < K; ++a) {
    kd[a] = __longlong_as_double(0x7ff0000000000000LL);
    ki[a] = 0x7fffffff;
  }
  if (active) {
    const int cx = rs_cell(p[0], inv_cs), cy = rs_cell(p[1], inv_cs), cz = rs_cell(p[2], inv_cs);
    for (int nb = sub; nb < 27; nb += S) {
      const int ix = cx + nb / 9 - 1, iy = cy + (nb / 3) % 3 - 1, iz = cz + nb % 3 - 1;
      if (ix < -kRsCellBias || ix >= kRsCellBias || iy < -kRsCellBias || iy >= kRsCellBias || iz < -kRsCellBias ||
          iz >= kRsCellBias)
        continue;
      const unsigned long long key = rs_cell_key(ix, iy, iz);
      const int b = rs_bucket(key, mask);
      const int e1 = bst[b + 1];
      for (int e = bst[b]; e < e1; ++e) {
        const RsLeafEntry& le = ent[e];
        if (le.key != key) continue;
        const double dx = p[0] - le.c[0], dy = p[1] - le.c[1], dz = p[2] - le.c[2];
        const double d2 = dx * dx + dy * dy + dz * dz;
        if (d2 <= kd[K - 1]) rs_kbest_insert<K>(kd, ki, d2, le.id);  // a tie may still win on the index
      }
    }
  }
  for (int off = 1; off < S; off <<= 1) {
    double od[K];
    int oi[K];
#pragma unroll
    for (int a = 0; a < K; ++a) {
      od[a] = __shfl_xor_sync(0xffffffffu, kd[a], off);
      oi[a] = __shfl_xor_sync(0xffffffffu, ki[a], off);
    }
#pragma unroll
    for (int a = 0; a < K; ++a) rs_kbest_insert<K>(kd, ki, od[a], oi[a]);
  }
#pragma unroll
  for (int a = 0; a < 8; ++a) {
    kd8[a] = a < K ? kd[a] : __longlong_as_double(0x7ff0000000000000LL);
    ki8[a] = a < K ? ki[a] : 0x7fffffff;
  }
}
struct RsPhoto {  // photometric inputs: world anchors and the scan range image
  const double* X;
  int M;
  const double* srange;
  const uint8_t* svalid;
  // device counts {confident model pixels, anchors} of an anchor pass enqueued just
  // before (frame batches, no host round trip): M is then min(counts[1], M) and a
  // model with fewer than min_residuals confident pixels ends the loop at once with
  // status 2, the host path's "too few confident pixels"
  const int* counts;
};

// kMinB = 1: one block per SM (255 registers; single registrations, whose grid-wide
// barriers cost less over fewer blocks).  kMinB = 2 (128 registers, a few spills in the
// state machine): frame batches, where two loops' blocks share each SM and hide each
// other's latency (config 3, 8 frames: 1,553 -> 1,715 registrations/s; one frame on
// 2 x 148 blocks is slower, 548 -> 497).
template <int kMinB>
__global__ void __launch_bounds__(kRsThreads, kMinB) k_reg_solve(RsGeo geo, RsPhoto ph, RegCam cam, RegSolveCfg cfg,
                                                         GeoTmp* __restrict__ gtmp, PhotoTmp* __restrict__ ptmp,
                                                         unsigned long long* __restrict__ gbits,
                                                         unsigned long long* __restrict__ pbits,
                                                         unsigned* __restrict__ hist, double* __restrict__ part,
                                                         int* __restrict__ pcnt, unsigned long long* __restrict__ pmm,
                                                         RegSolveState* st) {
  cg::grid_group grid = cg::this_grid();
  if (ph.counts) {
    if (ph.counts[0] < cfg.min_residuals) {  // (uniform over the grid: no block reaches a grid barrier)
      if (blockIdx.x == 0 && threadIdx.x == 0) st->status = 2;
      return;
    }
    ph.M = min(ph.counts[1], ph.M);
  }
  __shared__ __align__(16) unsigned sh[kRsBins];
  __shared__ double sred[kRsThreads / 32][kRsAcc];
  __shared__ double sfin[2 * kRsAcc];
  __shared__ unsigned s_part[kRsThreads / 32];
  __shared__ int s_bin, s_before;
  __shared__ unsigned long long s_min[kRsThreads / 32];
  __shared__ unsigned long long s_pub[20];
  static_assert(offsetof(RegSolveLM, pub_med) + 2 * sizeof(double) <= 20 * 8, "published fields in the first 20 words");
  __shared__ RegSolveLM s_lm;  // block 0: the LM state during the launch
  auto publish = [&]() {  // block 0, thread 0: the next evaluation's words to every block
    for (int q = 0; q < 20; ++q)
      reinterpret_cast<unsigned long long*>(st)[q] = reinterpret_cast<const unsigned long long*>(&s_lm)[q];
  };
  const int G = gridDim.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gtid = blockIdx.x * kRsThreads + tid, nthr = G * kRsThreads;
  const int kmax = min(min(cfg.assoc_k, geo.n_leaves), 8);
  // the leaf grid is constant for the launch: stage it in shared memory when it fits
  extern __shared__ __align__(16) unsigned char rs_dyn[];
  const int* s_bst = geo.bstart;
  const RsLeafEntry* s_ent = geo.ent;
  if (geo.staged) {
    int* b = reinterpret_cast<int*>(rs_dyn);
    RsLeafEntry* en = reinterpret_cast<RsLeafEntry*>(rs_dyn + ((size_t)(geo.mask + 2) * 4 + 15) / 16 * 16);
    for (int q = threadIdx.x; q <= geo.mask + 1; q += kRsThreads) b[q] = geo.bstart[q];
    const double* src = reinterpret_cast<const double*>(geo.ent);
    double* dst = reinterpret_cast<double*>(en);
    for (int q = threadIdx.x; q < geo.n_leaves * (int)(sizeof(RsLeafEntry) / 8); q += kRsThreads) dst[q] = src[q];
    s_bst = b;
    s_ent = en;
    __syncthreads();
  }
  if (blockIdx.x == 0 && tid == 0) {
    s_lm = *static_cast<const RegSolveLM*>(st);  // (initial pose from the host)
    s_lm.it_total = 0;
    s_lm.status = 0;
    s_lm.n_eval = 0;
    s_lm.last_m[0] = s_lm.last_m[1] = 0;
    s_lm.last_r2[0] = s_lm.last_r2[1] = 0.0;
    for (int a = 0; a < 2; ++a)
      for (int f = 0; f < 2; ++f) {
        st->vmin[a][f] = ~0ull;
        st->ncand[a][f] = 0;
      }
    rs_begin_phase(&s_lm, cfg, 0);
    publish();
  }
#ifdef SS_RS_PROF
  unsigned long long rs_prof[10] = {}, rs_last = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(rs_last));
#endif
  for (int e = 0;; ++e) {
    grid.sync();
    RS_MARK(0);
    RS_SUB(-1);
    // the published evaluation (P, floors, flags, reuse: the first 20 words of the state),
    // loaded by one warp in parallel instead of ~18 dependent volatile loads per thread
    if (tid < 20) s_pub[tid] = ((volatile unsigned long long*)st)[tid];
    __syncthreads();
    const RegSolveState* vs = reinterpret_cast<const RegSolveState*>(s_pub);
    if (vs->action == RS_DONE) {
      if (blockIdx.x == 0 && tid == 0) *static_cast<RegSolveLM*>(st) = s_lm;  // results for the host
#ifdef SS_RS_PROF
      if (blockIdx.x == 0 && threadIdx.x == 0)
        printf("RSPROF evals %d step+sync %llu resid %llu count %llu median %llu accum %llu part %llu sync %llu final %llu"
               " | sub %llu %llu %llu %llu %llu %llu | state %llu zero %llu\n",
               e, rs_prof[0], rs_prof[1], rs_prof[2], rs_prof[3], rs_prof[4], rs_prof[5], rs_prof[6], rs_prof[7],
               g_rs_sub[0], g_rs_sub[1], g_rs_sub[2], g_rs_sub[3], g_rs_sub[4], g_rs_sub[5], g_rs_sub[6],
               g_rs_sub[7]);
      if (blockIdx.x == 0 && threadIdx.x == 0)
        for (int q = 0; q < 8; ++q) g_rs_sub[q] = 0;
#endif
      break;
    }
    PoseK P;
    for (int q = 0; q < 9; ++q) P.R[q] = vs->P[q];
    for (int q = 0; q < 3; ++q) P.t[q] = vs->P[9 + q];
    const double fgeo = vs->fg, fph = vs->fp;
    const int objective_only = vs->objective_only;
    const int fam_on[2] = {vs->eval_geo && geo.n_leaves > 0, vs->eval_photo};
    RS_SUB(6);
    const int par = e & 1;
    // zero the next evaluation's scratch
    unsigned* Hnext = hist + (size_t)(par ^ 1) * 2 * kRsPasses * kRsBins;
    for (int i = gtid; i < 2 * kRsPasses * kRsBins; i += nthr) Hnext[i] = 0u;
    if (gtid == 0)
      for (int f = 0; f < 2; ++f) {
        st->vmin[par ^ 1][f] = ~0ull;
        st->ncand[par ^ 1][f] = 0;
      }
    for (int f = 0; f < 2; ++f) {
      if (!fam_on[f]) continue;  // uniform across the grid
      double acc[kRsAcc];
#pragma unroll
      for (int q = 0; q < kRsAcc; ++q) acc[q] = 0.0;
      unsigned* Hc = hist + ((size_t)par * 2 + f) * kRsPasses * kRsBins;
      unsigned long long* bits = f == 0 ? gbits : pbits;
      const int n = f == 0 ? geo.n_scan : ph.M;
      RS_SUB(7);
      // a family evaluated at exactly this pose by the previous (trial) evaluation keeps
      // its residuals (gtmp / ptmp, bits), count and median: only the trim floor differs
      int m = 0;
      double med = 0.0;
      if (vs->reuse[f]) {
        m = vs->pub_m[f];
        med = vs->pub_med[f];
      } else {
        // --- residuals
        int okc = 0;
        unsigned long long vlo = ~0ull, vhi = 0ull;  // this thread's smallest / largest valid |r| pattern
        if (f == 0) {
          // k nearest usable leaf centroids within the gate, then the leaf whose plane
          // is closest (registration.py:249-265); leaves staged through shared memory
          // S consecutive lanes share one scan point (n_scan <= grid threads, checked by
          // the host), each visiting every S-th cell of the point's 27-cell
          // neighbourhood in the leaf grid; their sorted k-best lists merge by
          // butterfly shuffles.  The lists live in registers (static indexing) and
          // order by (d2, leaf index), so the result does not depend on visit order.
          const int S = rs_geo_stride(n, nthr);
          const int i = gtid / S, sub = gtid & (S - 1);
          double p[3] = {0, 0, 0}, q3[3] = {0, 0, 0};
          if (i < n) {
            for (int c = 0; c < 3; ++c) q3[c] = geo.scan[3 * i + c];
            for (int c = 0; c < 3; ++c)
              p[c] = P.R[3 * c] * q3[0] + P.R[3 * c + 1] * q3[1] + P.R[3 * c + 2] * q3[2] + P.t[c];
          }
          double kd[8];
          int ki[8];
          switch (kmax) {  // (uniform)
  #define RS_KNN_CASE(K) \
    case K:              \
      rs_knn<K>(p, i < n, sub, S, s_bst, s_ent, geo.mask, geo.inv_cs, kd, ki); \
      break;
            RS_KNN_CASE(1)
            RS_KNN_CASE(2)
            RS_KNN_CASE(3)
            RS_KNN_CASE(4)
            RS_KNN_CASE(5)
            RS_KNN_CASE(6)
            RS_KNN_CASE(7)
            default:
              rs_knn<8>(p, i < n, sub, S, s_bst, s_ent, geo.mask, geo.inv_cs, kd, ki);
  #undef RS_KNN_CASE
          }
          bool ok = false;
          GeoTmp g{};
          if (i < n && sub == 0) {
            const double gate2 = cfg.assoc_gate * cfg.assoc_gate;
            double best = __longlong_as_double(0x7ff0000000000000LL);
            int bl = -1;
  #pragma unroll
            for (int a = 0; a < 8; ++a) {
              if (a >= kmax || !(kd[a] < gate2)) continue;  // beyond distance_upper_bound
              const double* nn = geo.nrm + 3 * ki[a];
              const double* cc = geo.cent + 3 * ki[a];
              const double pd = fabs(nn[0] * (p[0] - cc[0]) + nn[1] * (p[1] - cc[1]) + nn[2] * (p[2] - cc[2]));
              if (pd < best) {
                best = pd;
                bl = ki[a];
              }
            }
            ok = kd[0] < gate2;
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
            const unsigned long long bv = ok ? (unsigned long long)__double_as_longlong(fabs(g.r)) : ~0ull;
            bits[i] = bv;
            if (ok) vlo = vhi = bv;
          }
          okc = ok;
        } else {
          // two anchors per pass (branch-free residuals interleave; M ~ 1-2x the grid's threads)
          for (int i = gtid; i < n; i += 2 * nthr) {
            const int i2 = i + nthr < n ? i + nthr : i;
            PhotoTmp t[2];
            bool ok[2];
            ok[0] = photo_resid_nb(ph.X, i, P, cam, ph.srange, ph.svalid, cfg.spread_gate, t[0]);
            ok[1] = photo_resid_nb(ph.X, i2, P, cam, ph.srange, ph.svalid, cfg.spread_gate, t[1]);
  #pragma unroll
            for (int a = 0; a < 2; ++a) {
              if (a == 1 && i2 == i) break;
              const int ia = a ? i2 : i;
              if (!ok[a]) t[a] = PhotoTmp{};
              ptmp[ia] = t[a];
              const unsigned long long bv = ok[a] ? (unsigned long long)__double_as_longlong(fabs(t[a].r)) : ~0ull;
              bits[ia] = bv;
              if (ok[a]) {
                vlo = min(vlo, bv);
                vhi = max(vhi, bv);
              }
              okc += ok[a];
            }
          }
        }
        RS_MARK(1);
        // (a per-block select from a shared-memory copy of all patterns, one grid barrier
        // instead of one per pass, measured slower: 42 vs 37 us per geometric evaluation --
        // shared-memory atomics on the clustered top digits and redundant passes)
        // the count comes out of the median's first histogram (one grid barrier fewer)
        (void)okc;
        (void)vlo;
        (void)vhi;
        RS_MARK(2);
        m = -1;
        med = rs_median(grid, bits, n, &m, f == 0 ? rs_geo_stride(n, nthr) : 1, 0ull, 0ull, Hc, st->cand[par][f], &st->ncand[par][f],
                        &st->vmin[par][f], sh, s_part, &s_bin, &s_before, s_min);
        if (blockIdx.x == 0 && tid == 0) {
          s_lm.cur_m[f] = m;
          s_lm.cur_med[f] = med;
        }
      }
      RS_MARK(3);
      if (m > 0) {  // else the family returns None (uniform); its partial sums stay zero
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
          acc[27] += hub_value(g.r, cfg.huber_geo);
          acc[30] += hub_value(g.r, cfg.huber_photo);
          acc[28] += 1.0;
          acc[29] += g.r * g.r;
          if (objective_only) continue;
          int k = 0;
          for (int a = 0; a < 6; ++a)
            for (int b2 = a; b2 < 6; ++b2) acc[k++] += w * J[a] * J[b2];
          for (int a = 0; a < 6; ++a) acc[21 + a] += w * J[a] * g.r;
        }
      } else {
        const double thr = fmax(cfg.trim_factor * med, fph);
        for (int i = gtid; i < n; i += nthr) {
          if (bits[i] == ~0ull) continue;
          // slot 30: Huber with huber_photo; slot 27: with huber_geo (positional pairing)
          photo_accum_one(ptmp[i], cam, thr, cfg.huber_photo, cfg.huber_geo, objective_only, acc);
        }
      }
      }
      RS_MARK(4);
      // --- per-block partial sums of this family; block 0 reduces them in block order
#pragma unroll
      for (int q = 0; q < 31; ++q) {
        double v = acc[q];
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
      RS_MARK(5);
    }
    grid.sync();
    RS_MARK(6);
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
      RS_MARK(7);
      if (tid == 0) {
        rs_step(&s_lm, cfg, sfin);
        publish();
      }
    }
  }
}

}  // namespace ss
