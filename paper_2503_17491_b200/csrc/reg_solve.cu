// Device-resident photometric Gauss-Newton / Levenberg loop: the whole
// register() iteration of the reference (registration.py:437-524, photometric
// phase) in ONE cooperative kernel, so no evaluation round-trips to the host.
//
//   per evaluation (pose P, trim floor fp, objective-only flag):
//     residuals of every anchor                 (_photo_system, :324-340)
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

struct RegSolveCfg {
  double huber, trim_factor, spread_gate, assoc_gate, trim_floor, tol, damping_init, damping_max;
  int max_iters, min_residuals;
};

constexpr int kRsThreads = 256;
constexpr int kRsBins = 4096;  // 12-bit digits
constexpr int kRsPasses = 6;   // bits 63-52, 51-40, 39-28, 27-16, 15-4, 3-0
constexpr int kRsCand = 256;   // a selected bin this small is finished by an exact in-block rank

enum { RS_EVAL = 0, RS_DONE = 1 };

struct RegSolveState {
  // published evaluation
  double P[12];
  double fp;
  int objective_only, action;
  // LM state (block 0, thread 0)
  double T[12], Ttry[12], H[36], b[6], delta[6];
  double lam, obj0, s, last_r2;
  int it_total, converged, status, stage, last_m, n_eval;
  unsigned long long vmin[2];
  int ncand[2];
  unsigned long long cand[2][kRsCand];
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

// Start outer iteration it_total + 1 (or finish): publishes a full evaluation at T.
__device__ void rs_begin_iteration(RegSolveState* st, const RegSolveCfg& cfg) {
  if (st->it_total >= cfg.max_iters) {
    st->action = RS_DONE;
    return;
  }
  st->it_total += 1;
  const double anneal = cfg.assoc_gate * pow(0.5, (double)st->it_total);
  st->fp = fmax(cfg.trim_floor, anneal);
  for (int q = 0; q < 12; ++q) st->P[q] = st->T[q];
  st->objective_only = 0;
  st->stage = 0;
  st->action = RS_EVAL;
}

// Inner LM loop: next trial pose, or the end of the iteration when damping is exhausted.
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
  st->action = RS_DONE;  // damping exhausted: keep the current estimate
}

// red: the evaluation's sums ([0:21] H upper, [21:27] b, [27] Huber, [28] m, [29] r^2).
__device__ void rs_step(RegSolveState* st, const RegSolveCfg& cfg, const double* red) {
  const int m = (int)llrint(red[28]);
  st->n_eval += 1;
  if (st->stage == 0) {
    int n_photo = 0;
    if (m > 0) {
      const double s = 1.0 / m;
      st->s = s;
      int k = 0;
      for (int a = 0; a < 6; ++a)
        for (int b = a; b < 6; ++b) {
          st->H[6 * a + b] = st->H[6 * b + a] = s * red[k];
          ++k;
        }
      for (int a = 0; a < 6; ++a) st->b[a] = s * red[21 + a];
      n_photo = m;
      st->last_r2 = red[29];
      st->last_m = m;
    }
    if (n_photo < cfg.min_residuals) {
      st->status = 1;  // RegistrationError: too few residuals survive association
      st->action = RS_DONE;
      return;
    }
    st->obj0 = st->s * red[27];
    rs_try(st, cfg);
    return;
  }
  // trial evaluation at Ttry
  if (m > 0 && st->s * red[27] <= st->obj0 + 1e-12) {
    for (int q = 0; q < 12; ++q) st->T[q] = st->Ttry[q];
    st->lam = fmax(st->lam * 0.25, cfg.damping_init);
    const double dn = sqrt(st->delta[0] * st->delta[0] + st->delta[1] * st->delta[1] + st->delta[2] * st->delta[2] +
                           st->delta[3] * st->delta[3] + st->delta[4] * st->delta[4] + st->delta[5] * st->delta[5]);
    if (dn < cfg.tol) {
      st->converged = 1;
      st->action = RS_DONE;
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

__global__ void __launch_bounds__(kRsThreads) k_reg_solve(const double* __restrict__ X, int M, RegCam cam,
                                                         const double* __restrict__ srange,
                                                         const uint8_t* __restrict__ svalid, RegSolveCfg cfg,
                                                         PhotoTmp* __restrict__ tmp,
                                                         unsigned long long* __restrict__ bits,
                                                         unsigned* __restrict__ hist, double* __restrict__ part,
                                                         int* __restrict__ pcnt, RegSolveState* st) {
  cg::grid_group grid = cg::this_grid();
  __shared__ unsigned sh[kRsBins];
  __shared__ double sred[kRsThreads / 32][30];
  __shared__ double sfin[32];
  __shared__ unsigned s_part[kRsThreads / 32];
  __shared__ int s_bin, s_before, s_m;
  __shared__ unsigned long long s_min[kRsThreads / 32];
  const int G = gridDim.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gtid = blockIdx.x * kRsThreads + tid, nthr = G * kRsThreads;
  if (blockIdx.x == 0 && tid == 0) {
    st->lam = cfg.damping_init;
    st->it_total = 0;
    st->converged = 0;
    st->status = 0;
    st->last_m = 0;
    st->last_r2 = 0.0;
    st->n_eval = 0;
    st->s = 0.0;
    st->vmin[0] = st->vmin[1] = ~0ull;
    rs_begin_iteration(st, cfg);
  }
  for (int e = 0;; ++e) {
    grid.sync();
    volatile RegSolveState* vs = st;
    if (vs->action == RS_DONE) break;
    PoseK P;
    for (int q = 0; q < 9; ++q) P.R[q] = vs->P[q];
    for (int q = 0; q < 3; ++q) P.t[q] = vs->P[9 + q];
    const double fp = vs->fp;
    const int objective_only = vs->objective_only;
    unsigned* Hc = hist + (size_t)(e & 1) * kRsPasses * kRsBins;        // this evaluation
    unsigned* Hn = hist + (size_t)((e + 1) & 1) * kRsPasses * kRsBins;  // the next one: zeroed now
    for (int i = gtid; i < kRsPasses * kRsBins; i += nthr) Hn[i] = 0u;
    if (gtid == 0) {
      st->vmin[(e + 1) & 1] = ~0ull;
      st->ncand[(e + 1) & 1] = 0;
    }
    // --- residuals
    int okc = 0;
    for (int i = gtid; i < M; i += nthr) {
      PhotoTmp t{};
      const bool ok = photo_resid_one(X, i, P, cam, srange, svalid, cfg.spread_gate, t);
      tmp[i] = t;
      bits[i] = ok ? (unsigned long long)__double_as_longlong(fabs(t.r)) : ~0ull;
      okc += ok;
    }
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
      for (int b = lane; b < G; b += 32) c += pcnt[b];
      c = __reduce_add_sync(0xffffffffu, c);
      if (lane == 0) s_m = c;
    }
    __syncthreads();
    const int m = s_m;
    // --- exact median of |r| (np.median): k-th smallest by grid-wide radix select
    double median = 0.0;
    if (m > 0) {
      const int k1 = (m % 2 == 0) ? m / 2 - 1 : m / 2;
      unsigned long long prefix = 0ull, mask = 0ull;
      int kk = k1, cnt_eq = 0;
      bool exact = false;  // prefix is the full k1-th value
      unsigned long long v2c = ~0ull;  // the next order statistic when it lies in the gathered bin
      for (int p = 0; p < kRsPasses; ++p) {
        const int shift = p < 5 ? 52 - 12 * p : 0;
        const int nb = p < 5 ? 12 : 4;
        const unsigned dmask = (1u << nb) - 1u;
        for (int j = tid; j < kRsBins; j += kRsThreads) sh[j] = 0u;
        __syncthreads();
        for (int i = gtid; i < M; i += nthr) {
          const unsigned long long b = bits[i];
          if (b != ~0ull && (b & mask) == prefix) atomicAdd(&sh[(unsigned)(b >> shift) & dmask], 1u);
        }
        __syncthreads();
        unsigned* Hp = Hc + p * kRsBins;
        for (int j = tid; j <= (int)dmask; j += kRsThreads)
          if (sh[j]) atomicAdd(&Hp[j], sh[j]);
        grid.sync();
        rs_find_bin(Hp, (int)dmask + 1, kk, &s_bin, &s_before, s_part);
        const int bin = s_bin;
        kk -= s_before;
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
          int* nc = &st->ncand[e & 1];
          unsigned long long* cand = st->cand[e & 1];
          for (int i = gtid; i < M; i += nthr) {
            const unsigned long long b = bits[i];
            if (b != ~0ull && (b & mask) == prefix) cand[atomicAdd(nc, 1)] = b;
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
          exact = false;
          __syncthreads();
          break;
        }
      }
      const double v1 = __longlong_as_double((long long)prefix);
      median = v1;
      if (m % 2 == 0) {
        // the next order statistic: v1 again if it repeats, else the smallest larger value
        const int n_le = exact ? (k1 - kk) + cnt_eq : 0;
        if (!exact && v2c != ~0ull) {
          median = (v1 + __longlong_as_double((long long)v2c)) / 2.0;
        } else if (exact && k1 + 1 < n_le) {
          median = v1;
        } else {
          unsigned long long mn = ~0ull;
          for (int i = gtid; i < M; i += nthr) {
            const unsigned long long b = bits[i];
            if (b != ~0ull && b > prefix) mn = min(mn, b);
          }
          for (int off = 16; off > 0; off >>= 1) mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, off));
          if (lane == 0) s_min[warp] = mn;
          __syncthreads();
          if (tid == 0) {
            for (int w = 1; w < kRsThreads / 32; ++w) mn = min(mn, s_min[w]);
            if (mn != ~0ull) atomicMin(&st->vmin[e & 1], mn);
          }
          grid.sync();
          const double v2 = __longlong_as_double((long long)((volatile RegSolveState*)st)->vmin[e & 1]);
          median = (v1 + v2) / 2.0;
        }
      }
    }
    // --- trim, Huber, normal equations
    double acc[30];
#pragma unroll
    for (int q = 0; q < 30; ++q) acc[q] = 0.0;
    if (m > 0) {
      const double thr = fmax(cfg.trim_factor * median, fp);
      for (int i = gtid; i < M; i += nthr)
        if (bits[i] != ~0ull) photo_accum_one(tmp[i], cam, thr, cfg.huber, objective_only, acc);
    }
#pragma unroll
    for (int q = 0; q < 30; ++q) {
      double v = acc[q];
      for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      if (lane == 0) sred[warp][q] = v;
    }
    __syncthreads();
    if (tid < 30) {
      double s = 0.0;
      for (int w = 0; w < kRsThreads / 32; ++w) s += sred[w][tid];
      part[(size_t)blockIdx.x * 32 + tid] = s;
    }
    grid.sync();
    if (blockIdx.x == 0) {
      // 8 strided partial sums per value, combined in a fixed order (deterministic)
      {
        const int q = tid & 31, g = tid >> 5;
        double s = 0.0;
        if (q < 30)
          for (int b = g; b < G; b += kRsThreads / 32) s += part[(size_t)b * 32 + q];
        if (q < 30) sred[g][q] = s;
      }
      __syncthreads();
      if (tid < 30) {
        double s = 0.0;
        for (int g = 0; g < kRsThreads / 32; ++g) s += sred[g][tid];
        sfin[tid] = s;
      }
      __syncthreads();
      if (tid == 0) rs_step(st, cfg, sfin);
    }
  }
}

}  // namespace ss
