// PCA leaf tree of the model points on the device (registration.py:98-164,
// build_leaf_tree / _push_leaf): planar leaves from recursive splits at the
// median projection on the principal axis, stopping when a node is flat
// (lambda_min / lambda_mid <= tau), small (<= leaf_size) or unsplittable.
//
// B200 design: the tree is built level by level.  One 256-thread block per
// node of the level computes, in float64, the mean and biased covariance
// (block reductions), the 3x3 eigen-decomposition (cyclic Jacobi), the exact
// median of the projections (block radix select on order-preserving 64-bit
// keys, 12-bit digits, finished by an in-block rank once <= 256 candidates
// remain) and a stable partition of the node's index segment (left part
// first, original order kept), so every node stays one contiguous segment of
// a permutation array.  The host reads one small record per node per level
// and lays out the next level (a dozen levels at config 3).
//
// The 3x3 eigen-decomposition follows LAPACK's dsyevd path (lapack_eig3.cuh)
// so principal axes carry the reference's signs: the sign decides which child
// receives the median point of an odd-sized split (Jacobi's signs moved 0.7 %
// of the config points and shifted joint-mode poses by 1 cm).  Leaves are
// numbered in level order rather than the reference's depth-first stack
// order (only tie-breaks of the nearest-leaf search can see that).
#include "common.cuh"
#include "lapack_eig3.cuh"

namespace ss {

constexpr int kLtThreads = 256;   // blocks of a level with many nodes
constexpr int kLtThreadsBig = 1024;  // blocks of the top levels (few, large nodes)
constexpr int kLtBins = 4096;
constexpr int kLtCand = 256;

struct LeafRec {
  double c[3], n[3];
  int split, nl, usable, pad;
};

// order-preserving key of a float64
__device__ __forceinline__ unsigned long long okey(double v) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(v);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double okey_inv(unsigned long long k) {
  const unsigned long long u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)u);
}

template <int NT>
__device__ double block_sum_d(double v, double* sred) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  __syncthreads();
  if (lane == 0) sred[warp] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < NT / 32; ++w) s += sred[w];
  return s;
}

// Cyclic Jacobi eigen-decomposition of a symmetric 3x3; ascending eigenvalues, columns of V.
__device__ void eig3(double a[3][3], double w[3], double V[3][3]) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) V[i][j] = i == j ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 60; ++sweep) {
    const double off = a[0][1] * a[0][1] + a[0][2] * a[0][2] + a[1][2] * a[1][2];
    const double dia = a[0][0] * a[0][0] + a[1][1] * a[1][1] + a[2][2] * a[2][2];
    if (off <= 1e-36 * dia || off == 0.0) break;
    for (int pq = 0; pq < 3; ++pq) {
      const int p = pq == 2 ? 1 : 0, q = pq == 0 ? 1 : 2;
      if (a[p][q] == 0.0) continue;
      const double th = (a[q][q] - a[p][p]) / (2.0 * a[p][q]);
      const double t = (th >= 0.0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
      const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
      for (int k = 0; k < 3; ++k) {  // A <- A J
        const double akp = a[k][p], akq = a[k][q];
        a[k][p] = c * akp - s * akq;
        a[k][q] = s * akp + c * akq;
      }
      for (int k = 0; k < 3; ++k) {  // A <- J^T A
        const double apk = a[p][k], aqk = a[q][k];
        a[p][k] = c * apk - s * aqk;
        a[q][k] = s * apk + c * aqk;
      }
      for (int k = 0; k < 3; ++k) {
        const double vkp = V[k][p], vkq = V[k][q];
        V[k][p] = c * vkp - s * vkq;
        V[k][q] = s * vkp + c * vkq;
      }
    }
  }
  int o[3] = {0, 1, 2};
  for (int i = 0; i < 3; ++i)
    for (int j = i + 1; j < 3; ++j)
      if (a[o[j]][o[j]] < a[o[i]][o[i]]) {
        const int t = o[i];
        o[i] = o[j];
        o[j] = t;
      }
  double W[3][3];
  for (int i = 0; i < 3; ++i) {
    w[i] = a[o[i]][o[i]];
    for (int k = 0; k < 3; ++k) W[k][i] = V[k][o[i]];
  }
  for (int i = 0; i < 3; ++i)
    for (int k = 0; k < 3; ++k) V[k][i] = W[k][i];
}

// Block-wide k-th smallest (0-based) of the keys of proj[0, n): returns the key.
// sint: [NT/32] warp partials, then broadcast slots at sint[NT/32 + 0..4].
template <int NT>
__device__ unsigned long long block_select(const double* __restrict__ proj, int n, int k, unsigned* hist,
                                           unsigned long long* cand, int* sint) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  unsigned long long prefix = 0ull, mask = 0ull;
  int kk = k;
  for (int p = 0; p < 6; ++p) {
    const int shift = p < 5 ? 52 - 12 * p : 0;
    const unsigned dmask = p < 5 ? 4095u : 15u;
    for (int j = tid; j < kLtBins; j += NT) hist[j] = 0u;
    __syncthreads();
    for (int j = tid; j < n; j += NT) {
      const unsigned long long key = okey(proj[j]);
      if ((key & mask) == prefix) atomicAdd(&hist[(unsigned)(key >> shift) & dmask], 1u);
    }
    __syncthreads();
    // bin holding rank kk: per-thread runs of 16 bins, block scan
    constexpr int PER = kLtBins / NT;
    unsigned loc = 0;
    for (int j = 0; j < PER; ++j) loc += hist[tid * PER + j];
    unsigned inc = loc;
    for (int off = 1; off < 32; off <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, inc, off);
      if (lane >= off) inc += y;
    }
    if (lane == 31) sint[warp] = (int)inc;
    __syncthreads();
    unsigned run = inc - loc;
    for (int w = 0; w < warp; ++w) run += (unsigned)sint[w];
    if ((unsigned)kk >= run && (unsigned)kk < run + loc) {
      for (int j = 0; j < PER; ++j) {
        const unsigned h = hist[tid * PER + j];
        if ((unsigned)kk < run + h) {
          sint[NT / 32] = tid * PER + j;
          sint[NT / 32 + 1] = (int)run;
          sint[NT / 32 + 2] = (int)h;
          break;
        }
        run += h;
      }
    }
    __syncthreads();
    const int bin = sint[NT / 32], cnt = sint[NT / 32 + 2];
    kk -= sint[NT / 32 + 1];
    prefix |= (unsigned long long)bin << shift;
    mask |= (unsigned long long)dmask << shift;
    __syncthreads();
    if (p == 5) return prefix;
    if (cnt <= kLtCand) {  // gather the few keys sharing the prefix and rank them
      if (tid == 0) sint[NT / 32 + 3] = 0;
      __syncthreads();
      for (int j = tid; j < n; j += NT) {
        const unsigned long long key = okey(proj[j]);
        if ((key & mask) == prefix) cand[atomicAdd(&sint[NT / 32 + 3], 1)] = key;
      }
      __syncthreads();
      for (int j = tid; j < cnt; j += NT) {
        const unsigned long long c = cand[j];
        int rank = 0;
        for (int q = 0; q < cnt; ++q) rank += (cand[q] < c) | ((cand[q] == c) & (q < j));
        if (rank == kk) sint[NT / 32 + 4] = j;
      }
      __syncthreads();
      const unsigned long long r = cand[sint[NT / 32 + 4]];
      __syncthreads();
      return r;
    }
  }
  return prefix;
}

// One node of a level by one block of NT threads (record -> out[node]).
template <int NT>
__device__ void leaf_node(int node, const double* __restrict__ pts, int* __restrict__ idx, int* __restrict__ tmp,
                          double* __restrict__ proj, const int2* __restrict__ nodes, double3 viewpoint,
                          int leaf_size, double tau, LeafRec* __restrict__ out) {
  __shared__ double sred[NT / 32];
  __shared__ double s_axis[3], s_n[3], s_w[3];
  __shared__ unsigned hist[kLtBins];
  __shared__ unsigned long long cand[kLtCand];
  __shared__ int sint[2 * (NT / 32) + 8];
  const int2 nd = nodes[node];
  const int b = nd.x, n = nd.y - nd.x;
  const int tid = threadIdx.x;
  // mean (registration.py:121)
  double sx = 0.0, sy = 0.0, sz = 0.0;
  for (int j = tid; j < n; j += NT) {
    const int i = idx[b + j];
    sx += pts[3 * i];
    sy += pts[3 * i + 1];
    sz += pts[3 * i + 2];
  }
  sx = block_sum_d<NT>(sx, sred);
  sy = block_sum_d<NT>(sy, sred);
  sz = block_sum_d<NT>(sz, sred);
  const double c[3] = {sx / n, sy / n, sz / n};
  LeafRec rec{};
  rec.c[0] = c[0];
  rec.c[1] = c[1];
  rec.c[2] = c[2];
  if (n < 3) {  // (:122-124)
    if (tid == 0) out[node] = rec;
    return;
  }
  // biased covariance (:125)
  double q[6] = {0, 0, 0, 0, 0, 0};
  for (int j = tid; j < n; j += NT) {
    const int i = idx[b + j];
    const double dx = pts[3 * i] - c[0], dy = pts[3 * i + 1] - c[1], dz = pts[3 * i + 2] - c[2];
    q[0] += dx * dx;
    q[1] += dx * dy;
    q[2] += dx * dz;
    q[3] += dy * dy;
    q[4] += dy * dz;
    q[5] += dz * dz;
  }
  for (int k = 0; k < 6; ++k) q[k] = block_sum_d<NT>(q[k], sred) / n;
  if (tid == 0) {
    const double a[3][3] = {{q[0], q[1], q[2]}, {q[1], q[3], q[4]}, {q[2], q[4], q[5]}};
    double w[3], V[3][3];
    if (!lapack3::eigh3(a, w, V)) {  // (dsteqr did not converge: not seen on covariances) -> Jacobi
      double aj[3][3] = {{q[0], q[1], q[2]}, {q[1], q[3], q[4]}, {q[2], q[4], q[5]}};
      eig3(aj, w, V);
    }
    for (int k = 0; k < 3; ++k) {
      s_w[k] = w[k];
      s_n[k] = V[k][0];
      s_axis[k] = V[k][2];
    }
  }
  __syncthreads();
  const double w0 = s_w[0], w1 = s_w[1];
  const bool flat = w1 <= 1e-12 || w0 / w1 <= tau;  // (:127)
  auto emit_leaf = [&](bool has_normal) {
    if (tid != 0) return;
    if (has_normal) {  // oriented toward the viewpoint (:151-160)
      double nn[3] = {s_n[0], s_n[1], s_n[2]};
      const double d = nn[0] * (viewpoint.x - c[0]) + nn[1] * (viewpoint.y - c[1]) + nn[2] * (viewpoint.z - c[2]);
      if (d < 0.0)
        for (int k = 0; k < 3; ++k) nn[k] = -nn[k];
      for (int k = 0; k < 3; ++k) rec.n[k] = nn[k];
      rec.usable = 1;
    }
    out[node] = rec;
  };
  if (flat || n <= leaf_size) {  // (:128-131)
    emit_leaf(w1 > 1e-12);
    return;
  }
  // projections on the principal axis and their median (:132-134)
  for (int j = tid; j < n; j += NT) {
    const int i = idx[b + j];
    proj[b + j] = (pts[3 * i] - c[0]) * s_axis[0] + (pts[3 * i + 1] - c[1]) * s_axis[1] +
                  (pts[3 * i + 2] - c[2]) * s_axis[2];
  }
  __syncthreads();
  const double* pr = proj + b;
  const int k1 = (n % 2 == 0) ? n / 2 - 1 : n / 2;
  const unsigned long long key1 = block_select<NT>(pr, n, k1, hist, cand, sint);
  double med = okey_inv(key1);
  if (n % 2 == 0) {
    // second middle value: key1 again if repeated, else the smallest larger key
    int le = 0;
    unsigned long long mn = ~0ull;
    for (int j = tid; j < n; j += NT) {
      const unsigned long long key = okey(pr[j]);
      le += key <= key1;
      if (key > key1) mn = min(mn, key);
    }
    for (int off = 16; off > 0; off >>= 1) {
      le += __shfl_xor_sync(0xffffffffu, le, off);
      mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, off));
    }
    __syncthreads();
    if ((tid & 31) == 0) {
      sint[tid >> 5] = le;
      cand[tid >> 5] = mn;
    }
    __syncthreads();
    le = 0;
    mn = ~0ull;
    for (int w = 0; w < NT / 32; ++w) {
      le += sint[w];
      mn = min(mn, cand[w]);
    }
    const double v2 = le > k1 + 1 ? med : okey_inv(mn);
    med = (med + v2) / 2.0;
    __syncthreads();
  }
  // left = proj <= med (:135); stable partition of the segment
  int nl = 0;
  for (int j = tid; j < n; j += NT) nl += pr[j] <= med;
  for (int off = 16; off > 0; off >>= 1) nl += __shfl_xor_sync(0xffffffffu, nl, off);
  __syncthreads();
  if ((tid & 31) == 0) sint[tid >> 5] = nl;
  __syncthreads();
  nl = 0;
  for (int w = 0; w < NT / 32; ++w) nl += sint[w];
  __syncthreads();
  if (nl == 0 || nl == n) {  // (:136-139)
    emit_leaf(true);
    return;
  }
  int base_l = 0, base_r = nl;
  const int lane = tid & 31, warp = tid >> 5;
  for (int s0 = 0; s0 < n; s0 += NT) {
    const int j = s0 + tid;
    const bool in = j < n;
    const bool left = in && pr[j] <= med;
    const unsigned bl = __ballot_sync(0xffffffffu, left), br = __ballot_sync(0xffffffffu, in && !left);
    if (lane == 0) {
      sint[warp] = __popc(bl);
      sint[NT / 32 + warp] = __popc(br);
    }
    __syncthreads();
    int ol = base_l, orr = base_r, tl = 0, tr = 0;
    for (int w = 0; w < NT / 32; ++w) {
      if (w < warp) {
        ol += sint[w];
        orr += sint[NT / 32 + w];
      }
      tl += sint[w];
      tr += sint[NT / 32 + w];
    }
    const unsigned lt = (1u << lane) - 1u;
    if (in) tmp[b + (left ? ol + __popc(bl & lt) : orr + __popc(br & lt))] = idx[b + j];
    base_l += tl;
    base_r += tr;
    __syncthreads();
  }
  for (int j = tid; j < n; j += NT) idx[b + j] = tmp[b + j];
  if (tid == 0) {
    rec.split = 1;
    rec.nl = nl;
    out[node] = rec;
  }
}

template <int NT>
__global__ void __launch_bounds__(NT) k_leaf_level(const double* __restrict__ pts, int* __restrict__ idx,
                                                   int* __restrict__ tmp, double* __restrict__ proj,
                                                   const int2* __restrict__ nodes, const int* __restrict__ n_nodes,
                                                   double3 viewpoint, int leaf_size, double tau,
                                                   LeafRec* __restrict__ out) {
  if ((int)blockIdx.x >= *n_nodes) return;  // grid sized by a bound on the level's node count
  leaf_node<NT>(blockIdx.x, pts, idx, tmp, proj, nodes, viewpoint, leaf_size, tau, out);
}

// Lay out the next level (children of split nodes, in node order) and append
// this level's leaves (in node order): one block of NT threads, counts scanned
// per thread run.
template <int NT>
__device__ void next_level_block(const int2* __restrict__ cur, int n_cur, const LeafRec* __restrict__ recs,
                                 int2* __restrict__ next, int* __restrict__ n_next_p, int2* __restrict__ leaf_seg,
                                 LeafRec* __restrict__ leaf_rec, int* __restrict__ n_leaves_p, int max_leaves,
                                 int* __restrict__ overflow) {
  __shared__ int s_c[NT], s_l[NT];
  const int tid = threadIdx.x;
  const int per = (n_cur + NT - 1) / NT;
  const int b = min(tid * per, n_cur), e = min(b + per, n_cur);
  int nc = 0, nl = 0;
  for (int i = b; i < e; ++i) {
    if (recs[i].split)
      nc += 2;
    else
      ++nl;
  }
  s_c[tid] = nc;
  s_l[tid] = nl;
  __syncthreads();
  for (int off = 1; off < NT; off <<= 1) {
    const int vc = tid >= off ? s_c[tid - off] : 0, vl = tid >= off ? s_l[tid - off] : 0;
    __syncthreads();
    s_c[tid] += vc;
    s_l[tid] += vl;
    __syncthreads();
  }
  const int leaf0 = *n_leaves_p;
  int oc = s_c[tid] - nc, ol = leaf0 + s_l[tid] - nl;
  for (int i = b; i < e; ++i) {
    const int2 nd = cur[i];
    const LeafRec& r = recs[i];
    if (r.split) {
      next[oc++] = make_int2(nd.x, nd.x + r.nl);
      next[oc++] = make_int2(nd.x + r.nl, nd.y);
    } else if (ol < max_leaves) {
      leaf_seg[ol] = nd;
      leaf_rec[ol] = r;
      ++ol;
    } else {
      *overflow = 1;
    }
  }
  __syncthreads();
  if (tid == NT - 1) {
    *n_next_p = s_c[NT - 1];
    *n_leaves_p = leaf0 + s_l[NT - 1];
  }
  __syncthreads();
}

__global__ void __launch_bounds__(1024) k_next_level(const int2* __restrict__ cur, const int* __restrict__ n_cur_p,
                                                     const LeafRec* __restrict__ recs, int2* __restrict__ next,
                                                     int* __restrict__ n_next_p, int2* __restrict__ leaf_seg,
                                                     LeafRec* __restrict__ leaf_rec, int* __restrict__ n_leaves_p,
                                                     int max_leaves, int* __restrict__ overflow) {
  next_level_block<1024>(cur, *n_cur_p, recs, next, n_next_p, leaf_seg, leaf_rec, n_leaves_p, max_leaves, overflow);
}

// point -> leaf: blockIdx.x = leaf, blockIdx.y = 1024-point chunk of its segment
// (flat leaves stop splitting early and can hold tens of thousands of points)
__global__ void k_leaf_assign(const int* __restrict__ idx, const int2* __restrict__ leaves, int nleaves,
                              int* __restrict__ point_leaf) {
  const int l = blockIdx.x;
  if (l >= nleaves) return;
  const int2 s = leaves[l];
  const int j0 = s.x + blockIdx.y * 1024;
  for (int j = j0 + threadIdx.x; j < min(s.y, j0 + 1024); j += blockDim.x) point_leaf[idx[j]] = l;
}

__global__ void k_iota(int n, int* __restrict__ v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = i;
}

}  // namespace ss
