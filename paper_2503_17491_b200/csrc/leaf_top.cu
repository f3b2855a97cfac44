// Top levels of the PCA leaf tree (registration.py:98-164) in ONE cooperative
// kernel.  The per-node kernel of leaf_tree.cu gives each node one block, so
// the first levels -- one node of all the model points, then 2, 4, ... --
// ran on a handful of SMs at a single SM's bandwidth (1.4 ms of a 2.2 ms
// build at config 3; the host runs levels 0-4 here, 1.73 -> 0.73 ms per build).  Here every block of the grid works on every level: a
// level's nodes get blocks in proportion to their sizes (at least one each),
// each block takes a contiguous chunk of its node's index segment, and the
// node-wide quantities are combined across the node's blocks between grid
// barriers:
//   mean, biased covariance        per-block partial sums, summed in block order
//   3x3 eigen-decomposition        redundantly per block (same inputs, same result)
//   median projection              radix select on order-preserving keys with
//                                  per-node global histograms; passes start at the
//                                  highest bit where the node's smallest and largest
//                                  keys differ, finished by an exact rank of <= 256
//                                  gathered candidates
//   stable partition               per-block left counts -> offsets, ballot scatter
// Decisions, records and the next level's layout follow leaf_tree.cu exactly
// (same leaf order, same stable partition); only float64 summation order differs.
#include <cooperative_groups.h>

namespace ss {

#ifdef SS_RS_PROF
#define LT_MARK(q)                                                 \
  if (b == 0 && tid == 0) {                                        \
    unsigned long long t_;                                         \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));         \
    lt_prof[q] += t_ - lt_last;                                    \
    lt_last = t_;                                                  \
  }
#else
#define LT_MARK(q)
#endif

constexpr int kLtTopThreads = 512;
constexpr int kLtTopMaxNodes = 128;  // levels run here while 2^level <= this (and < the grid)

struct LtTopWs {
  double* part;              // [G][9] per-block partial sums: mean [0:3], covariance [3:9]
  unsigned long long* pmm;   // [G][2] per-block key min / max
  int* pcnt;                 // [G] per-block left counts
  unsigned* hist;            // [3][kLtTopMaxNodes][kLtBins] rotating per-node histograms
  unsigned long long* cand;  // [kLtTopMaxNodes][kLtCand]
  int* ncand;                // [kLtTopMaxNodes]
  unsigned long long* vmin;  // [kLtTopMaxNodes]
  int* more;                 // [2] nodes still selecting after a round
};

inline size_t lt_top_ws_bytes(int G) {
  return (size_t)G * (9 * 8 + 16 + 4) + (size_t)3 * kLtTopMaxNodes * kLtBins * 4 +
         (size_t)kLtTopMaxNodes * (kLtCand * 8 + 4 + 8) + 8 + 256;
}

template <int NT>
__device__ __forceinline__ double lt_block_sum(double v, double* sred) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  __syncthreads();
  if (lane == 0) sred[warp] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < NT / 32; ++w) s += sred[w];
  return s;
}

__global__ void __launch_bounds__(kLtTopThreads, 1)
    k_leaf_top(const double* __restrict__ pts, int* __restrict__ idx, int* __restrict__ tmp, double* __restrict__ proj,
               int2* __restrict__ nodes0, int2* __restrict__ nodes1, int* __restrict__ counts,
               LeafRec* __restrict__ recs, int2* __restrict__ leaf_seg, LeafRec* __restrict__ leaf_rec,
               int cap_leaves, double3 vp, int leaf_size, double tau, int levels, LtTopWs ws) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  constexpr int NT = kLtTopThreads, NW = NT / 32;
  __shared__ unsigned sh[kLtBins];
  __shared__ double sred[NW];
  __shared__ int2 s_nd[kLtTopMaxNodes];
  __shared__ int s_bst[kLtTopMaxNodes + 1];
  __shared__ int s_node, s_j, s_nb;
  __shared__ double s_c[3], s_axis[3], s_n[3], s_w[2];
  __shared__ int sint[2 * NW + 8];
  __shared__ unsigned long long s_mm[2 * NW];
  const int G = gridDim.x, b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#ifdef SS_RS_PROF
  unsigned long long lt_prof[12] = {}, lt_last = 0;
  if (b == 0 && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(lt_last));
#endif
  for (int level = 0; level < levels; ++level) {
    const int par = level & 1;
    int2* cur = par ? nodes1 : nodes0;
    int2* nxt = par ? nodes0 : nodes1;
    const int K = ((volatile int*)counts)[par];
    if (K == 0) {  // (uniform) the tree is complete: the host's next level must see no nodes either
      if (b == 0 && tid == 0) counts[par ^ 1] = 0;
      break;
    }
    // --- blocks -> nodes: one each, the rest in proportion to node size
    for (int k = tid; k < K; k += NT) s_nd[k] = cur[k];
    __syncthreads();
    if (tid == 0) {
      long long T = 0;
      for (int k = 0; k < K; ++k) T += s_nd[k].y - s_nd[k].x;
      long long P = 0;
      for (int k = 0; k < K; ++k) {
        s_bst[k] = k + (int)(T > 0 ? (long long)(G - K) * P / T : 0);
        P += s_nd[k].y - s_nd[k].x;
      }
      s_bst[K] = G;
      int k = 0;
      while (k + 1 < K && s_bst[k + 1] <= b) ++k;
      s_node = k;
      s_j = b - s_bst[k];
      s_nb = s_bst[k + 1] - s_bst[k];
    }
    __syncthreads();
    LT_MARK(0);
    const int k = s_node, j = s_nb > 0 ? s_j : 0, nb = max(s_nb, 1), b0 = s_bst[k];
    const int x = s_nd[k].x, n = s_nd[k].y - s_nd[k].x;
    const int c0 = x + (int)((long long)n * j / nb), c1 = x + (int)((long long)n * (j + 1) / nb);
    unsigned* Hn[3];
    for (int q = 0; q < 3; ++q) Hn[q] = ws.hist + ((size_t)q * kLtTopMaxNodes + k) * kLtBins;
    // --- S1: mean partials; clear the node's first histogram and candidate state
    {
      double sx = 0.0, sy = 0.0, sz = 0.0;
      for (int p = c0 + tid; p < c1; p += NT) {
        const int i = idx[p];
        sx += pts[3 * i];
        sy += pts[3 * i + 1];
        sz += pts[3 * i + 2];
      }
      sx = lt_block_sum<NT>(sx, sred);
      sy = lt_block_sum<NT>(sy, sred);
      sz = lt_block_sum<NT>(sz, sred);
      if (tid == 0) {
        ws.part[9 * b] = sx;
        ws.part[9 * b + 1] = sy;
        ws.part[9 * b + 2] = sz;
      }
      for (int q = j * NT + tid; q < kLtBins; q += nb * NT) Hn[0][q] = 0u;
      if (j == 0 && tid == 0) {
        ws.ncand[k] = 0;
        ws.vmin[k] = ~0ull;
      }
      if (b == 0 && tid == 0) ws.more[0] = ws.more[1] = 0;
    }
    LT_MARK(1);
    grid.sync();
    LT_MARK(2);
    // --- S2: mean, covariance partials
    if (warp == 0) {  // node sums of the block partials: lane-strided, fixed butterfly (deterministic)
      double sx = 0.0, sy = 0.0, sz = 0.0;
      for (int r = lane; r < nb; r += 32) {
        sx += ws.part[9 * (b0 + r)];
        sy += ws.part[9 * (b0 + r) + 1];
        sz += ws.part[9 * (b0 + r) + 2];
      }
      for (int off = 16; off > 0; off >>= 1) {
        sx += __shfl_xor_sync(0xffffffffu, sx, off);
        sy += __shfl_xor_sync(0xffffffffu, sy, off);
        sz += __shfl_xor_sync(0xffffffffu, sz, off);
      }
      if (lane == 0) {
        s_c[0] = sx / n;
        s_c[1] = sy / n;
        s_c[2] = sz / n;
      }
    }
    __syncthreads();
    const double c[3] = {s_c[0], s_c[1], s_c[2]};
    bool done = n < 3;  // (:122-124) centroid only, no normal
    {
      double q6[6] = {0, 0, 0, 0, 0, 0};
      if (!done)
        for (int p = c0 + tid; p < c1; p += NT) {
          const int i = idx[p];
          const double dx = pts[3 * i] - c[0], dy = pts[3 * i + 1] - c[1], dz = pts[3 * i + 2] - c[2];
          q6[0] += dx * dx;
          q6[1] += dx * dy;
          q6[2] += dx * dz;
          q6[3] += dy * dy;
          q6[4] += dy * dz;
          q6[5] += dz * dz;
        }
      for (int q = 0; q < 6; ++q) q6[q] = lt_block_sum<NT>(q6[q], sred);
      if (tid == 0)
        for (int q = 0; q < 6; ++q) ws.part[9 * b + 3 + q] = q6[q];
    }
    LT_MARK(3);
    grid.sync();
    LT_MARK(2);
    // --- S3: covariance, eigenvectors, leaf test, projections and their key range
    LeafRec rec{};
    rec.c[0] = c[0];
    rec.c[1] = c[1];
    rec.c[2] = c[2];
    if (!done && warp == 0) {
      double q6[6] = {0, 0, 0, 0, 0, 0};
      for (int r = lane; r < nb; r += 32)
        for (int q = 0; q < 6; ++q) q6[q] += ws.part[9 * (b0 + r) + 3 + q];
      for (int off = 16; off > 0; off >>= 1)
        for (int q = 0; q < 6; ++q) q6[q] += __shfl_xor_sync(0xffffffffu, q6[q], off);
      for (int q = 0; q < 6; ++q) q6[q] /= n;
      if (lane == 0) {
        const double a[3][3] = {{q6[0], q6[1], q6[2]}, {q6[1], q6[3], q6[4]}, {q6[2], q6[4], q6[5]}};
        double w[3], V[3][3];
        if (!lapack3::eigh3(a, w, V)) {
          double aj[3][3] = {{q6[0], q6[1], q6[2]}, {q6[1], q6[3], q6[4]}, {q6[2], q6[4], q6[5]}};
          eig3(aj, w, V);
        }
        for (int q = 0; q < 3; ++q) {
          s_n[q] = V[q][0];
          s_axis[q] = V[q][2];
        }
        s_w[0] = w[0];
        s_w[1] = w[1];
      }
    }
    __syncthreads();
    LT_MARK(4);
    auto leaf_record = [&](bool has_normal) {
      if (has_normal) {  // oriented toward the viewpoint (:151-160)
        double nn[3] = {s_n[0], s_n[1], s_n[2]};
        const double d = nn[0] * (vp.x - c[0]) + nn[1] * (vp.y - c[1]) + nn[2] * (vp.z - c[2]);
        if (d < 0.0)
          for (int q = 0; q < 3; ++q) nn[q] = -nn[q];
        for (int q = 0; q < 3; ++q) rec.n[q] = nn[q];
        rec.usable = 1;
      }
    };
    if (done) {
      if (j == 0 && tid == 0) recs[k] = rec;
    } else {
      const double w0 = s_w[0], w1 = s_w[1];
      if ((w1 <= 1e-12 || w0 / w1 <= tau) || n <= leaf_size) {  // (:127-131)
        done = true;
        leaf_record(w1 > 1e-12);
        if (j == 0 && tid == 0) recs[k] = rec;
      }
    }
    unsigned long long kmn = ~0ull, kmx = 0ull;
    if (!done) {
      const double a0 = s_axis[0], a1 = s_axis[1], a2 = s_axis[2];
      for (int p = c0 + tid; p < c1; p += NT) {
        const int i = idx[p];
        const double v = (pts[3 * i] - c[0]) * a0 + (pts[3 * i + 1] - c[1]) * a1 + (pts[3 * i + 2] - c[2]) * a2;
        proj[p] = v;
        const unsigned long long key = okey(v);
        kmn = min(kmn, key);
        kmx = max(kmx, key);
      }
    }
    for (int off = 16; off > 0; off >>= 1) {
      kmn = min(kmn, __shfl_xor_sync(0xffffffffu, kmn, off));
      kmx = max(kmx, __shfl_xor_sync(0xffffffffu, kmx, off));
    }
    if (lane == 0) {
      s_mm[2 * warp] = kmn;
      s_mm[2 * warp + 1] = kmx;
    }
    __syncthreads();
    if (tid == 0) {
      for (int w = 0; w < NW; ++w) {
        kmn = min(kmn, s_mm[2 * w]);
        kmx = max(kmx, s_mm[2 * w + 1]);
      }
      ws.pmm[2 * b] = kmn;
      ws.pmm[2 * b + 1] = kmx;
    }
    LT_MARK(5);
    grid.sync();
    LT_MARK(2);
    // --- S4: median of the projections (:132-134), rounds of radix passes
    if (warp == 0) {
      kmn = ~0ull;
      kmx = 0ull;
      for (int r = lane; r < nb; r += 32) {
        kmn = min(kmn, ws.pmm[2 * (b0 + r)]);
        kmx = max(kmx, ws.pmm[2 * (b0 + r) + 1]);
      }
      for (int off = 16; off > 0; off >>= 1) {
        kmn = min(kmn, __shfl_xor_sync(0xffffffffu, kmn, off));
        kmx = max(kmx, __shfl_xor_sync(0xffffffffu, kmx, off));
      }
      if (lane == 0) {
        s_mm[0] = kmn;
        s_mm[1] = kmx;
      }
    }
    __syncthreads();
    kmn = s_mm[0];
    kmx = s_mm[1];
    __syncthreads();
    const int k1 = (n % 2 == 0) ? n / 2 - 1 : n / 2;
    int kk = k1, cnt_eq = 0, top = kmn == kmx ? -1 : 63 - __clzll(kmn ^ kmx);
    unsigned long long mask = top < 0 ? ~0ull : (top == 63 ? 0ull : ~((2ull << top) - 1ull));
    unsigned long long prefix = kmn & mask;
    bool exact = top < 0, selecting = !done && top >= 0;
    unsigned long long v2c = ~0ull;
    if (!done && top < 0) cnt_eq = n;  // every key equal
    for (int round = 0;; ++round) {
      const int lo = max(top - 11, 0);
      const unsigned dmask = selecting ? (1u << (top - lo + 1)) - 1u : 0u;
      unsigned* H = Hn[round % 3];
      bool gathering = false;
      int cnt_bin = 0;
      if (selecting) {
        for (int q = tid; q <= (int)dmask; q += NT) sh[q] = 0u;
        __syncthreads();
        for (int p = c0 + tid; p < c1; p += NT) {
          const unsigned long long key = okey(proj[p]);
          if ((key & mask) == prefix) atomicAdd(&sh[(unsigned)(key >> lo) & dmask], 1u);
        }
        __syncthreads();
        for (int q = tid; q <= (int)dmask; q += NT)
          if (sh[q]) atomicAdd(&H[q], sh[q]);
        for (int q = j * NT + tid; q < kLtBins; q += nb * NT) Hn[(round + 1) % 3][q] = 0u;
      }
      LT_MARK(6);
      grid.sync();
      LT_MARK(2);
      if (selecting) {
        // bin of H holding rank kk (per-thread runs of PER bins, block scan)
        constexpr int PER = kLtBins / NT;
        unsigned loc[PER], sum = 0;
#pragma unroll
        for (int q = 0; q < PER; ++q) {
          const int bin = tid * PER + q;
          loc[q] = bin <= (int)dmask ? ((volatile unsigned*)H)[bin] : 0u;
          sum += loc[q];
        }
        unsigned inc = sum;
        for (int off = 1; off < 32; off <<= 1) {
          const unsigned y = __shfl_up_sync(0xffffffffu, inc, off);
          if (lane >= off) inc += y;
        }
        if (lane == 31) sint[warp] = (int)inc;
        __syncthreads();
        unsigned run = inc - sum;
        for (int w = 0; w < warp; ++w) run += (unsigned)sint[w];
        if ((unsigned)kk >= run && (unsigned)kk < run + sum) {
#pragma unroll
          for (int q = 0; q < PER; ++q) {
            if ((unsigned)kk < run + loc[q]) {
              sint[NW] = tid * PER + q;
              sint[NW + 1] = (int)run;
              sint[NW + 2] = (int)loc[q];
              break;
            }
            run += loc[q];
          }
        }
        __syncthreads();
        const int bin = sint[NW];
        kk -= sint[NW + 1];
        cnt_bin = sint[NW + 2];
        prefix |= (unsigned long long)bin << lo;
        mask |= (unsigned long long)dmask << lo;
        __syncthreads();
        if (lo == 0) {
          cnt_eq = cnt_bin;
          exact = true;
          selecting = false;
        } else if (cnt_bin <= kLtCand) {
          gathering = true;
          for (int p = c0 + tid; p < c1; p += NT) {
            const unsigned long long key = okey(proj[p]);
            if ((key & mask) == prefix) ws.cand[(size_t)k * kLtCand + atomicAdd(&ws.ncand[k], 1)] = key;
          }
          selecting = false;
        } else {
          top = lo - 1;
          if (j == 0 && tid == 0) atomicAdd(&ws.more[round & 1], 1);
        }
      }
      if (b == 0 && tid == 0) ws.more[(round + 1) & 1] = 0;
      LT_MARK(7);
      grid.sync();
      LT_MARK(2);
      if (gathering) {  // rank the candidates exactly (every block of the node, same result)
        const unsigned long long* cd = ws.cand + (size_t)k * kLtCand;
        if (tid == 0) {
          sint[NW + 3] = -1;
          sint[NW + 4] = -1;
        }
        __syncthreads();
        for (int q = tid; q < cnt_bin; q += NT) {
          const unsigned long long cq = ((volatile const unsigned long long*)cd)[q];
          int lt = 0, eqb = 0;
          for (int t = 0; t < cnt_bin; ++t) {
            const unsigned long long ct = ((volatile const unsigned long long*)cd)[t];
            lt += ct < cq;
            eqb += (ct == cq) & (t < q);
          }
          const int rank = lt + eqb;
          if (rank == kk) sint[NW + 3] = q;
          if (rank == kk + 1) sint[NW + 4] = q;
        }
        __syncthreads();
        prefix = ((volatile const unsigned long long*)cd)[sint[NW + 3]];
        v2c = sint[NW + 4] < 0 ? ~0ull : ((volatile const unsigned long long*)cd)[sint[NW + 4]];
        __syncthreads();
      }
      if (((volatile int*)ws.more)[round & 1] == 0) break;  // (uniform: read after the barrier)
    }
    LT_MARK(8);
    // second middle value for even sizes: v1 again if repeated, else the smallest larger key
    double med = 0.0;
    bool need_min = false;
    if (!done) {
      med = okey_inv(prefix);
      if (n % 2 == 0) {
        if (!exact && v2c != ~0ull)
          med = (med + okey_inv(v2c)) / 2.0;
        else if (!(exact && k1 + 1 < (k1 - kk) + cnt_eq))
          need_min = true;
      }
      if (need_min) {
        unsigned long long mn = ~0ull;
        for (int p = c0 + tid; p < c1; p += NT) {
          const unsigned long long key = okey(proj[p]);
          if (key > prefix) mn = min(mn, key);
        }
        for (int off = 16; off > 0; off >>= 1) mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, off));
        if (lane == 0) s_mm[warp] = mn;
        __syncthreads();
        if (tid == 0) {
          for (int w = 0; w < NW; ++w) mn = min(mn, s_mm[w]);
          if (mn != ~0ull) atomicMin(&ws.vmin[k], mn);
        }
      }
    }
    LT_MARK(9);
    grid.sync();
    LT_MARK(2);
    if (need_min) med = (med + okey_inv(((volatile unsigned long long*)ws.vmin)[k])) / 2.0;
    // --- S5: left = proj <= med (:135), counts per block
    {
      int nl = 0;
      if (!done)
        for (int p = c0 + tid; p < c1; p += NT) nl += proj[p] <= med;
      nl = __reduce_add_sync(0xffffffffu, nl);
      if (lane == 0) sint[warp] = nl;
      __syncthreads();
      if (tid == 0) {
        int t = 0;
        for (int w = 0; w < NW; ++w) t += sint[w];
        ws.pcnt[b] = t;
      }
    }
    LT_MARK(10);
    grid.sync();
    LT_MARK(2);
    bool split = false;
    if (!done) {
      if (warp == 0) {
        int bf = 0, tot = 0;
        for (int r = lane; r < nb; r += 32) {
          const int v = ws.pcnt[b0 + r];
          bf += r < j ? v : 0;
          tot += v;
        }
        bf = __reduce_add_sync(0xffffffffu, bf);
        tot = __reduce_add_sync(0xffffffffu, tot);
        if (lane == 0) {
          sint[2 * NW] = bf;
          sint[2 * NW + 1] = tot;
        }
      }
      __syncthreads();
      const int before = sint[2 * NW], nl = sint[2 * NW + 1];
      __syncthreads();
      if (nl == 0 || nl == n) {  // (:136-139)
        leaf_record(true);
        if (j == 0 && tid == 0) recs[k] = rec;
      } else {
        split = true;
        int base_l = x + before, base_r = x + nl + (c0 - x - before);
        for (int s0 = c0; s0 < c1; s0 += NT) {
          const int p = s0 + tid;
          const bool in = p < c1;
          const bool left = in && proj[p] <= med;
          const unsigned bl = __ballot_sync(0xffffffffu, left), br = __ballot_sync(0xffffffffu, in && !left);
          __syncthreads();
          if (lane == 0) {
            sint[warp] = __popc(bl);
            sint[NW + warp] = __popc(br);
          }
          __syncthreads();
          int ol = base_l, orr = base_r, tl = 0, tr = 0;
          for (int w = 0; w < NW; ++w) {
            if (w < warp) {
              ol += sint[w];
              orr += sint[NW + w];
            }
            tl += sint[w];
            tr += sint[NW + w];
          }
          const unsigned lt = (1u << lane) - 1u;
          if (in) tmp[left ? ol + __popc(bl & lt) : orr + __popc(br & lt)] = idx[p];
          base_l += tl;
          base_r += tr;
        }
        if (j == 0 && tid == 0) {
          rec.split = 1;
          rec.nl = nl;
          recs[k] = rec;
        }
      }
    }
    LT_MARK(11);
    grid.sync();
    LT_MARK(2);
    // --- S6: copy the partitioned chunk back; block 0 lays out the next level
    if (split)
      for (int p = c0 + tid; p < c1; p += NT) idx[p] = tmp[p];
    if (b == 0 && tid == 0) {
      int nn = 0, nlv = counts[2];
      for (int q = 0; q < K; ++q) {
        const LeafRec r = recs[q];
        const int2 nd = s_nd[q];
        if (r.split) {
          nxt[nn++] = make_int2(nd.x, nd.x + r.nl);
          nxt[nn++] = make_int2(nd.x + r.nl, nd.y);
        } else if (nlv < cap_leaves) {
          leaf_seg[nlv] = nd;
          leaf_rec[nlv] = r;
          ++nlv;
        } else {
          counts[3] = 1;
        }
      }
      counts[par ^ 1] = nn;
      counts[2] = nlv;
    }
    grid.sync();
    LT_MARK(2);
  }
#ifdef SS_RS_PROF
  if (b == 0 && tid == 0)
    printf("LTPROF setup %llu s1 %llu syncs %llu s2 %llu eig %llu proj %llu hist %llu find+gather %llu rank %llu "
           "vmin %llu nl %llu scatter %llu\n", lt_prof[0], lt_prof[1], lt_prof[2], lt_prof[3], lt_prof[4],
           lt_prof[5], lt_prof[6], lt_prof[7], lt_prof[8], lt_prof[9], lt_prof[10], lt_prof[11]);
#endif
}

// The remaining levels (many nodes) in one cooperative kernel: each block takes
// nodes grid-stride, one node at a time (leaf_node, as k_leaf_level does),
// block 0 lays out the next level between grid barriers.  Runs until a level
// has no node (or max_levels); counts[4] = the first level not processed.
__global__ void __launch_bounds__(kLtTopThreads, 1)
    k_leaf_rest(const double* __restrict__ pts, int* __restrict__ idx, int* __restrict__ tmp, double* __restrict__ proj,
                int2* __restrict__ nodes0, int2* __restrict__ nodes1, int* __restrict__ counts,
                LeafRec* __restrict__ recs, int2* __restrict__ leaf_seg, LeafRec* __restrict__ leaf_rec,
                int cap_leaves, double3 vp, int leaf_size, double tau, int level0, int max_levels) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  int level = level0;
  for (; level < level0 + max_levels; ++level) {
    const int par = level & 1;
    const int2* cur = par ? nodes1 : nodes0;
    int2* nxt = par ? nodes0 : nodes1;
    const int K = ((volatile int*)counts)[par];
    if (K == 0) break;  // (uniform)
    for (int node = blockIdx.x; node < K; node += gridDim.x) {
      leaf_node<kLtTopThreads>(node, pts, idx, tmp, proj, cur, vp, leaf_size, tau, recs);
      __syncthreads();  // (leaf_node's shared memory is reused by the next node)
    }
    grid.sync();
    if (blockIdx.x == 0)
      next_level_block<kLtTopThreads>(cur, K, recs, nxt, counts + (par ^ 1), leaf_seg, leaf_rec, counts + 2,
                                      cap_leaves, counts + 3);
    grid.sync();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) counts[4] = level;
}

}  // namespace ss
