// Segment-parallel forward for renders with few, long tile lists (config 2:
// 1,024 tiles of ~1,000 entries against ~2,400 resident warps).
//
// Reference behaviour: rasterizer.py:402-452 (_chunk_transmittance and the
// blend loop of _render_tile_lists).  Entry k of a pixel's list contributes
// iff its transmittance before it, T_before(k) = prod_{m<k} (1 - alpha_m),
// is >= min_transmittance; the blend is front to back.  The only carried
// state is T, so a list cut into segments of kSegChunks x 32 entries can be
// blended segment by segment in parallel and combined afterwards:
//
//   pass 1 (k_fwd_seg<1>)     every (tile, segment) slot, one warp each: the
//                             segment's blend of every pixel from T = 1, no
//                             termination -> per pixel the segment's
//                             transmittance Tend, the local T before its last
//                             contributing entry Tx, the partial D, O, N and
//                             the last contributing position; the
//                             contribution bitmask words.
//   pass 2 (k_fwd_seg_combine) per tile and pixel, segments in order:
//                             T_in(s+1) = T_in(s) Tend(s), D += T_in(s) D(s)
//                             ...; the pixel terminates inside segment s iff
//                             T_in(s) Tx(s) < min_T (T before the segment's
//                             last contributing entry: T is monotone).  Writes
//                             the state before every segment boundary (the
//                             segment backward starts there) and the final
//                             images of the pixels that never terminate;
//                             lists the (tile, segment) slots holding a
//                             termination.
//   pass 3 (k_fwd_seg<3>)     those slots: the terminating pixels re-blend
//                             their segment sequentially from the state pass
//                             2 recorded, with the reference's cut-off, and
//                             write their final images, bitmask words and the
//                             later boundary states.
// Products of segment transmittances round differently from one sequential
// product (float32, ~1e-7 relative): only a pixel whose T crosses min_T
// within that margin can decide differently -- the parity protocol's flagged
// pixels.
namespace ss {

constexpr int kSegFields = 8;  // Tend, Tx, D, O, N0, N1, N2, last (int bits)

// segment slot index, unique over (tile, segment) (see seg_state for the chunk offsets)
__device__ __forceinline__ size_t seg_slot(int cbase, int seg, int t) {
  return (size_t)((cbase + seg * kSegChunks) / kSegChunks + t);
}

template <int kPass>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, SS_FWD_MINB)
    k_fwd_seg(BlendParams bp, const int* __restrict__ tile_ptr, const int* __restrict__ chunk_ptr,
              const int* __restrict__ pairs, const SplatRec* __restrict__ rec, const SplatRec64* __restrict__ rec64,
              float* __restrict__ out_D, float* __restrict__ out_N, float* __restrict__ out_O,
              float* __restrict__ out_T, int* __restrict__ out_last, unsigned* __restrict__ bitmask,
              float* __restrict__ segpart, const int* __restrict__ term_seg, const int* __restrict__ overflow,
              const int* __restrict__ slots, int* __restrict__ counter, const int* __restrict__ nslots) {
  pdl_wait();
  constexpr int TS = 8, PPL = 2;
  if (*overflow) return;
  __shared__ __align__(16) float stage[kWarpsPerBlock][32 * kStride];
  __shared__ __align__(16) RawEntry raw_all[kWarpsPerBlock][2][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const CamK& k = bp.cam;
  const size_t P = (size_t)k.W * k.H;
  float* st = stage[warp];
  for (int code = next_tile(counter, slots, nslots, lane); code >= 0; code = next_tile(counter, slots, nslots, lane)) {
    const int t = code >> 16, seg = code & 0xffff;
    const int tr = t / k.tx, tc = t % k.tx;
    TileFrame f;
    tile_frame<TS>(k, tr, tc, f);
    Pix px[PPL];
    float T[PPL], D[PPL], O[PPL], N[PPL][3], Tx[PPL];
    int last[PPL];
    bool live[PPL], mine[PPL];
    float xm = 0.f, ym = 0.f;
#pragma unroll
    for (int j = 0; j < PPL; ++j) {
      pixel_geo<TS>(k, tr, tc, lane + 32 * j, f, px[j]);
      const size_t p = (size_t)px[j].row * k.W + px[j].col;
      T[j] = 1.f; D[j] = 0.f; O[j] = 0.f; N[j][0] = N[j][1] = N[j][2] = 0.f;
      Tx[j] = 1.f;
      last[j] = 0;
      mine[j] = kPass == 1 ? true : (px[j].inside && term_seg[p] == seg);
      if (kPass == 3 && mine[j]) {  // the state before this segment (pass 2)
        T[j] = out_T[p];
        D[j] = out_D[p];
        O[j] = out_O[p];
        N[j][0] = out_N[3 * p];
        N[j][1] = out_N[3 * p + 1];
        N[j][2] = out_N[3 * p + 2];
        last[j] = out_last[p];
      }
      // (pass 3 may start below the cut-off: the previous segment's last entry took T
      // under it and this segment holds the first entry that no longer contributes)
      live[j] = mine[j] && px[j].ray_ok && (kPass == 1 || T[j] >= bp.min_T);
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
    unsigned long long PP[PPL / 2][6];
#pragma unroll
    for (int q = 0; q < 6; ++q) PP[0][q] = pack2(px[0].p[q], px[1].p[q]);
    const int lo = tile_ptr[t], L = tile_ptr[t + 1] - lo;
    const int cbase = chunk_ptr[t];
    const int nch = (L + 31) / 32;
    const int c0 = seg * kSegChunks, c1 = min(c0 + kSegChunks, nch);
    int sid_cur = c0 * 32 + lane < L ? pairs[lo + c0 * 32 + lane] : -1;
    if (sid_cur >= 0) prefetch_entry(&raw_all[warp][0][lane], sid_cur, rec, rec64);
    __pipeline_commit();
    int sid_next = (c0 + 1) * 32 + lane < L ? pairs[lo + (c0 + 1) * 32 + lane] : -1;
    for (int chunk = c0; chunk < c1; ++chunk) {
      const int base = chunk * 32;
      const int slot = (chunk - c0) & 1;
      if (sid_next >= 0 && chunk + 1 < c1) prefetch_entry(&raw_all[warp][slot ^ 1][lane], sid_next, rec, rec64);
      __pipeline_commit();
      const int sid_after = base + 64 + lane < L ? pairs[lo + base + 64 + lane] : -1;
      __pipeline_wait_prior(1);
      if (sid_cur >= 0) stage_entry<true>(st + lane * kStride, sid_cur, raw_all[warp][slot][lane], f, xm, ym);
      __syncwarp();
      sid_cur = sid_next;
      sid_next = sid_after;
      const int cnt = min(32, L - base);
      unsigned word[PPL] = {0u, 0u}, cw[PPL] = {0u, 0u};
      for (int i = 0; i < cnt; ++i) {
        const float* e = st + i * kStride;
        const float4 q0 = *reinterpret_cast<const float4*>(e);
        const float4 q1 = *reinterpret_cast<const float4*>(e + 4);
        const unsigned long long q = cone2(q0, q1, PP[0]);
        cw[0] = __funnelshift_l((unsigned)q, cw[0], 1);
        cw[1] = __funnelshift_l((unsigned)(q >> 32), cw[1], 1);
      }
#pragma unroll
      for (int j = 0; j < PPL; ++j) cw[j] = __brev(cw[j]) >> (32 - cnt);
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
          Tx[j] = T[j];
          const float w = h.alpha * T[j];
          D[j] += w * h.lam;
          O[j] += w;
          N[j][0] += w * x.n[0];
          N[j][1] += w * x.n[1];
          N[j][2] += w * x.n[2];
          T[j] *= (1.f - h.alpha);
          word[j] |= 1u << i;
          last[j] = base + i + 1;
          if (kPass == 3 && T[j] < bp.min_T) {  // the reference's cut-off (T before the next entry)
            live[j] = false;
            m = 0u;
          }
        }
      }
#pragma unroll
      for (int j = 0; j < PPL; ++j)
        if (mine[j]) bitmask[(size_t)(cbase + chunk) * (TS * TS) + lane + 32 * j] = word[j];
      __syncwarp();
      // pass 3: once every pixel of the slot has hit the cut-off the rest of the segment is
      // beyond their last contributions (the backward masks those chunks by `last`)
      if (kPass == 3 && !__any_sync(0xffffffffu, live[0] || live[1])) break;
    }
    __pipeline_wait_prior(0);
    __syncwarp();
    if (kPass == 1) {
      float* sp = segpart + seg_slot(cbase, seg, t) * (kSegFields * 64);
#pragma unroll
      for (int j = 0; j < PPL; ++j) {
        const int q = lane + 32 * j;
        sp[q] = T[j];
        sp[64 + q] = Tx[j];
        sp[128 + q] = D[j];
        sp[192 + q] = O[j];
        sp[256 + q] = N[j][0];
        sp[320 + q] = N[j][1];
        sp[384 + q] = N[j][2];
        sp[448 + q] = __int_as_float(last[j]);
      }
    } else {
      const int nseg = (nch + kSegChunks - 1) / kSegChunks;
#pragma unroll
      for (int j = 0; j < PPL; ++j) {
        if (!mine[j]) continue;
        const int q = lane + 32 * j;
        const size_t p = (size_t)px[j].row * k.W + px[j].col;
        out_D[p] = D[j];
        out_O[p] = O[j];
        out_N[3 * p] = N[j][0];
        out_N[3 * p + 1] = N[j][1];
        out_N[3 * p + 2] = N[j][2];
        out_T[p] = T[j];
        out_last[p] = last[j];
        bp.fin[p] = D[j];
        bp.fin[P + p] = O[j];
        bp.fin[2 * P + p] = N[j][0];
        bp.fin[3 * P + p] = N[j][1];
        bp.fin[4 * P + p] = N[j][2];
        for (int s2 = seg + 1; s2 < nseg; ++s2) {  // later boundaries: the final state
          float* sg = seg_state(bp.segst, cbase, s2 * kSegChunks);
          sg[q] = T[j];
          sg[64 + q] = D[j];
          sg[128 + q] = O[j];
          sg[192 + q] = N[j][0];
          sg[256 + q] = N[j][1];
          sg[320 + q] = N[j][2];
        }
      }
    }
  }
}

// Pass 2: one warp per tile (grid-stride), two pixels per lane.  The segments'
// partials are loaded kComb segments at a time ahead of the sequential combine
// (one dependent round trip per batch, not per segment: the longest lists have
// ~40 segments and set the kernel's duration).
constexpr int kComb = 4;

__global__ void __launch_bounds__(128) k_fwd_seg_combine(BlendParams bp, int ntiles, const int* __restrict__ tile_ptr,
                                                         const int* __restrict__ chunk_ptr,
                                                         const float* __restrict__ segpart, float* __restrict__ out_D,
                                                         float* __restrict__ out_N, float* __restrict__ out_O,
                                                         float* __restrict__ out_T, int* __restrict__ out_last,
                                                         int* __restrict__ term_seg, int* __restrict__ slots3,
                                                         int* __restrict__ nslots3, const int* __restrict__ overflow) {
  pdl_wait();
  constexpr int TS = 8, PPL = 2;
  if (*overflow) return;
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  const CamK& k = bp.cam;
  const size_t P = (size_t)k.W * k.H;
  for (int t = gw; t < ntiles; t += nw) {
    const int tr = t / k.tx, tc = t % k.tx;
    const int L = tile_ptr[t + 1] - tile_ptr[t];
    const int cbase = chunk_ptr[t];
    const int nseg = ((L + 31) / 32 + kSegChunks - 1) / kSegChunks;
    float T[PPL], D[PPL], O[PPL], N[PPL][3];
    int last[PPL], ts[PPL];
    bool in[PPL];
#pragma unroll
    for (int j = 0; j < PPL; ++j) {
      const int q = lane + 32 * j;
      in[j] = tr * TS + q / TS < k.H && tc * TS + q % TS < k.W;
      T[j] = 1.f; D[j] = O[j] = N[j][0] = N[j][1] = N[j][2] = 0.f;
      last[j] = 0;
      ts[j] = in[j] ? -2 : -1;  // -2: still combining
    }
    for (int s0 = 0; s0 < nseg; s0 += kComb) {
      float v[kComb][PPL][kSegFields];
#pragma unroll
      for (int b = 0; b < kComb; ++b) {
        const float* sp = segpart + seg_slot(cbase, min(s0 + b, nseg - 1), t) * (kSegFields * 64);
#pragma unroll
        for (int j = 0; j < PPL; ++j)
#pragma unroll
          for (int f = 0; f < kSegFields; ++f) v[b][j][f] = sp[64 * f + lane + 32 * j];
      }
#pragma unroll
      for (int b = 0; b < kComb; ++b) {
        const int s = s0 + b;
        if (s >= nseg) break;
#pragma unroll
        for (int j = 0; j < PPL; ++j) {
          if (ts[j] != -2) continue;
          const int q = lane + 32 * j;
          if (s > 0) {
            float* sg = seg_state(bp.segst, cbase, s * kSegChunks);
            sg[q] = T[j];
            sg[64 + q] = D[j];
            sg[128 + q] = O[j];
            sg[192 + q] = N[j][0];
            sg[256 + q] = N[j][1];
            sg[320 + q] = N[j][2];
          }
          if (T[j] * v[b][j][1] < bp.min_T) {  // the cut-off falls inside segment s: pass 3
            ts[j] = s;
            continue;
          }
          D[j] = fmaf(T[j], v[b][j][2], D[j]);
          O[j] = fmaf(T[j], v[b][j][3], O[j]);
          N[j][0] = fmaf(T[j], v[b][j][4], N[j][0]);
          N[j][1] = fmaf(T[j], v[b][j][5], N[j][1]);
          N[j][2] = fmaf(T[j], v[b][j][6], N[j][2]);
          const int l = __float_as_int(v[b][j][7]);
          if (l) last[j] = l;
          T[j] *= v[b][j][0];
        }
      }
      if (!__any_sync(0xffffffffu, ts[0] == -2 || ts[1] == -2)) break;
    }
#pragma unroll
    for (int j = 0; j < PPL; ++j) {
      if (!in[j]) continue;
      if (ts[j] == -2) ts[j] = -1;
      const int q = lane + 32 * j;
      const size_t p = (size_t)(tr * TS + q / TS) * k.W + tc * TS + q % TS;
      out_D[p] = D[j];  // (for a terminating pixel: the state pass 3 starts from)
      out_O[p] = O[j];
      out_N[3 * p] = N[j][0];
      out_N[3 * p + 1] = N[j][1];
      out_N[3 * p + 2] = N[j][2];
      out_T[p] = T[j];
      out_last[p] = last[j];
      term_seg[p] = ts[j];
      if (ts[j] < 0) {
        bp.fin[p] = D[j];
        bp.fin[P + p] = O[j];
        bp.fin[2 * P + p] = N[j][0];
        bp.fin[3 * P + p] = N[j][1];
        bp.fin[4 * P + p] = N[j][2];
      }
    }
    // one pass-3 slot per distinct terminating segment of the tile
    unsigned pend0 = __ballot_sync(0xffffffffu, ts[0] >= 0), pend1 = __ballot_sync(0xffffffffu, ts[1] >= 0);
    while (pend0 | pend1) {
      const int v = pend0 ? __shfl_sync(0xffffffffu, ts[0], __ffs(pend0) - 1)
                          : __shfl_sync(0xffffffffu, ts[1], __ffs(pend1) - 1);
      if (lane == 0) slots3[atomicAdd(nslots3, 1)] = (t << 16) | v;
      pend0 &= ~__ballot_sync(0xffffffffu, ts[0] == v);
      pend1 &= ~__ballot_sync(0xffffffffu, ts[1] == v);
    }
  }
}

}  // namespace ss
