// C ABI of the B200 hot path (declared in include/splat_b200.h).
// Unity build: the kernel sources are included here so the library is one
// translation unit without relocatable device code.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <new>
#include <vector>

#include "binning.cu"
#include "blend.cu"
#include "blend_seg.cu"
#include "keyframe.cu"
#include "densify.cu"
#include "leaf_tree.cu"
#include "leaf_top.cu"
#include "loss.cu"
#include "reg_solve.cu"  // includes registration.cu

using namespace ss;

namespace {

// numpy-style float modulo on the host (np.mod semantics)
double host_py_mod(double a, double b) {
  double m = std::fmod(a, b);
  if (m != 0.0 && ((b < 0.0) != (m < 0.0))) m += b;
  return m;
}

// Camera constants with the reference's operation order
// (geometry.py:95-109, 160-174; rasterizer.py:252-276).
int make_camk(const ss_camera* c, int T, double pad_px, CamK& k) {
  if (!c || c->width < 2 || c->height < 2) return SS_ERR_INVALID_ARGUMENT;
  if (!(c->az_max > c->az_min && c->el_max > c->el_min)) return SS_ERR_INVALID_ARGUMENT;
  if (T != 8 && T != 16) return SS_ERR_UNSUPPORTED;
  double fov_h = c->az_max - c->az_min, fov_v = c->el_max - c->el_min;
  k.W = c->width;
  k.H = c->height;
  k.T = T;
  k.tx = (c->width + T - 1) / T;
  k.ty = (c->height + T - 1) / T;
  k.fx = (double)(-(c->width - 1)) / fov_h;
  k.fy = (double)(-(c->height - 1)) / fov_v;
  k.cx = 0.5 * c->width * (1.0 + (c->az_max + c->az_min) / fov_h);
  k.cy = 0.5 * c->height * (1.0 + (c->el_max + c->el_min) / fov_v);
  volatile double fu = k.fx * c->az_max;
  volatile double fv = k.fy * c->el_max;
  double first_u = fu + k.cx, first_v = fv + k.cy;
  k.off_u = host_py_mod(first_u + 0.5, 1.0) - 0.5;
  k.off_v = host_py_mod(first_v + 0.5, 1.0) - 0.5;
  k.pad_az = pad_px * (1.0 / std::fabs(k.fx));
  k.pad_el = pad_px * (1.0 / std::fabs(k.fy));
  return SS_OK;
}

template <typename T>
int grow(T*& ptr, size_t& cap, size_t need, cudaStream_t s) {
  if (need <= cap && ptr) return SS_OK;
  if (ptr) cudaFreeAsync(ptr, s);
  ptr = nullptr;
  size_t c = need + need / 4 + 64;
  if (cudaMallocAsync((void**)&ptr, c * sizeof(T), s) != cudaSuccess) {
    cap = 0;
    return SS_ERR_CUDA;
  }
  cap = c;
  return SS_OK;
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

SplatsK to_k(const ss_splats* s) {
  SplatsK k;
  k.n = s->n;
  k.centers = s->centers;
  k.raw_ta = s->raw_t_alpha;
  k.raw_tb = s->raw_t_beta;
  k.log_scales = s->log_scales;
  k.logit_opacity = s->logit_opacity;
  return k;
}

// FP32 FMA throughput probe (roofline denominator; MEASURED_PEAKS.json has no FP32 figure).
__global__ void k_ffma_probe(float* out, int iters, float a, float b) {
  float x0 = threadIdx.x * 1e-3f, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6,
        x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
      x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
    }
  }
  float s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 12345.f) out[0] = s;
}

// totals[0..1] and status/overflow (misc[0..1]) into mapped host memory.
__global__ void k_publish_totals(const long long* __restrict__ totals, const int* __restrict__ misc,
                                 volatile long long* __restrict__ host) {
  if (threadIdx.x == 0) {
    host[0] = totals[0];
    host[1] = totals[1];
    host[3] = totals[2];  // longest tile list
    const long long sm = (long long)(unsigned)misc[0] | ((long long)(unsigned)misc[1] << 32);
    host[2] = sm;
    __threadfence_system();
  }
}

}  // namespace

struct ss_records {
  CamK cam{};
  PoseK pose{};
  BlendParams bp{};
  int n = 0, ntiles = 0, valid = 0, pending = 0;
  int deterministic = 0;  // backward: fixed-order gradient reduction (ss_records_set_deterministic)
  int split_target = 0;   // work slots beyond one per tile (k_tile_order)
  bool captured = false;  // last forward was recorded into a CUDA graph
  float* pacc = nullptr;  // deterministic mode: per list position accumulators
  size_t cap_pacc = 0;
  uint32_t epoch = 0;
  long long n_pairs = 0, n_chunks = 0;
  long long cap_pairs = 0;  // speculative pair capacity of the current forward
  long long want_pairs = 0; // capacity requested for the next forward
  // per splat
  SplatRec* rec = nullptr;
  size_t cap_rec = 0;
  SplatRec64* rec64 = nullptr;
  size_t cap_rec64 = 0;
  unsigned long long* key64 = nullptr;
  size_t cap_key64 = 0;
  uint32_t* key32 = nullptr;
  size_t cap_key32 = 0;
  int4* rect = nullptr;
  size_t cap_rect = 0;
  uint32_t* bsum = nullptr;  // per preprocess block pair counts -> offsets
  size_t cap_bsum = 0;
  uint32_t* mat = nullptr;  // pair blocks x tiles histogram -> offsets
  size_t cap_mat = 0;
  // per camera / tile
  double2* tint = nullptr;  // tx column + ty row intervals
  size_t cap_tint = 0;
  int* tiles = nullptr;  // tile_ptr | chunk_ptr | tile_count | (unused) | long_list | order (2) | order_fwd
  size_t cap_tiles = 0;
  // pairs: emitted (tile, splat) and the bucketed per-tile lists
  uint32_t* ptile = nullptr;
  size_t cap_ptile = 0;
  uint32_t* psplat = nullptr;
  size_t cap_psplat = 0;
  uint32_t* pbucket = nullptr;
  size_t cap_pbucket = 0;
  int* pairs = nullptr;  // == pbucket: final per-tile lists
  unsigned* bitmask = nullptr;
  size_t cap_bitmask = 0;
  // segment-parallel backward (few tiles): recorded pixel states, finals, work slots
  bool seg = false;
  bool hyb = false;  // many tiles: segment slots for the long lists, whole-tile slots for the rest
  float* segst = nullptr;
  size_t cap_segst = 0;
  float* fin = nullptr;
  size_t cap_fin = 0;
  int* segorder = nullptr;
  size_t cap_segorder = 0;
  // segment-parallel forward (few tiles): per-segment partial blends, the terminating
  // segment of every pixel, and the slots of the recompute pass
  float* segpart = nullptr;
  size_t cap_segpart = 0;
  int* term_seg = nullptr;
  size_t cap_term_seg = 0;
  int* seg3 = nullptr;
  size_t cap_seg3 = 0;
  int* misc = nullptr;  // [0] status, [1] overflow, [2] n_long, [4..9] blend counters
  size_t cap_misc = 0;
  long long* totals = nullptr;
  size_t cap_totals = 0;
  // per pixel
  float* Tf = nullptr;
  size_t cap_Tf = 0;
  int* last = nullptr;
  size_t cap_last = 0;
  float* acc = nullptr;
  size_t cap_acc = 0;
  // Buffer generation: bumped whenever any device buffer above moved (a grow() freed
  // and reallocated it).  CUDA graphs captured over these records hold the old
  // pointers, so their owners key the graphs on this counter.
  unsigned long long generation = 0;
  uintptr_t buf_sig = 0;
  void note_buffers() {
    const void* bufs[] = {rec, rec64, key64, key32, rect, bsum, mat, tint, tiles, ptile, psplat, pbucket, bitmask,
                          misc, totals, Tf, last, acc, pacc, segst, fin, segorder, segpart, term_seg, seg3};
    uintptr_t h = 1469598103934665603ull;
    for (const void* b : bufs) h = (h ^ (uintptr_t)b) * 1099511628211ull;
    if (h != buf_sig) {
      buf_sig = h;
      ++generation;
    }
  }
  long long* h_totals = nullptr;  // mapped pinned: pairs, chunks, status | overflow, longest list
  long long last_max_list = 0;  // longest tile list of the last checked forward (diagnostics)
  long long* d_h_totals = nullptr;  // its device alias
  cudaEvent_t done = nullptr;
  cudaEvent_t fwd_end = nullptr;  // forward kernels finished (side-stream fork point)
  cudaEvent_t long_fork = nullptr, long_join = nullptr;  // block-per-tile forward on `side`
  cudaEvent_t sort_fork = nullptr, sort_join = nullptr;  // big-list tile sort on `side`
  cudaStream_t side = nullptr;    // publishes the totals off the compute stream
  // optional per-stage CUDA-event timing (bench.py roofline), stream-ordered
  bool profiling = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev_used;
  cudaEvent_t take_event() {
    if (!ev_pool.empty()) {
      cudaEvent_t e = ev_pool.back();
      ev_pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
};

namespace {
// Stage markers around each kernel when profiling is enabled.
struct StageTimer {
  ss_records* r;
  int stage;
  cudaStream_t s;
  cudaEvent_t a = nullptr, b = nullptr;
  bool on = false;
  StageTimer(ss_records* r_, int st, cudaStream_t s_) : r(r_), stage(st), s(s_) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cs);
    on = r->profiling && cs == cudaStreamCaptureStatusNone;  // (no timing events inside a graph)
    if (on) {
      a = r->take_event();
      b = r->take_event();
      cudaEventRecord(a, s);
    }
  }
  ~StageTimer() {
    if (on) {
      cudaEventRecord(b, s);
      r->ev_used.push_back({stage, {a, b}});
    }
  }
};
enum { ST_PREPROCESS, ST_EMIT, ST_BUCKET, ST_TILE_SORT, ST_UNUSED, ST_FORWARD, ST_BACKWARD, ST_FINALIZE, ST_COUNT };

// Launch with programmatic stream serialization (PDL): the kernel's blocks may be
// scheduled while the previous kernel on the stream drains; every kernel launched
// this way starts with pdl_wait().  `allow` = false where the kernel follows a
// cross-stream event wait or sits between profiling events.  SS_PDL=0 disables.
bool pdl_enabled() {
  static const bool on = !std::getenv("SS_PDL") || std::atoi(std::getenv("SS_PDL")) != 0;
  return on;
}
template <typename... KArgs, typename... Args>
cudaError_t pdl_launch(bool allow, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = (allow && pdl_enabled()) ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// Contributions U: the contribution bits of each pixel up to its last contributing list
// position (the segment forward leaves words past a pixel's cut-off that no pass reads:
// the backward masks them the same way).  One warp per tile.
__global__ void k_count_contrib(CamK k, int ntiles, const int* __restrict__ tile_ptr, const int* __restrict__ chunk_ptr,
                                const int* __restrict__ last, const unsigned* __restrict__ bm,
                                unsigned long long* out) {
  const int lane = threadIdx.x & 31;
  const int TT = k.T * k.T;
  unsigned long long c = 0;
  for (int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < ntiles; t += (gridDim.x * blockDim.x) >> 5) {
    const int tr = t / k.tx, tc = t % k.tx;
    const int nch = (tile_ptr[t + 1] - tile_ptr[t] + 31) / 32;
    const int cbase = chunk_ptr[t];
    for (int q = lane; q < TT; q += 32) {
      const int row = tr * k.T + q / k.T, col = tc * k.T + q % k.T;
      if (row >= k.H || col >= k.W) continue;
      const int l = last[(size_t)row * k.W + col];
      for (int ch = 0; ch < nch && ch * 32 < l; ++ch) {
        const int r = l - ch * 32;
        const unsigned mask = r >= 32 ? 0xffffffffu : ((1u << r) - 1u);
        c += __popc(bm[(size_t)(cbase + ch) * TT + q] & mask);
      }
    }
  }
  for (int off = 16; off > 0; off >>= 1) c += __shfl_xor_sync(0xffffffffu, c, off);
  if (lane == 0) atomicAdd(out, c);
}

void set_smem_attrs() {
  static bool done = false;
  if (done) return;
  const int bytes = (int)(sizeof(uint32_t) * kMaxTiles);
  cudaFuncSetAttribute(k_tile_hist_blocks, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaFuncSetAttribute(k_tile_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(2 * bytes + (size_t)kPairChunkMany * 6));
  cudaFuncSetAttribute(k_bin_count, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * bytes + 16);
  cudaFuncSetAttribute(k_bin_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(2 * bytes + (size_t)kBinStage * 6));
  cudaFuncSetAttribute(k_backward<8, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBwdDynSmem);
  cudaFuncSetAttribute(k_backward<8, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBwdDynSmem);
  cudaFuncSetAttribute(k_backward<8, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBwdDynSmem);
  cudaFuncSetAttribute(k_tile_sort_big<kTileSortBig>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)sort_smem_bytes<kTileSortBig, 1024>());
  cudaFuncSetAttribute(k_tile_sort_big<kTileSortHuge>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)sort_smem_bytes<kTileSortHuge, 1024>());
  cudaFuncSetAttribute(k_backward<16, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBwdDynSmem);
  done = true;
}
}  // namespace

// (ss_host_stage_f64 below)
// DST: 0 no copy, 1 float64 copy, 2 float32 (round to nearest, as the device conversion);
// FP: accumulate the fingerprint (weights w = (m ^ (m >> 29)) | 1, m = i * K: one 64-bit
// multiply per value, two accumulators so the adds do not chain; the scalar form measured
// faster on the GPU box's host than a 32-bit-half form the compiler vectorises with SSE2)
template <int DST, bool FP>
static uint64_t host_stage(const double* __restrict__ src, void* __restrict__ dst, int64_t n, int64_t base) {
  constexpr uint64_t K = 0x9E3779B97F4A7C15ull;
  const uint64_t* x = reinterpret_cast<const uint64_t*>(src);
  if (!FP) {
    for (int64_t k = 0; k < n; ++k) {
      if (DST == 1) static_cast<uint64_t*>(dst)[k] = x[k];
      if (DST == 2) static_cast<float*>(dst)[k] = (float)src[k];
    }
    return 0;
  }
  uint64_t m = (uint64_t)base * K, a0 = 0, a1 = 0;
  int64_t k = 0;
  for (; k + 2 <= n; k += 2) {
    const uint64_t v0 = x[k], v1 = x[k + 1];
    if (DST == 1) {
      static_cast<uint64_t*>(dst)[k] = v0;
      static_cast<uint64_t*>(dst)[k + 1] = v1;
    } else if (DST == 2) {
      static_cast<float*>(dst)[k] = (float)src[k];
      static_cast<float*>(dst)[k + 1] = (float)src[k + 1];
    }
    const uint64_t m1 = m + K;
    a0 += v0 * ((m ^ (m >> 29)) | 1ull);
    a1 += v1 * ((m1 ^ (m1 >> 29)) | 1ull);
    m = m1 + K;
  }
  if (k < n) {
    if (DST == 1) static_cast<uint64_t*>(dst)[k] = x[k];
    if (DST == 2) static_cast<float*>(dst)[k] = (float)src[k];
    a0 += x[k] * ((m ^ (m >> 29)) | 1ull);
  }
  return a0 + a1;
}

extern "C" {

const char* ss_version(void) { return "paper_2503_17491_b200 0.2 (sm_100a)"; }

ss_records* ss_records_create(void) {
  ss_records* r = new (std::nothrow) ss_records();
  if (!r) return nullptr;
  // mapped pinned memory: the forward publishes its totals with a kernel store,
  // not a device-to-host copy (a copy would queue behind the caller's bulk
  // downloads on the D2H copy engine and stall the compute stream)
  if (cudaHostAlloc((void**)&r->h_totals, 4 * sizeof(long long), cudaHostAllocMapped) != cudaSuccess ||
      cudaHostGetDevicePointer((void**)&r->d_h_totals, r->h_totals, 0) != cudaSuccess) {
    if (r->h_totals) cudaFreeHost(r->h_totals);
    delete r;
    return nullptr;
  }
  cudaEventCreateWithFlags(&r->done, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&r->fwd_end, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&r->long_fork, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&r->long_join, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&r->sort_fork, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&r->sort_join, cudaEventDisableTiming);
  cudaStreamCreateWithFlags(&r->side, cudaStreamNonBlocking);
  return r;
}

void ss_records_destroy(ss_records* r, void* stream) {
  if (!r) return;
  cudaStream_t s = (cudaStream_t)stream;
  // work queued on the side stream (totals publication, big-list sort, long-list
  // forward) may still read these buffers and the mapped host words
  if (r->side) cudaStreamSynchronize(r->side);
  void* bufs[] = {r->rec,    r->rec64,   r->key64, r->key32,  r->rect, r->bsum, r->mat, r->tint,
                  r->tiles,  r->ptile,   r->psplat, r->pbucket, r->bitmask, r->misc, r->totals,
                  r->Tf,     r->last,    r->acc,     r->pacc,  r->segst, r->fin, r->segorder,
                  r->segpart, r->term_seg, r->seg3};
  for (void* b : bufs)
    if (b) cudaFreeAsync(b, s);
  cudaStreamSynchronize(s);
  for (auto& u : r->ev_used) {
    cudaEventDestroy(u.second.first);
    cudaEventDestroy(u.second.second);
  }
  for (auto e : r->ev_pool) cudaEventDestroy(e);
  if (r->done) cudaEventDestroy(r->done);
  if (r->fwd_end) cudaEventDestroy(r->fwd_end);
  if (r->long_fork) cudaEventDestroy(r->long_fork);
  if (r->long_join) cudaEventDestroy(r->long_join);
  if (r->sort_fork) cudaEventDestroy(r->sort_fork);
  if (r->sort_join) cudaEventDestroy(r->sort_join);
  if (r->side) cudaStreamDestroy(r->side);
  if (r->h_totals) cudaFreeHost(r->h_totals);
  delete r;
}

// Enqueue a complete forward render; no host synchronisation.  The caller
// checks capacity with ss_records_check (and re-runs on SS_ERR_CAPACITY).
int ss_render_forward(const ss_camera* cam, const double* pose_Rt, const ss_splats* splats, const ss_raster_cfg* cfg,
                      float* out_range, float* out_normal, float* out_opacity, ss_records* rec, void* stream) {
  if (!cam || !pose_Rt || !splats || !cfg || !rec || !out_range || !out_normal || !out_opacity)
    return SS_ERR_INVALID_ARGUMENT;
  if (splats->n < 0) return SS_ERR_INVALID_ARGUMENT;
  cudaStream_t s = (cudaStream_t)stream;
  CamK k;
  int st = make_camk(cam, cfg->tile_size, cfg->bbox_pad_px, k);
  if (st) return st;
  rec->valid = 0;
  rec->pending = 1;
  rec->cam = k;
  for (int q = 0; q < 9; ++q) rec->pose.R[q] = pose_Rt[q];
  for (int q = 0; q < 3; ++q) rec->pose.t[q] = pose_Rt[9 + q];
  rec->bp.cam = k;
  rec->bp.alpha_cutoff = (float)cfg->alpha_cutoff;
  rec->bp.alpha_clamp = (float)cfg->alpha_clamp;
  rec->bp.min_T = (float)cfg->min_transmittance;
  rec->bp.denom_eps = (float)cfg->denom_eps;
  RasterK rk{cfg->alpha_cutoff, cfg->alpha_clamp, cfg->min_transmittance, cfg->denom_eps, cfg->cutoff_sigma};
  const int n = splats->n;
  const int ntiles = k.tx * k.ty;
  const size_t P = (size_t)k.W * k.H;
  const int TT = k.T * k.T;
  rec->n = n;
  rec->ntiles = ntiles;
  long long cap = std::max<long long>(rec->want_pairs, std::max<long long>(8LL * n, 65536));
  if (cap > 0x7fff0000LL) cap = 0x7fff0000LL;
  rec->cap_pairs = cap;
  const int nb = (n + 255) / 256;
  if (ntiles > kMaxTiles) return SS_ERR_UNSUPPORTED;
  const int pchunk = num_sms() * 16 > ntiles ? kPairChunkFew : kPairChunkMany;
  const int pblocks = (int)((cap + pchunk - 1) / pchunk);
  const int nbb = std::max(1, (n + kBinSplats - 1) / kBinSplats);  // direct binning blocks
  if (grow(rec->rec, rec->cap_rec, (size_t)n + 1, s) || grow(rec->rec64, rec->cap_rec64, (size_t)n + 1, s) ||
      grow(rec->key64, rec->cap_key64, (size_t)n + 1, s) || grow(rec->key32, rec->cap_key32, (size_t)n + 1, s) ||
      grow(rec->rect, rec->cap_rect, (size_t)n + 1, s) || grow(rec->bsum, rec->cap_bsum, (size_t)nb + 1, s) ||
      grow(rec->mat, rec->cap_mat, (size_t)std::max(pblocks, nbb) * ntiles, s) ||
      grow(rec->tint, rec->cap_tint, (size_t)(k.tx + k.ty), s) ||
      grow(rec->tiles, rec->cap_tiles, (size_t)8 * (ntiles + 1), s) ||
      grow(rec->ptile, rec->cap_ptile, (size_t)cap, s) || grow(rec->psplat, rec->cap_psplat, (size_t)cap, s) ||
      grow(rec->pbucket, rec->cap_pbucket, (size_t)cap, s) ||
      grow(rec->bitmask, rec->cap_bitmask, ((size_t)cap / 32 + ntiles + 1) * TT, s) ||
      grow(rec->misc, rec->cap_misc, 16, s) || grow(rec->totals, rec->cap_totals, 3, s) ||
      grow(rec->Tf, rec->cap_Tf, P, s) || grow(rec->last, rec->cap_last, P, s))
    return SS_ERR_CUDA;
  rec->note_buffers();
  int* tile_ptr = rec->tiles;
  int* chunk_ptr = rec->tiles + (ntiles + 1);
  int* tile_count = rec->tiles + 2 * (ntiles + 1);
  int* long_list = rec->tiles + 4 * (ntiles + 1);
  int* order = rec->tiles + 5 * (ntiles + 1);  // up to 2 * ntiles work slots
  int* counters = rec->misc + 4;  // [0] forward, [1] backward tile tickets, [2] work slots
  // fewer tiles than resident blend warps (4 blocks x 4 warps per SM): split the longest in two
  // (not in deterministic mode: both halves of a split tile would write one list position)
  // With few tiles the backward walks segments of kSegChunks chunks of each list in
  // parallel (instead of splitting tiles into pixel halves): the forward records
  // the per-pixel state at the segment boundaries.
  const bool seg = SS_SEG_MODE && k.T == 8 && (SS_SEG_ALWAYS || num_sms() * 16 > ntiles);
  rec->seg = seg;
  // Many tiles: the backward walks the tiles as whole-tile slots, or -- when the longest
  // list exceeds twice the pairs per resident warp, so that the longest tile's walk would
  // set the kernel's duration -- every list in segments from states the forward recorded
  // (config-4a maps, lists up to ~3,700 entries: backward 320 -> 212 us).  Decided on the
  // device from this render's lists (k_tile_order), so the same inputs always take the
  // same path.  SS_HYBRID=0: the plain whole-tile backward (A/B).
  static const bool hyb_on = !std::getenv("SS_HYBRID") || std::atoi(std::getenv("SS_HYBRID")) != 0;
  const bool hyb = SS_SEG_MODE && k.T == 8 && !seg && hyb_on;
  rec->hyb = hyb;
  const int split_target = (k.T == 8 && !rec->deterministic && !seg) ? std::max(0, num_sms() * 16 - ntiles) : 0;
  rec->split_target = split_target;
  // segment-parallel forward (blend_seg.cu) wherever the backward walks segments
  // (SS_SEG_FWD=0: the block-per-tile forward instead, for A/B)
  static const bool seg_fwd_on = !std::getenv("SS_SEG_FWD") || std::atoi(std::getenv("SS_SEG_FWD")) != 0;
  const bool seg_fwd = seg && seg_fwd_on;
  if (seg || hyb) {
    const size_t nchunk = (size_t)cap / 32 + ntiles + 1;
    const size_t nsegs = nchunk / kSegChunks + (size_t)ntiles + 2;
    if (grow(rec->segst, rec->cap_segst, (nchunk / kSegChunks + 2) * 6 * 64, s) ||
        grow(rec->fin, rec->cap_fin, (size_t)5 * P, s) ||
        grow(rec->segorder, rec->cap_segorder, nchunk / kSegChunks + 2 * (size_t)ntiles + 2, s))
      return SS_ERR_CUDA;
    if (seg_fwd && (grow(rec->segpart, rec->cap_segpart, nsegs * kSegFields * 64, s) ||
                    grow(rec->term_seg, rec->cap_term_seg, P, s) || grow(rec->seg3, rec->cap_seg3, nsegs, s)))
      return SS_ERR_CUDA;
  }
  rec->note_buffers();
  rec->bp.segst = (seg || hyb) ? rec->segst : nullptr;
  rec->bp.fin = (seg || hyb) ? rec->fin : nullptr;
  rec->bp.seg_min = rec->misc + 4 + 9;  // (k_tile_order's threshold, counters[9])
  // ... and hand the long lists to the block-per-tile forward: every list of >= SS_LONG_MIN
  // entries when tiles are few, only the tail (>= SS_LONG_MIN_MANY) when they are many
  const bool few_tiles = num_sms() * 16 > ntiles;
  const int long_min = few_tiles ? SS_LONG_MIN : SS_LONG_MIN_MANY;
  const int long_target = (k.T == 8 && !seg_fwd && (few_tiles || SS_LONG_MIN_MANY > 0)) ? SS_LONG_TARGET : 0;
  int* status = rec->misc;
  int* overflow = rec->misc + 1;
  int* n_long = rec->misc + 2;
  double2* colt = rec->tint;
  double2* rowt = rec->tint + k.tx;

  PoseK pk = rec->pose;
  SplatsK sk = to_k(splats);
  const bool pa = !rec->profiling;  // (PDL launches: not between profiling events)
  {
    StageTimer tm(rec, ST_PREPROCESS, s);
    const int nti = std::max(std::max(k.tx + k.ty, ntiles), 16);
    SS_CUDA_TRY(pdl_launch(pa, k_tile_intervals, dim3((nti + 127) / 128), dim3(128), 0, s, k, colt, rowt, rec->misc, rec->totals, tile_count, ntiles));
    if (n > 0)
      SS_CUDA_TRY(pdl_launch(pa, k_preprocess, dim3(nb), dim3(256), 0, s, sk, pk, k, rk, colt, rowt, rec->rec, rec->rec64, rec->key64, rec->key32,
                                      rec->rect, rec->bsum, status));
  }
#if SS_DIRECT_BIN
  // direct binning: tile histograms and buckets straight from the splats' tile rectangles
  const size_t hsm = sizeof(uint32_t) * ntiles;
  set_smem_attrs();
  {
    StageTimer tm(rec, ST_EMIT, s);
    SS_CUDA_TRY(pdl_launch(pa, k_bin_count, dim3(nbb), dim3(1024), sizeof(int) * (k.tx + 1) * (k.ty + 1), s, n, rec->rect,
                           k.tx, k.ty, rec->mat));
  }
  {
    StageTimer tm(rec, ST_BUCKET, s);
    SS_CUDA_TRY(pdl_launch(pa, k_tile_prefix, dim3((ntiles + 31) / 32), dim3(dim3(32, 32)), 0, s, rec->totals, cap, ntiles, rec->mat, tile_count, pchunk, nbb));
    SS_CUDA_TRY(pdl_launch(pa, k_scan_tiles, dim3(1), dim3(1024), 0, s, ntiles, tile_count, tile_ptr, chunk_ptr, rec->totals, long_list, n_long, cap, overflow, 1));
    SS_CUDA_TRY(pdl_launch(pa, k_bin_scatter, dim3(nbb), dim3(1024), 2 * hsm + (size_t)kBinStage * 6, s, n, rec->rect, k.tx,
                           ntiles, rec->mat, nbb, tile_ptr, tile_count, rec->pbucket, overflow));
  }
#else
  if (n > 0) {
    StageTimer tm(rec, ST_EMIT, s);
    SS_CUDA_TRY(pdl_launch(pa, k_scan_blocks, dim3(1), dim3(1024), 0, s, nb, rec->bsum, rec->totals));
    SS_CUDA_TRY(pdl_launch(pa, k_emit, dim3(nb), dim3(256), 0, s, n, rec->rect, rec->bsum, k.tx, cap, rec->ptile, rec->psplat, overflow));
  }
  {
    StageTimer tm(rec, ST_BUCKET, s);
    const size_t hsm = sizeof(uint32_t) * ntiles;
    set_smem_attrs();
    SS_CUDA_TRY(pdl_launch(pa, k_tile_hist_blocks, dim3(pblocks), dim3(1024), hsm, s, rec->ptile, rec->totals, cap, ntiles, rec->mat, overflow, pchunk));
    SS_CUDA_TRY(pdl_launch(pa, k_tile_prefix, dim3((ntiles + 31) / 32), dim3(dim3(32, 32)), 0, s, rec->totals, cap, ntiles, rec->mat, tile_count, pchunk, 0));
    SS_CUDA_TRY(pdl_launch(pa, k_scan_tiles, dim3(1), dim3(1024), 0, s, ntiles, tile_count, tile_ptr, chunk_ptr, rec->totals, long_list, n_long, cap, overflow, 0));
    SS_CUDA_TRY(pdl_launch(pa, k_tile_scatter, dim3(pblocks), dim3(1024), 2 * hsm + (size_t)pchunk * 6, s, rec->ptile,
                           rec->psplat, rec->totals, cap, ntiles, rec->mat, tile_ptr, rec->pbucket, overflow, pchunk,
                           tile_count));
  }
#endif
  {
    StageTimer tm(rec, ST_TILE_SORT, s);
    // lists over kTileSortMax (listed by k_scan_tiles) sort on the side stream while the
    // regular ones sort here (a regular tile whose equal-key runs defeat the shared-memory
    // sort merge-sorts in place); the blend kernels' work order only needs the list
    // lengths, so it is built on the side stream too
    SS_CUDA_TRY(cudaEventRecord(rec->sort_fork, s));
    SS_CUDA_TRY(cudaStreamWaitEvent(rec->side, rec->sort_fork, 0));
    // dense maps (more than SS_HUGE_SORT splats per tile: lists beyond 8,192 likely) take
    // the 16,384-entry variant; the sorted lists are the same either way
    const bool huge = (long long)n > (long long)SS_HUGE_SORT * ntiles;
    if (huge)
      k_tile_sort_big<kTileSortHuge><<<num_sms(), 1024, sort_smem_bytes<kTileSortHuge, 1024>(), rec->side>>>(
          tile_ptr, rec->pbucket, rec->ptile, rec->key32, rec->key64, long_list, n_long);
    else
      k_tile_sort_big<kTileSortBig><<<num_sms(), 1024, sort_smem_bytes<kTileSortBig, 1024>(), rec->side>>>(
          tile_ptr, rec->pbucket, rec->ptile, rec->key32, rec->key64, long_list, n_long);
    k_tile_order<<<1, 1024, 0, rec->side>>>(ntiles, tile_ptr, order + 2 * (ntiles + 1), order, counters,
                                            split_target, long_target, long_min,
                                            (seg || hyb) ? rec->segorder : nullptr, seg ? 0 : SS_SEG_MIN_LIST,
                                            num_sms() * SS_BWD_MINB * kWarpsPerBlock, rec->totals);
    SS_CUDA_TRY(cudaEventRecord(rec->sort_join, rec->side));
    if (num_sms() * 16 <= ntiles)
      SS_CUDA_TRY(pdl_launch(pa, k_tile_sort<128>, dim3(ntiles), dim3(128), 0, s, tile_ptr, rec->pbucket, rec->ptile, rec->key32, rec->key64, overflow));
    else
      SS_CUDA_TRY(pdl_launch(pa, k_tile_sort<256>, dim3(ntiles), dim3(256), 0, s, tile_ptr, rec->pbucket, rec->ptile, rec->key32, rec->key64, overflow));
    SS_CUDA_TRY(cudaStreamWaitEvent(s, rec->sort_join, 0));
  }
  rec->pairs = (int*)rec->pbucket;
  const int blocks = std::min((ntiles + kWarpsPerBlock - 1) / kWarpsPerBlock, num_sms() * 8);
  {
    StageTimer tmf(rec, ST_FORWARD, s);
    if (long_target) {  // the longest tiles, one block each, concurrently on the side stream
      SS_CUDA_TRY(cudaEventRecord(rec->long_fork, s));
      SS_CUDA_TRY(cudaStreamWaitEvent(rec->side, rec->long_fork, 0));
      k_forward_long<<<std::min(long_target, num_sms() * SS_LONG_BPS), 128, kLongSmem, rec->side>>>(
          rec->bp, tile_ptr, chunk_ptr, rec->pairs, rec->rec, rec->rec64, out_range, out_normal, out_opacity,
          rec->Tf, rec->last, rec->bitmask, overflow, order + 2 * (ntiles + 1), counters + 4, counters + 5);
      SS_CUDA_TRY(cudaEventRecord(rec->long_join, rec->side));
    }
    if (seg_fwd) {
      // pass 1 over the (tile, segment) slots k_seg_order listed, pass 2 per tile, pass 3
      // over the slots pass 2 listed (counters [6] / [8] tickets, [7] pass-3 slot count)
      const int pblk = num_sms() * SS_FWD_MINB;
      SS_CUDA_TRY(pdl_launch(false, k_fwd_seg<1>, dim3(pblk), dim3(kWarpsPerBlock * 32), 0, s, 
          rec->bp, tile_ptr, chunk_ptr, rec->pairs, rec->rec, rec->rec64, out_range, out_normal, out_opacity, rec->Tf,
          rec->last, rec->bitmask, rec->segpart, rec->term_seg, overflow, rec->segorder, counters + 6, counters + 2));
      SS_CUDA_TRY(pdl_launch(pa, k_fwd_seg_combine, dim3((ntiles + kWarpsPerBlock - 1) / kWarpsPerBlock), dim3(kWarpsPerBlock * 32), 0, s, 
          rec->bp, ntiles, tile_ptr, chunk_ptr, rec->segpart, out_range, out_normal, out_opacity, rec->Tf, rec->last,
          rec->term_seg, rec->seg3, counters + 7, overflow));
      SS_CUDA_TRY(pdl_launch(pa, k_fwd_seg<3>, dim3(pblk), dim3(kWarpsPerBlock * 32), 0, s, 
          rec->bp, tile_ptr, chunk_ptr, rec->pairs, rec->rec, rec->rec64, out_range, out_normal, out_opacity, rec->Tf,
          rec->last, rec->bitmask, rec->segpart, rec->term_seg, overflow, rec->seg3, counters + 8, counters + 7));
    } else if (k.T == 8)
      SS_CUDA_TRY(pdl_launch(false, k_forward<8, false>, dim3(blocks), dim3(kWarpsPerBlock * 32), 0, s, rec->bp, ntiles, tile_ptr, chunk_ptr, rec->pairs, rec->rec,
                                                          rec->rec64, out_range, out_normal, out_opacity, rec->Tf,
                                                          rec->last, rec->bitmask, overflow, order + 2 * (ntiles + 1),
                                                          counters, counters + 3));
    else
      SS_CUDA_TRY(pdl_launch(false, k_forward<16, false>, dim3(blocks), dim3(kWarpsPerBlock * 32), 0, s, rec->bp, ntiles, tile_ptr, chunk_ptr, rec->pairs, rec->rec,
                                                           rec->rec64, out_range, out_normal, out_opacity, rec->Tf,
                                                           rec->last, rec->bitmask, overflow, order + 2 * (ntiles + 1),
                                                          counters, counters + 3));
    if (long_target) SS_CUDA_TRY(cudaStreamWaitEvent(s, rec->long_join, 0));
  }
  SS_CUDA_TRY(cudaGetLastError());
  // The totals go to mapped host memory from a side stream: that kernel's
  // store crosses PCIe and would otherwise hold the compute stream behind the
  // caller's bulk copies.  Under CUDA-graph capture the completion event cannot
  // be waited on from the host: the kernel stays on the captured stream and
  // ss_records_check synchronises the device instead.
  cudaStreamCaptureStatus capst = cudaStreamCaptureStatusNone;
  SS_CUDA_TRY(cudaStreamIsCapturing(s, &capst));
  rec->captured = capst != cudaStreamCaptureStatusNone;
  if (rec->captured) {
    k_publish_totals<<<1, 32, 0, s>>>(rec->totals, rec->misc, rec->d_h_totals);
  } else {
    SS_CUDA_TRY(cudaEventRecord(rec->fwd_end, s));
    SS_CUDA_TRY(cudaStreamWaitEvent(rec->side, rec->fwd_end, 0));
    k_publish_totals<<<1, 32, 0, rec->side>>>(rec->totals, rec->misc, rec->d_h_totals);
    SS_CUDA_TRY(cudaEventRecord(rec->done, rec->side));
  }
  SS_CUDA_TRY(cudaGetLastError());
  return SS_OK;
}

// Completes a forward: waits (wait=1) or polls (wait=0, SS_ERR_CAPACITY
// never raised before completion) for its counters.  Returns SS_ERR_CAPACITY
// when the speculative pair capacity was too small (the next forward on
// these records will allocate enough; re-run it), or the device status.
__global__ void k_sticky_or(const int* __restrict__ flag, int* __restrict__ sticky) {
  if (*flag) *sticky = 1;
}

int ss_records_sticky_overflow(const ss_records* rec, int32_t* sticky, void* stream) {
  if (!rec || !sticky || !rec->misc) return SS_ERR_INVALID_ARGUMENT;
  k_sticky_or<<<1, 1, 0, (cudaStream_t)stream>>>(rec->misc + 1, sticky);
  SS_CUDA_TRY(cudaGetLastError());
  return SS_OK;
}

int ss_records_reserve(ss_records* rec, int64_t n_pairs) {
  if (!rec || n_pairs < 0) return SS_ERR_INVALID_ARGUMENT;
  rec->want_pairs = std::max<long long>(rec->want_pairs, n_pairs);
  return SS_OK;
}

int ss_records_generation(const ss_records* rec, uint64_t* generation) {
  if (!rec || !generation) return SS_ERR_INVALID_ARGUMENT;
  *generation = rec->generation;
  return SS_OK;
}

int ss_records_set_deterministic(ss_records* rec, int32_t deterministic) {
  if (!rec) return SS_ERR_INVALID_ARGUMENT;
  rec->deterministic = deterministic ? 1 : 0;
  return SS_OK;
}

int ss_records_check(ss_records* rec, int wait) {
  if (!rec) return SS_ERR_INVALID_ARGUMENT;
  if (!rec->pending) return rec->valid ? SS_OK : SS_ERR_STALE_RECORDS;
  if (rec->captured) {
    if (!wait) return SS_OK;
    SS_CUDA_TRY(cudaDeviceSynchronize());
  } else if (wait) {
    SS_CUDA_TRY(cudaEventSynchronize(rec->done));
  } else if (cudaEventQuery(rec->done) != cudaSuccess) {
    return SS_OK;
  }
  rec->pending = 0;
  const int dev_status = ((int*)(rec->h_totals + 2))[0];
  const int overflow = ((int*)(rec->h_totals + 2))[1];
  rec->n_pairs = rec->h_totals[0];
  rec->n_chunks = rec->h_totals[1];
  rec->last_max_list = rec->h_totals[3];
  if (dev_status) return dev_status;
  if (overflow || rec->n_pairs > rec->cap_pairs) {
    rec->want_pairs = rec->n_pairs + rec->n_pairs / 4 + 1024;
    return SS_ERR_CAPACITY;
  }
  rec->want_pairs = std::max(rec->want_pairs, rec->n_pairs + rec->n_pairs / 8);
  rec->valid = 1;
  return SS_OK;
}

int ss_records_counts(const ss_records* rec, int64_t* n_pairs, int32_t* tiles_x, int32_t* tiles_y) {
  if (rec && rec->pending) {
    int cs = ss_records_check(const_cast<ss_records*>(rec), 1);
    if (cs) return cs;
  }
  if (!rec || !rec->valid) return SS_ERR_STALE_RECORDS;
  if (n_pairs) *n_pairs = rec->n_pairs;
  if (tiles_x) *tiles_x = rec->cam.tx;
  if (tiles_y) *tiles_y = rec->cam.ty;
  return SS_OK;
}

int ss_records_export(const ss_records* rec, int64_t* tile_ptr, int64_t* pair_splats, void* stream) {
  if (rec && rec->pending) {
    int cs = ss_records_check(const_cast<ss_records*>(rec), 1);
    if (cs) return cs;
  }
  if (!rec || !rec->valid) return SS_ERR_STALE_RECORDS;
  cudaStream_t s = (cudaStream_t)stream;
  int nt = rec->ntiles + 1;
  if (tile_ptr) k_widen_i32<<<(nt + 255) / 256, 256, 0, s>>>(nt, rec->tiles, (long long*)tile_ptr);
  if (pair_splats && rec->n_pairs > 0)
    k_widen_i32<<<(int)((rec->n_pairs + 255) / 256), 256, 0, s>>>((int)rec->n_pairs, rec->pairs,
                                                                   (long long*)pair_splats);
  SS_CUDA_TRY(cudaGetLastError());
  return SS_OK;
}

int ss_records_pixel_state(const ss_records* rec, float* final_T, int32_t* last, void* stream) {
  if (rec && rec->pending) {
    int cs = ss_records_check(const_cast<ss_records*>(rec), 1);
    if (cs) return cs;
  }
  if (!rec || !rec->valid) return SS_ERR_STALE_RECORDS;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t P = (size_t)rec->cam.W * rec->cam.H;
  if (final_T) SS_CUDA_TRY(cudaMemcpyAsync(final_T, rec->Tf, P * sizeof(float), cudaMemcpyDeviceToDevice, s));
  if (last) SS_CUDA_TRY(cudaMemcpyAsync(last, rec->last, P * sizeof(int), cudaMemcpyDeviceToDevice, s));
  return SS_OK;
}

// The blend half of the backward: per-splat accumulators from the pixel gradients.
static int backward_blend(ss_records* rec, const ss_splats* splats, const float* dD, const float* dN,
                          const float* dO, cudaStream_t s) {
  const int n = rec->n;
  // acc is all-zero between backward passes: zeroed once when (re)allocated, and
  // k_finalize clears every row it consumes (no per-call 32 MB memset)
  {
    float* before = rec->acc;
    if (grow(rec->acc, rec->cap_acc, (size_t)n * kAcc, s)) return SS_ERR_CUDA;
    if (rec->acc != before) SS_CUDA_TRY(cudaMemsetAsync(rec->acc, 0, sizeof(float) * rec->cap_acc, s));
    rec->note_buffers();
  }
  const int ntiles = rec->ntiles;
  const int* tile_ptr = rec->tiles;
  const int* chunk_ptr = rec->tiles + (ntiles + 1);
  set_smem_attrs();
  float* pacc = nullptr;
  if (rec->deterministic) {
    if (grow(rec->pacc, rec->cap_pacc, (size_t)rec->cap_pairs * kAcc, s)) return SS_ERR_CUDA;
    pacc = rec->pacc;
    rec->note_buffers();
    SS_CUDA_TRY(pdl_launch(!rec->profiling, k_zero_pacc, dim3(num_sms() * 4), dim3(256), 0, s, (float4*)pacc, rec->totals, rec->cap_pairs));
  }
  const int blocks = std::min((ntiles + rec->split_target + kWarpsPerBlock - 1) / kWarpsPerBlock, num_sms() * 8);
  int* order = rec->tiles + 5 * (ntiles + 1);
  int* counters = rec->misc + 4;
  const bool pa = !rec->profiling;
  StageTimer tm(rec, ST_BACKWARD, s);
  if (rec->cam.T == 8 && (rec->seg || rec->hyb))  // segment / whole-tile slots: persistent warps
    SS_CUDA_TRY(pdl_launch(pa, k_backward<8, false, true>, dim3(num_sms() * SS_BWD_MINB), dim3(kWarpsPerBlock * 32), kBwdDynSmem, s, 
        rec->bp, ntiles, tile_ptr, chunk_ptr, rec->pairs, rec->rec, rec->rec64, rec->Tf, rec->last, rec->bitmask, dD,
        dN, dO, rec->acc, rec->misc + 1, rec->segorder, counters + 1, counters + 2, pacc));
  else if (rec->cam.T == 8)
    SS_CUDA_TRY(pdl_launch(pa, rec->split_target ? k_backward<8, true, false> : k_backward<8, false, false>,
                           dim3(blocks), dim3(kWarpsPerBlock * 32), kBwdDynSmem, s, rec->bp, ntiles, tile_ptr,
                           chunk_ptr, rec->pairs, rec->rec, rec->rec64, rec->Tf, rec->last, rec->bitmask, dD, dN, dO,
                           rec->acc, rec->misc + 1, order, counters + 1, counters + 2, pacc));
  else
    SS_CUDA_TRY(pdl_launch(pa, k_backward<16, false, false>, dim3(blocks), dim3(kWarpsPerBlock * 32), kBwdDynSmem, s, 
        rec->bp, ntiles, tile_ptr, chunk_ptr, rec->pairs, rec->rec, rec->rec64, rec->Tf, rec->last, rec->bitmask, dD,
        dN, dO, rec->acc, rec->misc + 1, order, counters + 1, counters + 2, pacc));
  SS_CUDA_TRY(cudaGetLastError());
  if (pacc)
    SS_CUDA_TRY(pdl_launch(pa, k_det_gather, dim3((n + 255) / 256), dim3(256), 0, s, n, rec->cam.tx, rec->rect, rec->key64, tile_ptr, rec->pairs, pacc,
                                                 rec->acc, rec->misc + 1));
  SS_CUDA_TRY(cudaGetLastError());
  return SS_OK;
}

// The finalize half on splats [begin, end): camera-frame -> world / raw gradients
// into rows begin..end-1 of `grads`, clearing the consumed accumulators.
static int backward_finalize(ss_records* rec, const ss_splats* splats, const float* d_scales_extra, float* grads,
                             int raw_space, int begin, int end, cudaStream_t s, const AdamK* adam = nullptr,
                             const float* adam_bias = nullptr, float* adam_m = nullptr, float* adam_v = nullptr,
                             double hinge_cap = 0.0, double hinge_w = 0.0, double* hinge_loss = nullptr) {
  if (end <= begin) return SS_OK;
  const int w = raw_space ? 12 : 15;
  SplatsK sk = to_k(splats);
  sk.n = end - begin;
  sk.centers += 3 * (size_t)begin;
  sk.raw_ta += 3 * (size_t)begin;
  sk.raw_tb += 3 * (size_t)begin;
  sk.log_scales += 2 * (size_t)begin;
  sk.logit_opacity += begin;
  StageTimer tm(rec, ST_FINALIZE, s);
  SS_CUDA_TRY(pdl_launch(!rec->profiling, k_finalize, dim3((sk.n + kFinBlock - 1) / kFinBlock), dim3(kFinBlock), 0, s,
      sk, rec->pose, rec->rec64 + begin, rec->acc + (size_t)begin * kAcc,
      d_scales_extra ? d_scales_extra + 2 * (size_t)begin : nullptr, grads ? grads + (size_t)begin * w : nullptr,
      raw_space, rec->misc + 5, adam ? *adam : AdamK{}, adam_bias, adam_m, adam_v, hinge_cap, hinge_w, hinge_loss));
  SS_CUDA_TRY(cudaGetLastError());
  return SS_OK;
}

static int backward_args(const ss_records* rec, const ss_splats* splats) {
  if (!rec) return SS_ERR_STALE_RECORDS;
  // A forward still in flight (or being captured into a CUDA graph) is fine:
  // stream order covers it and the kernels skip work if its capacity
  // overflowed; completed forwards must have been valid.
  if (!rec->pending && !rec->valid) return SS_ERR_STALE_RECORDS;
  if (!splats || splats->n != rec->n) return SS_ERR_STALE_RECORDS;
  return SS_OK;
}

int ss_render_backward(const ss_records* rec_c, const ss_splats* splats, const float* dD, const float* dN,
                       const float* dO, const float* d_scales_extra, float* grads, int raw_space, void* stream) {
  ss_records* rec = const_cast<ss_records*>(rec_c);
  int st = backward_args(rec, splats);
  if (st) return st;
  if (!dD || !dN || !dO || !grads) return SS_ERR_INVALID_ARGUMENT;
  cudaStream_t s = (cudaStream_t)stream;
  if (rec->n == 0) return SS_OK;
  st = backward_blend(rec, splats, dD, dN, dO, s);
  if (st) return st;
  return backward_finalize(rec, splats, d_scales_extra, grads, raw_space, 0, rec->n, s);
}

int ss_render_backward_blend(const ss_records* rec_c, const ss_splats* splats, const float* dD, const float* dN,
                             const float* dO, void* stream) {
  ss_records* rec = const_cast<ss_records*>(rec_c);
  int st = backward_args(rec, splats);
  if (st) return st;
  if (!dD || !dN || !dO) return SS_ERR_INVALID_ARGUMENT;
  if (rec->n == 0) return SS_OK;
  return backward_blend(rec, splats, dD, dN, dO, (cudaStream_t)stream);
}

int ss_render_finalize(const ss_records* rec_c, const ss_splats* splats, const float* d_scales_extra, float* grads,
                       int raw_space, int32_t begin, int32_t end, void* stream) {
  ss_records* rec = const_cast<ss_records*>(rec_c);
  int st = backward_args(rec, splats);
  if (st) return st;
  if (!grads || begin < 0 || end > rec->n || begin > end) return SS_ERR_INVALID_ARGUMENT;
  // row chunks start on kFinBlock boundaries: the kernel's vector loads stay 16-byte aligned
  if (begin % kFinBlock != 0) return SS_ERR_INVALID_ARGUMENT;
  if (!rec->acc || rec->cap_acc < (size_t)rec->n * kAcc) return SS_ERR_STALE_RECORDS;  // no blend pass yet
  return backward_finalize(rec, splats, d_scales_extra, grads, raw_space, begin, end, (cudaStream_t)stream);
}

// Host staging for the reference-signature drop-in (rasterizer.py, engine.splats_to_device):
// one pass over n float64 values that copies them into the pinned upload buffer, as float64
// or rounded to float32 (dst may be null) and returns their content fingerprint (fp may be
// null: conversion only), the wrapping sum of the values' bit patterns times odd weights of
// the global index i = base + k, so fingerprints of disjoint chunks add.  No
// GPU work; callers run chunks on host threads.
int ss_host_stage_f64(const double* src, void* dst, int32_t dst_f32, int64_t n, int64_t base, uint64_t* fp) {
  if ((!src && n > 0) || n < 0 || base < 0 || (!dst && !fp)) return SS_ERR_INVALID_ARGUMENT;
  uint64_t r = 0;
  if (!dst)
    r = host_stage<0, true>(src, nullptr, n, base);
  else if (!fp)  // conversion only
    r = dst_f32 ? host_stage<2, false>(src, dst, n, base) : host_stage<1, false>(src, dst, n, base);
  else
    r = dst_f32 ? host_stage<2, true>(src, dst, n, base) : host_stage<1, true>(src, dst, n, base);
  if (fp) *fp = r;
  return SS_OK;
}

int ss_fp32_peak_tflops(double* tflops, void* stream) {
  if (!tflops) return SS_ERR_INVALID_ARGUMENT;
  cudaStream_t s = (cudaStream_t)stream;
  int dev = 0, sms = 0;
  SS_CUDA_TRY(cudaGetDevice(&dev));
  SS_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  float* out = nullptr;
  SS_CUDA_TRY(cudaMallocAsync((void**)&out, sizeof(float), s));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8, threads = 256, iters = 2048;
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0, s);
    k_ffma_probe<<<blocks, threads, 0, s>>>(out, iters, 0.999f, 1e-4f);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best) best = ms;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFreeAsync(out, s);
  *tflops = 2.0 * 8 * 16 * (double)iters * blocks * threads / (best * 1e-3) / 1e12;
  return SS_OK;
}

int ss_records_profile(ss_records* rec, int enable) {
  if (!rec) return SS_ERR_INVALID_ARGUMENT;
  rec->profiling = enable != 0;
  return SS_OK;
}

int ss_records_stage_times(ss_records* rec, double* ms, int32_t* launches, int32_t n_stages) {
  if (!rec || !ms || n_stages < ST_COUNT) return SS_ERR_INVALID_ARGUMENT;
  for (int q = 0; q < n_stages; ++q) {
    ms[q] = 0.0;
    if (launches) launches[q] = 0;
  }
  for (auto& u : rec->ev_used) {
    cudaEventSynchronize(u.second.second);
    float t = 0.f;
    cudaEventElapsedTime(&t, u.second.first, u.second.second);
    ms[u.first] += t;
    if (launches) launches[u.first] += 1;
    rec->ev_pool.push_back(u.second.first);
    rec->ev_pool.push_back(u.second.second);
  }
  rec->ev_used.clear();
  return SS_OK;
}

int ss_records_work(const ss_records* rec, int64_t* evaluations, int64_t* contributions, void* stream) {
  if (rec && rec->pending) {
    int cs = ss_records_check(const_cast<ss_records*>(rec), 1);
    if (cs) return cs;
  }
  if (!rec || !rec->valid) return SS_ERR_STALE_RECORDS;
  cudaStream_t s = (cudaStream_t)stream;
  // E = sum over tiles of (pixels in the tile) x (list length), U = popcount of the contribution masks
  std::vector<int> tp(rec->ntiles + 1);
  SS_CUDA_TRY(cudaMemcpyAsync(tp.data(), rec->tiles, sizeof(int) * (rec->ntiles + 1),
                              cudaMemcpyDeviceToHost, s));
  unsigned long long* d_u = nullptr;
  SS_CUDA_TRY(cudaMallocAsync((void**)&d_u, sizeof(unsigned long long), s));
  SS_CUDA_TRY(cudaMemsetAsync(d_u, 0, sizeof(unsigned long long), s));
  if (rec->n_chunks > 0)
    k_count_contrib<<<148 * 4, 256, 0, s>>>(rec->cam, rec->ntiles, rec->tiles, rec->tiles + (rec->ntiles + 1), rec->last,
                                            rec->bitmask, d_u);
  unsigned long long hu = 0;
  SS_CUDA_TRY(cudaMemcpyAsync(&hu, d_u, sizeof(hu), cudaMemcpyDeviceToHost, s));
  SS_CUDA_TRY(cudaFreeAsync(d_u, s));
  SS_CUDA_TRY(cudaStreamSynchronize(s));
  long long E = 0;
  const CamK& k = rec->cam;
  for (int t = 0; t < rec->ntiles; ++t) {
    int tr = t / k.tx, tc = t % k.tx;
    long long ph = std::min(k.T, k.H - tr * k.T), pw = std::min(k.T, k.W - tc * k.T);
    E += ph * pw * (long long)(tp[t + 1] - tp[t]);
  }
  if (evaluations) *evaluations = E;
  if (contributions) *contributions = (int64_t)hu;
  return SS_OK;
}

// ---- photometric registration ------------------------------------------------
namespace {
int make_regcam(const ss_camera* c, RegCam& r) {
  CamK k;
  const int st = make_camk(c, 8, 0.5, k);
  if (st) return st;
  r.W = k.W;
  r.H = k.H;
  r.fx = k.fx;
  r.fy = k.fy;
  r.cx = k.cx;
  r.cy = k.cy;
  r.off_u = k.off_u;
  r.off_v = k.off_v;
  return SS_OK;
}
bool full_circle(const ss_camera* c) {  // geometry.py:117-121
  const double fov = c->az_max - c->az_min;
  const double pitch = fov / (c->width - 1);
  return fov + pitch >= 2.0 * SS_PI - 0.5 * pitch;
}
}  // namespace

size_t ss_anchor_workspace_bytes(int32_t width, int32_t height) {
  const size_t P = (size_t)width * height;
  return P * 10 + ((P + 255) / 256 + 1) * 4 + 64;
}

namespace {
// sample_model's anchors enqueued on s; *counts_dev = the device counts {confident pixels, anchors}
int reg_anchors_enqueue(const ss_camera* geo_cam, const float* D, const float* O, const double* pose_Rt,
                        double vis_opacity, double spread_gate, int32_t thin, double* X_out, int32_t cap,
                        int** counts_dev, void* workspace, cudaStream_t s) {
  RegCam rc;
  int st = make_regcam(geo_cam, rc);
  if (st) return st;
  const int P = rc.W * rc.H;
  const int nb = (P + 255) / 256;
  unsigned char* w = (unsigned char*)workspace;
  double* depth = (double*)w;
  uint8_t* m = (uint8_t*)(w + (size_t)P * 8);
  uint8_t* keep = m + P;
  uint32_t* bsum = (uint32_t*)(((uintptr_t)(keep + P) + 15) & ~(uintptr_t)15);
  int* counts = (int*)(bsum + nb + 1);
  PoseK pk;
  for (int q = 0; q < 9; ++q) pk.R[q] = pose_Rt[q];
  for (int q = 0; q < 3; ++q) pk.t[q] = pose_Rt[9 + q];
  k_anchor_depth<<<nb, 256, 0, s>>>(P, D, O, vis_opacity, depth, m);
  k_anchor_keep<<<nb, 256, 0, s>>>(rc.W, rc.H, full_circle(geo_cam) ? 1 : 0, spread_gate, depth, m, keep, bsum);
  k_excl_scan_small<<<1, 1024, 0, s>>>(nb, bsum);
  k_anchor_emit<<<nb, 256, 0, s>>>(rc.W, rc.H, rc, pk, thin, depth, keep, bsum, X_out, cap, counts);
  SS_CUDA_TRY(cudaGetLastError());
  *counts_dev = counts;
  return SS_OK;
}
}  // namespace

int ss_reg_anchors(const ss_camera* geo_cam, const float* D, const float* O, const double* pose_Rt,
                   double vis_opacity, double spread_gate, int32_t thin, double* X_out, int32_t cap,
                   int32_t* counts_out, void* workspace, void* stream) {
  if (!geo_cam || !D || !O || !pose_Rt || !X_out || !counts_out || !workspace || thin < 1)
    return SS_ERR_INVALID_ARGUMENT;
  cudaStream_t s = (cudaStream_t)stream;
  int* counts = nullptr;
  int st = reg_anchors_enqueue(geo_cam, D, O, pose_Rt, vis_opacity, spread_gate, thin, X_out, cap, &counts,
                               workspace, s);
  if (st) return st;
  SS_CUDA_TRY(cudaMemcpyAsync(counts_out, counts, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
  SS_CUDA_TRY(cudaStreamSynchronize(s));
  return SS_OK;
}

int ss_range_image(const ss_camera* cam, const double* pts, int32_t n, double* range_out, uint8_t* valid_out,
                   void* stream) {
  if (!cam || (!pts && n > 0) || !range_out || !valid_out || n < 0) return SS_ERR_INVALID_ARGUMENT;
  RegCam rc;
  int st = make_regcam(cam, rc);
  if (st) return st;
  cudaStream_t s = (cudaStream_t)stream;
  const int P = rc.W * rc.H;
  unsigned long long* img = (unsigned long long*)range_out;
  // +inf bit pattern in every pixel, then scatter-min of the point ranges
  const double inf = __builtin_inf();
  unsigned long long infbits;
  std::memcpy(&infbits, &inf, sizeof(infbits));
  SS_CUDA_TRY(cudaMemsetAsync(img, 0, sizeof(double) * P, s));
  k_fill_u64<<<(P + 255) / 256, 256, 0, s>>>(P, img, infbits);
  if (n > 0) k_range_scatter<<<(n + 255) / 256, 256, 0, s>>>(pts, n, rc, img);
  k_range_finish<<<(P + 255) / 256, 256, 0, s>>>(P, img, valid_out);
  SS_CUDA_TRY(cudaGetLastError());
  return SS_OK;
}

size_t ss_photo_workspace_bytes(int32_t M) { return (size_t)(M > 0 ? M : 1) * (sizeof(PhotoTmp) + 8) + 512; }

int ss_photo_system(const double* X_w, int32_t M, const double* scan_range, const uint8_t* scan_valid,
                    const ss_camera* cam, const double* T_Rt, double trim_floor, const ss_reg_cfg* cfg,
                    int32_t objective_only, double* out30, void* workspace, void* stream) {
  if (!X_w || M <= 0 || !scan_range || !scan_valid || !cam || !T_Rt || !cfg || !out30 || !workspace)
    return SS_ERR_INVALID_ARGUMENT;
  RegCam rc;
  int st = make_regcam(cam, rc);
  if (st) return st;
  cudaStream_t s = (cudaStream_t)stream;
  unsigned char* w = (unsigned char*)workspace;
  PhotoTmp* tmp = (PhotoTmp*)w;
  unsigned long long* bits = (unsigned long long*)(w + (size_t)M * sizeof(PhotoTmp));
  double* dev_out = (double*)(w + (size_t)M * (sizeof(PhotoTmp) + 8));
  double* median = dev_out + 30;
  int* n_ok = (int*)(median + 1);
  PoseK pk;
  for (int q = 0; q < 9; ++q) pk.R[q] = T_Rt[q];
  for (int q = 0; q < 3; ++q) pk.t[q] = T_Rt[9 + q];
  SS_CUDA_TRY(cudaMemsetAsync(dev_out, 0, sizeof(double) * 32 + 16, s));
  const int nb = (M + 255) / 256;
  k_photo_resid<<<nb, 256, 0, s>>>(X_w, M, pk, rc, scan_range, scan_valid, cfg->spread_gate, tmp, bits, n_ok);
  k_photo_median<<<1, 1024, 0, s>>>(bits, M, n_ok, median);
  k_photo_accum<<<nb, 256, 0, s>>>(M, rc, tmp, bits, median, cfg->trim_factor, trim_floor, cfg->huber_photo,
                                    objective_only, dev_out);
  SS_CUDA_TRY(cudaGetLastError());
  SS_CUDA_TRY(cudaMemcpyAsync(out30, dev_out, sizeof(double) * 30, cudaMemcpyDeviceToHost, s));
  SS_CUDA_TRY(cudaStreamSynchronize(s));
  return SS_OK;
}

size_t ss_reg_solve_workspace_bytes(int32_t n_leaves, int32_t n_geo_scan, int32_t M) {
  const size_t g = (size_t)(n_geo_scan > 0 ? n_geo_scan : 1), m = (size_t)(M > 0 ? M : 1);
  const size_t l = (size_t)(n_leaves > 0 ? n_leaves : 1);
  return g * (sizeof(GeoTmp) + 8) + m * (sizeof(PhotoTmp) + 8) + (size_t)4 * kRsPasses * kRsBins * 4 +
         (size_t)1024 * 2 * kRsAcc * 8 + 1024 * 4 + 1024 * 16 + sizeof(RegSolveState) + (kRsGridBuckets + 1) * 4 +
         l * (sizeof(RsLeafEntry) + 4) + 1024 + sizeof(ss_reg_out) + 32;
}

namespace {
// Packs the final loop state into the public result record (one thread).
__global__ void k_reg_out(const RegSolveState* __restrict__ st, ss_reg_out* __restrict__ out) {
  for (int q = 0; q < 12; ++q) out->T[q] = st->T[q];
  out->r2[0] = st->last_r2[0];
  out->r2[1] = st->last_r2[1];
  out->info[0] = st->it_total;
  out->info[1] = st->converged;
  out->info[2] = st->last_m[0];
  out->info[3] = st->last_m[1];
  out->info[4] = st->n_eval;
  out->info[5] = st->status;
}

// Enqueues the loop on `s` with at most max_blocks blocks (0: one per SM) and the packing
// of its result into out_dev (device memory; may be the workspace's tail).
int reg_solve_launch(const double* leaf_centroids, const double* leaf_normals, int32_t n_leaves,
                     const double* geo_scan, int32_t n_geo_scan, const double* X_w, int32_t M,
                     const double* scan_range, const uint8_t* scan_valid, const ss_camera* cam, const double* T0_Rt,
                     const ss_reg_solve_cfg* cfg, int32_t max_blocks, ss_reg_out* out_dev, void* workspace,
                     cudaStream_t s, const int* dev_counts = nullptr);
}  // namespace

int ss_reg_solve(const double* leaf_centroids, const double* leaf_normals, int32_t n_leaves, const double* geo_scan,
                 int32_t n_geo_scan, const double* X_w, int32_t M, const double* scan_range,
                 const uint8_t* scan_valid, const ss_camera* cam, const double* T0_Rt, const ss_reg_solve_cfg* cfg,
                 double* T_out_Rt, int32_t* info6, double* r2_out2, void* workspace, void* stream) {
  if (!T_out_Rt || !info6 || !r2_out2 || !workspace) return SS_ERR_INVALID_ARGUMENT;
  cudaStream_t s = (cudaStream_t)stream;
  ss_reg_out* od = (ss_reg_out*)((unsigned char*)workspace +
                                 ss_reg_solve_workspace_bytes(n_leaves, n_geo_scan, M) - sizeof(ss_reg_out) - 16);
  od = (ss_reg_out*)(((uintptr_t)od) & ~(uintptr_t)15);
  int st = reg_solve_launch(leaf_centroids, leaf_normals, n_leaves, geo_scan, n_geo_scan, X_w, M, scan_range,
                            scan_valid, cam, T0_Rt, cfg, 0, od, workspace, s);
  if (st) return st;
  ss_reg_out out{};
  SS_CUDA_TRY(cudaMemcpyAsync(&out, od, sizeof(out), cudaMemcpyDeviceToHost, s));
  SS_CUDA_TRY(cudaStreamSynchronize(s));
  for (int q = 0; q < 12; ++q) T_out_Rt[q] = out.T[q];
  for (int q = 0; q < 6; ++q) info6[q] = out.info[q];
  r2_out2[0] = out.r2[0];
  r2_out2[1] = out.r2[1];
  return out.info[5] ? SS_ERR_REGISTRATION : SS_OK;
}

int ss_reg_solve_async(const double* leaf_centroids, const double* leaf_normals, int32_t n_leaves,
                       const double* geo_scan, int32_t n_geo_scan, const double* X_w, int32_t M,
                       const double* scan_range, const uint8_t* scan_valid, const ss_camera* cam, const double* T0_Rt,
                       const ss_reg_solve_cfg* cfg, int32_t max_blocks, ss_reg_out* out_host, void* workspace,
                       void* stream) {
  if (!out_host || !workspace || max_blocks < 0) return SS_ERR_INVALID_ARGUMENT;
  cudaStream_t s = (cudaStream_t)stream;
  ss_reg_out* od = (ss_reg_out*)((unsigned char*)workspace +
                                 ss_reg_solve_workspace_bytes(n_leaves, n_geo_scan, M) - sizeof(ss_reg_out) - 16);
  od = (ss_reg_out*)(((uintptr_t)od) & ~(uintptr_t)15);
  int st = reg_solve_launch(leaf_centroids, leaf_normals, n_leaves, geo_scan, n_geo_scan, X_w, M, scan_range,
                            scan_valid, cam, T0_Rt, cfg, max_blocks, od, workspace, s);
  if (st) return st;
  SS_CUDA_TRY(cudaMemcpyAsync(out_host, od, sizeof(ss_reg_out), cudaMemcpyDeviceToHost, s));
  return SS_OK;
}

int ss_register_photo_batch(int32_t B, const ss_camera* geo_cam, const ss_camera* cam, const ss_splats* splats,
                            const ss_raster_cfg* rcfg, ss_records* const* recs, void* const* streams,
                            const double* poses0_Rt, const double* scan_pts, const int32_t* scan_offsets,
                            int32_t thin, double vis_opacity, double spread_gate, const ss_reg_solve_cfg* cfg,
                            int32_t max_blocks, float* render_buf, double* scan_range, uint8_t* scan_valid,
                            double* anchors, int32_t anchor_cap, void* anchor_ws, size_t anchor_ws_stride,
                            void* solve_ws, size_t solve_ws_stride, ss_reg_out* out_host) {
  if (B < 0 || !geo_cam || !cam || !splats || !rcfg || !recs || !streams || !poses0_Rt || !scan_offsets || !cfg ||
      !render_buf || !scan_range || !scan_valid || !anchors || !anchor_ws || !solve_ws || !out_host || thin < 1 ||
      anchor_cap < 1)
    return SS_ERR_INVALID_ARGUMENT;
  if (cfg->mode != 0) return SS_ERR_UNSUPPORTED;  // photometric only (the other modes: the Python batch path)
  const size_t Pg = (size_t)geo_cam->width * geo_cam->height, P = (size_t)cam->width * cam->height;
  static const bool timing = std::getenv("SS_BATCH_TIMING") != nullptr;  // phase host timestamps (diagnostics)
  // SS_BATCH_PHASED: anchors counted on the host between the phases (A/B)
  static const bool phased = std::getenv("SS_BATCH_PHASED") != nullptr;
  auto now = []() { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
  const double t0 = timing ? now() : 0.0;
  auto frame_render = [&](int b) -> int {
    cudaStream_t s = (cudaStream_t)streams[b];
    float* D = render_buf + (size_t)b * 5 * Pg;
    return ss_render_forward(geo_cam, poses0_Rt + 12 * b, splats, rcfg, D, D + Pg, D + 4 * Pg, recs[b], s);
  };
  auto frame_out_dev = [&](int b) {
    unsigned char* ws = (unsigned char*)solve_ws + b * solve_ws_stride;
    return (ss_reg_out*)(((uintptr_t)(ws + solve_ws_stride - sizeof(ss_reg_out) - 16)) & ~(uintptr_t)15);
  };
  // anchors and loop of frame b on its stream; with dev_counts the loop reads the anchor
  // counts on the device (M = anchor_cap sizes its workspace only)
  auto frame_loop = [&](int b, int32_t M, const int* dev_counts) -> int {
    cudaStream_t s = (cudaStream_t)streams[b];
    ss_reg_out* od = frame_out_dev(b);
    int st = reg_solve_launch(nullptr, nullptr, 0, nullptr, 0, anchors + (size_t)b * anchor_cap * 3, M,
                              scan_range + (size_t)b * P, scan_valid + (size_t)b * P, cam, poses0_Rt + 12 * b, cfg,
                              max_blocks, od, (unsigned char*)solve_ws + b * solve_ws_stride, s, dev_counts);
    if (st) return st;
    SS_CUDA_TRY(cudaMemcpyAsync(out_host + b, od, sizeof(ss_reg_out), cudaMemcpyDeviceToHost, s));
    return (int)SS_OK;
  };
  auto frame_anchors = [&](int b, int** counts_dev) -> int {
    float* D = render_buf + (size_t)b * 5 * Pg;
    return reg_anchors_enqueue(geo_cam, D, D + 4 * Pg, poses0_Rt + 12 * b, vis_opacity, spread_gate, thin,
                               anchors + (size_t)b * anchor_cap * 3, anchor_cap, counts_dev,
                               (unsigned char*)anchor_ws + b * anchor_ws_stride, (cudaStream_t)streams[b]);
  };
  auto frame_scan = [&](int b) -> int {
    const int32_t n = scan_offsets[b + 1] - scan_offsets[b];
    return ss_range_image(cam, scan_pts + 3 * (size_t)scan_offsets[b], n, scan_range + (size_t)b * P,
                          scan_valid + (size_t)b * P, streams[b]);
  };
  // one frame start to finish with host reads (the phased schedule, and the re-run of a
  // frame whose render outgrew its records' speculative capacity)
  auto frame_sync = [&](int b) -> int {
    int st = ss_records_check(recs[b], 1);
    for (int attempt = 0; st == SS_ERR_CAPACITY && attempt < 3; ++attempt) {  // rare: re-render at the exact size
      st = frame_render(b);
      if (!st) st = ss_records_check(recs[b], 1);
    }
    if (st) return st;
    int* cd = nullptr;
    st = frame_anchors(b, &cd);
    if (st) return st;
    int32_t counts[2] = {0, 0};
    SS_CUDA_TRY(cudaMemcpyAsync(counts, cd, sizeof(counts), cudaMemcpyDeviceToHost, (cudaStream_t)streams[b]));
    SS_CUDA_TRY(cudaStreamSynchronize((cudaStream_t)streams[b]));
    if (counts[0] < cfg->min_residuals) {  // the reference's "too few confident pixels"
      ss_reg_out bad{};
      for (int q = 0; q < 12; ++q) bad.T[q] = poses0_Rt[12 * b + q];
      bad.info[5] = 2;
      out_host[b] = bad;
      return (int)SS_OK;
    }
    return frame_loop(b, counts[1], nullptr);
  };
  double t1 = 0.0, t2 = 0.0;
  // 1. every frame's render and scan range image, each on its own stream
  for (int b = 0; b < B; ++b) {
    int st = frame_render(b);
    if (!st) st = frame_scan(b);
    if (st) return st;
  }
  t1 = timing ? now() : 0.0;
  if (!phased) {
    // 2. every frame's anchors, then 3. every frame's loop, all enqueued with no host
    // round trip: the loops read the anchor counts on the device.  (Loops are enqueued
    // after all anchors: a loop started beside the remaining renders slows them more
    // than it gains -- per-frame render/anchors/loop chains measured 1,201 against
    // 1,399 registrations/s at 8 frames.)
    std::vector<int*> cd(B, nullptr);
    for (int b = 0; b < B; ++b) {
      const int st = frame_anchors(b, &cd[b]);
      if (st) return st;
    }
    for (int b = 0; b < B; ++b) {
      const int st = frame_loop(b, anchor_cap, cd[b]);
      if (st) return st;
    }
    t2 = timing ? now() : 0.0;
    for (int b = 0; b < B; ++b) SS_CUDA_TRY(cudaStreamSynchronize((cudaStream_t)streams[b]));
    // a render that overflowed its speculative pair capacity skipped its blend: redo that frame
    for (int b = 0; b < B; ++b) {
      int st = ss_records_check(recs[b], 1);
      if (st == SS_ERR_CAPACITY) {
        st = frame_render(b);
        if (!st) st = frame_sync(b);
        if (st) return st;
        SS_CUDA_TRY(cudaStreamSynchronize((cudaStream_t)streams[b]));
      } else if (st) {
        return st;
      }
    }
  } else {
    // 2. every frame's anchors with a host read of its counts, then 3. the loops
    std::vector<int32_t> M(B, -1);
    for (int b = 0; b < B; ++b) {
      int st = ss_records_check(recs[b], 1);
      for (int attempt = 0; st == SS_ERR_CAPACITY && attempt < 3; ++attempt) {
        st = frame_render(b);
        if (!st) st = ss_records_check(recs[b], 1);
      }
      if (st) return st;
      int* c = nullptr;
      st = frame_anchors(b, &c);
      if (st) return st;
      int32_t counts[2] = {0, 0};
      SS_CUDA_TRY(cudaMemcpyAsync(counts, c, sizeof(counts), cudaMemcpyDeviceToHost, (cudaStream_t)streams[b]));
      SS_CUDA_TRY(cudaStreamSynchronize((cudaStream_t)streams[b]));
      if (counts[0] < cfg->min_residuals) {  // the reference's "too few confident pixels"
        ss_reg_out bad{};
        for (int q = 0; q < 12; ++q) bad.T[q] = poses0_Rt[12 * b + q];
        bad.info[5] = 2;
        out_host[b] = bad;
      } else {
        M[b] = counts[1];
      }
    }
    for (int b = 0; b < B; ++b) {
      if (M[b] < 0) continue;
      const int st = frame_loop(b, M[b], nullptr);
      if (st) return st;
    }
    t2 = timing ? now() : 0.0;
    for (int b = 0; b < B; ++b) SS_CUDA_TRY(cudaStreamSynchronize((cudaStream_t)streams[b]));
  }
  if (timing)
    std::fprintf(stderr, "photo_batch B=%d (%s): enqueued %.3f ms, +%.3f, done +%.3f\n", B, phased ? "phased" : "async",
                 t1 - t0, t2 - t1, now() - t2);
  return SS_OK;
}

namespace {
int reg_solve_launch(const double* leaf_centroids, const double* leaf_normals, int32_t n_leaves,
                     const double* geo_scan, int32_t n_geo_scan, const double* X_w, int32_t M,
                     const double* scan_range, const uint8_t* scan_valid, const ss_camera* cam, const double* T0_Rt,
                     const ss_reg_solve_cfg* cfg, int32_t max_blocks, ss_reg_out* out_dev, void* workspace,
                     cudaStream_t s, const int* dev_counts) {
  if (!cam || !T0_Rt || !cfg || !workspace) return SS_ERR_INVALID_ARGUMENT;
  if (cfg->mode < 0 || cfg->mode > 3 || cfg->max_iters < 0 || cfg->assoc_k < 1) return SS_ERR_INVALID_ARGUMENT;
  // the association keeps register-resident k-best lists of at most 8 leaves
  if (cfg->mode != 0 && cfg->assoc_k > 8) return SS_ERR_UNSUPPORTED;
  const bool need_geo = cfg->mode != 0, need_photo = cfg->mode != 1;
  if (need_geo && (n_leaves < 0 || n_geo_scan < 0 || (n_leaves > 0 && (!leaf_centroids || !leaf_normals)) ||
                   (n_geo_scan > 0 && !geo_scan)))
    return SS_ERR_INVALID_ARGUMENT;
  if (need_photo && (M < 0 || (M > 0 && (!X_w || !scan_range || !scan_valid)))) return SS_ERR_INVALID_ARGUMENT;
  RegCam rc;
  int st = make_regcam(cam, rc);
  if (st) return st;
  // leaf grid buckets: a power of two >= 2 n_leaves in [64, kRsGridBuckets]; staged in
  // shared memory when it fits beside the kernel's static shared memory
  const int nl = need_geo ? n_leaves : 0;
  int nbk = 64;
  while (nbk < kRsGridBuckets && nbk < 2 * nl) nbk *= 2;
  const int gmask = nbk - 1;
  const size_t gsmem = rs_grid_smem_bytes(nl, gmask);
  const bool staged = nl > 0 && gsmem <= (size_t)96 * 1024;
  const size_t dyn = staged ? gsmem : 0;
  // batches (max_blocks given) run the 2-blocks-per-SM build of the loop
  const void* kfn = max_blocks > 0 ? (const void*)k_reg_solve<2> : (const void*)k_reg_solve<1>;
  if (dyn > 0) SS_CUDA_TRY(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
  int occ = 0;
  SS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, kRsThreads, dyn));
  if (occ < 1) return SS_ERR_CUDA;
  const int G = std::min(max_blocks > 0 ? std::min(max_blocks, occ * num_sms()) : num_sms(), 1024);
  const int ng = need_geo ? n_geo_scan : 0, m = need_photo ? M : 0;
  if (ng > G * kRsThreads) return SS_ERR_UNSUPPORTED;  // one scan point per thread
  unsigned char* w = (unsigned char*)workspace;
  auto take = [&](size_t bytes) {
    unsigned char* p = (unsigned char*)(((uintptr_t)w + 15) & ~(uintptr_t)15);
    w = p + bytes;
    return p;
  };
  GeoTmp* gtmp = (GeoTmp*)take((size_t)std::max(ng, 1) * sizeof(GeoTmp));
  unsigned long long* gbits = (unsigned long long*)take((size_t)std::max(ng, 1) * 8);
  PhotoTmp* ptmp = (PhotoTmp*)take((size_t)std::max(m, 1) * sizeof(PhotoTmp));
  unsigned long long* pbits = (unsigned long long*)take((size_t)std::max(m, 1) * 8);
  unsigned* hist = (unsigned*)take((size_t)4 * kRsPasses * kRsBins * 4);
  double* part = (double*)take((size_t)1024 * 2 * kRsAcc * 8);
  int* pcnt = (int*)take(1024 * 4);
  unsigned long long* pmm = (unsigned long long*)take(1024 * 16);
  RegSolveState* state = (RegSolveState*)take(sizeof(RegSolveState));
  int* bstart = (int*)take((size_t)(kRsGridBuckets + 1) * 4);
  RsLeafEntry* ent = (RsLeafEntry*)take((size_t)std::max(nl, 1) * sizeof(RsLeafEntry));
  int* lbucket = (int*)take((size_t)std::max(nl, 1) * 4);
  const double inv_cs = rs_inv_cell(cfg->assoc_gate);
  if (nl > 0) {
    k_leaf_grid<<<1, 1024, 0, s>>>(leaf_centroids, nl, inv_cs, gmask, bstart, ent, lbucket);
    SS_CUDA_TRY(cudaGetLastError());
  }
  // the first evaluation's histograms start zeroed; later evaluations zero the next set themselves
  SS_CUDA_TRY(cudaMemsetAsync(hist, 0, (size_t)4 * kRsPasses * kRsBins * 4, s));
  RegSolveState init{};
  for (int q = 0; q < 12; ++q) init.T[q] = T0_Rt[q];
  SS_CUDA_TRY(cudaMemcpyAsync(state, &init, sizeof(init), cudaMemcpyHostToDevice, s));
  RegSolveCfg k;
  k.huber_photo = cfg->huber_photo;
  k.huber_geo = cfg->huber_geo;
  k.trim_factor = cfg->trim_factor;
  k.spread_gate = cfg->spread_gate;
  k.assoc_gate = cfg->assoc_gate;
  k.floor_photo = cfg->trim_floor_photo;
  k.floor_geo = cfg->trim_floor_geo;
  k.tol = cfg->tol;
  k.damping_init = cfg->damping_init;
  k.damping_max = cfg->damping_max;
  k.max_iters = cfg->max_iters;
  k.min_residuals = cfg->min_residuals;
  k.assoc_k = cfg->assoc_k;
  k.mode = cfg->mode;
  RsGeo geo{leaf_centroids, leaf_normals, nl, geo_scan, ng, bstart, ent, inv_cs, gmask, staged ? 1 : 0};
  RsPhoto ph{X_w, m, scan_range, scan_valid, need_photo ? dev_counts : nullptr};
  void* args[] = {(void*)&geo, (void*)&ph, (void*)&rc, (void*)&k, (void*)&gtmp, (void*)&ptmp,
                  (void*)&gbits, (void*)&pbits, (void*)&hist, (void*)&part, (void*)&pcnt, (void*)&pmm, (void*)&state};
  SS_CUDA_TRY(cudaLaunchCooperativeKernel(kfn, dim3(G), dim3(kRsThreads), args, dyn, s));
  k_reg_out<<<1, 1, 0, s>>>(state, out_dev);
  SS_CUDA_TRY(cudaGetLastError());
  return SS_OK;
}
}  // namespace

int ss_spawn_weights(int32_t width, int32_t height, int32_t wrap, const double* range, const uint8_t* valid,
                     double* w_out, void* stream) {
  if (width < 1 || height < 1 || !range || !valid || !w_out) return SS_ERR_INVALID_ARGUMENT;
  const int P = width * height;
  k_spawn_weights<<<(P + 255) / 256, 256, 0, (cudaStream_t)stream>>>(width, height, wrap ? 1 : 0, range, valid, w_out);
  SS_CUDA_TRY(cudaGetLastError());
  return SS_OK;
}

int ss_densify_mask(int32_t n_pixels, const double* kf_range, const uint8_t* kf_valid, const float* render_range,
                    const float* render_opacity, double densify_opacity, double densify_range_err, uint8_t* mask_out,
                    void* stream) {
  if (n_pixels < 0 || (n_pixels > 0 && (!kf_range || !kf_valid || !render_range || !render_opacity || !mask_out)))
    return SS_ERR_INVALID_ARGUMENT;
  if (n_pixels == 0) return SS_OK;
  k_densify_mask<<<(n_pixels + 255) / 256, 256, 0, (cudaStream_t)stream>>>(
      n_pixels, kf_range, kf_valid, render_range, render_opacity, densify_opacity, densify_range_err, mask_out);
  SS_CUDA_TRY(cudaGetLastError());
  return SS_OK;
}

int ss_spawn_splats(const ss_camera* cam, const double* kf_range, const double* kf_normal, const uint8_t* kf_nvalid,
                    const double* pose_Rt, const int64_t* pixels, int32_t m, double footprint_gain,
                    double scale_floor, double opacity_init, float* centers, float* raw_t_alpha, float* raw_t_beta,
                    float* log_scales, float* logit_opacity, void* stream) {
  if (!cam || !pose_Rt || m < 0) return SS_ERR_INVALID_ARGUMENT;
  if (m == 0) return SS_OK;
  if (!kf_range || !kf_normal || !kf_nvalid || !pixels || !centers || !raw_t_alpha || !raw_t_beta || !log_scales ||
      !logit_opacity || !(opacity_init > 0.0 && opacity_init < 1.0))
    return SS_ERR_INVALID_ARGUMENT;
  CamK ck;
  const int st = make_camk(cam, 8, 0.5, ck);
  if (st) return st;
  SpawnK k;
  k.W = ck.W;
  k.fx = ck.fx;
  k.fy = ck.fy;
  k.cx = ck.cx;
  k.cy = ck.cy;
  k.off_u = ck.off_u;
  k.off_v = ck.off_v;
  for (int q = 0; q < 9; ++q) k.R[q] = pose_Rt[q];
  for (int q = 0; q < 3; ++q) k.t[q] = pose_Rt[9 + q];
  k.gain = footprint_gain;
  k.floor_ = scale_floor;
  k.opacity = opacity_init;
  k_spawn<<<(m + 255) / 256, 256, 0, (cudaStream_t)stream>>>(m, (const long long*)pixels, k, kf_range, kf_normal,
                                                             kf_nvalid, centers, raw_t_alpha, raw_t_beta, log_scales,
                                                             logit_opacity);
  SS_CUDA_TRY(cudaGetLastError());
  return SS_OK;
}

size_t ss_prune_workspace_bytes(int32_t n) {
  const size_t m = (size_t)(n > 0 ? n : 1);
  return m * 4 + ((m + 255) / 256) * 4 + 64;
}

int ss_prune_flags(int32_t n, const float* logit_opacity, double prune_opacity, int32_t* n_keep_out, void* workspace,
                   void* stream) {
  if (n < 0 || !n_keep_out || (n > 0 && (!logit_opacity || !workspace))) return SS_ERR_INVALID_ARGUMENT;
  if (n == 0) {
    *n_keep_out = 0;
    return SS_OK;
  }
  cudaStream_t s = (cudaStream_t)stream;
  uint32_t* keep = (uint32_t*)workspace;
  uint32_t* bsum = keep + n;
  const int nb = (n + 255) / 256;
  k_prune_flags<<<nb, 256, 0, s>>>(n, logit_opacity, prune_opacity, keep, bsum);
  std::vector<uint32_t> h(nb);
  SS_CUDA_TRY(cudaMemcpyAsync(h.data(), bsum, sizeof(uint32_t) * nb, cudaMemcpyDeviceToHost, s));
  SS_CUDA_TRY(cudaStreamSynchronize(s));
  uint32_t run = 0;
  for (int b = 0; b < nb; ++b) {
    const uint32_t c = h[b];
    h[b] = run;
    run += c;
  }
  SS_CUDA_TRY(cudaMemcpyAsync(bsum, h.data(), sizeof(uint32_t) * nb, cudaMemcpyHostToDevice, s));
  SS_CUDA_TRY(cudaStreamSynchronize(s));
  *n_keep_out = (int32_t)run;
  return SS_OK;
}

int ss_prune_compact(int32_t n, int32_t width, const float* src, float* dst, const void* workspace, void* stream) {
  if (n < 0 || width < 1 || (n > 0 && (!src || !dst || !workspace))) return SS_ERR_INVALID_ARGUMENT;
  if (n == 0) return SS_OK;
  const uint32_t* keep = (const uint32_t*)workspace;
  const uint32_t* boff = keep + n;
  k_compact_f32<<<(n + 255) / 256, 256, 0, (cudaStream_t)stream>>>(n, width, keep, boff, src, dst);
  SS_CUDA_TRY(cudaGetLastError());
  return SS_OK;
}

int ss_smooth_range_image(int32_t width, int32_t height, int32_t wrap, const double* range, const uint8_t* valid,
                          double* out, void* stream) {
  if (width < 1 || height < 1 || !range || !valid || !out) return SS_ERR_INVALID_ARGUMENT;
  const int P = width * height;
  k_smooth_range<<<(P + 255) / 256, 256, 0, (cudaStream_t)stream>>>(width, height, wrap ? 1 : 0, range, valid, out);
  SS_CUDA_TRY(cudaGetLastError());
  return SS_OK;
}

int ss_range_image_normals(const ss_camera* cam, const double* range, const uint8_t* valid, double* normal_out,
                           uint8_t* ok_out, void* stream) {
  if (!cam || !range || !valid || !normal_out || !ok_out) return SS_ERR_INVALID_ARGUMENT;
  CamK k;
  const int st = make_camk(cam, 8, 0.5, k);
  if (st) return st;
  const int P = k.W * k.H;
  k_range_normals<<<(P + 255) / 256, 256, 0, (cudaStream_t)stream>>>(k, full_circle(cam) ? 1 : 0, range, valid,
                                                                     normal_out, ok_out);
  SS_CUDA_TRY(cudaGetLastError());
  return SS_OK;
}

size_t ss_leaf_tree_workspace_bytes(int32_t n) {
  const size_t m = (size_t)(n > 0 ? n : 1);
  return m * (4 + 4 + 8 + 2 * 8 + sizeof(LeafRec) + 8 + sizeof(LeafRec)) + lt_top_ws_bytes(num_sms()) + 1024;
}

int ss_leaf_tree_build(const double* pts, int32_t n, const double* viewpoint3, int32_t leaf_size, double tau,
                       int32_t max_leaves, double* centroids_out, double* normals_out, int32_t* sizes_out,
                       uint8_t* usable_out, int32_t* point_leaf_out, int32_t* n_leaves_out, void* workspace,
                       void* stream) {
  if (!pts || n <= 0 || !viewpoint3 || leaf_size < 0 || max_leaves <= 0 || !centroids_out || !normals_out ||
      !sizes_out || !usable_out || !point_leaf_out || !n_leaves_out || !workspace)
    return SS_ERR_INVALID_ARGUMENT;
  cudaStream_t s = (cudaStream_t)stream;
  unsigned char* w = (unsigned char*)workspace;
  auto take = [&](size_t bytes) {
    unsigned char* p = (unsigned char*)(((uintptr_t)w + 15) & ~(uintptr_t)15);
    w = p + bytes;
    return p;
  };
  // a node is split only when larger than leaf_size: a level holds at most 2n/(leaf_size+1) + 2 nodes
  const int cap_nodes = std::min(n, 2 * (n / (leaf_size + 1)) + 2);
  const int cap_leaves = std::min(max_leaves, n);
  int* idx = (int*)take((size_t)n * 4);
  int* tmp = (int*)take((size_t)n * 4);
  double* proj = (double*)take((size_t)n * 8);
  int2* nodes[2] = {(int2*)take((size_t)cap_nodes * 8), (int2*)take((size_t)cap_nodes * 8)};
  LeafRec* recs = (LeafRec*)take((size_t)cap_nodes * sizeof(LeafRec));
  int2* leaf_seg = (int2*)take((size_t)cap_leaves * 8);
  LeafRec* leaf_rec = (LeafRec*)take((size_t)cap_leaves * sizeof(LeafRec));
  int* counts = (int*)take(32);  // [0] nodes of level parity 0, [1] parity 1, [2] leaves, [3] overflow, [4] level
  // top levels (node bound 2^level below the grid): one cooperative kernel, all SMs per level
  const int G = num_sms();
  int top_levels = 0;
  // (measured at config 3: levels 0-4 here, 1.73 -> 0.73 ms; deeper levels have enough
  // nodes for the per-node kernel, whose cost falls with the node size)
  while (top_levels < 5 && (1 << top_levels) <= std::min(kLtTopMaxNodes, G - 1)) ++top_levels;
  LtTopWs tws{};
  tws.part = (double*)take((size_t)G * 9 * 8);
  tws.pmm = (unsigned long long*)take((size_t)G * 16);
  tws.pcnt = (int*)take((size_t)G * 4);
  tws.hist = (unsigned*)take((size_t)3 * kLtTopMaxNodes * kLtBins * 4);
  tws.cand = (unsigned long long*)take((size_t)kLtTopMaxNodes * kLtCand * 8);
  tws.ncand = (int*)take((size_t)kLtTopMaxNodes * 4);
  tws.vmin = (unsigned long long*)take((size_t)kLtTopMaxNodes * 8);
  tws.more = (int*)take(8);
  k_iota<<<(n + 255) / 256, 256, 0, s>>>(n, idx);
  const int init[4] = {1, 0, 0, 0};
  const int2 root = make_int2(0, n);
  SS_CUDA_TRY(cudaMemcpyAsync(counts, init, sizeof(init), cudaMemcpyHostToDevice, s));
  SS_CUDA_TRY(cudaMemcpyAsync(nodes[0], &root, sizeof(root), cudaMemcpyHostToDevice, s));
  const double3 vp = make_double3(viewpoint3[0], viewpoint3[1], viewpoint3[2]);
  // Levels run back to back without host round trips: each level's grid is a
  // bound on its node count (blocks past the actual count exit), the next
  // level is laid out on the device; the host checks for leftovers at the end.
  int level = 0;
  bool tree_done = false;
  if (top_levels > 0) {
    int occ = 0;
    SS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_leaf_top, kLtTopThreads, 0));
    if (occ < 1) return SS_ERR_CUDA;
    const double* a_pts = pts;
    int *a_idx = idx, *a_tmp = tmp, *a_counts = counts;
    double* a_proj = proj;
    int2 *a_n0 = nodes[0], *a_n1 = nodes[1], *a_seg = leaf_seg;
    LeafRec *a_recs = recs, *a_lrec = leaf_rec;
    int a_cap = cap_leaves, a_ls = leaf_size, a_lv = top_levels;
    double a_tau = tau;
    double3 a_vp = vp;
    void* args[] = {(void*)&a_pts, (void*)&a_idx, (void*)&a_tmp, (void*)&a_proj, (void*)&a_n0, (void*)&a_n1,
                    (void*)&a_counts, (void*)&a_recs, (void*)&a_seg, (void*)&a_lrec, (void*)&a_cap, (void*)&a_vp,
                    (void*)&a_ls, (void*)&a_tau, (void*)&a_lv, (void*)&tws};
    SS_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)k_leaf_top, dim3(G), dim3(kLtTopThreads), args, 0, s));
    level = top_levels;
    // every further level in one more cooperative launch (one block per node, grid-stride)
    int occ2 = 0;
    SS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, k_leaf_rest, kLtTopThreads, 0));
    if (occ2 >= 1) {
      int a_l0 = level, a_max = 64;
      void* args2[] = {(void*)&a_pts, (void*)&a_idx, (void*)&a_tmp, (void*)&a_proj, (void*)&a_n0, (void*)&a_n1,
                       (void*)&a_counts, (void*)&a_recs, (void*)&a_seg, (void*)&a_lrec, (void*)&a_cap, (void*)&a_vp,
                       (void*)&a_ls, (void*)&a_tau, (void*)&a_l0, (void*)&a_max};
      SS_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)k_leaf_rest, dim3(G), dim3(kLtTopThreads), args2, 0, s));
      int h5[5];
      SS_CUDA_TRY(cudaMemcpyAsync(h5, counts, sizeof(h5), cudaMemcpyDeviceToHost, s));
      SS_CUDA_TRY(cudaStreamSynchronize(s));
      if (h5[3]) return SS_ERR_CAPACITY;
      level = h5[4];
      tree_done = h5[level & 1] == 0;  // else nodes remain past max_levels: the level loop below
    }
  }
  for (int batch = 0; !tree_done; ++batch) {
    const int depth = batch == 0 ? std::max(1, 2 + (int)std::ceil(std::log2((double)n + 1.0)) - level) : 8;
    for (int q = 0; q < depth; ++q, ++level) {
      const int par = level & 1;
      const long long bound = std::min<long long>(level < 30 ? (1LL << level) : cap_nodes, cap_nodes);
      if (bound < num_sms())  // top levels: few large nodes, 1024 threads each
        k_leaf_level<kLtThreadsBig><<<(int)bound, kLtThreadsBig, 0, s>>>(pts, idx, tmp, proj, nodes[par],
                                                                         counts + par, vp, leaf_size, tau, recs);
      else
        k_leaf_level<kLtThreads><<<(int)bound, kLtThreads, 0, s>>>(pts, idx, tmp, proj, nodes[par], counts + par,
                                                                   vp, leaf_size, tau, recs);
      k_next_level<<<1, 1024, 0, s>>>(nodes[par], counts + par, recs, nodes[par ^ 1], counts + (par ^ 1), leaf_seg,
                                      leaf_rec, counts + 2, cap_leaves, counts + 3);
      SS_CUDA_TRY(cudaGetLastError());
    }
    int h[4];
    SS_CUDA_TRY(cudaMemcpyAsync(h, counts, sizeof(h), cudaMemcpyDeviceToHost, s));
    SS_CUDA_TRY(cudaStreamSynchronize(s));
    if (h[3]) return SS_ERR_CAPACITY;
    if (h[level & 1] == 0) break;  // no node left at the next level
  }
  int nl_total = 0;
  SS_CUDA_TRY(cudaMemcpyAsync(&nl_total, counts + 2, sizeof(int), cudaMemcpyDeviceToHost, s));
  SS_CUDA_TRY(cudaStreamSynchronize(s));
  std::vector<LeafRec> hr(nl_total);
  std::vector<int2> hs(nl_total);
  SS_CUDA_TRY(cudaMemcpyAsync(hr.data(), leaf_rec, sizeof(LeafRec) * nl_total, cudaMemcpyDeviceToHost, s));
  SS_CUDA_TRY(cudaMemcpyAsync(hs.data(), leaf_seg, sizeof(int2) * nl_total, cudaMemcpyDeviceToHost, s));
  SS_CUDA_TRY(cudaStreamSynchronize(s));
  int max_seg = 1;
  for (int i = 0; i < nl_total; ++i) max_seg = std::max(max_seg, hs[i].y - hs[i].x);
  k_leaf_assign<<<dim3(std::max(nl_total, 1), (max_seg + 1023) / 1024), 256, 0, s>>>(idx, leaf_seg, nl_total,
                                                                                     point_leaf_out);
  SS_CUDA_TRY(cudaGetLastError());
  SS_CUDA_TRY(cudaStreamSynchronize(s));
  for (int i = 0; i < nl_total; ++i) {
    for (int k = 0; k < 3; ++k) {
      centroids_out[3 * i + k] = hr[i].c[k];
      normals_out[3 * i + k] = hr[i].n[k];
    }
    sizes_out[i] = hs[i].y - hs[i].x;
    usable_out[i] = (uint8_t)hr[i].usable;
  }
  *n_leaves_out = nl_total;
  return SS_OK;
}

int ss_scale_loss(const float* log_scales, int32_t n, double cap, double w_scale, float* d_scales_extra,
                  double* loss_out, void* stream) {
  if (n < 0 || (n > 0 && (!log_scales || !d_scales_extra || !loss_out))) return SS_ERR_INVALID_ARGUMENT;
  if (n == 0) return SS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  k_scale_loss<<<(n + 255) / 256, 256, 0, s>>>(n, log_scales, cap, w_scale, d_scales_extra, loss_out);
  SS_CUDA_TRY(cudaGetLastError());
  return SS_OK;
}

int ss_adam_step_dev(float* centers, float* raw_t_alpha, float* raw_t_beta, float* log_scales, float* logit_opacity,
                     const float* grads, float* m, float* v, int32_t n, int32_t* t_dev, float* bias_ws,
                     const double* lrs5, double beta1, double beta2, double eps, double log_scale_lo,
                     double log_scale_hi, void* stream) {
  if (n < 0 || !t_dev || !bias_ws || !lrs5) return SS_ERR_INVALID_ARGUMENT;
  if (n == 0) return SS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  AdamK a;
  a.p[0] = centers;
  a.p[1] = raw_t_alpha;
  a.p[2] = raw_t_beta;
  a.p[3] = log_scales;
  a.p[4] = logit_opacity;
  for (int q = 0; q < 5; ++q) a.lr[q] = (float)lrs5[q];
  a.b1 = (float)beta1;
  a.b2 = (float)beta2;
  a.eps = (float)eps;
  a.b1c = a.b2c = 1.f;
  a.lo = (float)log_scale_lo;
  a.hi = (float)log_scale_hi;
  k_adam_tick<<<1, 1, 0, s>>>(t_dev, beta1, beta2, bias_ws);
  k_adam_dev<<<(n + 255) / 256, 256, 0, s>>>(n, a, bias_ws, grads, m, v);
  SS_CUDA_TRY(cudaGetLastError());
  return SS_OK;
}

int ss_render_finalize_adam_dev(const ss_records* rec, const ss_splats* splats, const float* d_scales_extra,
                                float* m, float* v, int32_t* t_dev, float* bias_ws, const double* lrs5,
                                double beta1, double beta2, double eps, double log_scale_lo, double log_scale_hi,
                                double scale_cap, double w_scale, double* scale_loss, void* stream) {
  if (!rec || !splats || !m || !v || !t_dev || !bias_ws || !lrs5) return SS_ERR_INVALID_ARGUMENT;
  ss_records* r = const_cast<ss_records*>(rec);
  if (splats->n != r->n) return SS_ERR_STALE_RECORDS;
  if (splats->n == 0) return SS_OK;
  if (!r->acc) return SS_ERR_STALE_RECORDS;
  cudaStream_t s = (cudaStream_t)stream;
  AdamK a;
  a.p[0] = const_cast<float*>(splats->centers);
  a.p[1] = const_cast<float*>(splats->raw_t_alpha);
  a.p[2] = const_cast<float*>(splats->raw_t_beta);
  a.p[3] = const_cast<float*>(splats->log_scales);
  a.p[4] = const_cast<float*>(splats->logit_opacity);
  for (int q = 0; q < 5; ++q) a.lr[q] = (float)lrs5[q];
  a.b1 = (float)beta1;
  a.b2 = (float)beta2;
  a.eps = (float)eps;
  a.b1c = a.b2c = 1.f;
  a.lo = (float)log_scale_lo;
  a.hi = (float)log_scale_hi;
  k_adam_tick<<<1, 1, 0, s>>>(t_dev, beta1, beta2, bias_ws);
  SS_CUDA_TRY(cudaGetLastError());
  return backward_finalize(r, splats, d_scales_extra, nullptr, 1, 0, splats->n, s, &a, bias_ws, m, v, scale_cap,
                           w_scale, scale_loss);
}

int ss_store_loss_parts(const double* parts4, double* history, int32_t* it_dev, int32_t cap, void* stream) {
  if (!parts4 || !history || !it_dev || cap < 0) return SS_ERR_INVALID_ARGUMENT;
  k_store_parts<<<1, 1, 0, (cudaStream_t)stream>>>(parts4, history, it_dev, cap);
  SS_CUDA_TRY(cudaGetLastError());
  return SS_OK;
}

int ss_adam_step(float* centers, float* raw_t_alpha, float* raw_t_beta, float* log_scales, float* logit_opacity,
                 const float* grads, float* m, float* v, int32_t n, int32_t t, const double* lrs5, double beta1,
                 double beta2, double eps, double log_scale_lo, double log_scale_hi, void* stream) {
  if (n < 0 || t < 1 || !lrs5) return SS_ERR_INVALID_ARGUMENT;
  if (n == 0) return SS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  AdamK a;
  a.p[0] = centers;
  a.p[1] = raw_t_alpha;
  a.p[2] = raw_t_beta;
  a.p[3] = log_scales;
  a.p[4] = logit_opacity;
  for (int q = 0; q < 5; ++q) a.lr[q] = (float)lrs5[q];
  a.b1 = (float)beta1;
  a.b2 = (float)beta2;
  a.eps = (float)eps;
  a.b1c = (float)(1.0 - std::pow(beta1, t));
  a.b2c = (float)(1.0 - std::pow(beta2, t));
  a.lo = (float)log_scale_lo;
  a.hi = (float)log_scale_hi;
  k_adam<<<(n + 255) / 256, 256, 0, s>>>(n, a, grads, m, v);
  SS_CUDA_TRY(cudaGetLastError());
  return SS_OK;
}

int ss_mapping_loss(int32_t width, int32_t height, const float* range, const float* normal, const float* opacity,
                    const float* kf_range, const uint8_t* kf_valid, const float* kf_normal, const uint8_t* kf_nvalid,
                    double w_opacity, double w_normal, double range_floor, float* dD, float* dN, float* dO,
                    double* parts4, void* stream) {
  if (width <= 0 || height <= 0) return SS_ERR_INVALID_ARGUMENT;
  cudaStream_t s = (cudaStream_t)stream;
  int P = width * height;
  int blocks = (P + 511) / 512;  // two pixels per thread
  if (blocks > num_sms() * 8) blocks = num_sms() * 8;
  SS_CUDA_TRY(pdl_launch(true, k_mapping_loss, dim3(blocks), dim3(256), 0, s, P, range, normal, opacity, kf_range,
                         kf_valid, kf_normal, kf_nvalid, w_opacity, w_normal, range_floor, dD, dN, dO, parts4));
  SS_CUDA_TRY(cudaGetLastError());
  return SS_OK;
}

}  // extern "C"
