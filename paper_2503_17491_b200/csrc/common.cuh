// Shared device-side definitions of the B200 Splat-LOAM hot path.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/splat_b200.h"

#define SS_PI 3.14159265358979323846

// Programmatic dependent launch: kernels of the render / backward / mapping step are
// launched with cudaLaunchAttributeProgrammaticStreamSerialization, so the next
// kernel's blocks are scheduled while the previous one drains; each of them waits
// here, first thing, until its predecessor has completed and its writes are visible
// (a no-op for an ordinary launch).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Camera constants in float64, computed on the host with the reference's
// operation order (geometry.py:95-109, 160-174; rasterizer.py:273-276).
struct CamK {
  int W, H, T, tx, ty;
  double fx, fy, cx, cy, off_u, off_v;
  double pad_az, pad_el;
};

// RasterConfig scalars (rasterizer.py:69-78)
struct RasterK {
  double alpha_cutoff, alpha_clamp, min_transmittance, denom_eps, cutoff_sigma;
};

struct PoseK {
  double R[9];  // row-major, sensor-in-world (se3.py:3-7)
  double t[3];
};

struct SplatsK {
  int n;
  const float* centers;
  const float* raw_ta;
  const float* raw_tb;
  const float* log_scales;
  const float* logit_opacity;
};

// Per-splat records written by the preprocess kernel and staged per
// (tile, splat) pair by the blend kernels (96 B per staged entry):
//   SplatRec   (float32, 16 B): r0 = (opacity, Kp, ncam.x, ncam.y)
//              Kp = 2 ln(opacity/alpha_cutoff) (+ tiny margin): alpha >= cutoff <=> sa^2+sb^2 <= K
//   SplatRec64 (float64, 80 B): Ba, Bb, Bc (camera frame) and ncam.z
struct SplatRec {
  float4 r0;
};
struct SplatRec64 {
  double2 v[5];  // Ba.xy | Ba.z Bb.x | Bb.yz | Bc.xy | Bc.z ncam.z
};

// --- IEEE float64 helpers with contraction disabled (bit-exact binning) ---
__device__ __forceinline__ double x_add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double x_sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double x_mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double x_div(double a, double b) { return __ddiv_rn(a, b); }

// np.mod semantics for floats: result carries the sign of the divisor.
__device__ __forceinline__ double py_mod(double a, double b) {
  double m = fmod(a, b);
  if (m != 0.0 && ((b < 0.0) != (m < 0.0))) m = x_add(m, b);
  return m;
}

// Angular interval of tile column / row from its first and last sample
// (rasterizer.py:278-294).
__device__ __forceinline__ void tile_col_interval(const CamK& k, int c, double& center, double& hw) {
  int f = c * k.T;
  int l = min(f + k.T, k.W) - 1;
  double a0 = x_div(x_sub(x_add((double)f, k.off_u), k.cx), k.fx);
  double a1 = x_div(x_sub(x_add((double)l, k.off_u), k.cx), k.fx);
  center = x_mul(0.5, x_add(a0, a1));
  hw = x_mul(0.5, fabs(x_sub(a0, a1)));
}
__device__ __forceinline__ void tile_row_interval(const CamK& k, int r, double& center, double& hw) {
  int f = r * k.T;
  int l = min(f + k.T, k.H) - 1;
  double e0 = x_div(x_sub(x_add((double)f, k.off_v), k.cy), k.fy);
  double e1 = x_div(x_sub(x_add((double)l, k.off_v), k.cy), k.fy);
  center = x_mul(0.5, x_add(e0, e1));
  hw = x_mul(0.5, fabs(x_sub(e0, e1)));
}

// Unit ray at continuous sample position (u, v) (geometry.py:123-127, 60-65).
__device__ __forceinline__ void ray_at(const CamK& k, double u, double v, double d[3]) {
  double az = (u - k.cx) / k.fx;
  double el = (v - k.cy) / k.fy;
  double sa, ca, se, ce;
  sincos(az, &sa, &ca);
  sincos(el, &se, &ce);
  d[0] = ce * ca;
  d[1] = ce * sa;
  d[2] = se;
}

#define SS_CUDA_TRY(expr)                          \
  do {                                             \
    cudaError_t _e = (expr);                       \
    if (_e != cudaSuccess) return SS_ERR_CUDA;     \
  } while (0)

// entries for a tile to count as long (k_tile_order -> k_forward_long)
#ifndef SS_LONG_MIN
#define SS_LONG_MIN 256
#endif

// segment-parallel backward when tiles are few (blend.cu kSegChunks)
#ifndef SS_SEG_MODE
#define SS_SEG_MODE 1
#endif
#ifndef SS_SEG_ALWAYS
#define SS_SEG_ALWAYS 0
#endif
#ifndef SS_HUGE_SORT
#define SS_HUGE_SORT 256  // the 16,384-entry list sort pass when splats > this x tiles
#endif
#ifndef SS_DIRECT_BIN
#define SS_DIRECT_BIN 1  // tile buckets straight from the splats' tile rectangles (no pair list)
#endif
#ifndef SS_SEG_MIN_LIST
#define SS_SEG_MIN_LIST -1  // many tiles: lists this long are walked in segments (-1: a fair share, see k_tile_order)
#endif
// with many tiles only lists of >= SS_LONG_MIN_MANY entries take the block kernel (0: none)
#ifndef SS_LONG_MIN_MANY
#define SS_LONG_MIN_MANY 1536  // (config-3 registration render: forward 224 -> 181 us; config 1 unchanged)
#endif
