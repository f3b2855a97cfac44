// FP32 FFMA peak microbenchmark for the roofline denominator (B200, sm_100a).
// Each thread runs 8 independent FMA chains so issue, not latency, bounds it.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void ffma_kernel(float* out, int iters, float a, float b) {
  float x0 = threadIdx.x * 1e-3f, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  float x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
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

// 3-register form: the multiplier is a per-thread register (no immediate/constant operand)
__global__ void ffma3_kernel(float* out, int iters, const float* ab) {
  float a = ab[threadIdx.x & 31], b = ab[32 + (threadIdx.x & 31)];
  float x0 = threadIdx.x * 1e-3f, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  float x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
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

int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  float *out, *ab; cudaMalloc(&out, 4); cudaMalloc(&ab, 256);
  float h[64]; for (int i = 0; i < 64; ++i) h[i] = (i < 32) ? 0.999f : 1e-4f;
  cudaMemcpy(ab, h, 256, cudaMemcpyHostToDevice);
  int blocks = p.multiProcessorCount * 8, threads = 256, iters = 4096;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int variant = 0; variant < 2; ++variant) {
    float best = 1e30f;
    for (int rep = 0; rep < 6; ++rep) {
      cudaEventRecord(e0);
      if (variant == 0) ffma_kernel<<<blocks, threads>>>(out, iters, 0.999f, 1e-4f);
      else ffma3_kernel<<<blocks, threads>>>(out, iters, ab);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (rep > 0 && ms < best) best = ms;
    }
    double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
    printf("{\"ffma_variant\": \"%s\", \"tflops\": %.2f, \"ms\": %.3f, \"sms\": %d}\n",
           variant == 0 ? "imm" : "reg3", flops / best / 1e9, best, p.multiProcessorCount);
  }
  return 0;
}
