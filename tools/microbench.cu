// microbench.cu -- measured B200 issue/pipe rates used by the "alu" roofline
// (DESIGN.md).  Each kernel runs 148*8 CTAs x 256 threads of independent
// chains; reports lane-ops per second.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb tools/microbench.cu
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 4096

__global__ void k_ex2(float* out, float s) {
  float a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = -1e-3f * (threadIdx.x + j);
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[j]));
  }
  float r = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) r += a[j];
  if (r == s) out[0] = r;
}

__global__ void k_ffma(float* out, float s) {
  float a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x + j;
  const float b = s, c = 1e-7f * s;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[j]) : "f"(b), "f"(c));
  }
  float r = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) r += a[j];
  if (r == s) out[0] = r;
}

__global__ void k_ffma2(float* out, float s) {
  float2 a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = make_float2(threadIdx.x + j, j);
  const float2 b = make_float2(s, s), c = make_float2(1e-7f * s, 2e-7f);
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = __ffma2_rn(a[j], b, c);
    asm volatile("" ::: "memory");
  }
  float r = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) r += a[j].x + a[j].y;
  if (r == s) out[0] = r;
}

// 1 ex2 : 2 FFMA2 (the scan forward's per-element mix without loads)
__global__ void k_mix(float* out, float s) {
  float e[8];
  float2 h[4];
#pragma unroll
  for (int j = 0; j < 8; ++j) e[j] = -1e-3f * (threadIdx.x + j);
#pragma unroll
  for (int j = 0; j < 4; ++j) h[j] = make_float2(j, j);
  const float2 b = make_float2(s, s);
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(e[j]));
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      h[j] = __ffma2_rn(make_float2(e[2 * j], e[2 * j + 1]), h[j], b);
      h[j] = __ffma2_rn(h[j], b, b);
    }
  }
  float r = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) r += h[j].x + h[j].y;
  if (r == s) out[0] = r;
}

template <typename K>
double run(K kern, const char* name, double ops_per_thread_iter, int blocks, float* d) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  kern<<<blocks, 256>>>(d, 3.f);
  cudaEventRecord(a);
  kern<<<blocks, 256>>>(d, 3.f);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  double ops = ops_per_thread_iter * ITERS * 256.0 * blocks;
  printf("{\"kernel\": \"%s\", \"ms\": %.4f, \"Gop_per_s\": %.1f, \"per_sm_per_clk_at_1965MHz\": %.2f}\n",
         name, ms, ops / ms / 1e6, ops / (ms * 1e-3) / 148 / 1.965e9);
  return ops / ms / 1e6;
}

int main() {
  float* d;
  cudaMalloc(&d, 4);
  const int blocks = 148 * 8;
  run(k_ex2, "mufu_ex2 (lane-ops)", 8, blocks, d);
  run(k_ffma, "ffma (lane-flops/2)", 8, blocks, d);
  run(k_ffma2, "ffma2 (lane-fma, 2 per instr)", 16, blocks, d);
  run(k_mix, "mix 8 ex2 + 8 ffma2 (ex2 count)", 8, blocks, d);
  return 0;
}
