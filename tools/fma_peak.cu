// FP32/FP64 FMA-pipe peak microbenchmark (sm_100a): FFMA (3-reg), FFMA2 (f32x2), DFMA.
// Used to record the FP32 roofline denominator (not in MEASURED_PEAKS.json).
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 4096
#define NACC 16

__global__ void k_ffma(float* out, float a, float b) {
  float acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; i++) acc[i] = threadIdx.x * 1e-3f + i;
  float x = a + threadIdx.x * 1e-6f, y = b;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < NACC; i++) acc[i] = fmaf(acc[i], x, y);
  }
  float s = 0; for (int i = 0; i < NACC; i++) s += acc[i];
  if (s == 12345.f) out[0] = s;
}

__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d;
}
__global__ void k_ffma2(float* out, float a, float b) {
  unsigned long long acc[NACC];
  for (int i = 0; i < NACC; i++) { float2 t = make_float2(threadIdx.x * 1e-3f + i, i); acc[i] = *(unsigned long long*)&t; }
  float2 xx = make_float2(a + threadIdx.x * 1e-6f, a), yy = make_float2(b, b);
  unsigned long long x = *(unsigned long long*)&xx, y = *(unsigned long long*)&yy;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < NACC; i++) acc[i] = ffma2(acc[i], x, y);
  }
  float s = 0; for (int i = 0; i < NACC; i++) { float2 t = *(float2*)&acc[i]; s += t.x + t.y; }
  if (s == 12345.f) out[0] = s;
}
__global__ void k_dfma(double* out, double a, double b) {
  double acc[NACC];
  for (int i = 0; i < NACC; i++) acc[i] = threadIdx.x * 1e-3 + i;
  double x = a + threadIdx.x * 1e-6, y = b;
  for (int it = 0; it < ITERS / 4; it++) {
#pragma unroll
    for (int i = 0; i < NACC; i++) acc[i] = fma(acc[i], x, y);
  }
  double s = 0; for (int i = 0; i < NACC; i++) s += acc[i];
  if (s == 12345.) out[0] = s;
}

int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int sms = p.multiProcessorCount;
  float* d; cudaMalloc(&d, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int threads = 256, blocks = sms * 8;
  for (int rep = 0; rep < 2; rep++) {
    double flops = 2.0 * NACC * (double)ITERS * threads * blocks;
    float ms;
    cudaEventRecord(e0); k_ffma<<<blocks, threads>>>(d, 0.999f, 1e-4f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); if (rep) printf("{\"op\": \"ffma\", \"tflops\": %.2f, \"ms\": %.3f}\n", flops / ms / 1e9, ms);
    cudaEventRecord(e0); k_ffma2<<<blocks, threads>>>(d, 0.999f, 1e-4f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); if (rep) printf("{\"op\": \"ffma2\", \"tflops\": %.2f, \"ms\": %.3f}\n", 2 * flops / ms / 1e9, ms);
    cudaEventRecord(e0); k_dfma<<<blocks, threads>>>((double*)d, 0.999, 1e-4); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); if (rep) printf("{\"op\": \"dfma\", \"tflops\": %.2f, \"ms\": %.3f}\n", flops / 4 / ms / 1e9, ms);
  }
  printf("sms %d clock_khz %d\n", sms, p.clockRate);
  return 0;
}
