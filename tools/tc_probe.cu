// Probe: tcgen05 kind::tf32 MMA, M=128 N=32 K=32, K-major SWIZZLE_NONE smem operands,
// accumulator in TMEM read back with tcgen05.ld.32x32b.x32.  Validates the descriptor
// encodings used by the fused scorer (csrc/kt_tc.cuh) against a CPU GEMM.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cmath>
#include <cuda_runtime.h>
#include "../paper_2102_04199_b200/csrc/kt_tc.cuh"

using namespace kt::tc;

constexpr int M = 128, N = 32, K = 32;

__global__ void probe(const float* A, const float* B, float* D, float* D3, float* D4) {
  __shared__ __align__(1024) float sa[M * K];
  __shared__ __align__(1024) float sb[N * K];
  __shared__ __align__(1024) float sa_lo[M * K];
  __shared__ __align__(1024) float sb_lo[N * K];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) tmem_alloc(&tmem_slot, 256);
  if (tid == 0) mbar_init(&bar, 1);
  // operands into the canonical K-major no-swizzle layout; A also split hi/lo
  for (int k = 0; k < K; ++k) {
    const float v = A[tid * K + k];
    const float hi = tf32_hi(v);
    sa[kmajor_offset(tid, k, K) / 4] = hi;
    sa_lo[kmajor_offset(tid, k, K) / 4] = v - hi;
  }
  if (tid < N)
    for (int k = 0; k < K; ++k) {
      const float v = B[tid * K + k];
      const float hi = tf32_hi(v);
      sb[kmajor_offset(tid, k, K) / 4] = hi;
      sb_lo[kmajor_offset(tid, k, K) / 4] = v - hi;
    }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  if (tid == 0) {
    const uint32_t idesc = idesc_tf32(M, N);
    // plain tf32 product into columns [0, 32), 3xTF32 into [32, 64)
    for (int kk = 0; kk < K / 8; ++kk)
      mma_tf32(tmem, kdesc(sa, K, kk), kdesc(sb, K, kk), idesc, kk > 0);
    int first = 1;
    for (int kk = 0; kk < K / 8; ++kk) {
      mma_tf32(tmem + 32, kdesc(sa, K, kk), kdesc(sb, K, kk), idesc, !first); first = 0;
      mma_tf32(tmem + 32, kdesc(sa, K, kk), kdesc(sb_lo, K, kk), idesc, 1);
      mma_tf32(tmem + 32, kdesc(sa_lo, K, kk), kdesc(sb, K, kk), idesc, 1);
    }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  float v[32];
  tmem_ld32(tmem + ((warp * 32) << 16), v);
  tmem_wait_ld();
  for (int j = 0; j < N; ++j) D[tid * N + j] = v[j];
  tmem_ld32(tmem + ((warp * 32) << 16) + 32, v);
  tmem_wait_ld();
  for (int j = 0; j < N; ++j) D3[tid * N + j] = v[j];
  // TS check: R = D3 (this thread's row) -> TMEM A operand (hi at col 64, lo at col 96),
  // D4 (col 128) = R * B^T via 3xTF32 with A read from TMEM
  float hi[32], lo[32];
  for (int j = 0; j < 32; ++j) { hi[j] = tf32_hi(v[j]); lo[j] = v[j] - hi[j]; }
  tmem_st32(tmem + ((warp * 32) << 16) + 64, hi);
  tmem_st32(tmem + ((warp * 32) << 16) + 96, lo);
  tmem_wait_st();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    const uint32_t idesc = idesc_tf32(M, N);
    for (int kk = 0; kk < 4; ++kk) {
      mma_tf32_ts(tmem + 128, tmem + 64 + 8 * kk, kdesc(sb, K, kk), idesc, kk > 0);
      mma_tf32_ts(tmem + 128, tmem + 64 + 8 * kk, kdesc(sb_lo, K, kk), idesc, 1);
      mma_tf32_ts(tmem + 128, tmem + 96 + 8 * kk, kdesc(sb, K, kk), idesc, 1);
    }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 1);
  tc_fence_after();
  tmem_ld32(tmem + ((warp * 32) << 16) + 128, v);
  tmem_wait_ld();
  for (int j = 0; j < N; ++j) D4[tid * N + j] = v[j];
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 256);
}

int main() {
  float *A, *B, *D, *D3, *D4;
  cudaMallocManaged(&A, M * K * 4); cudaMallocManaged(&B, N * K * 4);
  cudaMallocManaged(&D, M * N * 4); cudaMallocManaged(&D3, M * N * 4); cudaMallocManaged(&D4, M * N * 4);
  srand(1);
  for (int i = 0; i < M * K; ++i) A[i] = (rand() / (float)RAND_MAX - 0.5f) * 2.0f;
  for (int i = 0; i < N * K; ++i) B[i] = (rand() / (float)RAND_MAX - 0.5f) * 2.0f;
  probe<<<1, 128>>>(A, B, D, D3, D4);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("{\"ok\": false, \"err\": \"%s\"}\n", cudaGetErrorString(e)); return 1; }
  double max1 = 0, max3 = 0, ref_max = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      double r = 0;
      for (int k = 0; k < K; ++k) r += (double)A[i * K + k] * (double)B[j * K + k];
      max1 = fmax(max1, fabs(D[i * N + j] - r));
      max3 = fmax(max3, fabs(D3[i * N + j] - r));
      ref_max = fmax(ref_max, fabs(r));
    }
  double max4 = 0, ref4 = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      double r = 0;
      for (int k = 0; k < K; ++k) r += (double)D3[i * N + k] * (double)B[j * K + k];
      max4 = fmax(max4, fabs(D4[i * N + j] - r));
      ref4 = fmax(ref4, fabs(r));
    }
  printf("{\"ok\": true, \"max_abs_err_tf32\": %.3e, \"max_abs_err_3xtf32\": %.3e, \"ref_max\": %.3e, "
         "\"ts_max_abs_err\": %.3e, \"ts_ref_max\": %.3e}\n", max1, max3, ref_max, max4, ref4);
  return 0;
}
