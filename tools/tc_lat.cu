// Microbenchmark: tcgen05.mma kind::tf32 latency / throughput at small N on one SM.
//   chain:  n MMAs (M=128, N, K=8) into one accumulator, commit, wait  -> cycles
//   indep:  the same n MMAs spread round-robin over A accumulators
//   ts:     A operand from TMEM instead of shared memory
//   ld:     tcgen05.ld 32x32b.x16 / .x32 + wait::ld, one warp
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tc_lat tools/tc_lat.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2102_04199_b200/csrc/kt_tc.cuh"

using namespace kt::tc;

struct Res {
  long long chain[4][7];
  long long indep2[4][7];
  long long indep4[4][7];
  long long ts[7];
  long long ld16, ld32, commit_only;
};

__global__ void lat(Res* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  float* sa = reinterpret_cast<float*>(sm);            // 128 x 8
  float* sb = sa + 128 * 8;                             // 256 x 8
  uint64_t* bar = reinterpret_cast<uint64_t*>(sb + 256 * 8);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 128 * 8 + 256 * 8; i += blockDim.x) sa[i] = 0.001f * (i % 7);
  if (warp == 0) tmem_alloc(slot, 512);
  if (tid == 0) mbar_init(bar, 1);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  const int ns[7] = {1, 2, 4, 8, 16, 32, 64};
  const int Ns[4] = {32, 64, 128, 256};
  uint32_t phase = 0;
  if (tid == 0) {
    for (int ni = 0; ni < 4; ++ni) {
      const int N = Ns[ni];
      const uint32_t id = idesc_tf32(128, N);
      for (int mode = 0; mode < 3; ++mode) {
        const int nacc = mode == 0 ? 1 : (mode == 1 ? 2 : 4);
        if (N * nacc > 512) {
          for (int j = 0; j < 7; ++j) (mode == 1 ? out->indep2 : out->indep4)[ni][j] = -1;
          continue;
        }
        for (int j = 0; j < 7; ++j) {
          long long best = 1LL << 60;
          for (int rep = 0; rep < 4; ++rep) {
            const long long t0 = clock64();
            for (int i = 0; i < ns[j]; ++i) {
              const int a = i % nacc;
              mma_tf32(tmem + N * a, kdesc(sa, 8, 0), kdesc(sb, 8, 0), id, i >= nacc);
            }
            mma_commit(bar);
            mbar_wait(bar, phase);
            phase ^= 1;
            const long long t1 = clock64();
            if (t1 - t0 < best) best = t1 - t0;
          }
          if (mode == 0) out->chain[ni][j] = best;
          if (mode == 1) out->indep2[ni][j] = best;
          if (mode == 2) out->indep4[ni][j] = best;
        }
      }
    }
    // TS: A from TMEM columns [256, 264), N = 32 into column 0
    const uint32_t id = idesc_tf32(128, 32);
    for (int j = 0; j < 7; ++j) {
      long long best = 1LL << 60;
      for (int rep = 0; rep < 4; ++rep) {
        const long long t0 = clock64();
        for (int i = 0; i < ns[j]; ++i) mma_tf32_ts(tmem, tmem + 256, kdesc(sb, 8, 0), id, i > 0);
        mma_commit(bar);
        mbar_wait(bar, phase);
        phase ^= 1;
        const long long t1 = clock64();
        if (t1 - t0 < best) best = t1 - t0;
      }
      out->ts[j] = best;
    }
    {
      long long best = 1LL << 60;
      for (int rep = 0; rep < 4; ++rep) {
        const long long t0 = clock64();
        mma_commit(bar);
        mbar_wait(bar, phase);
        phase ^= 1;
        const long long t1 = clock64();
        if (t1 - t0 < best) best = t1 - t0;
      }
      out->commit_only = best;
    }
  }
  __syncthreads();
  tc_fence_after();
  if (warp == 0) {
    float v[32];
    long long b16 = 1LL << 60, b32 = 1LL << 60;
    for (int rep = 0; rep < 4; ++rep) {
      long long t0 = clock64();
      tmem_ld16(tmem, v);
      tmem_wait_ld();
      long long t1 = clock64();
      if (v[3] == 12345.f) out->ld16 = 0;
      if (t1 - t0 < b16) b16 = t1 - t0;
      t0 = clock64();
      tmem_ld32(tmem, v);
      tmem_wait_ld();
      t1 = clock64();
      if (v[5] == 12345.f) out->ld16 = 0;
      if (t1 - t0 < b32) b32 = t1 - t0;
    }
    if (tid == 0) {
      out->ld16 = b16;
      out->ld32 = b32;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

int main() {
  Res* d;
  cudaMalloc(&d, sizeof(Res));
  const int smem = (128 * 8 + 256 * 8) * 4 + 64;
  cudaFuncSetAttribute(lat, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  lat<<<1, 128, smem>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return 1;
  }
  Res h;
  cudaMemcpy(&h, d, sizeof(Res), cudaMemcpyDeviceToHost);
  const int ns[7] = {1, 2, 4, 8, 16, 32, 64};
  const int Ns[4] = {32, 64, 128, 256};
  printf("# tcgen05.mma kind::tf32 M=128 K=8, cycles from first issue to commit-wait return (min of 4)\n");
  printf("| N | mode | n=1 | 2 | 4 | 8 | 16 | 32 | 64 |\n|---|---|---|---|---|---|---|---|---|\n");
  for (int ni = 0; ni < 4; ++ni) {
    const char* names[3] = {"chain (1 acc)", "2 accs", "4 accs"};
    long long* rows[3] = {h.chain[ni], h.indep2[ni], h.indep4[ni]};
    for (int m = 0; m < 3; ++m) {
      printf("| %d | %s |", Ns[ni], names[m]);
      for (int j = 0; j < 7; ++j) printf(" %lld |", rows[m][j]);
      printf("\n");
    }
  }
  printf("| 32 | TS chain |");
  for (int j = 0; j < 7; ++j) printf(" %lld |", h.ts[j]);
  printf("\n\ncommit+wait with nothing outstanding: %lld cycles\n", h.commit_only);
  printf("tcgen05.ld x16 + wait: %lld cycles; x32 + wait: %lld cycles\n", h.ld16, h.ld32);
  (void)ns;
  return 0;
}
