// Microbenchmark 2: per-instruction cost of tcgen05.mma at small N when the whole
// warp runs the issue loop (descriptors warp-uniform, one elected lane issues),
// kind::tf32 (K=8) vs kind::f16 (K=16), SS and TS; and tcgen05.ld throughput.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tc_lat2 tools/tc_lat2.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2102_04199_b200/csrc/kt_tc.cuh"

using namespace kt::tc;


__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
  return (1u << 4) | (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(M >> 4) << 24);
}

__device__ __forceinline__ void mma_f16_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_f16_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
      "r"(a), "l"(b), "r"(id), "r"(acc));
}

constexpr int NREP = 64;

struct Res {
  long long t[8][4];  // [test][N index]
  long long ld_cycles, ld_bytes;
};

// KIND 0 = tf32 SS, 1 = f16 SS, 2 = f16 TS, 3 = tf32 TS; NACC accumulators round-robin
template <int KIND, int N, int NACC>
__device__ __forceinline__ long long run(uint32_t tmem, uint64_t da, uint64_t db, uint64_t* bar, uint32_t& phase) {
  constexpr uint32_t idt = (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(N >> 3) << 17) | (8u << 24);
  constexpr uint32_t idf = idesc_f16(128, N);
  long long best = 1LL << 60;
  for (int rep = 0; rep < 3; ++rep) {
    __syncwarp();
    const long long t0 = clock64();
    if (elect_one()) {
#pragma unroll
      for (int i = 0; i < NREP; ++i) {
        const uint32_t d = tmem + (i % NACC) * 128;
        const uint32_t acc = i >= NACC;
        if (KIND == 0) mma_tf32(d, da, db, idt, acc);
        if (KIND == 1) mma_f16_ss(d, da, db, idf, acc);
        if (KIND == 2) mma_f16_ts(d, tmem + 384, db, idf, acc);
        if (KIND == 3) mma_tf32_ts(d, tmem + 384, db, idt, acc);
      }
      mma_commit(bar);
    }
    __syncwarp();
    mbar_wait(bar, phase);
    phase ^= 1;
    const long long t1 = clock64();
    if (t1 - t0 < best) best = t1 - t0;
  }
  return best;
}

template <int KIND, int NACC>
__device__ void row(long long* t, uint32_t tmem, uint64_t da, uint64_t db, uint64_t* bar, uint32_t& phase) {
  t[0] = run<KIND, 32, NACC>(tmem, da, db, bar, phase);
  t[1] = run<KIND, 64, NACC>(tmem, da, db, bar, phase);
  t[2] = run<KIND, 128, NACC>(tmem, da, db, bar, phase);
  t[3] = (KIND >= 2 || NACC > 1) ? -1 : run<KIND, 256, NACC>(tmem, da, db, bar, phase);
}

__global__ void lat(Res* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  float* sa = reinterpret_cast<float*>(sm);  // 128 x 32 B
  float* sb = sa + 128 * 8;                  // 256 x 32 B
  uint64_t* bar = reinterpret_cast<uint64_t*>(sb + 256 * 8);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 128 * 8 + 256 * 8; i += blockDim.x) sa[i] = 0.0f;
  if (warp == 0) tmem_alloc(slot, 512);
  if (tid == 0) mbar_init(bar, 1);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  uint32_t phase = 0;
  if (warp == 0) {
    const uint64_t da = kdesc(sa, 8, 0), db = kdesc(sb, 8, 0);
    row<0, 1>(out->t[0], tmem, da, db, bar, phase);
    row<1, 1>(out->t[1], tmem, da, db, bar, phase);
    row<2, 1>(out->t[2], tmem, da, db, bar, phase);
    row<1, 2>(out->t[3], tmem, da, db, bar, phase);
    row<0, 2>(out->t[4], tmem, da, db, bar, phase);
    row<3, 1>(out->t[5], tmem, da, db, bar, phase);
    row<1, 3>(out->t[6], tmem, da, db, bar, phase);
  }
  __syncthreads();
  tc_fence_after();
  // TMEM load throughput: all 4 warps, 64 x (ld.x32 + wait) each
  {
    float acc = 0.f;
    __syncthreads();
    const long long t0 = clock64();
    for (int i = 0; i < 64; ++i) {
      float v[32];
      tmem_ld32(tmem + ((warp * 32) << 16) + (i & 7) * 32, v);
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 32; ++j) acc += v[j];
    }
    __syncthreads();
    const long long t1 = clock64();
    if (tid == 0) {
      out->ld_cycles = t1 - t0;
      out->ld_bytes = 4LL * 64 * 32 * 32 * 4;
    }
    if (acc == 123.f) out->ld_bytes = 0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

// Contention: warp 0 issues NREP MMAs (TS or SS, N=32) while warps 4..7 run
// tcgen05.ld / tcgen05.st loops on other TMEM columns (mode 1 ld only, 2 st only, 3 both).
template <bool TS>
__global__ void contend(long long* out, int mode) {
  extern __shared__ __align__(1024) unsigned char sm[];
  float* sa = reinterpret_cast<float*>(sm);
  float* sb = sa + 128 * 8;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sb + 256 * 8);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  volatile int* stop = reinterpret_cast<volatile int*>(slot + 1);
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 128 * 8 + 256 * 8; i += blockDim.x) sa[i] = 0.0f;
  if (warp == 0) tmem_alloc(slot, 512);
  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 2, 1);
    *stop = 0;
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (warp == 0) {
    const uint64_t da = kdesc(sa, 8, 0), db = kdesc(sb, 8, 0);
    constexpr uint32_t idf = idesc_f16(128, 32);
    for (int i = 0; i < 2000; ++i) __nanosleep(100);  // let the traffic warps ramp up
    __syncwarp();
    const long long t0 = clock64();
    if (elect_one()) {
#pragma unroll
      for (int i = 0; i < NREP; ++i) {
        if (TS) mma_f16_ts(tmem, tmem + 480, db, idf, i > 0);
        else mma_f16_ss(tmem, da, db, idf, i > 0);
      }
      mma_commit(bar);
    }
    __syncwarp();
    mbar_wait(bar, 0);
    const long long t1 = clock64();
    if (tid == 0) {
      out[0] = t1 - t0;
      *stop = 1;
    }
  } else if (warp >= 4 && mode != 0) {
    const uint32_t lane = static_cast<uint32_t>(((warp & 3) * 32) << 16);
    float v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = j;
    long long n = 0;
    if (mode == 4) {  // spin on an mbarrier phase that never completes
      uint64_t* never = bar + 2;
      while (!*stop) {
        uint32_t ok;
        asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.b32 %0, 1, 0, P;\n\t}"
                     : "=r"(ok) : "r"(smem_u32(never)), "r"(0u) : "memory");
        ++n;
      }
    }
    if (mode == 5) {  // shared-memory load/store traffic
      float* buf = reinterpret_cast<float*>(bar + 4) + (warp - 4) * 1024;
      float a = 0.f;
      while (!*stop) {
        for (int r = 0; r < 8; ++r) {
          volatile float* src = buf + 4 * ((tid & 31) + 32 * (r & 7));
          volatile float* dst = buf + 4 * ((tid & 31) + 32 * ((r + 1) & 7));
          const float x0 = src[0], x1 = src[1], x2 = src[2], x3 = src[3];
          a += x0;
          dst[0] = x1;
          dst[1] = x2;
          dst[2] = x3;
          dst[3] = x0;
          ++n;
        }
      }
      if (a == 1.f) n = 0;
    }
    while (mode < 4 && !*stop) {
      for (int r = 0; r < 8; ++r) {
        const uint32_t c = tmem + lane + 128 + 32 * r;
        if (mode & 1) {
          tmem_ld32(c, v);
          tmem_wait_ld();
        }
        if (mode & 2) {
          tmem_st32(c, v);
          tmem_wait_st();
        }
        ++n;
      }
    }
    if ((tid & 31) == 0) out[warp] = n;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

// The scorer's per-chunk MMA sequence in isolation: G1 = 2 K-steps x 3 terms (TS, N=32,
// B = W1 hi/lo, K=16 layout) into D1[q&1], G2 = 4 K-steps x 3 terms (TS, N=32, B = W2 hi/lo,
// K=32 layout) into D2[q&1], optional commits after each group.  No consumers.
template <int COMMITS, bool ALT_B, int FENCE = 0, int DATA = 0>
__global__ void seq(long long* out, int nq) {
  extern __shared__ __align__(1024) unsigned char sm[];
  float* b1h = reinterpret_cast<float*>(sm);
  float* b1l = b1h + 32 * 16;
  float* b2h = b1l + 32 * 16;
  float* b2l = b2h + 32 * 32;
  uint64_t* bars = reinterpret_cast<uint64_t*>(b2l + 32 * 32);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bars + 8);
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 3 * 1024; i += blockDim.x) {
    const float r = DATA ? (float)((i * 2654435761u) % 20011) / 20011.0f - 0.5f : 0.001f * (i % 5);
    b1h[i] = DATA ? tf32_hi(r) : r;
  }
  if (warp == 0) tmem_alloc(slot, 512);
  if (tid == 0)
    for (int i = 0; i < 8; ++i) mbar_init(&bars[i], 1);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (DATA) {  // random values in every TMEM column this benchmark reads
    float v[32];
    for (int c = 0; c < 16; ++c) {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = tf32_hi((float)(((tid * 131 + c * 977 + j * 7919) % 10007)) / 10007.0f - 0.3f);
      tmem_st32(tmem + ((warp * 32) << 16) + 32 * c, v);
    }
    tmem_wait_st();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  if (warp == 0) {
    constexpr uint32_t id32 = (1u << 4) | (2u << 7) | (2u << 10) | (4u << 17) | (8u << 24);
    __syncwarp();
    const long long t0 = clock64();
    if (elect_one()) {
      for (int q = 0; q < nq; ++q) {
        const int s = q & 3, b = q & 1;
        if (FENCE == 1) tc_fence_after();
        if (FENCE == 2) {
          mbar_arrive(&bars[5]);
          mbar_wait(&bars[5], q & 1);
          tc_fence_after();
        }
        const uint32_t xh = tmem + 32 * s, xl = xh + 16, d1 = tmem + 128 + 32 * b;
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          mma_tf32_ts(d1, xh + 8 * kk, kdesc(b1h, 16, kk), id32, kk > 0);
          mma_tf32_ts(d1, xh + 8 * kk, kdesc(ALT_B ? b1l : b1h, 16, kk), id32, 1);
          mma_tf32_ts(d1, xl + 8 * kk, kdesc(b1h, 16, kk), id32, 1);
        }
        if (COMMITS) mma_commit(&bars[0]);
        if (COMMITS > 1) mma_commit(&bars[1]);
        if (FENCE == 1) tc_fence_after();
        if (FENCE == 2) {
          mbar_arrive(&bars[6]);
          mbar_wait(&bars[6], q & 1);
          tc_fence_after();
        }
        const uint32_t rh = tmem + 192 + 64 * b, rl = rh + 32, d2 = tmem + 320 + 32 * b;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          mma_tf32_ts(d2, rh + 8 * kk, kdesc(b2h, 32, kk), id32, kk > 0);
          mma_tf32_ts(d2, rh + 8 * kk, kdesc(ALT_B ? b2l : b2h, 32, kk), id32, 1);
          mma_tf32_ts(d2, rl + 8 * kk, kdesc(b2h, 32, kk), id32, 1);
        }
        if (COMMITS) mma_commit(&bars[2]);
      }
      mma_commit(&bars[7]);
    }
    __syncwarp();
    mbar_wait(&bars[7], 0);
    const long long t1 = clock64();
    if (tid == 0) out[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

// Latency of tcgen05.st / tcgen05.ld (+wait) issued by warp 4 while warp 0 streams MMAs
// (busy = 1) or not (busy = 0).  out[1] = st+wait cycles, out[2] = ld+wait cycles.
__global__ void stlat(long long* out, int busy) {
  extern __shared__ __align__(1024) unsigned char sm[];
  float* sb = reinterpret_cast<float*>(sm);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sb + 256 * 8);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bars + 4);
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 256 * 8; i += blockDim.x) sb[i] = 0.f;
  if (warp == 0) tmem_alloc(slot, 512);
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (warp == 0) {
    constexpr uint32_t id32 = (1u << 4) | (2u << 7) | (2u << 10) | (4u << 17) | (8u << 24);
    if (busy && elect_one()) {
      for (int i = 0; i < 512; ++i) mma_tf32_ts(tmem, tmem + 480, kdesc(sb, 8, 0), id32, i > 0);
      mma_commit(&bars[0]);
    }
    __syncwarp();
    if (busy) mbar_wait(&bars[0], 0);
  } else if (warp == 4) {
    for (int i = 0; i < 200; ++i) __nanosleep(10);
    float v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = j;
    const uint32_t lane = 0;
    long long t0 = clock64();
    for (int r = 0; r < 8; ++r) {
      tmem_st16(tmem + lane + 256 + 16 * r, v);
      tmem_wait_st();
    }
    long long t1 = clock64();
    for (int r = 0; r < 8; ++r) {
      tmem_ld16(tmem + lane + 256 + 16 * r, v);
      tmem_wait_ld();
    }
    long long t2 = clock64();
    if (tid == 128) {
      out[1] = (t1 - t0) / 8;
      out[2] = (t2 - t1) / 8;
      out[3] = (long long)v[3];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

// Round trip: MMA warp issues a group of G TS MMAs (N=32) + commit -> bar0; warp 4 waits
// bar0 (optionally tcgen05.ld of the accumulator), arrives bar1; MMA warp waits bar1; repeat.
template <int G, bool LD, bool ST = false, int NCONS = 1>
__global__ void roundtrip(long long* out, int iters) {
  extern __shared__ __align__(1024) unsigned char sm[];
  float* sb = reinterpret_cast<float*>(sm);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sb + 256 * 8);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bars + 4);
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 256 * 8; i += blockDim.x) sb[i] = 0.f;
  if (warp == 0) tmem_alloc(slot, 512);
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], NCONS);
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (warp == 0) {
    constexpr uint32_t id32 = (1u << 4) | (2u << 7) | (2u << 10) | (4u << 17) | (8u << 24);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (it) {
        mbar_wait(&bars[1], (it - 1) & 1);
        __syncwarp();
        tc_fence_after();
      }
      if (elect_one()) {
#pragma unroll
        for (int i = 0; i < G; ++i) mma_tf32_ts(tmem, tmem + 480, kdesc(sb, 8, 0), id32, i > 0);
        mma_commit(&bars[0]);
      }
      __syncwarp();
    }
    mbar_wait(&bars[1], (iters - 1) & 1);
    const long long t1 = clock64();
    if (tid == 0) out[0] = t1 - t0;
  } else if (warp >= 4 && warp < 4 + NCONS) {
    float v[16];
    float acc = 0.f;
    const uint32_t lane = static_cast<uint32_t>(((warp & 3) * 32) << 16);
    for (int it = 0; it < iters; ++it) {
      mbar_wait(&bars[0], it & 1);
      __syncwarp();
      tc_fence_after();
      if (LD) {
        tmem_ld16(tmem + lane, v);
        tmem_wait_ld();
        acc += v[0];
      }
      if (ST) {
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = 0.001f * j;
        tmem_st16(tmem + lane + 480, v);
        tmem_st16(tmem + lane + 496, v);
        tmem_wait_st();
      }
      tc_fence_before();
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(&bars[1]);
    }
    if (acc == 1234.f) out[5] = 1;
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
  const char* names[7] = {"tf32 SS K8 chain", "f16 SS K16 chain", "f16 TS K16 chain", "f16 SS 2 accs",
                          "tf32 SS 2 accs", "tf32 TS K8 chain", "f16 SS 3 accs"};
  printf("# cycles per tcgen05.mma (M=128), %d back-to-back, whole-warp issue loop + elect\n", NREP);
  printf("| test | N=32 | N=64 | N=128 | N=256 |\n|---|---|---|---|---|\n");
  for (int t = 0; t < 7; ++t) {
    printf("| %s |", names[t]);
    for (int n = 0; n < 4; ++n) printf(" %.1f |", h.t[t][n] < 0 ? -1.0 : double(h.t[t][n]) / NREP);
    printf("\n");
  }
  printf("\ntcgen05.ld 32x32b.x32 + wait, 4 warps x 64: %lld cycles for %lld bytes = %.1f B/cycle\n", h.ld_cycles,
         h.ld_bytes, double(h.ld_bytes) / h.ld_cycles);
  long long* dc;
  cudaMalloc(&dc, 16 * sizeof(long long));
  for (int ts = 0; ts < 2; ++ts) {
    for (int mode = 0; mode < 6; ++mode) {
      cudaMemset(dc, 0, 16 * sizeof(long long));
      if (ts) {
        cudaFuncSetAttribute(contend<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem + 64 + 4 * 4096 * 4);
        contend<true><<<1, 256, smem + 64 + 4 * 4096 * 4>>>(dc, mode);
      } else {
        cudaFuncSetAttribute(contend<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem + 64 + 4 * 4096 * 4);
        contend<false><<<1, 256, smem + 64 + 4 * 4096 * 4>>>(dc, mode);
      }
      if (cudaDeviceSynchronize() != cudaSuccess) {
        printf("contend error\n");
        return 1;
      }
      long long hc[16];
      cudaMemcpy(hc, dc, sizeof(hc), cudaMemcpyDeviceToHost);
      const char* mn[6] = {"none", "ld", "st", "ld+st", "mbarrier-spin", "smem ld/st"};
      printf("%s N=32 MMA with TMEM %s traffic on 4 warps: %.1f cycles/MMA (traffic ops %lld)\n", ts ? "TS" : "SS",
             mn[mode], double(hc[0]) / NREP, hc[4] + hc[5] + hc[6] + hc[7]);
    }
  }
  {
    const int smem2 = (3 * 1024) * 4 + 128;
    long long hc;
    int grid = 1;
    auto go = [&](auto kern, const char* name) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2);
      kern<<<grid, 128, smem2>>>(dc, 64);
      if (cudaDeviceSynchronize() != cudaSuccess) {
        printf("seq error\n");
        return;
      }
      cudaMemcpy(&hc, dc, sizeof(hc), cudaMemcpyDeviceToHost);
      printf("chunk sequence (18 TS MMAs, N=32) %s, grid %d: %.1f cycles/chunk\n", name, grid, double(hc) / 64);
    };
    go(seq<0, true>, "no commits");
    go(seq<2, true>, "3 commits/chunk");
    go(seq<2, false>, "3 commits/chunk, B hi only");
    go(seq<2, true, 1>, "3 commits + fence::after_thread_sync per group");
    go(seq<2, true, 2>, "3 commits + mbarrier arrive/wait + fence per group");
    go(seq<2, true, 0, 1>, "3 commits/chunk, random data");
    grid = 148;
    go(seq<2, true>, "3 commits/chunk");
    go(seq<2, true, 0, 1>, "3 commits/chunk, random data");
    grid = 296;
    go(seq<2, true>, "3 commits/chunk");
  }
  for (int busy = 0; busy < 2; ++busy) {
    const int sm3 = 256 * 8 * 4 + 128;
    cudaFuncSetAttribute(stlat, cudaFuncAttributeMaxDynamicSharedMemorySize, sm3);
    stlat<<<1, 256, sm3>>>(dc, busy);
    if (cudaDeviceSynchronize() != cudaSuccess) {
      printf("stlat error\n");
      return 1;
    }
    long long hc[4];
    cudaMemcpy(hc, dc, sizeof(hc), cudaMemcpyDeviceToHost);
    printf("tcgen05.st.x16+wait %lld cycles, tcgen05.ld.x16+wait %lld cycles (MMA stream %s)\n", hc[1], hc[2],
           busy ? "queued (512 TS MMAs)" : "idle");
  }
  {
    const int sm3 = 256 * 8 * 4 + 128;
    int rgrid = 1, rthreads = 256;
    auto rt = [&](auto kern, const char* name) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, sm3);
      kern<<<rgrid, rthreads, sm3>>>(dc, 64);
      if (cudaDeviceSynchronize() != cudaSuccess) {
        printf("roundtrip error\n");
        return;
      }
      long long hc;
      cudaMemcpy(&hc, dc, sizeof(hc), cudaMemcpyDeviceToHost);
      printf("round trip %s (grid %d, %d threads): %.1f cycles/iteration\n", name, rgrid, rthreads, double(hc) / 64);
    };
    rt(roundtrip<1, false>, "1 MMA");
    rt(roundtrip<6, false>, "6 MMAs");
    rt(roundtrip<12, false>, "12 MMAs");
    rt(roundtrip<6, true>, "6 MMAs + ld");
    rt(roundtrip<12, true>, "12 MMAs + ld");
    rt(roundtrip<12, true, true, 4>, "12 MMAs + ld + st of the A columns, 4 consumer warps");
    rt(roundtrip<12, true, false, 4>, "12 MMAs + ld, 4 consumer warps");
    rthreads = 416;
    rt(roundtrip<6, false, false, 8>, "6 MMAs, 8 consumer warps");
    rt(roundtrip<6, false, false, 4>, "6 MMAs, 4 consumer warps");
    rgrid = 148;
    rt(roundtrip<6, false, false, 8>, "6 MMAs, 8 consumer warps");
    rt(roundtrip<6, false, false, 1>, "6 MMAs, 1 consumer warp");
  }
  return 0;
}
