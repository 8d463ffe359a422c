// sm_100a tensor-core helpers: tcgen05 MMA (kind::tf32, cta_group::1), TMEM
// allocation / loads, mbarriers, descriptors.  Inline PTX only.
//
// Operand layout: K-major, SWIZZLE_NONE ("interleaved") canonical layout.  An
// operand tile of R rows x K fp32 is stored as 8-row x 16-byte core matrices:
//   byte(row, k) = ((row / 8) * (K / 4) + k / 4) * 128 + (row % 8) * 16 + (k % 4) * 4
// so K-adjacent core matrices are 128 B apart (LBO) and 8-row groups are
// K * 32 B apart (SBO).  One kind::tf32 MMA consumes K = 8 (two core matrices);
// K-step kk starts at byte 256 * kk.
//
// 3xTF32: A*B ~= Ah*Bh + Ah*Bl + Al*Bh with Xh = rna_tf32(X), Xl = X - Xh, all
// accumulated in fp32 in TMEM -- fp32-level accuracy on the tensor pipe.
#pragma once

#ifndef KT_WAIT_SLEEP
#define KT_WAIT_SLEEP 20
#endif
#if !defined(KT_WAIT_HINT) && !defined(KT_WAIT_SPIN)
#define KT_WAIT_HINT 1000000  // ns: waiting threads are parked by the hardware
#endif

#include <cuda_runtime.h>
#include <stdint.h>

namespace kt {
namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__host__ __device__ __forceinline__ int kmajor_offset(int row, int k, int K) {
  return ((row >> 3) * (K >> 2) + (k >> 2)) * 128 + (row & 7) * 16 + (k & 3) * 4;
}

// Shared-memory matrix descriptor (SmemDescriptor, sm100 version 1, no swizzle).
__device__ __forceinline__ uint64_t kdesc(const void* tile, int K, int kk) {
  const uint32_t addr = smem_u32(tile) + 256u * kk;
  const uint64_t lbo = 128u >> 4;
  const uint64_t sbo = (static_cast<uint32_t>(K) * 32u) >> 4;
  return static_cast<uint64_t>((addr >> 4) & 0x3FFFu) | (lbo << 16) | (sbo << 32) | (1ull << 46);
}

// Instruction descriptor: F32 accumulate, TF32 A/B, both K-major, dense.
__host__ __device__ __forceinline__ uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}

__device__ __forceinline__ float tf32_hi(float v) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
  return __uint_as_float(r);
}

// Truncating split (one LOP3): hi keeps the 10 explicit tf32 mantissa bits, and
// lo = v - hi is exact in fp32, so hi + lo == v; the tensor core then sees lo to
// 11 significant bits (split error <= 2^-21 |v|, fp32-level).  For the hot loops.
__device__ __forceinline__ float tf32_trunc(float v) { return __uint_as_float(__float_as_uint(v) & 0xffffe000u); }

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, int accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
      :
      : "r"(d_tmem), "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

// A operand from TMEM (lane = row, column = k; K-step kk at column offset 8*kk).
__device__ __forceinline__ void mma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                            int accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n"
      :
      : "r"(d_tmem), "r"(a_tmem), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
               :
               : "r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" : : "r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t phase);

// Blocking wait with a suspend-time hint: a thread whose phase is not complete is
// parked by the hardware (woken on completion) instead of spinning through issue
// slots its SMSP neighbours need.  KT_TEST_FIRST: probe with test_wait first.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
#if defined(KT_TEST_FIRST) && KT_TEST_FIRST
  if (mbar_test(bar, phase)) return;
#endif
#if defined(KT_WAIT_HINT)
  // hardware-suspended wait: the thread parks until the phase completes (or the hint expires)
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n"
      :
      : "r"(smem_u32(bar)), "r"(phase), "r"(KT_WAIT_HINT)
      : "memory");
#else
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, P1;\n\t}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  // not complete yet: back off between probes so a waiting warp does not take the
  // issue slots its SMSP neighbours on the critical path need
  while (!ok) {
    __nanosleep(KT_WAIT_SLEEP);
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, P1;\n\t}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  }
#endif
}

// Wait for a phase that is typically far off (a warp idle for most of a tile): probe, then
// sleep between probes, so the waiting warp issues a handful of instructions instead of
// spinning through try_wait retries in its SMSP neighbours' issue slots.
template <int SLEEP_NS>
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t phase);

// Non-blocking probe: true once the phase with parity `phase` has completed.
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, P1;\n\t}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}

template <int SLEEP_NS>
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t phase) {
  while (!mbar_test(bar, phase)) __nanosleep(SLEEP_NS);
}

// generic-proxy smem writes -> visible to the tensor core (async proxy)
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
#ifndef KT_DBG_NO_FENCE
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
#else
__device__ __forceinline__ void tc_fence_before() { asm volatile("" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("" ::: "memory"); }
#endif

// Whole warp: allocate ncols (power of 2 >= 32) TMEM columns; base address -> *slot.
__device__ __forceinline__ void tmem_alloc(uint32_t* slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
               :
               : "r"(smem_u32(slot)), "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" : : "r"(taddr), "r"(ncols) : "memory");
}

// Warp-collective: lane l of warp w reads TMEM lane (32*(w%4) + l), 32 consecutive
// 32-bit columns starting at taddr's column (taddr's lane field = 32*(w%4)).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// Warp-collective load of 16 consecutive columns of this thread's TMEM lane.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// Warp-collective store of 32 consecutive columns of this thread's TMEM lane.
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
      :
      : "r"(taddr), "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
        "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
        "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
        "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
        "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
        "r"(__float_as_uint(v[15])), "r"(__float_as_uint(v[16])), "r"(__float_as_uint(v[17])),
        "r"(__float_as_uint(v[18])), "r"(__float_as_uint(v[19])), "r"(__float_as_uint(v[20])),
        "r"(__float_as_uint(v[21])), "r"(__float_as_uint(v[22])), "r"(__float_as_uint(v[23])),
        "r"(__float_as_uint(v[24])), "r"(__float_as_uint(v[25])), "r"(__float_as_uint(v[26])),
        "r"(__float_as_uint(v[27])), "r"(__float_as_uint(v[28])), "r"(__float_as_uint(v[29])),
        "r"(__float_as_uint(v[30])), "r"(__float_as_uint(v[31]))
      : "memory");
}

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
      :
      : "r"(taddr), "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
        "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
        "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7]))
      : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
      :
      : "r"(taddr), "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
        "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
        "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
        "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
        "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
        "r"(__float_as_uint(v[15]))
      : "memory");
}

__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// K-major layout with a padded K-chunk stride (lbo bytes, multiple of 16): used
// for operands written column-wise by many threads, to spread shared-memory banks.
__host__ __device__ __forceinline__ int kmajor_offset_lbo(int row, int k, int K, int lbo) {
  return (row >> 3) * (K >> 2) * lbo + (k >> 2) * lbo + (row & 7) * 16 + (k & 3) * 4;
}

__device__ __forceinline__ uint64_t kdesc_lbo(const void* tile, int K, int kk, int lbo) {
  const uint32_t addr = smem_u32(tile) + 2u * lbo * kk;
  const uint64_t l = static_cast<uint32_t>(lbo) >> 4;
  const uint64_t sbo = (static_cast<uint32_t>(K >> 2) * lbo) >> 4;
  return static_cast<uint64_t>((addr >> 4) & 0x3FFFu) | (l << 16) | (sbo << 32) | (1ull << 46);
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" : : "r"(smem_u32(bar)) : "memory");
}

// One arrive per warp (the barrier counts warps, not threads): 128 per-thread
// arrives on one mbarrier serialise in the shared-memory atomic unit and stall
// the tensor core's shared-memory operand reads behind them.
__device__ __forceinline__ void warp_arrive(uint64_t* bar) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive(bar);
}

// Named barrier over `count` threads (ids 1..15; 0 is __syncthreads).
__device__ __forceinline__ void named_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" : : "r"(id), "r"(count) : "memory");
}

// One lane of a converged warp (elect.sync): the single-thread tcgen05.mma / commit
// issue idiom that keeps the warp's descriptors in uniform registers.
__device__ __forceinline__ bool elect_one() {
  uint32_t p = 0;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(p));
  return p != 0;
}

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

}  // namespace tc
}  // namespace kt
