// Head engine on flat parameter vectors: head_loss_grad (model.py:358-389),
// head_hvp (model.py:392-432), the per-task MAML outer gradient
// (meta.py:167-196, inside meta_step 223-257) and fine_tune_embedded
// (meta.py:274-282).
//
// One CTA owns one flat head vector theta (<= KT_HEAD_MAX floats, in shared
// memory) and streams the rows (embeddings) through in chunks of RC rows, so
// any row count works; gradients accumulate per-thread-owned entries in a
// fixed order (deterministic).  MAML: one CTA per task computes
//   theta' = theta - alpha grad L_s(theta) (inner_steps times),
//   g = grad L_q(theta') [ , v <- v - alpha H_s(theta_k) v  (second order) ]
// and writes g; kt_task_sum adds the per-task rows in a fixed order (fp64),
// after which the outer update theta - beta * sum is one kt_sgd (on one GPU)
// or an NCCL all-reduce of the sum followed by kt_sgd (data parallel).
#include <cooperative_groups.h>
#include <cstdlib>

#include "kt_graph.cuh"

namespace kt {

int check_dims(const kt_dims& d);

namespace meta {

#ifndef KT_META_NT
#define KT_META_NT 256
#endif
constexpr int NT = KT_META_NT;  // threads per CTA (one head vector per CTA)
constexpr int HMAX = 2 * KT_MAX_DIM;  // widest head vector (input 2 d_L)

struct Head {
  int nh;
  int dim[KT_MAX_LAYERS + 2];
  int ow[KT_MAX_LAYERS + 1], ob[KT_MAX_LAYERS + 1];  // offsets into the flat head vector
  int P;
  int HS;  // scratch row stride (widest layer, padded to 4)
  int RC;  // rows per chunk
};

__host__ __device__ inline Head head_of(const kt_dims& d, int rc = 8) {
  Head h;
  h.nh = d.n_head;
  int w = 1;
  for (int i = 0; i <= d.n_head; ++i) {
    h.dim[i] = d.head[i];
    w = d.head[i] > w ? d.head[i] : w;
  }
  for (int i = 0; i < d.n_head; ++i) {
    h.ow[i] = d.off_hw[i] - d.off_head;
    h.ob[i] = d.off_hb[i] - d.off_head;
  }
  h.P = d.n_head_params;
  h.HS = (w + 3) & ~3;
  h.RC = rc;
  return h;
}

// Row-chunk scratch carved arithmetically from one base pointer (no pointer
// arrays -> no local-memory indirection in the hot loops):
//   A(0..nh) activations, Z(0..nh-1) pre-activations, [TA(0..nh) tangents,]
//   D(0..1) deltas [, D(2..3) tangent deltas] -- each RC x HS -- then NT floats.
struct Scratch {
  float* base;
  int blk, nh, hvp;
  __device__ __forceinline__ float* A(int i) const { return base + i * blk; }
  __device__ __forceinline__ float* Z(int i) const { return base + (nh + 1 + i) * blk; }
  __device__ __forceinline__ float* TA(int i) const { return base + (2 * nh + 1 + i) * blk; }
  __device__ __forceinline__ float* D(int j) const { return base + ((hvp ? 3 * nh + 2 : 2 * nh + 1) + j) * blk; }
  __device__ __forceinline__ float* red() const { return base + ((hvp ? 3 * nh + 2 : 2 * nh + 1) + (hvp ? 4 : 2)) * blk; }
  // reduction-split partial sums, slice s (KS_MAX slices of a row chunk)
  __device__ __forceinline__ float* part(int s) const { return red() + NT + s * blk; }
};

constexpr int KS_MAX = 4;  // reduction slices of the split forward / propagate (warp-level split)
__host__ __device__ inline int scratch_floats(const Head& h, bool hvp) {
  return ((h.nh + 1) + h.nh + (hvp ? h.nh + 1 : 0) + (hvp ? 4 : 2) + KS_MAX) * h.RC * h.HS + NT;
}

__device__ __forceinline__ Scratch carve(float* p, const Head& h, bool hvp) {
  return Scratch{p, h.RC * h.HS, h.nh, hvp ? 1 : 0};
}

// Deterministic CTA sum: a fixed butterfly inside each warp, then warp 0 combines the warp
// sums with the same butterfly (a fixed tree, so the result does not depend on timing).
__device__ __forceinline__ float block_sum(float v, float* red) {
  static_assert(NT % 32 == 0 && NT / 32 <= 32, "block_sum: whole warps, at most 32");
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
  if (lane == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    float s = lane < NT / 32 ? red[lane] : 0.0f;
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) s += __shfl_xor_sync(0xffffffffu, s, m);
    if (lane == 0) red[NT / 32] = s;
  }
  __syncthreads();
  const float s = red[NT / 32];
  __syncthreads();
  return s;
}

// grad (and mse) of the head MSE at theta over n rows; if v != nullptr computes
// the Hessian-vector product H(theta) v instead (forward-over-reverse, ReLU masks
// constant).  Rows are u[ridx[r]] (or u[r]) and labels y[ridx[r]] (or y[r]).
// out (h.P floats, smem) is overwritten.  Returns the mse.
__device__ float head_pass_scalar(const Head& h, const float* th, const float* v, const float* u,
                                  const int64_t* ridx, const float* y, int n, float* out, const Scratch& S,
                                  int n_norm) {
  const int nh = h.nh, HS = h.HS, RC = h.RC;
  const bool hvp = v != nullptr;
  for (int e = threadIdx.x; e < h.P; e += NT) out[e] = 0.0f;
  float sq_local = 0.0f;
  const float two_n = 2.0f / static_cast<float>(n_norm);
  for (int r0 = 0; r0 < n; r0 += RC) {
    const int nr = n - r0 < RC ? n - r0 : RC;
    __syncthreads();
    {
      const int d0 = h.dim[0];
      float* A0 = S.A(0);
      float* T0 = hvp ? S.TA(0) : nullptr;
      for (int e = threadIdx.x; e < nr * d0; e += NT) {
        const int r = e / d0, c = e - r * d0;
        const int64_t row = ridx ? ridx[r0 + r] : r0 + r;
        A0[r * HS + c] = u[row * d0 + c];
        if (hvp) T0[r * HS + c] = 0.0f;
      }
    }
    __syncthreads();
    // forward
    for (int i = 0; i < nh; ++i) {
      const int din = h.dim[i], dout = h.dim[i + 1];
      const float* __restrict__ W = th + h.ow[i];
      const float* __restrict__ b = th + h.ob[i];
      const float* __restrict__ Ai = S.A(i);
      float* __restrict__ Zi = S.Z(i);
      float* __restrict__ An = S.A(i + 1);
      const bool last = i == nh - 1;
      if (!hvp) {
        for (int e = threadIdx.x; e < nr * dout; e += NT) {
          const int r = e / dout, c = e - r * dout;
          const float* a = Ai + r * HS;
          float acc = b[c];
          for (int k = 0; k < din; ++k) acc = fmaf(a[k], W[k * dout + c], acc);
          Zi[r * HS + c] = acc;
          An[r * HS + c] = last ? acc : fmaxf(acc, 0.0f);
        }
      } else {
        const float* __restrict__ vW = v + h.ow[i];
        const float* __restrict__ TAi = S.TA(i);
        float* __restrict__ TAn = S.TA(i + 1);
        for (int e = threadIdx.x; e < nr * dout; e += NT) {
          const int r = e / dout, c = e - r * dout;
          const float* a = Ai + r * HS;
          const float* ta = TAi + r * HS;
          float acc = b[c], t = v[h.ob[i] + c];
          for (int k = 0; k < din; ++k) {
            const float w = W[k * dout + c];
            acc = fmaf(a[k], w, acc);
            t = fmaf(ta[k], w, fmaf(a[k], vW[k * dout + c], t));
          }
          Zi[r * HS + c] = acc;
          An[r * HS + c] = last ? acc : fmaxf(acc, 0.0f);
          TAn[r * HS + c] = (last || acc > 0.0f) ? t : 0.0f;
        }
      }
      __syncthreads();
    }
    // output deltas (model.py:382-383 / 422-423)
    {
      const float* An = S.A(nh);
      float* D0 = S.D(0);
      for (int r = threadIdx.x; r < nr; r += NT) {
        const int64_t row = ridx ? ridx[r0 + r] : r0 + r;
        const float resid = An[r * HS] - y[row];
        sq_local += resid * resid;
        D0[r * HS] = two_n * resid;
        if (hvp) S.D(2)[r * HS] = two_n * S.TA(nh)[r * HS];
      }
    }
    __syncthreads();
    // backward
    int cur = 0;
    for (int i = nh - 1; i >= 0; --i) {
      const int din = h.dim[i], dout = h.dim[i + 1];
      const bool last = i == nh - 1;
      float* __restrict__ da = S.D(cur);
      float* __restrict__ dn = S.D(cur ^ 1);
      float* __restrict__ tda = hvp ? S.D(2 + cur) : nullptr;
      float* __restrict__ tdn = hvp ? S.D(2 + (cur ^ 1)) : nullptr;
      const float* __restrict__ Zi = S.Z(i);
      const float* __restrict__ Ai = S.A(i);
      const float* __restrict__ TAi = hvp ? S.TA(i) : nullptr;
      if (!last) {  // dz = da * (z > 0)
        for (int e = threadIdx.x; e < nr * dout; e += NT) {
          const int r = e / dout, c = e - r * dout;
          if (!(Zi[r * HS + c] > 0.0f)) {
            da[r * HS + c] = 0.0f;
            if (hvp) tda[r * HS + c] = 0.0f;
          }
        }
        __syncthreads();
      }
      // out_w += A^T dz (grad) | TA^T dz + A^T tdz (hvp); out_b += sum dz | sum tdz
      float* gw = out + h.ow[i];
      for (int e = threadIdx.x; e < din * dout; e += NT) {
        const int k = e / dout, c = e - k * dout;
        float acc = gw[e];
        if (hvp) {
          for (int r = 0; r < nr; ++r)
            acc = fmaf(TAi[r * HS + k], da[r * HS + c], fmaf(Ai[r * HS + k], tda[r * HS + c], acc));
        } else {
          for (int r = 0; r < nr; ++r) acc = fmaf(Ai[r * HS + k], da[r * HS + c], acc);
        }
        gw[e] = acc;
      }
      for (int c = threadIdx.x; c < dout; c += NT) {
        float acc = out[h.ob[i] + c];
        const float* src = hvp ? tda : da;
        for (int r = 0; r < nr; ++r) acc += src[r * HS + c];
        out[h.ob[i] + c] = acc;
      }
      // propagate: da' = dz W^T ; tda' = tdz W^T + dz vW^T
      if (i > 0) {
        const float* __restrict__ W = th + h.ow[i];
        const float* __restrict__ vW = hvp ? v + h.ow[i] : nullptr;
        for (int e = threadIdx.x; e < nr * din; e += NT) {
          const int r = e / din, k = e - r * din;
          const float* dr = da + r * HS;
          const float* wk = W + k * dout;
          float acc = 0.0f, tacc = 0.0f;
          if (hvp) {
            const float* tdr = tda + r * HS;
            const float* vk = vW + k * dout;
            for (int c = 0; c < dout; ++c) {
              acc = fmaf(dr[c], wk[c], acc);
              tacc = fmaf(tdr[c], wk[c], fmaf(dr[c], vk[c], tacc));
            }
            tdn[r * HS + k] = tacc;
          } else {
            for (int c = 0; c < dout; ++c) acc = fmaf(dr[c], wk[c], acc);
          }
          dn[r * HS + k] = acc;
        }
      }
      __syncthreads();
      cur ^= 1;
    }
  }
  const float sq = block_sum(sq_local, S.red());
  return sq / static_cast<float>(n_norm);
}


#ifdef KT_META_TRACE
__device__ long long g_mt[512];
__device__ int g_mt_n;
#define MT()                                                                   \
  do {                                                                         \
    if (blockIdx.x == 0 && threadIdx.x == 0 && g_mt_n < 255) {                 \
      g_mt[2 * g_mt_n] = __LINE__;                                             \
      g_mt[2 * g_mt_n + 1] = clock64();                                        \
      ++g_mt_n;                                                                \
    }                                                                          \
  } while (0)
extern "C" int kt_meta_trace_read(void* host) {
  return static_cast<int>(cudaMemcpyFromSymbol(host, g_mt, sizeof(g_mt)));
}
#else
#define MT() \
  do {       \
  } while (0)
#endif

__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ uint32_t sa32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init1(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa32(bar)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// global -> shared bulk copy (bytes % 16 == 0, 16-byte aligned), completion on bar
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa32(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   sa32(dst)),
               "l"(src), "r"(bytes), "r"(sa32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t ph) {
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(sa32(bar)), "r"(ph)
        : "memory");
}
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
#ifndef KT_HEAD_WSPLIT
#define KT_HEAD_WSPLIT 1
#endif
// work items of a 2-row x 4-column tiling of an (nr2 x width) block, rounded up to whole warps
// (each warp then works on one reduction slice)
__device__ __forceinline__ int ncg_items(int width, int nr2) { return (((width >> 2) * (nr2 >> 1)) + 31) & ~31; }
__device__ __forceinline__ float ks_sum(float v, int ks, unsigned gm) {
  for (int o = 1; o < ks; o <<= 1) v += __shfl_xor_sync(gm, v, o);
  return v;
}
// dst[0..n) = src (+ scale * add): 16-byte pieces with every load of a thread in flight
// (n multiple of 4 and 16-byte aligned pointers; the tail in scalars otherwise)
__device__ __forceinline__ void vcopy(float* dst, const float* src, int n, const float* add = nullptr,
                                      float scale = 0.0f) {
  const bool al = ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src) |
                    reinterpret_cast<uintptr_t>(add)) & 15) == 0;
  const int n4 = al ? n >> 2 : 0;
#pragma unroll 4
  for (int e = threadIdx.x; e < n4; e += NT) {
    float4 v = ld4(src + 4 * e);
    if (add) {
      const float4 a = ld4(add + 4 * e);
      v = make_float4(v.x - scale * a.x, v.y - scale * a.y, v.z - scale * a.z, v.w - scale * a.w);
    }
    st4(dst + 4 * e, v);
  }
  for (int e = 4 * n4 + threadIdx.x; e < n; e += NT) dst[e] = add ? src[e] - scale * add[e] : src[e];
}

// Register-tiled pass (all hidden widths and the input width multiples of 4,
// single-output last layer): same arithmetic contract as head_pass_scalar.
//   forward   2 rows x 4 cols per thread, float4 weight loads
//   dW        4 x 4 (k, c) tile per thread, float4 row loads, summed over the chunk rows in order
//   propagate 2 rows x 4 k per thread, float4 loads along c
// Rows r0 .. r0 + nr of u (through ridx) into A(0), padded to a pair with a zero row.
__device__ __forceinline__ void load_rows(const Head& h, const float* u, const int64_t* ridx, int r0, int nr,
                                          const Scratch& S, bool hvp) {
  const int d4 = h.dim[0] >> 2, nr2 = (nr + 1) & ~1, HS = h.HS;
  float* A0 = S.A(0);
  for (int e = threadIdx.x; e < nr2 * d4; e += NT) {
    const int r = e / d4, c = (e - r * d4) * 4;
    float4 val = make_float4(0.f, 0.f, 0.f, 0.f);
    if (r < nr) {
      const int64_t row = ridx ? ridx[r0 + r] : r0 + r;
      val = *reinterpret_cast<const float4*>(u + row * h.dim[0] + c);
    }
    st4(A0 + r * HS + c, val);
    if (hvp) st4(S.TA(0) + r * HS + c, make_float4(0.f, 0.f, 0.f, 0.f));
  }
}

// a0_ready: the caller already loaded the first row chunk (load_rows) and synchronised.
// upd (single row chunk only, n <= RC): out receives upd - ualpha * gradient, the SGD step
// fused into the gradient's only write (upd may be th itself: each element is read once,
// by the thread that writes it, after the pass's last read of th)
__device__ float head_pass_tiled(const Head& h, const float* th, const float* v, const float* u,
                                 const int64_t* ridx, const float* y, int n, float* out, const Scratch& S,
                                 int n_norm, bool a0_ready = false, const float* upd = nullptr,
                                 float ualpha = 0.0f) {
  const int nh = h.nh, HS = h.HS, RC = h.RC;
  const bool hvp = v != nullptr;
  const int tid = threadIdx.x;
  // (no zero pass: the first row chunk writes every gradient element, later chunks add)
  float sq_local = 0.0f;
  const float two_n = 2.0f / static_cast<float>(n_norm);
  for (int r0 = 0; r0 < n; r0 += RC) {
    const int nr = n - r0 < RC ? n - r0 : RC;
    const int nr2 = (nr + 1) & ~1;  // rows padded to pairs (pad row is zero)
    const bool first = r0 == 0;
    __syncthreads();
    if (!(first && a0_ready)) {
      load_rows(h, u, ridx, r0, nr, S, hvp);
      __syncthreads();
    }
    MT();
    // ---- forward
    for (int i = 0; i < nh; ++i) {
      const int din = h.dim[i], dout = h.dim[i + 1];
      const float* __restrict__ W = th + h.ow[i];
      const float* __restrict__ b = th + h.ob[i];
      const float* __restrict__ Ai = S.A(i);
      float* __restrict__ Zi = S.Z(i);
      float* __restrict__ An = S.A(i + 1);
      const bool last = i == nh - 1;
      if (last) {  // dout == 1: eight adjacent lanes per row, k strided by 8, fixed xor tree
        for (int e = tid; e < 8 * nr2; e += NT) {
          const int r = e >> 3, j = e & 7;
          const unsigned gm = 0xFFu << (tid & 24);
          float acc = 0.0f, t = 0.0f;
          for (int k = j; k < din; k += 8) {
            acc = fmaf(Ai[r * HS + k], W[k], acc);
            if (hvp) t = fmaf(S.TA(i)[r * HS + k], W[k], fmaf(Ai[r * HS + k], v[h.ow[i] + k], t));
          }
          acc = ks_sum(acc, 8, gm);
          if (hvp) t = ks_sum(t, 8, gm);
          if (j == 0) {
            acc += b[0];
            Zi[r * HS] = acc;
            An[r * HS] = acc;
            if (hvp) S.TA(i + 1)[r * HS] = t + v[h.ob[i]];
          }
        }
      } else if (!hvp && KT_HEAD_WSPLIT && (ncg_items(dout, nr2) * KS_MAX <= NT) && din % (4 * KS_MAX) == 0) {
        // few rows: the k range is split over KS_MAX thread slices (a warp's lanes share a
        // slice, so their W reads stay row-contiguous), partial sums go to shared memory, and
        // a second phase adds them in slice order, then the bias and the ReLU
        const int ncg = dout >> 2, items = ncg * (nr2 >> 1), ip = ncg_items(dout, nr2), kl = din / KS_MAX;
        for (int it = tid; it < ip * KS_MAX; it += NT) {
          const int sl = it / ip, item = it - sl * ip;
          if (item >= items) continue;
          const int c = (item % ncg) * 4, r = (item / ncg) * 2;
          float4 a0 = make_float4(0.f, 0.f, 0.f, 0.f), a1 = a0;
          const float* x0 = Ai + r * HS;
          const float* x1 = x0 + HS;
#pragma unroll 4
          for (int k = sl * kl; k < (sl + 1) * kl; ++k) {
            const float4 w = ld4(W + k * dout + c);
            const float p = x0[k], q = x1[k];
            a0.x = fmaf(p, w.x, a0.x); a0.y = fmaf(p, w.y, a0.y); a0.z = fmaf(p, w.z, a0.z); a0.w = fmaf(p, w.w, a0.w);
            a1.x = fmaf(q, w.x, a1.x); a1.y = fmaf(q, w.y, a1.y); a1.z = fmaf(q, w.z, a1.z); a1.w = fmaf(q, w.w, a1.w);
          }
          st4(S.part(sl) + r * HS + c, a0);
          st4(S.part(sl) + (r + 1) * HS + c, a1);
        }
        __syncthreads();
        for (int e = tid; e < nr2 * ncg; e += NT) {
          const int r = e / ncg, c = (e - r * ncg) * 4;
          float4 a = ld4(b + c);
#pragma unroll
          for (int sl = 0; sl < KS_MAX; ++sl) {
            const float4 q = ld4(S.part(sl) + r * HS + c);
            a = make_float4(a.x + q.x, a.y + q.y, a.z + q.z, a.w + q.w);
          }
          st4(Zi + r * HS + c, a);
          st4(An + r * HS + c, make_float4(fmaxf(a.x, 0.f), fmaxf(a.y, 0.f), fmaxf(a.z, 0.f), fmaxf(a.w, 0.f)));
        }
      } else {
        const int ncg = dout >> 2;
        const float* __restrict__ vW = hvp ? v + h.ow[i] : nullptr;
        const float* __restrict__ TAi = hvp ? S.TA(i) : nullptr;
        for (int it = tid; it < ncg * (nr2 >> 1); it += NT) {
          const int c = (it % ncg) * 4, r = (it / ncg) * 2;
          const float4 bb = ld4(b + c);
          float4 a0 = bb, a1 = bb;
          float4 t0 = make_float4(0.f, 0.f, 0.f, 0.f), t1 = t0;
          if (hvp) t0 = t1 = ld4(v + h.ob[i] + c);
          const float* x0 = Ai + r * HS;
          const float* x1 = x0 + HS;
#pragma unroll 4
          for (int k = 0; k < din; ++k) {
            const float4 w = ld4(W + k * dout + c);
            const float p = x0[k], q = x1[k];
            a0.x = fmaf(p, w.x, a0.x); a0.y = fmaf(p, w.y, a0.y); a0.z = fmaf(p, w.z, a0.z); a0.w = fmaf(p, w.w, a0.w);
            a1.x = fmaf(q, w.x, a1.x); a1.y = fmaf(q, w.y, a1.y); a1.z = fmaf(q, w.z, a1.z); a1.w = fmaf(q, w.w, a1.w);
            if (hvp) {
              const float4 vw = ld4(vW + k * dout + c);
              const float tp = TAi[r * HS + k], tq = TAi[(r + 1) * HS + k];
              t0.x = fmaf(tp, w.x, fmaf(p, vw.x, t0.x)); t0.y = fmaf(tp, w.y, fmaf(p, vw.y, t0.y));
              t0.z = fmaf(tp, w.z, fmaf(p, vw.z, t0.z)); t0.w = fmaf(tp, w.w, fmaf(p, vw.w, t0.w));
              t1.x = fmaf(tq, w.x, fmaf(q, vw.x, t1.x)); t1.y = fmaf(tq, w.y, fmaf(q, vw.y, t1.y));
              t1.z = fmaf(tq, w.z, fmaf(q, vw.z, t1.z)); t1.w = fmaf(tq, w.w, fmaf(q, vw.w, t1.w));
            }
          }
          st4(Zi + r * HS + c, a0);
          st4(Zi + (r + 1) * HS + c, a1);
          const float4 z0 = make_float4(fmaxf(a0.x, 0.f), fmaxf(a0.y, 0.f), fmaxf(a0.z, 0.f), fmaxf(a0.w, 0.f));
          const float4 z1 = make_float4(fmaxf(a1.x, 0.f), fmaxf(a1.y, 0.f), fmaxf(a1.z, 0.f), fmaxf(a1.w, 0.f));
          st4(An + r * HS + c, z0);
          st4(An + (r + 1) * HS + c, z1);
          if (hvp) {
            float* TAn = S.TA(i + 1);
            st4(TAn + r * HS + c, make_float4(a0.x > 0.f ? t0.x : 0.f, a0.y > 0.f ? t0.y : 0.f,
                                              a0.z > 0.f ? t0.z : 0.f, a0.w > 0.f ? t0.w : 0.f));
            st4(TAn + (r + 1) * HS + c, make_float4(a1.x > 0.f ? t1.x : 0.f, a1.y > 0.f ? t1.y : 0.f,
                                                    a1.z > 0.f ? t1.z : 0.f, a1.w > 0.f ? t1.w : 0.f));
          }
        }
      }
      __syncthreads();
      MT();
    }
    // ---- output deltas; the pad row (if any) gets zero deltas
    {
      const float* An = S.A(nh);
      float* D0 = S.D(0);
      for (int r = tid; r < nr2; r += NT) {
        float d = 0.0f, td = 0.0f;
        if (r < nr) {
          const int64_t row = ridx ? ridx[r0 + r] : r0 + r;
          const float resid = An[r * HS] - y[row];
          sq_local += resid * resid;
          d = two_n * resid;
          if (hvp) td = two_n * S.TA(nh)[r * HS];
        }
        D0[r * HS] = d;
        if (hvp) S.D(2)[r * HS] = td;
      }
    }
    __syncthreads();
    MT();
    // ---- backward
    int cur = 0;
    for (int i = nh - 1; i >= 0; --i) {
      const int din = h.dim[i], dout = h.dim[i + 1];
      const bool last = i == nh - 1;
      float* __restrict__ da = S.D(cur);
      float* __restrict__ dn = S.D(cur ^ 1);
      float* __restrict__ tda = hvp ? S.D(2 + cur) : nullptr;
      float* __restrict__ tdn = hvp ? S.D(2 + (cur ^ 1)) : nullptr;
      const float* __restrict__ Zi = S.Z(i);
      const float* __restrict__ Ai = S.A(i);
      const float* __restrict__ TAi = hvp ? S.TA(i) : nullptr;
      // (layers below the last: da arrives already masked by (z > 0), see the propagate)
      float* gw = out + h.ow[i];
      if (last) {  // dout == 1: gW[k] += sum_r A[r][k] dz[r]
        for (int k = tid; k < din; k += NT) {
          float acc = first ? 0.0f : gw[k];
          for (int r = 0; r < nr; ++r)
            acc = hvp ? fmaf(TAi[r * HS + k], da[r * HS], fmaf(Ai[r * HS + k], tda[r * HS], acc))
                      : fmaf(Ai[r * HS + k], da[r * HS], acc);
          gw[k] = upd ? upd[gw - out + k] - ualpha * acc : acc;
        }
      } else {
        const int ncg = dout >> 2;
        for (int it = tid; it < (din >> 2) * ncg; it += NT) {
          const int c = (it % ncg) * 4, k = (it / ncg) * 4;
          float4 g[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) g[j] = first ? make_float4(0.f, 0.f, 0.f, 0.f) : ld4(gw + (k + j) * dout + c);
          for (int r = 0; r < nr; ++r) {
            const float4 a = ld4(Ai + r * HS + k);
            const float4 d = ld4(da + r * HS + c);
            const float av[4] = {a.x, a.y, a.z, a.w};
            if (!hvp) {
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                g[j].x = fmaf(av[j], d.x, g[j].x); g[j].y = fmaf(av[j], d.y, g[j].y);
                g[j].z = fmaf(av[j], d.z, g[j].z); g[j].w = fmaf(av[j], d.w, g[j].w);
              }
            } else {  // hvp: TA^T dz + A^T tdz
              const float4 ta = ld4(TAi + r * HS + k);
              const float4 td = ld4(tda + r * HS + c);
              const float tv[4] = {ta.x, ta.y, ta.z, ta.w};
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                g[j].x = fmaf(tv[j], d.x, fmaf(av[j], td.x, g[j].x));
                g[j].y = fmaf(tv[j], d.y, fmaf(av[j], td.y, g[j].y));
                g[j].z = fmaf(tv[j], d.z, fmaf(av[j], td.z, g[j].z));
                g[j].w = fmaf(tv[j], d.w, fmaf(av[j], td.w, g[j].w));
              }
            }
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            float4 o = g[j];
            if (upd) {
              const float4 b = ld4(upd + (gw - out) + (k + j) * dout + c);
              o = make_float4(b.x - ualpha * o.x, b.y - ualpha * o.y, b.z - ualpha * o.z, b.w - ualpha * o.w);
            }
            st4(gw + (k + j) * dout + c, o);
          }
        }
      }
      for (int c = tid; c < dout; c += NT) {
        float acc = first ? 0.0f : out[h.ob[i] + c];
        const float* src = hvp ? tda : da;
        for (int r = 0; r < nr; ++r) acc += src[r * HS + c];
        out[h.ob[i] + c] = upd ? upd[h.ob[i] + c] - ualpha * acc : acc;
      }
      const bool wsplit = i > 0 && !last && !hvp && KT_HEAD_WSPLIT &&
                          ncg_items(din, nr2) * KS_MAX <= NT && dout % (4 * KS_MAX) == 0;
      if (wsplit) {  // da' = dz W^T with the column range split over KS_MAX thread slices
        const float* __restrict__ W = th + h.ow[i];
        const int nkg = din >> 2, items = nkg * (nr2 >> 1), ip = ncg_items(din, nr2), cl = dout / KS_MAX;
        for (int it = tid; it < ip * KS_MAX; it += NT) {
          const int sl = it / ip, item = it - sl * ip;
          if (item >= items) continue;
          const int k = (item % nkg) * 4, r = (item / nkg) * 2;
          float a[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
          const int crot = k % cl;  // rotated start inside the slice (bank spread, fixed order)
          for (int cc = 0; cc < cl; cc += 4) {
            const int c = sl * cl + (cc + crot < cl ? cc + crot : cc + crot - cl);
            const float4 d0 = ld4(da + r * HS + c), d1 = ld4(da + (r + 1) * HS + c);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float4 w = ld4(W + (k + j) * dout + c);
              a[0][j] += d0.x * w.x + d0.y * w.y + d0.z * w.z + d0.w * w.w;
              a[1][j] += d1.x * w.x + d1.y * w.y + d1.z * w.z + d1.w * w.w;
            }
          }
          st4(S.part(sl) + r * HS + k, make_float4(a[0][0], a[0][1], a[0][2], a[0][3]));
          st4(S.part(sl) + (r + 1) * HS + k, make_float4(a[1][0], a[1][1], a[1][2], a[1][3]));
        }
        __syncthreads();
        // slice sums in order, then dz of layer i - 1 = da' * (z_{i-1} > 0)
        const float* Zp = S.Z(i - 1);
        for (int e = tid; e < nr2 * nkg; e += NT) {
          const int r = e / nkg, k = (e - r * nkg) * 4;
          float4 a = ld4(S.part(0) + r * HS + k);
#pragma unroll
          for (int sl = 1; sl < KS_MAX; ++sl) {
            const float4 q = ld4(S.part(sl) + r * HS + k);
            a = make_float4(a.x + q.x, a.y + q.y, a.z + q.z, a.w + q.w);
          }
          const float4 z = ld4(Zp + r * HS + k);
          st4(dn + r * HS + k, make_float4(z.x > 0.f ? a.x : 0.f, z.y > 0.f ? a.y : 0.f, z.z > 0.f ? a.z : 0.f,
                                           z.w > 0.f ? a.w : 0.f));
        }
      }
      if (i > 0 && !wsplit) {  // da' = dz W^T ; tda' = tdz W^T + dz vW^T   (2 rows x 4 k per thread)
        const float* __restrict__ W = th + h.ow[i];
        const float* __restrict__ vW = hvp ? v + h.ow[i] : nullptr;
        const int nkg = din >> 2;
        for (int it = tid; it < nkg * (nr2 >> 1); it += NT) {
          const int k = (it % nkg) * 4, r = (it / nkg) * 2;
          float a[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
          float t[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
          if (last) {  // dout == 1
            const float d0 = da[r * HS], d1 = da[(r + 1) * HS];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              a[0][j] = d0 * W[k + j];
              a[1][j] = d1 * W[k + j];
              if (hvp) {
                t[0][j] = fmaf(tda[r * HS], W[k + j], d0 * vW[k + j]);
                t[1][j] = fmaf(tda[(r + 1) * HS], W[k + j], d1 * vW[k + j]);
              }
            }
          } else {
            // rows k..k+3 of W are read at column c: threads on consecutive k quads start at
            // different column quads (rotated, fixed order per output) so their 16-byte reads
            // spread over the banks instead of all hitting column c's
            const int crot = k % dout;
            for (int cc = 0; cc < dout; cc += 4) {
              const int c = cc + crot < dout ? cc + crot : cc + crot - dout;
              const float4 d0 = ld4(da + r * HS + c), d1 = ld4(da + (r + 1) * HS + c);
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const float4 w = ld4(W + (k + j) * dout + c);
                a[0][j] += d0.x * w.x + d0.y * w.y + d0.z * w.z + d0.w * w.w;
                a[1][j] += d1.x * w.x + d1.y * w.y + d1.z * w.z + d1.w * w.w;
                if (hvp) {
                  const float4 vw = ld4(vW + (k + j) * dout + c);
                  const float4 e0 = ld4(tda + r * HS + c), e1 = ld4(tda + (r + 1) * HS + c);
                  t[0][j] += e0.x * w.x + e0.y * w.y + e0.z * w.z + e0.w * w.w + d0.x * vw.x + d0.y * vw.y +
                             d0.z * vw.z + d0.w * vw.w;
                  t[1][j] += e1.x * w.x + e1.y * w.y + e1.z * w.z + e1.w * w.w + d1.x * vw.x + d1.y * vw.y +
                             d1.z * vw.z + d1.w * vw.w;
                }
              }
            }
          }
          // dz of layer i - 1 = da' * (z_{i-1} > 0), applied here (no separate masking phase)
          const float* Zp = S.Z(i - 1);
          const float4 z0 = ld4(Zp + r * HS + k), z1 = ld4(Zp + (r + 1) * HS + k);
          const float m0[4] = {z0.x, z0.y, z0.z, z0.w}, m1[4] = {z1.x, z1.y, z1.z, z1.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if (!(m0[j] > 0.0f)) a[0][j] = t[0][j] = 0.0f;
            if (!(m1[j] > 0.0f)) a[1][j] = t[1][j] = 0.0f;
          }
          st4(dn + r * HS + k, make_float4(a[0][0], a[0][1], a[0][2], a[0][3]));
          st4(dn + (r + 1) * HS + k, make_float4(a[1][0], a[1][1], a[1][2], a[1][3]));
          if (hvp) {
            st4(tdn + r * HS + k, make_float4(t[0][0], t[0][1], t[0][2], t[0][3]));
            st4(tdn + (r + 1) * HS + k, make_float4(t[1][0], t[1][1], t[1][2], t[1][3]));
          }
        }
      }
      __syncthreads();
      MT();
      cur ^= 1;
    }
  }
  const float sq = block_sum(sq_local, S.red());
  return sq / static_cast<float>(n_norm);
}

__device__ __forceinline__ bool tiled_ok(const Head& h) {
  if (h.dim[h.nh] != 1 || (h.dim[0] & 3) || (h.RC & 1)) return false;
  for (int i = 1; i < h.nh; ++i)
    if (h.dim[i] & 3) return false;
  return true;
}

// n rows; the loss is the mean over n_norm rows (n_norm = n unless the rows are one
// share of a larger batch split over a cluster)
__device__ float head_pass(const Head& h, const float* th, const float* v, const float* u, const int64_t* ridx,
                           const float* y, int n, float* out, const Scratch& S, int n_norm = 0,
                           bool a0_ready = false, const float* upd = nullptr, float ualpha = 0.0f) {
  if (n_norm <= 0) n_norm = n;
  return tiled_ok(h) ? head_pass_tiled(h, th, v, u, ridx, y, n, out, S, n_norm, a0_ready, upd, ualpha)
                     : head_pass_scalar(h, th, v, u, ridx, y, n, out, S, n_norm);
}

struct TaskSet {
  const float* u;         // (N_rows, d0) embeddings
  const float* y;         // (N_rows,) normalised labels
  const int64_t* s_off;   // (T+1) support row offsets into s_idx
  const int64_t* s_idx;
  const int64_t* q_off;
  const int64_t* q_idx;
};

__global__ void __launch_bounds__(NT)
maml_task_kernel(kt_dims dims, int rc, const float* __restrict__ theta, TaskSet ts, int T, float alpha,
                 int inner_steps, int first_order, float* __restrict__ theta_ws, float* __restrict__ g_out,
                 float* __restrict__ loss_out) {
  extern __shared__ __align__(16) float sm[];
  pdl_launch_dependents();  // task_sum may launch now and wait for this grid
  pdl_wait();               // theta: the previous step's update
  MT();
  const Head h = head_of(dims, rc);
  const int P4 = (h.P + 3) & ~3;
  float* th = sm;             // current theta_k
  float* th1 = th + P4;       // next theta / theta_0 for HVP
  float* gb = th1 + P4;       // support gradient / HVP output
  float* vb = gb + P4;        // query gradient v
  const Scratch S = carve(vb + P4, h, !first_order);
  const int t = blockIdx.x;
  if (t >= T) return;
  const int64_t s0 = ts.s_off[t], ns = ts.s_off[t + 1] - s0;
  const int64_t q0 = ts.q_off[t], nq = ts.q_off[t + 1] - q0;
  // theta: one bulk copy (TMA engine) while the threads stage the support set's first rows
  __shared__ __align__(8) uint64_t tbar;
  const bool bulk = (reinterpret_cast<uintptr_t>(theta) & 15) == 0;
  const uint32_t tb = static_cast<uint32_t>(h.P * 4) & ~15u;
  if (threadIdx.x == 0 && bulk) {
    mbar_init1(&tbar);
    bulk_g2s(th, theta, tb, &tbar);
  }
  if (bulk) {
    for (int e = static_cast<int>(tb >> 2) + threadIdx.x; e < h.P; e += NT) th[e] = theta[e];
  } else {
    vcopy(th, theta, h.P);
  }
  const bool pre = tiled_ok(h);
  if (pre) load_rows(h, ts.u, ts.s_idx + s0, 0, static_cast<int>(ns < h.RC ? ns : h.RC), S, false);
  __syncthreads();
  if (bulk) mbar_wait_parity(&tbar, 0);
  MT();
  float ls0 = 0.0f;
  float* cur = th;
  float* nxt = th1;
  for (int k = 0; k < inner_steps; ++k) {
    if (!first_order && inner_steps > 1)
      for (int e = threadIdx.x; e < h.P; e += NT) theta_ws[(static_cast<int64_t>(t) * inner_steps + k) * h.P + e] = cur[e];
    // one row chunk: the pass writes nxt = cur - alpha * grad directly
    const bool fused = pre && ns <= h.RC;
    const float ls = head_pass(h, cur, nullptr, ts.u, ts.s_idx + s0, ts.y, static_cast<int>(ns), fused ? nxt : gb,
                               S, 0, pre && k == 0, fused ? cur : nullptr, alpha);
    if (k == 0) ls0 = ls;
    __syncthreads();
    MT();
    if (!fused) {
      vcopy(nxt, cur, h.P, gb, alpha);
      __syncthreads();
      MT();
    }
    float* tmp = cur; cur = nxt; nxt = tmp;
  }
  const float lq = head_pass(h, cur, nullptr, ts.u, ts.q_idx + q0, ts.y, static_cast<int>(nq), vb, S);
  __syncthreads();
  MT();
  if (!first_order) {
    for (int k = inner_steps - 1; k >= 0; --k) {
      // theta_k -> nxt
      for (int e = threadIdx.x; e < h.P; e += NT)
        nxt[e] = inner_steps > 1 ? theta_ws[(static_cast<int64_t>(t) * inner_steps + k) * h.P + e] : theta[e];
      __syncthreads();
      MT();
      head_pass(h, nxt, vb, ts.u, ts.s_idx + s0, ts.y, static_cast<int>(ns), gb, S);
      __syncthreads();
      MT();
      vcopy(vb, vb, h.P, gb, alpha);
      __syncthreads();
      MT();
    }
  }
  vcopy(g_out + static_cast<int64_t>(t) * h.P, vb, h.P);
  MT();
  if (threadIdx.x == 0) {
    loss_out[2 * t] = ls0;
    loss_out[2 * t + 1] = lq;
  }
}

// sum_out[p] = sum_t g[t][p] (fixed order, fp64 accumulate); stats = (sum ls, sum lq)
__global__ void task_sum_kernel(const float* __restrict__ g, int T, int P, float* __restrict__ sum_out,
                                const float* __restrict__ losses, double* __restrict__ stats, float beta = 0.0f,
                                float* __restrict__ theta = nullptr) {
  pdl_launch_dependents();
  pdl_wait();  // g / losses: the task kernel (PDL launch in kt_maml_step)
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < P) {
    double s = 0.0;
    for (int t = 0; t < T; ++t) s += static_cast<double>(g[static_cast<int64_t>(t) * P + p]);
    sum_out[p] = static_cast<float>(s);
    if (theta) theta[p] = theta[p] - beta * static_cast<float>(s);  // kt_sgd's arithmetic (kt_maml_step)
  }
  if (stats && blockIdx.x == 0 && threadIdx.x < 2) {
    double s = 0.0;
    for (int t = 0; t < T; ++t) s += static_cast<double>(losses[2 * t + threadIdx.x]);
    stats[threadIdx.x] = s;
  }
}

// head_loss_grad / head_hvp / fine-tune: one CTA on one theta.
__global__ void __launch_bounds__(NT)
head_kernel(kt_dims dims, int rc, const float* __restrict__ theta, const float* __restrict__ v,
            const float* __restrict__ u, const float* __restrict__ y, int n, int steps, float alpha,
            float* __restrict__ out, float* __restrict__ mse_out) {
  extern __shared__ __align__(16) float sm[];
  const Head h = head_of(dims, rc);
  const int P4 = (h.P + 3) & ~3;
  float* th = sm;
  float* gb = th + P4;
  float* vb = gb + P4;
  const bool hvp = v != nullptr;
  const Scratch S = carve(vb + P4, h, hvp);
  for (int e = threadIdx.x; e < h.P; e += NT) {
    th[e] = theta[e];
    if (hvp) vb[e] = v[e];
  }
  __syncthreads();
  MT();
  if (steps <= 0) {  // single evaluation: grad (or hvp) -> out
    const float mse = head_pass(h, th, hvp ? vb : nullptr, u, nullptr, y, n, gb, S);
    __syncthreads();
    MT();
    for (int e = threadIdx.x; e < h.P; e += NT) out[e] = gb[e];
    if (threadIdx.x == 0 && mse_out) mse_out[0] = mse;
    return;
  }
  for (int s = 0; s < steps; ++s) {  // fine_tune_embedded: theta -= alpha * grad, `steps` times
    const float mse = head_pass(h, th, nullptr, u, nullptr, y, n, gb, S);
    __syncthreads();
    MT();
    vcopy(th, th, h.P, gb, alpha);
    if (threadIdx.x == 0 && mse_out) mse_out[s] = mse;
    __syncthreads();
  }
  for (int e = threadIdx.x; e < h.P; e += NT) out[e] = th[e];
}

// fine_tune_embedded over a thread-block cluster: CTA c of C owns rows [c n / C, (c+1) n / C)
// and parameter slice [c P / C, (c+1) P / C).  Per step every CTA computes its rows'
// gradient share (scaled by the full batch: the mean is over n), then reduces its
// parameter slice over the C shares read from the peers' shared memory (distributed
// shared memory, fixed CTA order), updates that slice, and finally gathers the other
// slices from their owners -- two cluster barriers per step, no global traffic.
__global__ void __launch_bounds__(NT)
fine_tune_cluster_kernel(kt_dims dims, int rc, const float* __restrict__ theta, const float* __restrict__ u,
                         const float* __restrict__ y, int n, int steps, float alpha, float* __restrict__ out,
                         float* __restrict__ mse_out) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(16) float sm[];
  __shared__ float s_mse;
  const Head h = head_of(dims, rc);
  const int P4 = (h.P + 3) & ~3;
  float* th = sm;
  float* gb = th + P4;
  const Scratch S = carve(gb + 2 * P4, h, false);
  const int C = static_cast<int>(cl.num_blocks()), c = static_cast<int>(cl.block_rank());
  const int r0 = static_cast<int>(static_cast<int64_t>(n) * c / C), r1 = static_cast<int>(static_cast<int64_t>(n) * (c + 1) / C);
  // parameter slices in whole float4 groups, so the distributed-shared-memory reduce and gather
  // move 16 bytes per remote access with all of a thread's loads in flight together
  const int G4 = P4 >> 2;
  const int q0 = static_cast<int>(static_cast<int64_t>(G4) * c / C), q1 = static_cast<int>(static_cast<int64_t>(G4) * (c + 1) / C);
  const int p0 = 4 * q0, p1 = 4 * q1 < h.P ? 4 * q1 : h.P;
  const int d0 = h.dim[0];
  for (int e = threadIdx.x; e < h.P; e += NT) th[e] = theta[e];
  // this CTA's rows never change across the steps: staged once when they fit one row chunk
  const bool rows_once = tiled_ok(h) && r1 > r0 && r1 - r0 <= h.RC;
  if (rows_once) load_rows(h, u + static_cast<int64_t>(r0) * d0, nullptr, 0, r1 - r0, S, false);
  __syncthreads();
  for (int st = 0; st < steps; ++st) {
    float part = 0.0f;
    if (r1 > r0) {
      part = head_pass(h, th, nullptr, u + static_cast<int64_t>(r0) * d0, nullptr, y + r0, r1 - r0, gb, S, n, rows_once);
    } else {
      for (int e = threadIdx.x; e < h.P; e += NT) gb[e] = 0.0f;
    }
    if (threadIdx.x == 0) s_mse = part;
    MT();
    cl.sync();  // every CTA's gradient share is complete
    MT();
    if (C == 8) {  // (the launch's cluster size for >= 64 rows: the peer loads unrolled)
      for (int e4 = q0 + static_cast<int>(threadIdx.x); e4 < q1; e4 += NT) {
        float4 v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = reinterpret_cast<const float4*>(cl.map_shared_rank(gb, q))[e4];
        float4 g = v[0];
#pragma unroll
        for (int q = 1; q < 8; ++q) {
          g.x += v[q].x;
          g.y += v[q].y;
          g.z += v[q].z;
          g.w += v[q].w;
        }
        float4* t = reinterpret_cast<float4*>(th) + e4;
        float4 tv = *t;
        tv.x -= alpha * g.x;
        tv.y -= alpha * g.y;
        tv.z -= alpha * g.z;
        tv.w -= alpha * g.w;
        *t = tv;
        // pushed into every peer's copy too (their slice c is read only after the next cluster
        // barrier and written only here), so no gather pass follows
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (q != c) reinterpret_cast<float4*>(cl.map_shared_rank(th, q))[e4] = tv;
      }
    } else {
      for (int e = p0 + static_cast<int>(threadIdx.x); e < p1; e += NT) {
        float g = 0.0f;
        for (int q = 0; q < C; ++q) g += cl.map_shared_rank(gb, q)[e];
        th[e] -= alpha * g;
      }
    }
    if (c == 0 && threadIdx.x == 0 && mse_out) {
      float m = 0.0f;
      for (int q = 0; q < C; ++q) m += *cl.map_shared_rank(&s_mse, q);
      mse_out[st] = m;
    }
    MT();
    cl.sync();  // every slice updated
    MT();
    if (C != 8) {  // (C == 8: the peers pushed their slices during the reduce)
      for (int q = 0; q < C; ++q) {  // the other slices, float4 groups
        if (q == c) continue;
        const int a0 = static_cast<int>(static_cast<int64_t>(G4) * q / C);
        const int a1 = static_cast<int>(static_cast<int64_t>(G4) * (q + 1) / C);
        const float4* src = reinterpret_cast<const float4*>(cl.map_shared_rank(th, q));
        float4* dst = reinterpret_cast<float4*>(th);
        for (int e4 = a0 + static_cast<int>(threadIdx.x); e4 < a1; e4 += NT) dst[e4] = src[e4];
      }
    }
    __syncthreads();
  }
  cl.sync();  // peers may still read this CTA's slice of theta
  for (int e = p0 + static_cast<int>(threadIdx.x); e < p1; e += NT) out[e] = th[e];
}

static size_t task_smem(const Head& h, bool so) { return sizeof(float) * (4 * ((h.P + 3) & ~3) + scratch_floats(h, so)); }
static size_t head_smem(const Head& h, bool hvp) { return sizeof(float) * (3 * ((h.P + 3) & ~3) + scratch_floats(h, hvp)); }

// Largest row chunk (<= cap) whose shared-memory footprint fits.
static Head fit_rows(const kt_dims& d, int cap, bool task, bool hvp) {
  for (int rc = cap; rc >= 1; rc >>= 1) {
    const Head h = head_of(d, rc);
    if ((task ? task_smem(h, hvp) : head_smem(h, hvp)) <= 220 * 1024) return h;
  }
  return head_of(d, 1);
}

static int check_head(const kt_dims& d) {
  KT_REQUIRE(d.n_head >= 1 && d.n_head <= KT_MAX_LAYERS + 1, KT_E_UNSUPPORTED, "head depth beyond limits");
  for (int i = 0; i <= d.n_head; ++i)
    KT_REQUIRE(d.head[i] >= 1 && d.head[i] <= HMAX, KT_E_UNSUPPORTED, "head width %d beyond %d", d.head[i], HMAX);
  KT_REQUIRE(d.head[d.n_head] == 1, KT_E_SHAPE, "head must end in one output");
  return KT_OK;
}

template <class K>
static int set_smem(K kernel, size_t smem, SmemAttr& cached) {
  KT_REQUIRE(smem <= 227 * 1024, KT_E_UNSUPPORTED, "head too large for shared memory (%zu bytes)", smem);
  cached.ensure(kernel, smem);
  return KT_OK;
}

}  // namespace meta
}  // namespace kt

extern "C" {

int kt_head_loss_grad(const kt_dims* dims, const float* theta, const float* u, const float* y, int64_t n,
                      float* grad_out, float* mse_out, void* stream) {
  using namespace kt;
  KT_REQUIRE(dims && theta && u && y && grad_out, KT_E_ARG, "kt_head_loss_grad: null pointer");
  KT_REQUIRE(n > 0, KT_E_EMPTY, "kt_head_loss_grad: empty batch");
  int rc = meta::check_head(*dims);
  if (rc) return rc;
  const meta::Head h = meta::fit_rows(*dims, 32, false, false);
  static SmemAttr cached;
  const size_t smem = meta::head_smem(h, false);
  rc = meta::set_smem(meta::head_kernel, smem, cached);
  if (rc) return rc;
  meta::head_kernel<<<1, meta::NT, smem, as_stream(stream)>>>(*dims, h.RC, theta, nullptr, u, y, (int)n, 0, 0.f,
                                                               grad_out, mse_out);
  note_launches(1);
  return check_launch("kt_head_loss_grad");
}

int kt_head_hvp(const kt_dims* dims, const float* theta, const float* u, const float* y, const float* v, int64_t n,
                float* hvp_out, void* stream) {
  using namespace kt;
  KT_REQUIRE(dims && theta && u && y && v && hvp_out, KT_E_ARG, "kt_head_hvp: null pointer");
  KT_REQUIRE(n > 0, KT_E_EMPTY, "kt_head_hvp: empty batch");
  int rc = meta::check_head(*dims);
  if (rc) return rc;
  const meta::Head h = meta::fit_rows(*dims, 32, false, true);
  static SmemAttr cached;
  const size_t smem = meta::head_smem(h, true);
  rc = meta::set_smem(meta::head_kernel, smem, cached);
  if (rc) return rc;
  meta::head_kernel<<<1, meta::NT, smem, as_stream(stream)>>>(*dims, h.RC, theta, v, u, y, (int)n, 0, 0.f, hvp_out,
                                                               nullptr);
  note_launches(1);
  return check_launch("kt_head_hvp");
}

int kt_fine_tune(const kt_dims* dims, const float* theta, const float* u, const float* y, int64_t n, float alpha,
                 int32_t steps, float* theta_out, float* mse_out, void* stream) {
  using namespace kt;
  KT_REQUIRE(dims && theta && u && y && theta_out, KT_E_ARG, "kt_fine_tune: null pointer");
  KT_REQUIRE(n > 0 && steps > 0, KT_E_EMPTY, "kt_fine_tune: nothing to do");
  int rc = meta::check_head(*dims);
  if (rc) return rc;
  const meta::Head h = meta::fit_rows(*dims, 32, false, false);
  const size_t smem = meta::head_smem(h, false);
  const char* one = getenv("KT_FT_ONE_CTA");
  int C = n >= 16 && !(one && one[0] == '1') ? (n >= 64 ? 8 : 4) : 1;
  const char* cs = getenv("KT_FT_CLUSTER");  // experiment hook: cluster size
  if (cs && atoi(cs) >= 1 && atoi(cs) <= 16) C = atoi(cs);
  if (C > 1) {  // rows and parameters split over a cluster (distributed shared memory)
    static SmemAttr ccached;
    rc = meta::set_smem(meta::fine_tune_cluster_kernel, smem, ccached);
    if (rc) return rc;
    if (C > 8) cudaFuncSetAttribute(meta::fine_tune_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(meta::NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = as_stream(stream);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, meta::fine_tune_cluster_kernel, *dims, h.RC, theta, u, y, (int)n,
                                             (int)steps, alpha, theta_out, mse_out);
    KT_REQUIRE(e == cudaSuccess, KT_E_CUDA, "kt_fine_tune: cluster launch failed (%s)", cudaGetErrorString(e));
  } else {
    static SmemAttr cached;
    rc = meta::set_smem(meta::head_kernel, smem, cached);
    if (rc) return rc;
    meta::head_kernel<<<1, meta::NT, smem, as_stream(stream)>>>(*dims, h.RC, theta, nullptr, u, y, (int)n, steps,
                                                                 alpha, theta_out, mse_out);
  }
  note_launches(1);
  return check_launch("kt_fine_tune");
}

int64_t kt_maml_workspace_bytes(const kt_dims* dims, int32_t T, int32_t inner_steps, int32_t first_order) {
  const int64_t P = dims->n_head_params;
  int64_t b = (int64_t)T * P * 4 + (int64_t)T * 2 * 4 + 64;
  if (!first_order && inner_steps > 1) b += (int64_t)T * inner_steps * P * 4;
  return b;
}

int kt_maml_tasks(const kt_dims* dims, const float* theta, const float* u, const float* y, const int64_t* s_off,
                  const int64_t* s_idx, const int64_t* q_off, const int64_t* q_idx, int32_t T, float alpha,
                  int32_t inner_steps, int32_t first_order, float* g_sum, double* stats, void* workspace,
                  int64_t workspace_bytes, void* stream) {
  using namespace kt;
  KT_REQUIRE(dims && theta && u && y && s_off && s_idx && q_off && q_idx && g_sum && workspace, KT_E_ARG,
             "kt_maml_tasks: null pointer");
  KT_REQUIRE(T > 0, KT_E_EMPTY, "kt_maml_tasks: empty task batch");
  KT_REQUIRE(inner_steps >= 1, KT_E_ARG, "kt_maml_tasks: inner_steps must be >= 1");
  KT_REQUIRE(workspace_bytes >= kt_maml_workspace_bytes(dims, T, inner_steps, first_order), KT_E_ARG,
             "kt_maml_tasks: workspace too small");
  int rc = meta::check_head(*dims);
  if (rc) return rc;
  const bool so = !first_order;
  const meta::Head h = meta::fit_rows(*dims, 8, true, so);
  static SmemAttr cached;
  const size_t smem = meta::task_smem(h, so);
  rc = meta::set_smem(meta::maml_task_kernel, smem, cached);
  if (rc) return rc;
  float* g = static_cast<float*>(workspace);
  float* losses = g + (int64_t)T * h.P;
  float* thws = losses + 2 * T;
  meta::TaskSet ts{u, y, s_off, s_idx, q_off, q_idx};
  cudaStream_t st = as_stream(stream);
  meta::maml_task_kernel<<<T, meta::NT, smem, st>>>(*dims, h.RC, theta, ts, T, alpha, inner_steps, first_order,
                                                    thws, g, losses);
  meta::task_sum_kernel<<<(h.P + 255) / 256, 256, 0, st>>>(g, T, h.P, g_sum, losses, stats);
  note_launches(2);
  return check_launch("kt_maml_tasks");
}

// Data-parallel meta_step in two halves whose composition is bit-identical to kt_maml_step
// on one GPU: every rank writes the per-task gradient rows of its contiguous task share,
// the rows are all-gathered in task order, and every rank sums all of them in task order.
int kt_maml_task_grads(const kt_dims* dims, const float* theta, const float* u, const float* y,
                       const int64_t* s_off, const int64_t* s_idx, const int64_t* q_off, const int64_t* q_idx,
                       int32_t T, float alpha, int32_t inner_steps, int32_t first_order, float* g_rows,
                       float* losses, void* workspace, int64_t workspace_bytes, void* stream) {
  using namespace kt;
  KT_REQUIRE(dims && theta && u && y && s_off && s_idx && q_off && q_idx && g_rows && losses && workspace, KT_E_ARG,
             "kt_maml_task_grads: null pointer");
  KT_REQUIRE(T > 0, KT_E_EMPTY, "kt_maml_task_grads: empty task batch");
  KT_REQUIRE(inner_steps >= 1, KT_E_ARG, "kt_maml_task_grads: inner_steps must be >= 1");
  KT_REQUIRE(workspace_bytes >= kt_maml_workspace_bytes(dims, T, inner_steps, first_order), KT_E_ARG,
             "kt_maml_task_grads: workspace too small");
  int rc = meta::check_head(*dims);
  if (rc) return rc;
  const bool so = !first_order;
  const meta::Head h = meta::fit_rows(*dims, 8, true, so);
  static SmemAttr cached;
  const size_t smem = meta::task_smem(h, so);
  rc = meta::set_smem(meta::maml_task_kernel, smem, cached);
  if (rc) return rc;
  meta::TaskSet ts{u, y, s_off, s_idx, q_off, q_idx};
  meta::maml_task_kernel<<<T, meta::NT, smem, as_stream(stream)>>>(*dims, h.RC, theta, ts, T, alpha, inner_steps,
                                                                   first_order, static_cast<float*>(workspace),
                                                                   g_rows, losses);
  note_launches(1);
  return check_launch("kt_maml_task_grads");
}

int kt_task_sum_update(const kt_dims* dims, const float* g_rows, const float* losses, int32_t T, float beta,
                       float* theta, float* g_sum, double* stats, void* stream) {
  using namespace kt;
  KT_REQUIRE(dims && g_rows && losses && g_sum, KT_E_ARG, "kt_task_sum_update: null pointer");
  KT_REQUIRE(T > 0, KT_E_EMPTY, "kt_task_sum_update: empty task batch");
  const int P = dims->n_head_params;
  meta::task_sum_kernel<<<(P + 255) / 256, 256, 0, as_stream(stream)>>>(g_rows, T, P, g_sum, losses, stats, beta,
                                                                       theta);
  note_launches(1);
  return check_launch("kt_task_sum_update");
}

int kt_maml_step(const kt_dims* dims, float* theta, const float* u, const float* y, const int64_t* s_off,
                 const int64_t* s_idx, const int64_t* q_off, const int64_t* q_idx, int32_t T, float alpha,
                 int32_t inner_steps, int32_t first_order, float beta, float* g_sum, double* stats, void* workspace,
                 int64_t workspace_bytes, void* stream) {
  using namespace kt;
  KT_REQUIRE(dims && theta && u && y && s_off && s_idx && q_off && q_idx && g_sum && workspace, KT_E_ARG,
             "kt_maml_step: null pointer");
  KT_REQUIRE(T > 0, KT_E_EMPTY, "kt_maml_step: empty task batch");
  KT_REQUIRE(inner_steps >= 1, KT_E_ARG, "kt_maml_step: inner_steps must be >= 1");
  KT_REQUIRE(workspace_bytes >= kt_maml_workspace_bytes(dims, T, inner_steps, first_order), KT_E_ARG,
             "kt_maml_step: workspace too small");
  int rc = meta::check_head(*dims);
  if (rc) return rc;
  const bool so = !first_order;
  const meta::Head h = meta::fit_rows(*dims, 8, true, so);
  static SmemAttr cached;
  const size_t smem = meta::task_smem(h, so);
  rc = meta::set_smem(meta::maml_task_kernel, smem, cached);
  if (rc) return rc;
  float* g = static_cast<float*>(workspace);
  float* losses = g + (int64_t)T * h.P;
  float* thws = losses + 2 * T;
  meta::TaskSet ts{u, y, s_off, s_idx, q_off, q_idx};
  cudaStream_t st = as_stream(stream);
  // both launched as programmatic dependents (PDL): each kernel's launch overlaps its predecessor
  cudaError_t e = launch_pdl(meta::maml_task_kernel, dim3(T), dim3(meta::NT), smem, st, *dims, h.RC, theta, ts, T,
                             alpha, inner_steps, first_order, thws, g, losses);
  KT_REQUIRE(e == cudaSuccess, KT_E_CUDA, "kt_maml_step: %s", cudaGetErrorString(e));
  // task sum (fixed order, fp64) and the outer update in one pass over the parameters
  e = launch_pdl(meta::task_sum_kernel, dim3((h.P + 255) / 256), dim3(256), 0, st, g, T, h.P, g_sum, losses, stats,
                 beta, theta);
  KT_REQUIRE(e == cudaSuccess, KT_E_CUDA, "kt_maml_step: %s", cudaGetErrorString(e));
  note_launches(2);
  return check_launch("kt_maml_step");
}

}  // extern "C"
