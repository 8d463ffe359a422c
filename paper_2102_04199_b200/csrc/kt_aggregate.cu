// Streaming aggregation kernels: the layer-by-layer form of embed_batch
// (model.py:185-194) for large batches, HBM-bound by design.
//
//   kt_gcn_layer  H_out = ReLU(A_hat . H_in . W) for every graph of a batch
//                 (gcn_forward model.py:127-133; the einsum of embed_batch
//                 model.py:189-191).  Segmented CSR: graphs own contiguous row
//                 ranges; the adjacency of a graph is one of a few patterns
//                 (batch_layout yields one per op type), staged in shared memory.
//                 Layer-1 input may be the raw fp64 features, z-normalised on the
//                 fly (model.py:108-112: masked rows only, others exactly 0).
//   kt_readout    u = [sum_n a * h_n, max_n h_n] per graph (aggregate
//                 model.py:136-141) as warp-shuffle segmented reductions.
//
// Data movement (kt_gcn_layer): a persistent CTA walks tiles of G graphs whose
// rows are one contiguous byte range, so a tile moves in ONE bulk copy each way
// (cp.async.bulk, the 1D TMA: global -> smem completing on an mbarrier, smem ->
// global as a bulk group), double-buffered so the next tile's load overlaps this
// tile's math.  Math per tile: neighbour aggregation A_hat . H_in from the staged
// rows into a transposed buffer (float4 channel quads), then the dense transform
// on the FP32 pipe as 4-row x 8-column FFMA2 register tiles, ReLU, into the
// staged output rows.  Algorithmic bytes per graph: n d_in sizeof(in) + n d_out 4.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdlib>

#include "kt_common.cuh"
#include "kt_tc.cuh"

namespace kt {
namespace agg {

constexpr int NT = 256;
constexpr int MAXPAT = 8;       // adjacency patterns per batch
constexpr int MAXPNNZ = 1024;   // nnz over all patterns
          // input ring stages (bulk loads in flight per CTA)

struct LayerArgs {
  const void* in;
  int in_f64;
  float* out;
  const float* W;
  const double* fmean;
  const double* fstd;
  int d_in, d_out, relu;
  int64_t B;
  int n_uniform;             // > 0: every graph has n_uniform rows (node_ptr NULL)
  const int64_t* node_ptr;   // segmented row ranges (B + 1)
  const int32_t* pat_id;     // per graph (NULL: pattern 0)
  int n_pat;
  const int32_t* pat_n;      // nodes per pattern
  const int32_t* pat_rp;     // concatenated local row_ptr, (n_p + 1) per pattern
  const int32_t* pat_col;    // concatenated local column ids
  const float* pat_val;      // fp32 of the fp64 normalised adjacency
  const uint8_t* pat_mask;   // concatenated per-pattern node masks (fp64 input only)
  int G;                     // graphs per tile
  int R;                     // max rows per tile (buffer capacity)
  int bulk;                  // rows are 16-byte multiples: bulk copies
  int l2pf;                  // pipelined kernels: L2 prefetch distance in tiles past the smem ring (0: off)
};

struct PatSmem {
  int n[MAXPAT], rp_off[MAXPAT], nz_off[MAXPAT], mask_off[MAXPAT];
};

__device__ __forceinline__ uint32_t s32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init1(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(bar)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_par(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n\tW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra W_%=;\n\t}\n" ::"r"(s32(bar)),
      "r"(parity)
      : "memory");
}
// 1D TMA: global -> shared, completion counted on the mbarrier (bytes % 16 == 0)
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   s32(dst)),
               "l"(src), "r"(bytes), "r"(s32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(s32(src)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// L2 prefetch of a byte range / a tensor-map box (no shared memory, no completion to wait on)
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(map), "r"(c0), "r"(c1)
               : "memory");
}
// 2-D TMA through a tensor map (coordinates: column, row)
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          s32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(s32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, int c0, int c1, const void* src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(map), "r"(c0),
               "r"(c1), "r"(s32(src))
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

__device__ __forceinline__ int64_t tile_row0(const LayerArgs& a, int64_t g0) {
  return a.node_ptr ? a.node_ptr[g0] : g0 * a.n_uniform;
}

__device__ __forceinline__ float4 ldg_stream(const float4* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}

constexpr int PF = 8;  // prefetched float4 per lane: 4 KB of the next graph per warp
constexpr int WPC = NT / 32;

// One warp per graph (grid-stride), no block-wide barriers: the warp prefetches
// the next graph's rows into registers (coalesced 16-byte loads, 4 KB in flight
// per warp) while it aggregates and transforms the current one out of its own
// shared-memory slab, and writes the output rows straight to HBM (each store
// instruction covers two adjacent 128-byte row segments).
template <int DIN_T, int DOUT_T>
__global__ void __launch_bounds__(NT, 2) gcn_layer_kernel(LayerArgs a) {
  extern __shared__ __align__(16) unsigned char smem_w[];
  __shared__ PatSmem P;
  __shared__ double s_mean[KT_MAX_DIM], s_rstd[KT_MAX_DIM];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int din = DIN_T ? DIN_T : a.d_in, dout = DOUT_T ? DOUT_T : a.d_out;
  const int dinp = (din + 3) & ~3;  // slab row stride (float4 aligned)
  const int maxn = a.R;             // rows of the largest graph
  // ---- carve: W | pattern CSR | per-warp slabs (X rows, aggregated rows) ----------------------
  float* sW = reinterpret_cast<float*>(smem_w);
  int* s_rp = reinterpret_cast<int*>(sW + ((din * dout + 3) & ~3));
  const int rp_cap = a.n_pat * (KT_MAX_NODES + 1);
  int* s_col = s_rp + ((rp_cap + 3) & ~3);
  float* s_val = reinterpret_cast<float*>(s_col + MAXPNNZ);
  uint8_t* s_mask = reinterpret_cast<uint8_t*>(s_val + MAXPNNZ);
  float* slab0 = reinterpret_cast<float*>(s_mask + ((a.n_pat * KT_MAX_NODES + 15) & ~15));
  const int slab = 2 * maxn * dinp;
  float* X = slab0 + warp * slab;
  float* AG = X + maxn * dinp;

  for (int i = tid; i < din * dout; i += NT) sW[i] = a.W[i];
  if (tid == 0) {
    int rp = 0, nz = 0, mk = 0;
    for (int p = 0; p < a.n_pat; ++p) {
      P.n[p] = a.pat_n[p];
      P.rp_off[p] = rp;
      P.nz_off[p] = nz;
      P.mask_off[p] = mk;
      nz += a.pat_rp[rp + P.n[p]];
      rp += P.n[p] + 1;
      mk += P.n[p];
    }
  }
  if (a.in_f64)
    for (int c = tid; c < din; c += NT) {
      s_mean[c] = a.fmean[c];
      s_rstd[c] = 1.0 / a.fstd[c];
    }
  __syncthreads();
  int tot_rp = 0, tot_nz = 0, tot_mask = 0;
  for (int p = 0; p < a.n_pat; ++p) {
    tot_rp += P.n[p] + 1;
    tot_mask += P.n[p];
    tot_nz += a.pat_rp[P.rp_off[p] + P.n[p]];
  }
  for (int i = tid; i < tot_rp; i += NT) s_rp[i] = a.pat_rp[i];
  for (int i = tid; i < tot_nz; i += NT) {
    s_col[i] = a.pat_col[i];
    s_val[i] = a.pat_val[i];
  }
  const bool masked = a.in_f64 && a.pat_mask;
  if (masked)
    for (int i = tid; i < tot_mask; i += NT) s_mask[i] = a.pat_mask[i];
  __syncthreads();

  const int esz = a.in_f64 ? 8 : 4;
  const bool vec_in = ((din * esz) & 15) == 0;
  // fast transform: 16 lanes x 2 output channels, half-warp h takes rows h, h+2, ...
  constexpr bool kFast = DOUT_T == 32 && DIN_T > 0 && (DIN_T % 4) == 0;
  float2 wreg[kFast ? DIN_T : 1];
  if constexpr (kFast) {
    const int c2 = 2 * (lane & 15);
#pragma unroll
    for (int k = 0; k < DIN_T; ++k) wreg[k] = make_float2(sW[k * 32 + c2], sW[k * 32 + c2 + 1]);
  }

  const int64_t nw = static_cast<int64_t>(gridDim.x) * WPC;
  int64_t g = static_cast<int64_t>(blockIdx.x) * WPC + warp;
  float4 pf[PF];
  int64_t pr0 = 0;
  int pn = 0;
  auto prefetch = [&](int64_t gg) {
    pr0 = tile_row0(a, gg);
    pn = static_cast<int>(tile_row0(a, gg + 1) - pr0);
    if (vec_in) {
      const float4* src = reinterpret_cast<const float4*>(static_cast<const unsigned char*>(a.in) + pr0 * din * esz);
      const int nq = pn * din * esz / 16;
#pragma unroll
      for (int i = 0; i < PF; ++i)
        if (i * 32 + lane < nq) pf[i] = ldg_stream(src + i * 32 + lane);
    }
  };
  if (g < a.B) prefetch(g);
  for (; g < a.B; g += nw) {
    const int64_t r0 = pr0;
    const int n = pn;
    const int p = a.pat_id ? a.pat_id[g] : 0;
    const int moff = P.mask_off[p];
    // ---- 1. current graph -> X slab (fp32; fp64 rows z-normalised, model.py:108-112) ----------
    auto put64 = [&](int e, double v) {
      const int r = e / din, c = e - r * din;
      const bool on = !masked || s_mask[moff + r];
      X[r * dinp + c] = on ? static_cast<float>((v - s_mean[c]) * s_rstd[c]) : 0.0f;
    };
    if (vec_in) {
      const int nq = n * din * esz / 16;
      const float4* src = reinterpret_cast<const float4*>(static_cast<const unsigned char*>(a.in) + r0 * din * esz);
#pragma unroll
      for (int i = 0; i < PF + 1; ++i) {
        // the first PF float4 per lane come from the prefetch registers, any rest from HBM
        for (int q = i * 32 + lane; q < (i < PF ? (i + 1) * 32 : nq) && q < nq; q += 32) {
          const float4 v = i < PF ? pf[i < PF ? i : 0] : ldg_stream(src + q);
          if (a.in_f64) {
            const double2 d = *reinterpret_cast<const double2*>(&v);
            put64(2 * q, d.x);
            put64(2 * q + 1, d.y);
          } else if (din == dinp) {
            *reinterpret_cast<float4*>(X + 4 * q) = v;
          } else {
            const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const int e = 4 * q + t, r = e / din;
              X[r * dinp + (e - r * din)] = vv[t];
            }
          }
        }
      }
    } else {
      for (int e = lane; e < n * din; e += 32) {
        if (a.in_f64) {
          put64(e, reinterpret_cast<const double*>(a.in)[r0 * din + e]);
        } else {
          const int r = e / din;
          X[r * dinp + (e - r * din)] = reinterpret_cast<const float*>(a.in)[r0 * din + e];
        }
      }
    }
    // ---- 2. start the next graph's loads (registers) before this graph's math ------------------
    if (g + nw < a.B) prefetch(g + nw);
    __syncwarp();
    // ---- 3. aggregation AG = A_hat X (float4 channel quads) ------------------------------------
    {
      const int* rp = s_rp + P.rp_off[p];
      const int nz0 = P.nz_off[p];
      const int nq = dinp >> 2;
      for (int item = lane; item < n * nq; item += 32) {
        const int r = item / nq, c0 = 4 * (item - r * nq);
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int j = rp[r]; j < rp[r + 1]; ++j) {
          const float v = s_val[nz0 + j];
          const float4 x = *reinterpret_cast<const float4*>(X + s_col[nz0 + j] * dinp + c0);
          acc.x = fmaf(v, x.x, acc.x);
          acc.y = fmaf(v, x.y, acc.y);
          acc.z = fmaf(v, x.z, acc.z);
          acc.w = fmaf(v, x.w, acc.w);
        }
        *reinterpret_cast<float4*>(AG + r * dinp + c0) = acc;
      }
    }
    __syncwarp();
    // ---- 4. transform + ReLU, rows straight to HBM --------------------------------------------
    float* out = a.out + r0 * dout;
    if constexpr (kFast) {
      // four rows per pass (r, r+2, r+4, r+6): independent FFMA2 chains for ILP
      const int c2 = 2 * (lane & 15), h = lane >> 4;
      for (int rb = h; rb < n; rb += 8) {
        float2 acc[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[i] = make_float2(0.f, 0.f);
#pragma unroll
        for (int k4 = 0; k4 < DIN_T / 4; ++k4) {
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int r = rb + 2 * i < n ? rb + 2 * i : rb;  // clamp: recompute a valid row, store skipped
            const float4 v = reinterpret_cast<const float4*>(AG + r * dinp)[k4];
            acc[i] = ffma2s(v.x, wreg[4 * k4 + 0], acc[i]);
            acc[i] = ffma2s(v.y, wreg[4 * k4 + 1], acc[i]);
            acc[i] = ffma2s(v.z, wreg[4 * k4 + 2], acc[i]);
            acc[i] = ffma2s(v.w, wreg[4 * k4 + 3], acc[i]);
          }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int r = rb + 2 * i;
          if (r < n) {
            float2 o = acc[i];
            if (a.relu) o = make_float2(fmaxf(o.x, 0.f), fmaxf(o.y, 0.f));
            __stcs(reinterpret_cast<float2*>(out + r * 32 + c2), o);
          }
        }
      }
    } else {
      for (int e = lane; e < n * dout; e += 32) {
        const int r = e / dout, c = e - r * dout;
        float acc = 0.f;
        for (int k = 0; k < din; ++k) acc = fmaf(AG[r * dinp + k], sW[k * dout + c], acc);
        out[e] = a.relu ? fmaxf(acc, 0.f) : acc;
      }
    }
    __syncwarp();  // slabs consumed before the next graph overwrites them
  }
}

// ---- readout: one warp per graph ------------------------------------------------------------
__global__ void __launch_bounds__(256) readout_kernel(const float* __restrict__ h, int d, int64_t B, int n_uniform,
                                                      const int64_t* __restrict__ node_ptr,
                                                      const float* __restrict__ aw, float* __restrict__ u) {
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int dq = d >> 2;
  const bool vec = (d & 3) == 0 && dq <= 32 && (32 % dq) == 0;
  for (int64_t g = warp0; g < B; g += nwarps) {
    const int64_t r0 = node_ptr ? node_ptr[g] : g * n_uniform;
    const int n = static_cast<int>((node_ptr ? node_ptr[g + 1] : r0 + n_uniform) - r0);
    if (vec) {
      // lane owns channel quad (lane % dq) of rows lane / dq, + 32 / dq, ...
      const int cq = lane % dq, rstep = 32 / dq;
      const float4 a4 = reinterpret_cast<const float4*>(aw)[cq];
      float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
      float4 mx = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
      const float4* base = reinterpret_cast<const float4*>(h + r0 * d);
      int r = lane / dq;
      if (n <= 8 * rstep) {  // the whole graph's loads in flight at once (predicated, 8 per lane)
        float4 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k)
          v[k] = r + k * rstep < n ? __ldcs(base + (r + k * rstep) * dq + cq) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (r + k * rstep < n) {
            s.x = fmaf(v[k].x, a4.x, s.x);
            s.y = fmaf(v[k].y, a4.y, s.y);
            s.z = fmaf(v[k].z, a4.z, s.z);
            s.w = fmaf(v[k].w, a4.w, s.w);
            mx.x = fmaxf(mx.x, v[k].x);
            mx.y = fmaxf(mx.y, v[k].y);
            mx.z = fmaxf(mx.z, v[k].z);
            mx.w = fmaxf(mx.w, v[k].w);
          }
        r = n;
      }
#pragma unroll 4
      for (; r < n; r += rstep) {
        const float4 v = __ldcs(base + r * dq + cq);  // streamed once: evict-first
        s.x = fmaf(v.x, a4.x, s.x);
        s.y = fmaf(v.y, a4.y, s.y);
        s.z = fmaf(v.z, a4.z, s.z);
        s.w = fmaf(v.w, a4.w, s.w);
        mx.x = fmaxf(mx.x, v.x);
        mx.y = fmaxf(mx.y, v.y);
        mx.z = fmaxf(mx.z, v.z);
        mx.w = fmaxf(mx.w, v.w);
      }
      for (int off = dq; off < 32; off <<= 1) {  // segmented shuffle reduction over row groups
        s.x += __shfl_xor_sync(0xffffffffu, s.x, off);
        s.y += __shfl_xor_sync(0xffffffffu, s.y, off);
        s.z += __shfl_xor_sync(0xffffffffu, s.z, off);
        s.w += __shfl_xor_sync(0xffffffffu, s.w, off);
        mx.x = fmaxf(mx.x, __shfl_xor_sync(0xffffffffu, mx.x, off));
        mx.y = fmaxf(mx.y, __shfl_xor_sync(0xffffffffu, mx.y, off));
        mx.z = fmaxf(mx.z, __shfl_xor_sync(0xffffffffu, mx.z, off));
        mx.w = fmaxf(mx.w, __shfl_xor_sync(0xffffffffu, mx.w, off));
      }
      if (lane < dq) {
        float4* uo = reinterpret_cast<float4*>(u + g * 2 * d);
        uo[lane] = s;
        uo[dq + lane] = mx;
      }
    } else {
      for (int c = lane; c < d; c += 32) {
        float s = 0.f, mx = -INFINITY;
        for (int r = 0; r < n; ++r) {
          const float v = h[(r0 + r) * d + c];
          s = fmaf(v, aw[c], s);
          mx = fmaxf(mx, v);
        }
        u[g * 2 * d + c] = s;
        u[g * 2 * d + d + c] = mx;
      }
    }
  }
}


constexpr int TC_ROWS = 128;

// ---- pipelined tensor-core layer: TMA-staged tiles, aggregate-then-transform --------------------
//
// out = ReLU((A Xn) W) for tiles of whole graphs (<= 128 rows, contiguous in HBM):
//   thread 0 (producer)  1-D bulk copies (cp.async.bulk, TMA engine) of the next S tiles'
//                        input rows into an S-stage shared-memory ring, one copy per tile;
//   row r (thread r)     sums a_rj * xn_j over its CSR row straight out of the staged tile
//                        (layer 1 z-normalises and masks the fp64 rows on the fly), splits
//                        the sum hi/lo and tcgen05.st's it into TMEM (the A operand);
//   elected thread       3 x K/8 tcgen05.mma kind::tf32 (3xTF32), D in TMEM;
//   row r                tcgen05.ld's D, applies ReLU, writes the row into an output
//                        staging tile; thread 0 bulk-stores the tile (one copy).
// Loads run S tiles ahead and stores drain asynchronously, so HBM traffic overlaps the
// aggregation / MMA of the tile in flight; three CTAs per SM (128 TMEM columns each).
// Aggregating first (A X) W is the order the reference's einsum takes for layer 1
// (SURVEY.md 8(a)); for layer 2 it equals A (H W) up to fp32 rounding.
//
// TM (uniform graphs, 128-byte rows): tiles move through 2-D tensor maps with the 128-byte
// swizzle instead of 1-D copies -- 16-byte piece c of tile row R sits at piece c ^ (R & 7)
// -- so the row-per-thread reads and writes are bank-conflict free with no register
// rotation (TMA undoes the swizzle on the way out).
template <int DIN, bool IN64, int S, int OB, bool TM, bool PF = false>  // PF: the L2 prefetch is compiled in
__global__ void __launch_bounds__(TC_ROWS, S == 1 ? 4 : 3)
    gcn_layer_pipe_kernel(LayerArgs a, int rp_cap, int nz_cap, const __grid_constant__ CUtensorMap tm_in,
                          const __grid_constant__ CUtensorMap tm_out) {
  constexpr int K = (DIN + 7) & ~7;
  constexpr int DOUT = 32;
  constexpr int ESZ = IN64 ? 8 : 4;
  constexpr int ROWB = DIN * ESZ;             // input row bytes (16-byte multiple)
  constexpr int STAGE = TC_ROWS * ROWB;       // input stage bytes
  static_assert(ROWB % 16 == 0, "bulk copies need 16-byte rows");
  static_assert(!TM || (ROWB == 128 && !IN64), "the swizzled path takes 128-byte fp32 rows");
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // swizzled tiles need 1024-byte aligned buffers (the host adds 1 KB of slack)
  unsigned char* smem = smem_raw + ((1024 - (s32(smem_raw) & 1023)) & 1023);
  unsigned char* stage0 = smem;
  float* outb0 = reinterpret_cast<float*>(stage0 + S * STAGE);
  float* bh = outb0 + OB * TC_ROWS * DOUT;
  float* bl = bh + DOUT * K;
  int* s_rp = reinterpret_cast<int*>(bl + DOUT * K);
  int* s_col = s_rp + ((rp_cap + 3) & ~3);
  float* s_val = reinterpret_cast<float*>(s_col + ((nz_cap + 3) & ~3));
  uint8_t* s_mask = reinterpret_cast<uint8_t*>(s_val + ((nz_cap + 3) & ~3));
  __shared__ PatSmem P;
  __shared__ float s_mean[KT_MAX_DIM], s_rstd[KT_MAX_DIM];
  __shared__ double d_mean[KT_MAX_DIM], d_rstd[KT_MAX_DIM];
  __shared__ __align__(8) uint64_t full[S];
  __shared__ __align__(8) uint64_t mma_bar;
  __shared__ uint32_t tmem_slot;
  __shared__ int s_gptr[TC_ROWS + 1];
  __shared__ float4 hub_s[TC_ROWS / 32][8];  // hub-row channel quads, per warp
  const int tid = threadIdx.x, warp = tid >> 5;
  (void)s_mean;
  (void)s_rstd;

  const int64_t n_tiles = (a.B + a.G - 1) / a.G;
  auto tile_rows = [&](int64_t t, int64_t& r0) {
    const int64_t g0 = t * a.G;
    const int64_t g1 = g0 + a.G < a.B ? g0 + a.G : a.B;
    r0 = tile_row0(a, g0);
    return static_cast<int>(tile_row0(a, g1) - r0);
  };
  auto issue_load = [&](int64_t t, int st) {
    int64_t r0;
    const int rows = tile_rows(t, r0);
    if constexpr (TM) {  // full box every time (rows past the end arrive zero-filled)
      mbar_expect(&full[st], static_cast<uint32_t>(a.G * a.n_uniform * ROWB));
      tma_load_2d(stage0 + st * STAGE, &tm_in, 0, static_cast<int>(r0), &full[st]);
    } else {
      const uint32_t bytes = static_cast<uint32_t>(rows) * ROWB;
      mbar_expect(&full[st], bytes);
      bulk_load(stage0 + st * STAGE, static_cast<const unsigned char*>(a.in) + r0 * ROWB, bytes, &full[st]);
    }
  };
  // more bytes in flight than the smem ring holds: the tile l2pf grid strides past a load is
  // pulled into L2 when that load is issued, so the ring refills from L2
  auto issue_prefetch = [&](int64_t t) {
    if (t >= n_tiles) return;
    int64_t r0;
    const int rows = tile_rows(t, r0);
    if constexpr (TM)
      tma_prefetch_2d(&tm_in, 0, static_cast<int>(r0));
    else
      bulk_prefetch_l2(static_cast<const unsigned char*>(a.in) + r0 * ROWB, static_cast<uint32_t>(rows) * ROWB);
  };

  // ---- setup ---------------------------------------------------------------------------------
  for (int e = tid; e < DOUT * K; e += TC_ROWS) {  // B = W^T: row n, column k
    const int n = e / K, k = e - n * K;
    const float v = k < DIN ? a.W[k * DOUT + n] : 0.0f;
    const float h = tc::tf32_trunc(v);
    const int off = tc::kmajor_offset(n, k, K) >> 2;
    bh[off] = h;
    bl[off] = v - h;
  }
  if (tid == 0) {
    int rp = 0, nz = 0, mk = 0;
    for (int p = 0; p < a.n_pat; ++p) {
      P.n[p] = a.pat_n[p];
      P.rp_off[p] = rp;
      P.nz_off[p] = nz;
      P.mask_off[p] = mk;
      nz += a.pat_rp[rp + P.n[p]];
      rp += P.n[p] + 1;
      mk += P.n[p];
    }
    for (int st = 0; st < S; ++st) mbar_init1(&full[st]);
    tc::mbar_init(&mma_bar, 1);
    tc::fence_async_smem();
    // the first S tiles start streaming while the rest of the setup runs
    for (int st = 0; st < S; ++st)
      if (blockIdx.x + static_cast<int64_t>(st) * gridDim.x < n_tiles)
        issue_load(blockIdx.x + static_cast<int64_t>(st) * gridDim.x, st);
    if constexpr (PF)
      for (int p = 0; p < a.l2pf; ++p) issue_prefetch(blockIdx.x + static_cast<int64_t>(S + p) * gridDim.x);
  }
  if (IN64)
    for (int c = tid; c < DIN; c += TC_ROWS) {
      d_mean[c] = a.fmean[c];
      d_rstd[c] = 1.0 / a.fstd[c];
    }
  if (warp == 0) tc::tmem_alloc(&tmem_slot, 128);
  __syncthreads();
  {
    int tot_rp = 0, tot_nz = 0, tot_mask = 0;
    for (int p = 0; p < a.n_pat; ++p) {
      tot_rp += P.n[p] + 1;
      tot_mask += P.n[p];
      tot_nz += a.pat_rp[P.rp_off[p] + P.n[p]];
    }
    for (int i = tid; i < tot_rp; i += TC_ROWS) s_rp[i] = a.pat_rp[i];
    for (int i = tid; i < tot_nz; i += TC_ROWS) {
      s_col[i] = a.pat_col[i];
      s_val[i] = a.pat_val[i];
    }
    if (IN64)
      for (int i = tid; i < tot_mask; i += TC_ROWS) s_mask[i] = a.pat_mask ? a.pat_mask[i] : 1;
  }
  if (IN64) {
    // drop masked columns from the CSR once (their normalised rows are exactly 0), so the
    // row loop never tests the mask
    __syncthreads();
    if (tid == 0) {
      int w = 0;
      for (int p = 0; p < a.n_pat; ++p) {
        int* rp = s_rp + P.rp_off[p];
        const int src0 = P.nz_off[p];
        P.nz_off[p] = w;
        int prev = rp[0];
        rp[0] = 0;
        for (int l = 0; l < P.n[p]; ++l) {
          const int e_end = rp[l + 1];
          for (int e = prev; e < e_end; ++e) {
            const int j = s_col[src0 + e];
            if (s_mask[P.mask_off[p] + j]) {
              s_col[w] = j;
              s_val[w] = s_val[src0 + e];
              ++w;
            }
          }
          prev = e_end;
          rp[l + 1] = w - P.nz_off[p];
        }
      }
    }
  }
  const int u_g = a.node_ptr ? 0 : tid / a.n_uniform;  // uniform graphs: fixed row -> graph map
  tc::fence_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tmem_slot;
  const uint32_t lane_addr = static_cast<uint32_t>((32 * warp) << 16);
  const uint32_t T_AH = 0, T_AL = 32, T_D = 64;  // D double-buffered: T_D + 32 (it & 1)
  const uint32_t idesc = tc::idesc_tf32(128, DOUT);

  // Epilogue of a tile whose MMA has completed: ReLU(D) -> output staging -> one bulk store.
  // Runs one tile behind the aggregation, so tile t's MMA overlaps tile t-1's epilogue.
  auto epilogue = [&](int64_t pit, int64_t pr0, int prows) {
    float* ob = outb0 + (pit % OB) * (TC_ROWS * DOUT);
    {
      float v[32];
      tc::tmem_ld32(tmem + lane_addr + T_D + 32 * static_cast<uint32_t>(pit & 1), v);
      tc::tmem_wait_ld();
      if (tid < prows) {
        float4* dst = reinterpret_cast<float4*>(ob + tid * DOUT);
        // rows are 128 B: store piece (q + r) % 8 at step q so that eight consecutive rows hit
        // eight different bank groups; the registers are rotated to match (barrel shift)
        const int orot = tid & 7;
#pragma unroll
        for (int sh = 1; sh < 8; sh <<= 1) {
          if (!TM && (orot & sh)) {
            float r[32];
#pragma unroll
            for (int c = 0; c < 8; ++c)
#pragma unroll
              for (int q = 0; q < 4; ++q) r[4 * c + q] = v[4 * ((c + sh) & 7) + q];
#pragma unroll
            for (int k = 0; k < 32; ++k) v[k] = r[k];
          }
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          float4 o = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
          if (a.relu) o = make_float4(fmaxf(o.x, 0.f), fmaxf(o.y, 0.f), fmaxf(o.z, 0.f), fmaxf(o.w, 0.f));
          dst[TM ? (q ^ orot) : ((q + orot) & 7)] = o;
        }
      }
    }
    fence_proxy_async();
    tc::tc_fence_before();
    __syncthreads();  // (C) staging tile complete; TMEM D reads done
    if (tid == 0) {
      if constexpr (TM)
        tma_store_2d(&tm_out, 0, static_cast<int>(pr0), ob);  // rows past the end are clipped
      else
        bulk_store(a.out + pr0 * DOUT, ob, static_cast<uint32_t>(prows) * DOUT * 4);
    }
  };

  int64_t it = 0, prev_r0 = 0;
  int prev_rows = 0;
  for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++it) {
    const int st = static_cast<int>(it % S);
    const int64_t g0 = t * a.G;
    const int ng = static_cast<int>((g0 + a.G < a.B ? g0 + a.G : a.B) - g0);
    int64_t r0;
    const int rows = tile_rows(t, r0);
    if (tid <= ng) s_gptr[tid] = static_cast<int>(tile_row0(a, g0 + tid) - r0);
    tc::mbar_wait(&full[st], static_cast<uint32_t>((it / S) & 1));
    __syncthreads();  // (A) s_gptr ready
    // ---- 1. y_r = sum_j a_rj xn_j out of the staged tile -> hi / lo -> TMEM -------------------------
    float y[K];
#pragma unroll
    for (int k = 0; k < K; ++k) y[k] = 0.0f;
    constexpr int NP = IN64 ? 1 : DIN / 4;
    static_assert(IN64 || (NP & (NP - 1)) == 0, "rotation needs a power-of-two piece count");
    const int rot = tid & (NP - 1);
    const unsigned char* tile = stage0 + st * STAGE;
    int p = 0, base = 0, e_lo = 0, e_hi = 0;
    if (tid < rows) {
      int my_g = u_g;
      if (a.node_ptr)
        while (my_g + 1 < ng && s_gptr[my_g + 1] <= tid) ++my_g;
      base = a.node_ptr ? s_gptr[my_g] : my_g * a.n_uniform;
      p = a.pat_id ? a.pat_id[g0 + my_g] : 0;
      e_lo = P.nz_off[p] + s_rp[P.rp_off[p] + tid - base];
      e_hi = P.nz_off[p] + s_rp[P.rp_off[p] + tid - base + 1];
    }
    // hub rows (star roots: 13 of a graph's 73 nonzeros) are summed by the whole warp
    // below, so the per-row loop runs <= HUB iterations
    // (layer 1: a root's neighbours are masked loop nodes, skipped cheaply in the row loop)
    constexpr int HUB = IN64 ? (1 << 30) : 4;
    const bool hub = e_hi - e_lo > HUB;
    {
      for (int e = hub ? e_hi : e_lo; e < e_hi; ++e) {
        const int j = s_col[e];
        const float w = s_val[e];
        if constexpr (IN64) {
          const double2* src = reinterpret_cast<const double2*>(tile + (base + j) * ROWB);
#pragma unroll
          for (int i = 0; i < DIN / 2; ++i) {
            const double2 d = src[i];
            const float x0 = static_cast<float>((d.x - d_mean[2 * i]) * d_rstd[2 * i]);
            const float x1 = static_cast<float>((d.y - d_mean[2 * i + 1]) * d_rstd[2 * i + 1]);
            y[2 * i] = fmaf(w, x0, y[2 * i]);
            y[2 * i + 1] = fmaf(w, x1, y[2 * i + 1]);
          }
        } else {
          // 16-byte pieces read in a per-row rotated order (piece (i + rot) % NP): eight
          // consecutive rows then hit eight different bank groups of the 128-byte rows
          const float4* src = reinterpret_cast<const float4*>(tile + (base + j) * ROWB);
          const int sw = TM ? ((base + j) & 7) : 0;
#pragma unroll
          for (int i = 0; i < NP; ++i) {
            const float4 v = TM ? src[i ^ sw] : src[(i + rot) & (NP - 1)];
            y[4 * i] = fmaf(w, v.x, y[4 * i]);
            y[4 * i + 1] = fmaf(w, v.y, y[4 * i + 1]);
            y[4 * i + 2] = fmaf(w, v.z, y[4 * i + 2]);
            y[4 * i + 3] = fmaf(w, v.w, y[4 * i + 3]);
          }
        }
      }
      if constexpr (!IN64 && !TM) {  // undo the rotation: piece c <- accumulator (c - rot) % NP (barrel shift)
#pragma unroll
        for (int sh = 1; sh < NP; sh <<= 1) {
          if (rot & sh) {
            float r[K];
#pragma unroll
            for (int c = 0; c < NP; ++c)
#pragma unroll
              for (int q = 0; q < 4; ++q) r[4 * c + q] = y[4 * ((c - sh) & (NP - 1)) + q];
#pragma unroll
            for (int k = 0; k < 4 * NP; ++k) y[k] = r[k];
          }
        }
      }
    }
    {  // hub rows: lane c sums feature c over the hub's edges (same edge order), then the
       // hub's lane collects the DIN sums by shuffles
      const int lane = tid & 31;
      unsigned hubs = __ballot_sync(0xffffffffu, hub);
      while (hubs) {
        const int src = __ffs(hubs) - 1;
        hubs &= hubs - 1;
        const int h_lo = __shfl_sync(0xffffffffu, e_lo, src), h_hi = __shfl_sync(0xffffffffu, e_hi, src);
        const int h_base = __shfl_sync(0xffffffffu, base, src);
        if constexpr (!IN64 && DIN == 32) {
          // lane = (edge group eg, channel quad q): float4 partial sums over edges eg, eg + 4,
          // ..., a fixed butterfly over the 4 edge groups, then the hub's lane reads the 8
          // quads from a per-warp scratch -- 4 edge steps per lane instead of 13
          const int q = lane & 7, eg = lane >> 3;
          float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
          for (int e = h_lo + eg; e < h_hi; e += 4) {
            const int R = h_base + s_col[e];
            const float w = s_val[e];
            const float4 v = reinterpret_cast<const float4*>(tile + R * ROWB)[TM ? (q ^ (R & 7)) : q];
            acc.x = fmaf(w, v.x, acc.x);
            acc.y = fmaf(w, v.y, acc.y);
            acc.z = fmaf(w, v.z, acc.z);
            acc.w = fmaf(w, v.w, acc.w);
          }
#pragma unroll
          for (int m = 8; m <= 16; m <<= 1) {
            acc.x += __shfl_xor_sync(0xffffffffu, acc.x, m);
            acc.y += __shfl_xor_sync(0xffffffffu, acc.y, m);
            acc.z += __shfl_xor_sync(0xffffffffu, acc.z, m);
            acc.w += __shfl_xor_sync(0xffffffffu, acc.w, m);
          }
          if (eg == 0) hub_s[warp][q] = acc;
          __syncwarp();
          if (lane == src)
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const float4 v = hub_s[warp][i];
              y[4 * i] = v.x;
              y[4 * i + 1] = v.y;
              y[4 * i + 2] = v.z;
              y[4 * i + 3] = v.w;
            }
          __syncwarp();
          continue;
        }
        float yc = 0.0f;
        if (lane < DIN)
          for (int e = h_lo; e < h_hi; ++e) {
            const int j = s_col[e];
            const float w = s_val[e];
            if constexpr (IN64) {
              const double d = reinterpret_cast<const double*>(tile + (h_base + j) * ROWB)[lane];
              yc = fmaf(w, static_cast<float>((d - d_mean[lane]) * d_rstd[lane]), yc);
            } else {
              const int R = h_base + j;
              const int c = TM ? ((((lane >> 2) ^ (R & 7)) << 2) | (lane & 3)) : lane;
              yc = fmaf(w, reinterpret_cast<const float*>(tile + R * ROWB)[c], yc);
            }
          }
#pragma unroll
        for (int k = 0; k < DIN; ++k) {
          const float v = __shfl_sync(0xffffffffu, yc, k);
          if (lane == src) y[k] = v;
        }
      }
    }
    if (it > 0) {  // MMA of the previous tile done: A free again, its D complete
      tc::mbar_wait(&mma_bar, static_cast<uint32_t>((it - 1) & 1));
      __syncwarp();
      tc::tc_fence_after();
    }
    {
      float hi[K], lo[K];
#pragma unroll
      for (int k = 0; k < K; k += 2) {  // remainders as packed fp32x2 subtractions
        hi[k] = tc::tf32_trunc(y[k]);
        hi[k + 1] = tc::tf32_trunc(y[k + 1]);
        const float2 l = fsub2(make_float2(y[k], y[k + 1]), make_float2(hi[k], hi[k + 1]));
        lo[k] = l.x;
        lo[k + 1] = l.y;
      }
#pragma unroll
      for (int k0 = 0; k0 + 16 <= K; k0 += 16) {
        tc::tmem_st16(tmem + lane_addr + T_AH + k0, hi + k0);
        tc::tmem_st16(tmem + lane_addr + T_AL + k0, lo + k0);
      }
      if constexpr (K % 16 == 8) {
        float h16[16], l16[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          h16[k] = k < 8 ? hi[K - 8 + k] : 0.f;
          l16[k] = k < 8 ? lo[K - 8 + k] : 0.f;
        }
        tc::tmem_st16(tmem + lane_addr + T_AH + K - 8, h16);
        tc::tmem_st16(tmem + lane_addr + T_AL + K - 8, l16);
      }
      tc::tmem_wait_st();
    }
    if (tid == 0) {
      if (OB == 1) bulk_wait_read0(); else bulk_wait_read1();  // staging buffer it % OB is free again
    }
    tc::tc_fence_before();
    __syncthreads();  // (B) stage consumed, A in TMEM
    // ---- 2. refill the stage; D = A W on the tensor cores ------------------------------------------
    if (warp == 0) {
      tc::tc_fence_after();
      if (tid == 0 && t + static_cast<int64_t>(S) * gridDim.x < n_tiles) {
        issue_load(t + static_cast<int64_t>(S) * gridDim.x, st);
        if constexpr (PF)
          if (a.l2pf > 0) issue_prefetch(t + static_cast<int64_t>(S + a.l2pf) * gridDim.x);
      }
      __syncwarp();
      if (tc::elect_one()) {
#pragma unroll
        for (int kk = 0; kk < K / 8; ++kk) {
          const uint32_t d = tmem + T_D + 32 * static_cast<uint32_t>(it & 1);
          tc::mma_tf32_ts(d, tmem + T_AH + 8 * kk, tc::kdesc(bh, K, kk), idesc, kk > 0);
          tc::mma_tf32_ts(d, tmem + T_AH + 8 * kk, tc::kdesc(bl, K, kk), idesc, 1);
          tc::mma_tf32_ts(d, tmem + T_AL + 8 * kk, tc::kdesc(bh, K, kk), idesc, 1);
        }
        tc::mma_commit(&mma_bar);
      }
      __syncwarp();
    }
    // ---- 3. the previous tile's epilogue while this tile's MMA runs ---------------------------
    if (it > 0) epilogue(it - 1, prev_r0, prev_rows);
    prev_r0 = r0;
    prev_rows = rows;
  }
  if (it > 0) {
    if (tid == 0) {
      if (OB == 1) bulk_wait_read0(); else bulk_wait_read1();
    }
    tc::mbar_wait(&mma_bar, static_cast<uint32_t>((it - 1) & 1));
    __syncwarp();
    tc::tc_fence_after();
    __syncthreads();  // (staging buffer free for every thread)
    epilogue(it - 1, prev_r0, prev_rows);
  }
  if (tid == 0) bulk_wait0();
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem, 128);
  }
}


// Row-major fp32 (rows x 32) tensor maps for the swizzled path: box = one tile of
// box_rows rows, 128-byte swizzle.  False if the driver entry point is unavailable.
static bool tensor_maps(const void* in, const void* out, int64_t rows, int box_rows, CUtensorMap* tin,
                        CUtensorMap* tout) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  static bool looked = false;
  if (!looked) {
    looked = true;
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  if (!encode || box_rows > 256 || rows >= (int64_t{1} << 31)) return false;
  const cuuint64_t dims[2] = {32, static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {32 * sizeof(float)};
  const cuuint32_t box[2] = {32, static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  auto mk = [&](CUtensorMap* m, const void* p) {
    return encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(p), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  };
  return mk(tin, in) && mk(tout, out);
}
}  // namespace agg
}  // namespace kt

using namespace kt;

extern "C" int kt_gcn_layer(const void* in, int32_t in_f64, const double* fmean, const double* fstd,
                            const float* W, int32_t d_in, int32_t d_out, int32_t relu, int64_t B,
                            int32_t nodes_per_graph, const int64_t* node_ptr, const int32_t* pat_id,
                            int32_t n_pat, const int32_t* pat_n, const int32_t* pat_rp, const int32_t* pat_col,
                            const float* pat_val, const uint8_t* pat_mask, int32_t pat_nnz, int32_t max_nodes,
                            float* out, void* stream) {
  KT_REQUIRE(in && W && out && pat_n && pat_rp && pat_col && pat_val, KT_E_ARG, "kt_gcn_layer: null pointer");
  KT_REQUIRE(B > 0, KT_E_EMPTY, "kt_gcn_layer: empty batch");
  KT_REQUIRE(d_in > 0 && d_out > 0 && d_in <= KT_MAX_DIM && d_out <= KT_MAX_DIM, KT_E_SHAPE,
             "kt_gcn_layer: layer widths must be in [1, %d]", KT_MAX_DIM);
  KT_REQUIRE(n_pat >= 1 && n_pat <= agg::MAXPAT, KT_E_UNSUPPORTED, "kt_gcn_layer: 1..%d adjacency patterns",
             agg::MAXPAT);
  KT_REQUIRE(nodes_per_graph > 0 || node_ptr, KT_E_ARG, "kt_gcn_layer: need nodes_per_graph or node_ptr");
  KT_REQUIRE(pat_nnz > 0 && pat_nnz <= agg::MAXPNNZ, KT_E_UNSUPPORTED, "kt_gcn_layer: <= %d adjacency nonzeros",
             agg::MAXPNNZ);
  KT_REQUIRE(!in_f64 || (fmean && fstd), KT_E_ARG, "kt_gcn_layer: fp64 input needs the feature norms");
  KT_REQUIRE(max_nodes > 0 && max_nodes <= KT_MAX_NODES, KT_E_SHAPE, "kt_gcn_layer: graphs of <= %d nodes",
             KT_MAX_NODES);
  agg::LayerArgs a{};
  a.in = in;
  a.in_f64 = in_f64;
  a.out = out;
  a.W = W;
  a.fmean = fmean;
  a.fstd = fstd;
  a.d_in = d_in;
  a.d_out = d_out;
  a.relu = relu;
  a.B = B;
  a.n_uniform = nodes_per_graph;
  a.node_ptr = nodes_per_graph > 0 ? nullptr : node_ptr;
  a.pat_id = pat_id;
  a.n_pat = n_pat;
  a.pat_n = pat_n;
  a.pat_rp = pat_rp;
  a.pat_col = pat_col;
  a.pat_val = pat_val;
  a.pat_mask = pat_mask;
  // per-warp slabs (X rows + aggregated rows, fp32) sized for the largest graph
  a.R = max_nodes;
  a.G = 1;
  a.bulk = 0;
  const int dinp = (d_in + 3) & ~3;
  const size_t smem = static_cast<size_t>((d_in * d_out + 3) & ~3) * 4 +
                      ((static_cast<size_t>(n_pat) * (KT_MAX_NODES + 1) + 3) & ~3) * 4 + agg::MAXPNNZ * 8 +
                      ((static_cast<size_t>(n_pat) * KT_MAX_NODES + 15) & ~15) +
                      static_cast<size_t>(agg::WPC) * 2 * max_nodes * dinp * 4;
  KT_REQUIRE(smem <= 200 * 1024, KT_E_UNSUPPORTED, "kt_gcn_layer: slabs do not fit shared memory (%zu B)", smem);
  const int64_t blocks = (B + agg::WPC - 1) / agg::WPC;
  const int grid = static_cast<int>(blocks < 4 * kNumSMs ? blocks : 4 * kNumSMs);
  auto launch = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    kern<<<grid, agg::NT, smem, as_stream(stream)>>>(a);
  };
  const bool tc_ok = d_out == 32 && ((d_in == 12 && in_f64) || (d_in == 32 && !in_f64)) &&
                     max_nodes <= agg::TC_ROWS &&
                     (reinterpret_cast<uintptr_t>(in) % 16 == 0) && (reinterpret_cast<uintptr_t>(out) % 16 == 0) &&
                     !(getenv("KT_AGG_FFMA") && getenv("KT_AGG_FFMA")[0] == '1');
  if (tc_ok) {
    // TMA-staged tiles of whole graphs (<= 128 rows), three CTAs per SM
    a.G = agg::TC_ROWS / max_nodes;
    const int rp_cap = n_pat * (max_nodes + 1), nz_cap = pat_nnz;
    const size_t csr = ((static_cast<size_t>(rp_cap) + 3) & ~3) * 4 + ((static_cast<size_t>(nz_cap) + 3) & ~3) * 8 +
                       static_cast<size_t>(n_pat) * max_nodes + 16;
    const int64_t tiles = (B + a.G - 1) / a.G;
    {
      // layer 2 (fp32 in): one tile of L2 prefetch past the ring, 0.77 -> 0.84 of HBM; layer 1
      // (fp64 in, three stages) already streams at 0.94 and loses with it (0.90)
      const char* pf = getenv(d_in == 12 ? "KT_AGG_L2PF1" : "KT_AGG_L2PF");
      a.l2pf = pf ? atoi(pf) : (d_in == 12 ? 0 : 1);
    }
    const char* sob_env = getenv("KT_AGG_SOB");
    const bool staged1 = d_in == 32 && nodes_per_graph > 0 && !(sob_env && sob_env[0] == '2');
    const int per_sm = staged1 ? 4 : 3;  // CTAs per SM that shared memory holds
    const int tgrid = static_cast<int>(tiles < per_sm * kNumSMs ? tiles : per_sm * kNumSMs);
    CUtensorMap tm_in{}, tm_out{};
    auto plaunch = [&](auto kern, int K, int stage_bytes, int S, int OB, bool tm) {
      // (the swizzled path aligns its buffers to 1 KB at run time: slack for that)
      const size_t psm = (tm ? 1024 : 0) + static_cast<size_t>(2 * 32 * K) * 4 + static_cast<size_t>(S) * stage_bytes +
                         static_cast<size_t>(OB) * agg::TC_ROWS * 32 * 4 + csr;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(psm));
      kern<<<tgrid, agg::TC_ROWS, psm, as_stream(stream)>>>(a, rp_cap, nz_cap, tm_in, tm_out);
    };
    if (d_in == 12) {
      plaunch(agg::gcn_layer_pipe_kernel<12, true, 3, 2, false>, 16, agg::TC_ROWS * 12 * 8, 3, 2, false);
    } else if (nodes_per_graph > 0 && agg::tensor_maps(in, out, B * nodes_per_graph, a.G * nodes_per_graph,
                                                       &tm_in, &tm_out) &&
               !(getenv("KT_AGG_NOTM") && getenv("KT_AGG_NOTM")[0] == '1')) {
      // one input stage + one output tile (the epilogue already runs a tile behind the MMA),
      // so four CTAs fit an SM: measured 0.77 of HBM peak against 0.75 for 2 x 1 at three
      // CTAs per SM (2 x 2 and 3 x 1 drop to two CTAs per SM: 0.41); KT_AGG_SOB=21 for A/B
      const char* sob = getenv("KT_AGG_SOB");
      if (sob && sob[0] == '2' && sob[1] == '1')
        plaunch(agg::gcn_layer_pipe_kernel<32, false, 2, 1, true, true>, 32, agg::TC_ROWS * 32 * 4, 2, 1, true);
      else
        plaunch(agg::gcn_layer_pipe_kernel<32, false, 1, 1, true, true>, 32, agg::TC_ROWS * 32 * 4, 1, 1, true);
    } else {
      plaunch(agg::gcn_layer_pipe_kernel<32, false, 3, 1, false>, 32, agg::TC_ROWS * 32 * 4, 3, 1, false);
    }
  } else if (d_in == 12 && d_out == 32) {
    launch(agg::gcn_layer_kernel<12, 32>);
  } else if (d_in == 32 && d_out == 32) {
    launch(agg::gcn_layer_kernel<32, 32>);
  } else {
    launch(agg::gcn_layer_kernel<0, 0>);
  }
  note_launches(1);
  return check_launch("kt_gcn_layer");
}

extern "C" int kt_readout(const float* h, int32_t d, int64_t B, int32_t nodes_per_graph, const int64_t* node_ptr,
                          const float* agg_w, float* u_out, void* stream) {
  KT_REQUIRE(h && agg_w && u_out, KT_E_ARG, "kt_readout: null pointer");
  KT_REQUIRE(B > 0, KT_E_EMPTY, "kt_readout: empty batch");
  KT_REQUIRE(d > 0, KT_E_SHAPE, "kt_readout: embedding width must be positive");
  KT_REQUIRE(nodes_per_graph > 0 || node_ptr, KT_E_ARG, "kt_readout: need nodes_per_graph or node_ptr");
  const int64_t warps = B;
#ifndef KT_RO_BPS
#define KT_RO_BPS 128  // readout CTAs per SM in the grid-stride launch (16: 0.86 of HBM, 64-128: 0.97, uncapped: 0.84)
#endif
  const int64_t blocks = (warps * 32 + 255) / 256;
  const int grid = static_cast<int>(blocks < KT_RO_BPS * kNumSMs ? blocks : KT_RO_BPS * kNumSMs);
  agg::readout_kernel<<<grid, 256, 0, as_stream(stream)>>>(h, d, B, nodes_per_graph,
                                                           nodes_per_graph > 0 ? nullptr : node_ptr, agg_w, u_out);
  note_launches(1);
  return check_launch("kt_readout");
}
