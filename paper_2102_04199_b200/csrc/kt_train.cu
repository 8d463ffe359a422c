// Training path: model.grad (model.py:218-285), sgd_step (model.py:288-310) and
// the batch-1 SGD loop of meta.pretrain (meta.py:104-123) on device.
//
// kt_grad: one warp per graph runs the forward with caches and the reverse
// pass (head -> readout with first-index argmax routing -> GCN), writing that
// graph's gradient contribution (already scaled by 2 (pred - y) / B, as the
// reference does) into a per-graph row of a workspace matrix.  A second kernel
// sums the rows in a fixed order in fp64 (deterministic, no atomics), chunking
// batches larger than the workspace.  kt_pretrain_sgd keeps the parameters in
// shared memory and runs the whole sequential SGD loop in one CTA.
#include <cstdlib>

#include "kt_graph.cuh"

namespace kt {

int check_dims(const kt_dims& d);

namespace train {

struct Slab {
  float* H[KT_MAX_LAYERS + 1];
  float* AH[KT_MAX_LAYERS];
  float* t0;
  float* t1;
  float* act[KT_MAX_LAYERS + 2];
  float* zh[KT_MAX_LAYERS + 1];
  float* da;
  float* dz;
  int* arg;
};

constexpr int HV = 2 * KT_MAX_DIM;  // head vector slot

__host__ __device__ inline int slab_floats(const kt_dims& d, int nmax, int D) {
  const int L = d.n_gcn, nh = d.n_head;
  return (2 * L + 3) * nmax * D + (2 * nh + 3) * HV + KT_MAX_DIM;
}

__device__ __forceinline__ Slab carve(float* base, const kt_dims& d, int nmax, int D) {
  Slab s;
  float* p = base;
  for (int l = 0; l <= d.n_gcn; ++l) { s.H[l] = p; p += nmax * D; }
  for (int l = 0; l < d.n_gcn; ++l) { s.AH[l] = p; p += nmax * D; }
  s.t0 = p; p += nmax * D;
  s.t1 = p; p += nmax * D;
  for (int i = 0; i <= d.n_head; ++i) { s.act[i] = p; p += HV; }
  for (int i = 0; i < d.n_head; ++i) { s.zh[i] = p; p += HV; }
  s.da = p; p += HV;
  s.dz = p; p += HV;
  s.arg = reinterpret_cast<int*>(p);
  return s;
}

// Forward with caches + reverse pass for one graph.  Writes this graph's
// gradient contribution to gout[0 .. n_params) (overwrites; zeros for gcn/agg
// in head-only scope) and returns the squared error.
template <class Grp>
__device__ float graph_grad(const Grp& G, const kt_dims& dims, const float* P, const GraphView& v,
                            const double* feats, const double* fmean, const double* fstd, float y, float inv_b,
                            bool head_only, const Slab& S, float* gout, int D) {
  const int L = dims.n_gcn, nh = dims.n_head, n = v.n;
  const int dl = dims.gcn[L];
  load_features(G, v, feats, dims.F, fmean, fstd, S.H[0], D);
  G.sync();
  for (int l = 0; l < L; ++l) {
    csr_aggregate(G, v, S.H[l], S.AH[l], dims.gcn[l], D);
    G.sync();
    dense(G, S.AH[l], P + dims.off_gcn[l], S.H[l + 1], n, dims.gcn[l], dims.gcn[l + 1], D, true);
    G.sync();
  }
  readout(G, S.H[L], n, dl, D, P + dims.off_agg, S.act[0], S.arg);
  G.sync();
  // head layers: four threads per output (k split four ways, quad shuffles), so the
  // 64-wide layers keep every thread of the group busy
  const unsigned qm = 0xFu << (G.r & 28);
  for (int i = 0; i < nh; ++i) {
    const int din = dims.head[i], dout = dims.head[i + 1];
    const float* W = P + dims.off_hw[i];
    const float* b = P + dims.off_hb[i];
    for (int e = G.r; e < 4 * dout; e += G.n) {
      const int c = e >> 2;
      float acc = 0.0f;
      for (int k = e & 3; k < din; k += 4) acc = fmaf(S.act[i][k], W[k * dout + c], acc);
      acc += __shfl_xor_sync(qm, acc, 1);
      acc += __shfl_xor_sync(qm, acc, 2);
      if ((e & 3) == 0) {
        acc += b[c];
        S.zh[i][c] = acc;
        S.act[i + 1][c] = i == nh - 1 ? acc : fmaxf(acc, 0.0f);
      }
    }
    G.sync();
  }
  const float pred = S.act[nh][0];
  const float err = pred - y;
  if (G.r == 0) S.da[0] = 2.0f * err * inv_b;
  G.sync();
  // head backward (model.py:258-265)
  for (int i = nh - 1; i >= 0; --i) {
    const int din = dims.head[i], dout = dims.head[i + 1];
    const float* W = P + dims.off_hw[i];
    for (int c = G.r; c < dout; c += G.n)
      S.dz[c] = (i == nh - 1 || S.zh[i][c] > 0.0f) ? S.da[c] : 0.0f;
    G.sync();
    float* gw = gout + dims.off_hw[i];
    for (int e = G.r; e < din * dout; e += G.n) {
      const int k = e / dout, c = e - (e / dout) * dout;
      gw[e] = S.act[i][k] * S.dz[c];
    }
    for (int c = G.r; c < dout; c += G.n) gout[dims.off_hb[i] + c] = S.dz[c];
    for (int e = G.r; e < 4 * din; e += G.n) {
      const int k = e >> 2;
      float acc = 0.0f;
      for (int c = e & 3; c < dout; c += 4) acc = fmaf(S.dz[c], W[k * dout + c], acc);
      acc += __shfl_xor_sync(qm, acc, 1);
      acc += __shfl_xor_sync(qm, acc, 2);
      if ((e & 3) == 0) S.da[k] = acc;
    }
    G.sync();
  }
  if (head_only) {
    for (int e = G.r; e < dims.off_head; e += G.n) gout[e] = 0.0f;
    return err * err;
  }
  // readout backward (model.py:268-276): weighted-sum path + first-argmax routing of the max path
  const float* agg = P + dims.off_agg;
  for (int c = G.r; c < dl; c += G.n) {
    float colsum = 0.0f;
    for (int r = 0; r < n; ++r) colsum += S.H[L][r * D + c];
    gout[dims.off_agg + c] = colsum * S.da[c];
  }
  for (int e = G.r; e < n * dl; e += G.n) {
    const int r = e / dl, c = e - (e / dl) * dl;
    S.t0[r * D + c] = agg[c] * S.da[c] + (r == S.arg[c] ? S.da[dl + c] : 0.0f);
  }
  G.sync();
  // GCN backward (model.py:279-284)
  for (int l = L - 1; l >= 0; --l) {
    const int din = dims.gcn[l], dout = dims.gcn[l + 1];
    for (int e = G.r; e < n * dout; e += G.n) {
      const int r = e / dout, c = e - (e / dout) * dout;
      if (!(S.H[l + 1][r * D + c] > 0.0f)) S.t0[r * D + c] = 0.0f;
    }
    G.sync();
    float* gw = gout + dims.off_gcn[l];
    for (int e = G.r; e < din * dout; e += G.n) {
      const int a = e / dout, c = e - (e / dout) * dout;
      float acc = 0.0f;
      for (int r = 0; r < n; ++r) acc = fmaf(S.AH[l][r * D + a], S.t0[r * D + c], acc);
      gw[e] = acc;
    }
    if (l > 0) {
      dense_t(G, S.t0, P + dims.off_gcn[l], S.t1, n, din, dout, D);
      G.sync();
      csr_aggregate(G, v, S.t1, S.t0, din, D);
    }
    G.sync();
  }
  return err * err;
}

constexpr int WARPS = 4;

__global__ void __launch_bounds__(WARPS * 32)
pergraph_kernel(kt_dims dims_p, const float* __restrict__ params, const double* __restrict__ fmean,
                const double* __restrict__ fstd, const double* __restrict__ feats, const uint8_t* __restrict__ mask,
                const int64_t* __restrict__ node_ptr, int npg, int nmax, const int32_t* __restrict__ row_ptr,
                const int32_t* __restrict__ col, const float* __restrict__ val, const int64_t* __restrict__ gidx,
                const float* __restrict__ y, int64_t b0, int64_t nb, float inv_b, int head_only, int D,
                float* __restrict__ pg_grad, float* __restrict__ pg_sq) {
  extern __shared__ __align__(16) float sm[];
  __shared__ kt_dims dims_s;  // (run-time indexed tables: shared memory, not the stack)
  __shared__ Slab slab_s[WARPS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) dims_s = dims_p;
  __syncthreads();
  const kt_dims& dims = dims_s;
  if (lane == 0) slab_s[warp] = carve(sm + warp * slab_floats(dims, nmax, D), dims, nmax, D);
  __syncthreads();
  const Slab& S = slab_s[warp];
  const WarpGroup W{lane};
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * WARPS + warp; i < nb;
       i += static_cast<int64_t>(gridDim.x) * WARPS) {
    const int64_t b = b0 + i;
    const int64_t g = gidx ? gidx[b] : b;
    const GraphView v = graph_view(g, node_ptr, npg, row_ptr, col, val, mask);
    const float sq = graph_grad(W, dims, params, v, feats, fmean, fstd, y[b], inv_b, head_only != 0, S,
                                pg_grad + i * dims.n_params, D);
    if (lane == 0) pg_sq[i] = sq;
    W.sync();
  }
}

// Small batches: one CTA (CT threads) per graph.  The same per-graph arithmetic as the
// warp form (each output element is still owned by one thread with a sequential inner
// loop), spread over 8x the threads, so a 512-graph batch fills the GPU.  The CTA stages
// the parameters in shared memory first (39 KB for the default dims): every layer's inner
// loops then read weights at shared-memory latency instead of L1/L2 latency.
#ifndef KT_GRAD_CT
#define KT_GRAD_CT 256
#endif
constexpr int CT = KT_GRAD_CT;

__global__ void __launch_bounds__(CT)
pergraph_cta_kernel(kt_dims dims_p, const float* __restrict__ params, const double* __restrict__ fmean,
                    const double* __restrict__ fstd, const double* __restrict__ feats,
                    const uint8_t* __restrict__ mask, const int64_t* __restrict__ node_ptr, int npg, int nmax,
                    const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                    const float* __restrict__ val, const int64_t* __restrict__ gidx, const float* __restrict__ y,
                    int64_t b0, int64_t nb, float inv_b, int head_only, int D, float* __restrict__ pg_grad,
                    float* __restrict__ pg_sq) {
  extern __shared__ __align__(16) float sm[];
  __shared__ kt_dims dims_s;  // (run-time indexed tables: shared memory, not the stack)
  __shared__ Slab slab_s;
  if (threadIdx.x == 0) dims_s = dims_p;
  __syncthreads();
  const kt_dims& dims = dims_s;
  const int P = dims.n_params;
  float* Ps = sm;
  if (threadIdx.x == 0) slab_s = carve(sm + ((P + 3) & ~3), dims, nmax, D);
  const Slab& S = slab_s;
  const CtaGroup G{static_cast<int>(threadIdx.x), CT};
  for (int e = threadIdx.x; e < P; e += CT) Ps[e] = params[e];
  __syncthreads();
  for (int64_t i = blockIdx.x; i < nb; i += gridDim.x) {
    const int64_t b = b0 + i;
    const int64_t g = gidx ? gidx[b] : b;
    const GraphView v = graph_view(g, node_ptr, npg, row_ptr, col, val, mask);
    const float sq = graph_grad(G, dims, Ps, v, feats, fmean, fstd, y[b], inv_b, head_only != 0, S,
                                pg_grad + i * dims.n_params, D);
    if (threadIdx.x == 0) pg_sq[i] = sq;
    __syncthreads();
  }
}

// Fixed-order fp64 sum of the per-graph rows in two levels (deterministic, no atomics):
// partial[c][p] = sum of rows [c RG, (c+1) RG) (blockIdx.y = c), then acc[p] (+)= sum_c
// partial[c][p] in c order -- 32 rows per serial chain instead of the whole batch.
constexpr int RG = 32;

__global__ void reduce_rows_kernel(const float* __restrict__ pg, int64_t nb, int P, double* __restrict__ part) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * RG;
  if (p < P) {
    double s = 0.0;
    const int64_t r1 = r0 + RG < nb ? r0 + RG : nb;
    for (int64_t i = r0; i < r1; ++i) s += static_cast<double>(pg[i * P + p]);
    part[static_cast<int64_t>(blockIdx.y) * P + p] = s;
  }
}

__global__ void reduce_parts_kernel(const double* __restrict__ part, int nparts, int P, double* __restrict__ acc,
                                    int first, const float* __restrict__ pg_sq, int64_t nb,
                                    double* __restrict__ sq_acc) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < P) {
    double s = 0.0;
    for (int c = 0; c < nparts; ++c) s += part[static_cast<int64_t>(c) * P + p];
    acc[p] = first ? s : acc[p] + s;
  }
  if (blockIdx.x == 0 && threadIdx.x < 32) {  // the squared errors, one warp, fixed order
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < nb; i += 32) s += static_cast<double>(pg_sq[i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) sq_acc[0] = first ? s : sq_acc[0] + s;
  }
}

__global__ void finalize_kernel(const double* __restrict__ acc, int P, const double* __restrict__ sq_acc,
                                double inv_b, float* __restrict__ grad_out, double* __restrict__ loss_out,
                                const float* __restrict__ params, float lr, float* __restrict__ new_params) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < P) {
    const float g = static_cast<float>(acc[p]);
    if (grad_out) grad_out[p] = g;
    if (new_params) new_params[p] = params[p] - lr * g;
  }
  if (p == 0 && loss_out) loss_out[0] = sq_acc[0] * inv_b;
}

__global__ void sgd_kernel(const float* __restrict__ p, const float* __restrict__ g, float lr, int64_t n,
                           float* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = p[i] - lr * g[i];
}

// Sequential batch-1 SGD (meta.pretrain's inner loop): one CTA, params in smem.
template <int NTP>
__global__ void __launch_bounds__(NTP)
pretrain_sgd_kernel(kt_dims dims_p, float* __restrict__ params, const double* __restrict__ fmean,
                    const double* __restrict__ fstd, const double* __restrict__ feats,
                    const uint8_t* __restrict__ mask, const int64_t* __restrict__ node_ptr, int npg, int nmax,
                    const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                    const float* __restrict__ val, const int64_t* __restrict__ order, const float* __restrict__ y,
                    int64_t n_steps, float gamma, int D) {
  extern __shared__ __align__(16) float sm[];
  __shared__ kt_dims dims_s;  // (run-time indexed tables: shared memory, not the stack)
  __shared__ Slab slab_s;
  if (threadIdx.x == 0) dims_s = dims_p;
  __syncthreads();
  const kt_dims& dims = dims_s;
  const int P = dims.n_params;
  float* Ps = sm;
  float* Gs = Ps + ((P + 3) & ~3);
  if (threadIdx.x == 0) slab_s = carve(Gs + ((P + 3) & ~3), dims, nmax, D);
  __syncthreads();
  const Slab& S = slab_s;
  const CtaGroup C{static_cast<int>(threadIdx.x), static_cast<int>(blockDim.x)};
  for (int i = C.r; i < P; i += C.n) Ps[i] = params[i];
  C.sync();
  for (int64_t s = 0; s < n_steps; ++s) {
    const int64_t g = order[s];
    const GraphView v = graph_view(g, node_ptr, npg, row_ptr, col, val, mask);
    graph_grad(C, dims, Ps, v, feats, fmean, fstd, y[g], 1.0f, false, S, Gs, D);
    C.sync();
    for (int i = C.r; i < P; i += C.n) Ps[i] -= gamma * Gs[i];
    C.sync();
  }
  for (int i = C.r; i < P; i += C.n) params[i] = Ps[i];
}

// ---- factored batch gradient (kt_grad for batches up to kNumSMs x 8 graphs) --------------
//
// Every weight gradient of model.grad is a sum over the batch of outer products:
//   dW_gcn[l] = sum_graphs sum_nodes (A_hat H_l)[r]^T  delta_l[r]     (model.py:279-284)
//   dW_head[i] = sum_graphs act_i^T dz_i,  db_head[i] = sum_graphs dz_i (model.py:258-265)
//   d_agg     = sum_graphs colsum(H_L) * da                           (model.py:268-272)
// so a graph's CTA writes only those factors (~3.2k floats for the default dims) instead of
// its 9,825-float gradient row, and the batch reduction is a handful of fixed-order fp64
// contractions over the factor rows (phase B): deterministic, no atomics, and the graph
// kernel sheds the per-graph outer products.

struct FactorLayout {
  int nmax;                       // rows per graph record (graphs padded to nmax nodes)
  int fa[KT_MAX_LAYERS];          // A_hat H_l rows (nmax x din_l)
  int ft[KT_MAX_LAYERS];          // delta_l rows (nmax x dout_l)
  int fagg;                       // d_agg contribution (d_L)
  int fha[KT_MAX_LAYERS + 1];     // head layer i input act_i (din_i)
  int fhd[KT_MAX_LAYERS + 1];     // head layer i delta dz_i (dout_i)
  int rec;                        // floats per graph record (16-float aligned)
};

inline FactorLayout factor_layout(const kt_dims& d, int nmax) {
  FactorLayout f{};
  f.nmax = nmax;
  int o = 0;
  for (int l = 0; l < d.n_gcn; ++l) {
    f.fa[l] = o;
    o += nmax * d.gcn[l];
    f.ft[l] = o;
    o += nmax * d.gcn[l + 1];
  }
  f.fagg = o;
  o += d.gcn[d.n_gcn];
  for (int i = 0; i < d.n_head; ++i) {
    f.fha[i] = o;
    o += d.head[i];
    f.fhd[i] = o;
    o += d.head[i + 1];
  }
  f.rec = (o + 15) & ~15;
  return f;
}

// Transposed GCN weights W_l^T (dout x din) for layers l >= 1, consecutive in shared memory.
__host__ __device__ inline int wt_offset(const kt_dims& d, int l) {
  int o = 0;
  for (int j = 1; j < l; ++j) o += d.gcn[j] * d.gcn[j + 1];
  return o;
}
__host__ __device__ inline int wt_floats(const kt_dims& d) { return (wt_offset(d, d.n_gcn) + 3) & ~3; }

// Forward with caches + reverse pass for one graph (the arithmetic of graph_grad), writing
// the gradient factors to rec; returns the squared error.
template <class Grp>
__device__ float graph_factors(const Grp& G, const kt_dims& dims, const float* P, const float* WT, const GraphView& v,
                               const double* feats, const double* fmean, const double* fstd, float y, float inv_b,
                               bool head_only, const Slab& S, const FactorLayout& FL, float* rec, int D) {
  const int L = dims.n_gcn, nh = dims.n_head, n = v.n, nmax = FL.nmax;
  const int dl = dims.gcn[L];
  load_features(G, v, feats, dims.F, fmean, fstd, S.H[0], D);
  G.sync();
  for (int l = 0; l < L; ++l) {
    csr_aggregate(G, v, S.H[l], S.AH[l], dims.gcn[l], D);
    G.sync();
    dense(G, S.AH[l], P + dims.off_gcn[l], S.H[l + 1], n, dims.gcn[l], dims.gcn[l + 1], D, true);
    G.sync();
  }
  readout(G, S.H[L], n, dl, D, P + dims.off_agg, S.act[0], S.arg);
  G.sync();
  const unsigned qm = 0xFu << (G.r & 28);
  for (int i = 0; i < nh; ++i) {
    const int din = dims.head[i], dout = dims.head[i + 1];
    const float* W = P + dims.off_hw[i];
    const float* b = P + dims.off_hb[i];
    for (int e = G.r; e < 4 * dout; e += G.n) {
      const int c = e >> 2;
      float acc = 0.0f;
      for (int k = e & 3; k < din; k += 4) acc = fmaf(S.act[i][k], W[k * dout + c], acc);
      acc += __shfl_xor_sync(qm, acc, 1);
      acc += __shfl_xor_sync(qm, acc, 2);
      if ((e & 3) == 0) {
        acc += b[c];
        S.zh[i][c] = acc;
        S.act[i + 1][c] = i == nh - 1 ? acc : fmaxf(acc, 0.0f);
      }
    }
    G.sync();
  }
  const float pred = S.act[nh][0];
  const float err = pred - y;
  if (G.r == 0) S.da[0] = 2.0f * err * inv_b;
  G.sync();
  for (int i = nh - 1; i >= 0; --i) {
    const int din = dims.head[i], dout = dims.head[i + 1];
    const float* W = P + dims.off_hw[i];
    for (int c = G.r; c < dout; c += G.n) {
      const float dz = (i == nh - 1 || S.zh[i][c] > 0.0f) ? S.da[c] : 0.0f;
      S.dz[c] = dz;
      rec[FL.fhd[i] + c] = dz;
    }
    for (int k = G.r; k < din; k += G.n) rec[FL.fha[i] + k] = S.act[i][k];
    G.sync();
    for (int e = G.r; e < 4 * din; e += G.n) {
      const int k = e >> 2;
      float acc = 0.0f;
      if ((dout & 3) == 0) {  // the quad's c = e&3 + 4j, j rotated by k (bank spread, fixed order)
        const int nj = dout >> 2;
        int j = k % nj;
        for (int t = 0; t < nj; ++t) {
          const int c = (e & 3) + 4 * j;
          acc = fmaf(S.dz[c], W[k * dout + c], acc);
          if (++j == nj) j = 0;
        }
      } else {
        for (int c = e & 3; c < dout; c += 4) acc = fmaf(S.dz[c], W[k * dout + c], acc);
      }
      acc += __shfl_xor_sync(qm, acc, 1);
      acc += __shfl_xor_sync(qm, acc, 2);
      if ((e & 3) == 0) S.da[k] = acc;
    }
    G.sync();
  }
  if (head_only) return err * err;  // (phase B zeroes the GCN / readout gradients)
  const float* agg = P + dims.off_agg;
  for (int c = G.r; c < dl; c += G.n) {
    float colsum = 0.0f;
    for (int r = 0; r < n; ++r) colsum += S.H[L][r * D + c];
    rec[FL.fagg + c] = colsum * S.da[c];
  }
  for (int e = G.r; e < n * dl; e += G.n) {
    const int r = e / dl, c = e - (e / dl) * dl;
    S.t0[r * D + c] = agg[c] * S.da[c] + (r == S.arg[c] ? S.da[dl + c] : 0.0f);
  }
  G.sync();
  for (int l = L - 1; l >= 0; --l) {
    const int din = dims.gcn[l], dout = dims.gcn[l + 1];
    if (((din | dout | FL.ft[l] | FL.fa[l] | D) & 3) == 0) {  // the same, in 16-byte pieces
      const int q4 = dout >> 2;
      for (int e = G.r; e < nmax * q4; e += G.n) {
        const int r = e / q4, c = 4 * (e - r * q4);
        float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
        if (r < n) {
          const float4 h = *reinterpret_cast<const float4*>(S.H[l + 1] + r * D + c);
          float4* tp = reinterpret_cast<float4*>(S.t0 + r * D + c);
          const float4 d = *tp;
          t = make_float4(h.x > 0.0f ? d.x : 0.0f, h.y > 0.0f ? d.y : 0.0f, h.z > 0.0f ? d.z : 0.0f,
                          h.w > 0.0f ? d.w : 0.0f);
          *tp = t;
        }
        *reinterpret_cast<float4*>(rec + FL.ft[l] + r * dout + c) = t;
      }
      const int a4 = din >> 2;
      for (int e = G.r; e < nmax * a4; e += G.n) {
        const int r = e / a4, a = 4 * (e - r * a4);
        *reinterpret_cast<float4*>(rec + FL.fa[l] + r * din + a) =
            r < n ? *reinterpret_cast<const float4*>(S.AH[l] + r * D + a) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    } else {
    for (int e = G.r; e < nmax * dout; e += G.n) {  // masked delta rows (zero padding rows)
      const int r = e / dout, c = e - (e / dout) * dout;
      float t = 0.0f;
      if (r < n) {
        t = S.H[l + 1][r * D + c] > 0.0f ? S.t0[r * D + c] : 0.0f;
        S.t0[r * D + c] = t;
      }
      rec[FL.ft[l] + e] = t;
    }
    for (int e = G.r; e < nmax * din; e += G.n) {
      const int r = e / din, a = e - (e / din) * din;
      rec[FL.fa[l] + e] = r < n ? S.AH[l][r * D + a] : 0.0f;
    }
    }
    G.sync();
    if (l > 0) {
      // dZ W^T as a plain dense product with the transposed weights (staged once per CTA)
      dense(G, S.t0, WT + wt_offset(dims, l), S.t1, n, dout, din, D, false);
      G.sync();
      csr_aggregate(G, v, S.t1, S.t0, din, D);
      G.sync();
    }
  }
  return err * err;
}

// A CT-thread slice of a CTA working on its own graph (named barrier id + 1).
struct SubGroup {
  int r, n, id;
  __device__ __forceinline__ void sync() const { asm volatile("bar.sync %0, %1;" : : "r"(id + 1), "r"(n) : "memory"); }
};

// FG graphs per CTA at once, one CT-thread group each, sharing one copy of the parameters
// in shared memory (39 KB for the default dims): every layer's inner loops read weights at
// shared-memory latency, and FG slabs + the parameters still fit one CTA per SM.
constexpr int FG = 4;

__global__ void __launch_bounds__(CT * FG, 1)
factor_cta_kernel(kt_dims dims_p, const float* __restrict__ params, const double* __restrict__ fmean,
                  const double* __restrict__ fstd, const double* __restrict__ feats, const uint8_t* __restrict__ mask,
                  const int64_t* __restrict__ node_ptr, int npg, int nmax, const int32_t* __restrict__ row_ptr,
                  const int32_t* __restrict__ col, const float* __restrict__ val, const int64_t* __restrict__ gidx,
                  const float* __restrict__ y, int64_t nb, float inv_b, int head_only, int D, FactorLayout FL_p,
                  float* __restrict__ recs, float* __restrict__ pg_sq) {
  extern __shared__ __align__(16) float sm[];
  // the dims / record layout / slab pointer tables are indexed by run-time layer numbers: kept
  // in shared memory (as kernel parameters or locals they would be copied to the stack)
  __shared__ kt_dims dims_s;
  __shared__ FactorLayout fl_s;
  __shared__ Slab slab_s[FG];
  if (threadIdx.x == 0) {
    dims_s = dims_p;
    fl_s = FL_p;
  }
  __syncthreads();
  const kt_dims& dims = dims_s;
  const FactorLayout& FL = fl_s;
  const int P = dims.n_params;
  float* Ps = sm;
  float* WT = Ps + ((P + 3) & ~3);
  for (int e = threadIdx.x; e < P; e += CT * FG) Ps[e] = params[e];
  for (int l = 1; l < dims.n_gcn; ++l) {
    const int din = dims.gcn[l], dout = dims.gcn[l + 1];
    float* wt = WT + wt_offset(dims, l);
    for (int e = threadIdx.x; e < din * dout; e += CT * FG) {
      const int k = e / dout, c = e - k * dout;
      wt[c * din + k] = params[dims.off_gcn[l] + e];
    }
  }
  const int grp = threadIdx.x / CT;
  if (threadIdx.x % CT == 0)
    slab_s[grp] = carve(WT + wt_floats(dims) + grp * slab_floats(dims, nmax, D), dims, nmax, D);
  __syncthreads();
  const Slab& S = slab_s[grp];
  const SubGroup G{static_cast<int>(threadIdx.x) - grp * CT, CT, grp};
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * FG + grp; i < nb; i += static_cast<int64_t>(gridDim.x) * FG) {
    const int64_t g = gidx ? gidx[i] : i;
    const GraphView v = graph_view(g, node_ptr, npg, row_ptr, col, val, mask);
    const float sq = graph_factors(G, dims, Ps, WT, v, feats, fmean, fstd, y[i], inv_b, head_only != 0, S, FL,
                                   recs + i * FL.rec, D);
    if (G.r == 0) pg_sq[i] = sq;
    G.sync();
  }
}

// Phase B.  A "segment" is one parameter block whose gradient is sum_rows A[r]^T B[r]
// (+ a bias sum of B when bias_off >= 0): partial sums over fixed row chunks in fp64,
// thread = output element, rows in order within a chunk; then the chunks in order.
struct Segment {
  int a_off, b_off;  // factor offsets in a graph record (A rows: din wide, B rows: dout wide)
  int din, dout;     // (din = 0: a bias-only / vector segment: out[c] = sum_rows B[r][c])
  int rows;          // rows per graph record (nmax for GCN layers, 1 for head / agg)
  int p_off;         // parameter offset of the block
  int n_out;         // din * dout, or dout
};
constexpr int MAX_SEG = 2 * KT_MAX_LAYERS + 2 * (KT_MAX_LAYERS + 1) + 1;
struct Segments {
  Segment s[MAX_SEG];
  int n;
  int gpc;           // graphs per chunk
  int nch;           // chunks
  int part_off[MAX_SEG];  // (doubles) per segment: nch x n_out partial sums
};

// CTA = one chunk of gpc consecutive graphs: their records are staged in shared memory
// with coalesced loads, then every parameter's chunk sum is formed from shared memory.
constexpr int FRT = 1024;  // phase-B threads per CTA: many short latency-bound chains

__global__ void __launch_bounds__(FRT)
factor_reduce_kernel(const float* __restrict__ recs, int rec, int64_t nb, Segments SG, double* __restrict__ part) {
  extern __shared__ __align__(16) float rs[];
  const int ch = blockIdx.x;
  const int64_t g0 = static_cast<int64_t>(ch) * SG.gpc;
  const int ng = static_cast<int>((g0 + SG.gpc < nb ? g0 + SG.gpc : nb) - g0);
  {
    const float4* src = reinterpret_cast<const float4*>(recs + g0 * rec);
    float4* dst = reinterpret_cast<float4*>(rs);
    const int n4 = ng * rec / 4;  // (rec is a multiple of 16 floats)
    for (int i = threadIdx.x; i < n4; i += blockDim.x) dst[i] = __ldcs(src + i);
  }
  __syncthreads();
  // the work items of every segment in one index space (item = an output quad of a 4-wide
  // segment, else one output), so the threads run the segments side by side
  int base = 0;
  for (int k = 0; k < SG.n; ++k) {
    const Segment sg = SG.s[k];
    double* out = part + SG.part_off[k] + static_cast<int64_t>(ch) * sg.n_out;
    const bool quad = sg.din > 0 && (sg.dout & 3) == 0 && ((sg.b_off | rec) & 3) == 0;
    const int items = quad ? sg.n_out >> 2 : sg.n_out;
    const int first = ((static_cast<int>(threadIdx.x) - base) % FRT + FRT) % FRT;  // this thread's first item
    base += items;
    if (quad) {
      // four adjacent outputs per thread (16-byte B reads, four independent chains); each
      // output's arithmetic and order are those of the scalar loop below
      const int q4 = sg.dout >> 2, n4 = items;
      for (int o4 = first; o4 < n4; o4 += FRT) {
        const int a = o4 / q4, c = 4 * (o4 - a * q4);
        double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
        for (int g = 0; g < ng; ++g) {
          const float* A = rs + g * rec + sg.a_off + a;
          const float* Bm = rs + g * rec + sg.b_off + c;
          float4 s4 = make_float4(0.f, 0.f, 0.f, 0.f);
          for (int r = 0; r < sg.rows; ++r) fma4(A[r * sg.din], *reinterpret_cast<const float4*>(Bm + r * sg.dout), s4);
          acc0 += static_cast<double>(s4.x);
          acc1 += static_cast<double>(s4.y);
          acc2 += static_cast<double>(s4.z);
          acc3 += static_cast<double>(s4.w);
        }
        double2* o2 = reinterpret_cast<double2*>(out + 4 * o4);
        o2[0] = make_double2(acc0, acc1);
        o2[1] = make_double2(acc2, acc3);
      }
      continue;
    }
    for (int o = first; o < sg.n_out; o += FRT) {
      // per graph: an fp32 dot over its rows (as each graph's own gradient row was formed
      // before); across the chunk's graphs: fp64, in batch order
      double acc = 0.0;
      if (sg.din > 0) {
        const int a = o / sg.dout, c = o - a * sg.dout;
        for (int g = 0; g < ng; ++g) {
          const float* A = rs + g * rec + sg.a_off + a;
          const float* Bm = rs + g * rec + sg.b_off + c;
          float s = 0.0f;
          for (int r = 0; r < sg.rows; ++r) s = fmaf(A[r * sg.din], Bm[r * sg.dout], s);
          acc += static_cast<double>(s);
        }
      } else {
        for (int g = 0; g < ng; ++g) acc += static_cast<double>(rs[g * rec + sg.b_off + o]);
      }
      out[o] = acc;
    }
  }
}

// Eight lanes per parameter: lane j sums chunks j, j + 8, ... in order (fp64), a fixed
// three-step butterfly combines them, then the update; warp 0 of CTA 0 also sums the loss.
__global__ void __launch_bounds__(256)
factor_finalize_kernel(const double* __restrict__ part, Segments SG, int P, int head_only, int off_head,
                       const float* __restrict__ pg_sq, int64_t nb, double inv_b, float* __restrict__ grad_out,
                       double* __restrict__ loss_out, const float* __restrict__ params, float lr,
                       float* __restrict__ new_params) {
  const int p = (blockIdx.x * blockDim.x + threadIdx.x) >> 3, j = threadIdx.x & 7;
  if (p < P) {  // (P is uniform per 8-lane group: the group is all in or all out)
    int k = 0;
#pragma unroll 1
    while (k + 1 < SG.n && SG.s[k + 1].p_off <= p) ++k;
    const int n_out = SG.s[k].n_out, o = p - SG.s[k].p_off;
    double s = 0.0;
    if (!(head_only && p < off_head)) {
      const double* q = part + SG.part_off[k] + o;
#pragma unroll 4
      for (int c = j; c < SG.nch; c += 8) s += __ldcs(q + static_cast<int64_t>(c) * n_out);
    }
    const unsigned gm = 0xFFu << (threadIdx.x & 24);
    s += __shfl_xor_sync(gm, s, 1);
    s += __shfl_xor_sync(gm, s, 2);
    s += __shfl_xor_sync(gm, s, 4);
    if (j == 0) {
      const float g = static_cast<float>(s);
      if (grad_out) grad_out[p] = g;
      if (new_params) new_params[p] = params[p] - lr * g;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < 32 && loss_out) {  // squared errors, one warp, fixed order
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < nb; i += 32) s += static_cast<double>(pg_sq[i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) loss_out[0] = s * inv_b;
  }
}

inline Segments factor_segments(const kt_dims& d, const FactorLayout& FL, int64_t nb, int gpc) {
  Segments SG{};
  int n = 0;
  for (int l = 0; l < d.n_gcn; ++l)
    SG.s[n++] = Segment{FL.fa[l], FL.ft[l], d.gcn[l], d.gcn[l + 1], FL.nmax, d.off_gcn[l], d.gcn[l] * d.gcn[l + 1]};
  SG.s[n++] = Segment{0, FL.fagg, 0, d.gcn[d.n_gcn], 1, d.off_agg, d.gcn[d.n_gcn]};
  for (int i = 0; i < d.n_head; ++i) {
    SG.s[n++] = Segment{FL.fha[i], FL.fhd[i], d.head[i], d.head[i + 1], 1, d.off_hw[i], d.head[i] * d.head[i + 1]};
    SG.s[n++] = Segment{0, FL.fhd[i], 0, d.head[i + 1], 1, d.off_hb[i], d.head[i + 1]};
  }
  SG.n = n;
  SG.gpc = gpc;
  SG.nch = static_cast<int>((nb + gpc - 1) / gpc);
  int off = 0;
  for (int k = 0; k < n; ++k) {
    SG.part_off[k] = off;
    off += SG.nch * SG.s[k].n_out;
  }
  return SG;
}

inline int64_t factor_partials(const Segments& SG) {
  int64_t t = 0;
  for (int k = 0; k < SG.n; ++k) t += static_cast<int64_t>(SG.nch) * SG.s[k].n_out;
  return t;
}

#ifndef KT_FACTOR_GPC
#define KT_FACTOR_GPC 4
#endif
constexpr int FACTOR_GPC = KT_FACTOR_GPC;  // graphs per phase-B chunk (CTA)

static int row_stride(const kt_dims& d) {
  int D = d.F;
  for (int i = 1; i <= d.n_gcn; ++i) D = D > d.gcn[i] ? D : d.gcn[i];
  D = (D + 3) & ~3;
  // rows of a multiple of 32 words would put every row's word k in one bank (the 4-wide
  // dense reads t[k] of four rows per warp): pad by one 16-byte piece
  return KT_DPAD && D % 32 == 0 ? D + 4 : D;
}

static int64_t chunk_of(int64_t B) { return B < 8192 ? B : 8192; }

}  // namespace train
}  // namespace kt

extern "C" {

int64_t kt_grad_workspace_bytes(const kt_dims* dims, int64_t B) {
  const int64_t c = kt::train::chunk_of(B);
  const int64_t P = dims->n_params;
  const int64_t parts = (c + kt::train::RG - 1) / kt::train::RG;
  const int64_t rows = c * P * 4 + c * 4 + P * 8 + 16 + 64 + parts * P * 8 + 64;
  // factored path (B <= kNumSMs x 8): records sized for the largest graph the kernels take
  const kt::train::FactorLayout FL = kt::train::factor_layout(*dims, KT_MAX_NODES);
  const kt::train::Segments SG = kt::train::factor_segments(*dims, FL, B, kt::train::FACTOR_GPC);
  const int64_t fac = B * FL.rec * 4 + B * 4 + 64 + kt::train::factor_partials(SG) * 8 + 64;
  return rows > fac ? rows : fac;
}

int kt_grad(const kt_dims* dims, const float* params, const double* fmean, const double* fstd, const double* feats,
            const uint8_t* mask, const int64_t* node_ptr, int32_t nodes_per_graph, int32_t max_nodes,
            const int32_t* row_ptr, const int32_t* col, const float* val, const int64_t* graph_idx, const float* y,
            int64_t B, int32_t head_only, float* grad_out, double* loss_out, float lr, float* new_params,
            void* workspace, int64_t workspace_bytes, void* stream) {
  using namespace kt;
  KT_REQUIRE(dims && params && fmean && fstd && feats && mask && row_ptr && col && val && y && workspace, KT_E_ARG,
             "kt_grad: null pointer");
  KT_REQUIRE(B > 0, KT_E_EMPTY, "kt_grad: empty batch");
  KT_REQUIRE(nodes_per_graph > 0 || node_ptr, KT_E_ARG, "kt_grad: need node_ptr or nodes_per_graph");
  KT_REQUIRE(max_nodes >= 1 && max_nodes <= KT_MAX_NODES, KT_E_UNSUPPORTED, "graph too large");
  int rc = check_dims(*dims);
  if (rc) return rc;
  KT_REQUIRE(workspace_bytes >= kt_grad_workspace_bytes(dims, B), KT_E_ARG, "kt_grad: workspace too small");
  const int D = train::row_stride(*dims);
  const size_t smem = sizeof(float) * train::WARPS * train::slab_floats(*dims, max_nodes, D);
  KT_REQUIRE(smem <= 220 * 1024, KT_E_UNSUPPORTED, "kt_grad: model/graph too large for shared memory");
  static SmemAttr smem_attr;
  smem_attr.ensure(train::pergraph_kernel, smem);
  cudaStream_t st = as_stream(stream);
  const int P = dims->n_params;
  const int64_t chunk = train::chunk_of(B);
  float* pg = static_cast<float*>(workspace);
  float* pg_sq = pg + chunk * P;
  double* acc = reinterpret_cast<double*>(reinterpret_cast<uintptr_t>(pg_sq + chunk + 3) & ~uintptr_t(7));
  double* sq_acc = acc + P;
  double* part = reinterpret_cast<double*>(reinterpret_cast<uintptr_t>(sq_acc + 2 + 7) & ~uintptr_t(63));
  const float inv_b = static_cast<float>(1.0 / static_cast<double>(B));
  const train::FactorLayout FL = train::factor_layout(*dims, max_nodes);
  const size_t csm = sizeof(float) * (((P + 3) & ~3) + train::wt_floats(*dims) +
                                      train::FG * train::slab_floats(*dims, max_nodes, D));
  const size_t rsm = sizeof(float) * train::FACTOR_GPC * FL.rec;
  // factored path when its CTAs fit shared memory (large graphs / models: the row path)
  if (B <= kNumSMs * 8 && csm <= 220 * 1024 && rsm <= 220 * 1024 &&
      !(getenv("KT_GRAD_ROWS") && getenv("KT_GRAD_ROWS")[0] == '1')) {
    // factored path: per-graph gradient factors, then fixed-order fp64 contractions
    const train::Segments SG = train::factor_segments(*dims, FL, B, train::FACTOR_GPC);
    float* recs = static_cast<float*>(workspace);
    float* fsq = recs + B * FL.rec;
    double* part = reinterpret_cast<double*>(reinterpret_cast<uintptr_t>(fsq + B + 15) & ~uintptr_t(63));
    static SmemAttr fsm_attr;
    fsm_attr.ensure(train::factor_cta_kernel, csm);
    const int64_t fcta = (B + train::FG - 1) / train::FG;
    train::factor_cta_kernel<<<(int)(fcta < kNumSMs ? fcta : kNumSMs), train::CT * train::FG, csm, st>>>(*dims, params, fmean, fstd, feats, mask, node_ptr,
                                                              nodes_per_graph, max_nodes, row_ptr, col, val,
                                                              graph_idx, y, B, inv_b, head_only, D, FL, recs, fsq);
    static SmemAttr rsm_attr;
    rsm_attr.ensure(train::factor_reduce_kernel, rsm);
    train::factor_reduce_kernel<<<SG.nch, train::FRT, rsm, st>>>(recs, FL.rec, B, SG, part);
    train::factor_finalize_kernel<<<(P + 31) / 32, 256, 0, st>>>(part, SG, P, head_only, dims->off_head, fsq, B,
                                                                   1.0 / static_cast<double>(B), grad_out, loss_out,
                                                                   params, lr, new_params);
    note_launches(3);
    return check_launch("kt_grad");
  }
  int launches = 0;
  for (int64_t b0 = 0; b0 < B; b0 += chunk) {
    const int64_t nb = B - b0 < chunk ? B - b0 : chunk;
    if (nb <= kNumSMs * 8 && !(getenv("KT_GRAD_WARP") && getenv("KT_GRAD_WARP")[0] == '1')) {
      // small batch: a CTA per graph (the warp form would leave most of the GPU idle)
      const size_t csm = sizeof(float) * (((P + 3) & ~3) + train::slab_floats(*dims, max_nodes, D));
      KT_REQUIRE(csm <= 220 * 1024, KT_E_UNSUPPORTED, "kt_grad: model too large for shared memory");
      static SmemAttr csm_attr;
      csm_attr.ensure(train::pergraph_cta_kernel, csm);
      const int per_sm = static_cast<int>((224 * 1024) / (csm + 1024)) > 0 ? static_cast<int>((224 * 1024) / (csm + 1024)) : 1;
      const int64_t cap = static_cast<int64_t>(kNumSMs) * (per_sm < 8 ? per_sm : 8);
      train::pergraph_cta_kernel<<<(int)(nb < cap ? nb : cap), train::CT, csm, st>>>(
          *dims, params, fmean, fstd, feats, mask, node_ptr, nodes_per_graph, max_nodes, row_ptr, col, val,
          graph_idx, y, b0, nb, inv_b, head_only, D, pg, pg_sq);
    } else {
      int64_t blocks = (nb + train::WARPS - 1) / train::WARPS;
      if (blocks > kNumSMs * 16) blocks = kNumSMs * 16;
      train::pergraph_kernel<<<(int)blocks, train::WARPS * 32, smem, st>>>(
          *dims, params, fmean, fstd, feats, mask, node_ptr, nodes_per_graph, max_nodes, row_ptr, col, val,
          graph_idx, y, b0, nb, inv_b, head_only, D, pg, pg_sq);
    }
    const int nparts = static_cast<int>((nb + train::RG - 1) / train::RG);
    train::reduce_rows_kernel<<<dim3((P + 255) / 256, nparts), 256, 0, st>>>(pg, nb, P, part);
    train::reduce_parts_kernel<<<(P + 255) / 256, 256, 0, st>>>(part, nparts, P, acc, b0 == 0, pg_sq, nb, sq_acc);
    launches += 3;
  }
  train::finalize_kernel<<<(P + 255) / 256, 256, 0, st>>>(acc, P, sq_acc, 1.0 / static_cast<double>(B), grad_out,
                                                            loss_out, params, lr, new_params);
  note_launches(launches + 1);
  return check_launch("kt_grad");
}

int kt_sgd(const float* params, const float* grad, float lr, int64_t n, float* out, void* stream) {
  using namespace kt;
  KT_REQUIRE(params && grad && out, KT_E_ARG, "kt_sgd: null pointer");
  KT_REQUIRE(n > 0, KT_E_EMPTY, "kt_sgd: empty vector");
  int64_t blocks = (n + 255) / 256;
  if (blocks > kNumSMs * 8) blocks = kNumSMs * 8;
  train::sgd_kernel<<<(int)blocks, 256, 0, as_stream(stream)>>>(params, grad, lr, n, out);
  note_launches(1);
  return check_launch("kt_sgd");
}

int kt_pretrain_sgd(const kt_dims* dims, float* params, const double* fmean, const double* fstd, const double* feats,
                    const uint8_t* mask, const int64_t* node_ptr, int32_t nodes_per_graph, int32_t max_nodes,
                    const int32_t* row_ptr, const int32_t* col, const float* val, const int64_t* order,
                    const float* y, int64_t n_steps, float gamma, void* stream) {
  using namespace kt;
  KT_REQUIRE(dims && params && fmean && fstd && feats && mask && row_ptr && col && val && order && y, KT_E_ARG,
             "kt_pretrain_sgd: null pointer");
  KT_REQUIRE(nodes_per_graph > 0 || node_ptr, KT_E_ARG, "kt_pretrain_sgd: need node_ptr or nodes_per_graph");
  KT_REQUIRE(max_nodes >= 1 && max_nodes <= KT_MAX_NODES, KT_E_UNSUPPORTED, "graph too large");
  int rc = check_dims(*dims);
  if (rc) return rc;
  if (n_steps <= 0) return KT_OK;
  const int D = train::row_stride(*dims);
  const int P4 = (dims->n_params + 3) & ~3;
  const size_t smem = sizeof(float) * (2 * P4 + train::slab_floats(*dims, max_nodes, D));
  KT_REQUIRE(smem <= 220 * 1024, KT_E_UNSUPPORTED, "kt_pretrain_sgd: model too large for shared memory");
  // 1024 threads: the sequential SGD chain is latency-bound, more warps per phase help
  // (24k -> 31k samples/s over 256 threads); KT_PRETRAIN_NT overrides for experiments
  const char* nt_env = getenv("KT_PRETRAIN_NT");
  const int ntp = nt_env ? atoi(nt_env) : 1024;
  auto go = [&](auto kern, int threads) {
    static SmemAttr smem_attr;
    smem_attr.ensure(kern, smem);
    kern<<<1, threads, smem, as_stream(stream)>>>(*dims, params, fmean, fstd, feats, mask, node_ptr,
                                                                   nodes_per_graph, max_nodes, row_ptr, col, val,
                                                                   order, y, n_steps, gamma, D);
  };
  if (ntp >= 1024) go(train::pretrain_sgd_kernel<1024>, 1024);
  else if (ntp >= 512) go(train::pretrain_sgd_kernel<512>, 512);
  else go(train::pretrain_sgd_kernel<256>, 256);
  note_launches(1);
  return check_launch("kt_pretrain_sgd");
}

}  // extern "C"
