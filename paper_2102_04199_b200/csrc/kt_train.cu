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
pergraph_kernel(kt_dims dims, const float* __restrict__ params, const double* __restrict__ fmean,
                const double* __restrict__ fstd, const double* __restrict__ feats, const uint8_t* __restrict__ mask,
                const int64_t* __restrict__ node_ptr, int npg, int nmax, const int32_t* __restrict__ row_ptr,
                const int32_t* __restrict__ col, const float* __restrict__ val, const int64_t* __restrict__ gidx,
                const float* __restrict__ y, int64_t b0, int64_t nb, float inv_b, int head_only, int D,
                float* __restrict__ pg_grad, float* __restrict__ pg_sq) {
  extern __shared__ __align__(16) float sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const Slab S = carve(sm + warp * slab_floats(dims, nmax, D), dims, nmax, D);
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
// loop), spread over 8x the threads, so a 512-graph batch fills the GPU.
#ifndef KT_GRAD_CT
#define KT_GRAD_CT 256
#endif
constexpr int CT = KT_GRAD_CT;

__global__ void __launch_bounds__(CT)
pergraph_cta_kernel(kt_dims dims, const float* __restrict__ params, const double* __restrict__ fmean,
                    const double* __restrict__ fstd, const double* __restrict__ feats,
                    const uint8_t* __restrict__ mask, const int64_t* __restrict__ node_ptr, int npg, int nmax,
                    const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                    const float* __restrict__ val, const int64_t* __restrict__ gidx, const float* __restrict__ y,
                    int64_t b0, int64_t nb, float inv_b, int head_only, int D, float* __restrict__ pg_grad,
                    float* __restrict__ pg_sq) {
  extern __shared__ __align__(16) float sm[];
  const Slab S = carve(sm, dims, nmax, D);
  const CtaGroup G{static_cast<int>(threadIdx.x), CT};
  for (int64_t i = blockIdx.x; i < nb; i += gridDim.x) {
    const int64_t b = b0 + i;
    const int64_t g = gidx ? gidx[b] : b;
    const GraphView v = graph_view(g, node_ptr, npg, row_ptr, col, val, mask);
    const float sq = graph_grad(G, dims, params, v, feats, fmean, fstd, y[b], inv_b, head_only != 0, S,
                                pg_grad + i * dims.n_params, D);
    if (threadIdx.x == 0) pg_sq[i] = sq;
    __syncthreads();
  }
}

// acc[p] (+)= sum_i pg[i][p] in fixed order, fp64
__global__ void reduce_kernel(const float* __restrict__ pg, int64_t nb, int P, double* __restrict__ acc, int first,
                              const float* __restrict__ pg_sq, double* __restrict__ sq_acc) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < P) {
    double s = 0.0;
    for (int64_t i = 0; i < nb; ++i) s += static_cast<double>(pg[i * P + p]);
    acc[p] = first ? s : acc[p] + s;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double s = 0.0;
    for (int64_t i = 0; i < nb; ++i) s += static_cast<double>(pg_sq[i]);
    sq_acc[0] = first ? s : sq_acc[0] + s;
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
pretrain_sgd_kernel(kt_dims dims, float* __restrict__ params, const double* __restrict__ fmean,
                    const double* __restrict__ fstd, const double* __restrict__ feats,
                    const uint8_t* __restrict__ mask, const int64_t* __restrict__ node_ptr, int npg, int nmax,
                    const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                    const float* __restrict__ val, const int64_t* __restrict__ order, const float* __restrict__ y,
                    int64_t n_steps, float gamma, int D) {
  extern __shared__ __align__(16) float sm[];
  const int P = dims.n_params;
  float* Ps = sm;
  float* Gs = Ps + ((P + 3) & ~3);
  const Slab S = carve(Gs + ((P + 3) & ~3), dims, nmax, D);
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

static int row_stride(const kt_dims& d) {
  int D = d.F;
  for (int i = 1; i <= d.n_gcn; ++i) D = D > d.gcn[i] ? D : d.gcn[i];
  return (D + 3) & ~3;
}

static int64_t chunk_of(int64_t B) { return B < 8192 ? B : 8192; }

}  // namespace train
}  // namespace kt

extern "C" {

int64_t kt_grad_workspace_bytes(const kt_dims* dims, int64_t B) {
  const int64_t c = kt::train::chunk_of(B);
  const int64_t P = dims->n_params;
  return c * P * 4 + c * 4 + P * 8 + 16 + 64;
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
  const float inv_b = static_cast<float>(1.0 / static_cast<double>(B));
  int launches = 0;
  for (int64_t b0 = 0; b0 < B; b0 += chunk) {
    const int64_t nb = B - b0 < chunk ? B - b0 : chunk;
    if (nb <= kNumSMs * 8 && !(getenv("KT_GRAD_WARP") && getenv("KT_GRAD_WARP")[0] == '1')) {
      // small batch: a CTA per graph (the warp form would leave most of the GPU idle)
      const size_t csm = sizeof(float) * train::slab_floats(*dims, max_nodes, D);
      static SmemAttr csm_attr;
      csm_attr.ensure(train::pergraph_cta_kernel, csm);
      train::pergraph_cta_kernel<<<(int)nb, train::CT, csm, st>>>(
          *dims, params, fmean, fstd, feats, mask, node_ptr, nodes_per_graph, max_nodes, row_ptr, col, val,
          graph_idx, y, b0, nb, inv_b, head_only, D, pg, pg_sq);
    } else {
      int64_t blocks = (nb + train::WARPS - 1) / train::WARPS;
      if (blocks > kNumSMs * 16) blocks = kNumSMs * 16;
      train::pergraph_kernel<<<(int)blocks, train::WARPS * 32, smem, st>>>(
          *dims, params, fmean, fstd, feats, mask, node_ptr, nodes_per_graph, max_nodes, row_ptr, col, val,
          graph_idx, y, b0, nb, inv_b, head_only, D, pg, pg_sq);
    }
    train::reduce_kernel<<<(P + 255) / 256, 256, 0, st>>>(pg, nb, P, acc, b0 == 0, pg_sq, sq_acc);
    launches += 2;
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
