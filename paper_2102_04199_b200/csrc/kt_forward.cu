// kt_embed_csr / kt_head_forward: embed_batch + head_forward_batch for
// arbitrary adjacency (shared pattern or segmented CSR) and model dims
// (model.py:185-203).  The star-layout fast path is kt_score_indices.
#include "kt_graph.cuh"

namespace kt {
namespace fwd {

constexpr int WARPS = 4;

__global__ void __launch_bounds__(WARPS * 32)
embed_kernel(kt_dims dims, const float* __restrict__ params, const double* __restrict__ fmean,
             const double* __restrict__ fstd, const double* __restrict__ feats, const uint8_t* __restrict__ mask,
             const int64_t* __restrict__ node_ptr, int npg, int max_nodes, const int32_t* __restrict__ row_ptr,
             const int32_t* __restrict__ col, const float* __restrict__ val, const int64_t* __restrict__ gidx,
             int64_t B, int D, float* __restrict__ u_out, float* __restrict__ z_out) {
  extern __shared__ __align__(16) float sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slab = 2 * max_nodes * D + 2 * 2 * KT_MAX_DIM;
  float* A = sm + warp * slab;
  float* Bf = A + max_nodes * D;
  float* h0 = Bf + max_nodes * D;
  float* h1 = h0 + 2 * KT_MAX_DIM;
  const int dl = dims.gcn[dims.n_gcn];
  const WarpGroup W{lane};
  for (int64_t g = static_cast<int64_t>(blockIdx.x) * WARPS + warp; g < B;
       g += static_cast<int64_t>(gridDim.x) * WARPS) {
    const GraphView v = graph_view(gidx ? gidx[g] : g, node_ptr, npg, row_ptr, col, val, mask);
    load_features(W, v, feats, dims.F, fmean, fstd, A, D);
    W.sync();
    for (int l = 0; l < dims.n_gcn; ++l) {
      csr_aggregate(W, v, A, Bf, dims.gcn[l], D);
      W.sync();
      dense(W, Bf, params + dims.off_gcn[l], A, v.n, dims.gcn[l], dims.gcn[l + 1], D, true);
      W.sync();
    }
    readout(W, A, v.n, dl, D, params + dims.off_agg, h0, static_cast<int*>(nullptr));
    W.sync();
    for (int c = lane; c < 2 * dl; c += 32) u_out[g * 2 * dl + c] = h0[c];
    if (z_out) {
      const float z = head_row(W, dims, params, h0, h1);
      if (lane == 0) z_out[g] = z;
    }
    W.sync();
  }
}

// Small batches (the single-graph API path, model.py:153-169): one CTA per graph so
// each output element of a layer gets its own thread.  Same per-element operation
// order as embed_kernel, so the two agree bit for bit.
constexpr int CTA_THREADS = 256;

__global__ void __launch_bounds__(CTA_THREADS)
embed_cta_kernel(kt_dims dims, const float* __restrict__ params, const double* __restrict__ fmean,
                 const double* __restrict__ fstd, const double* __restrict__ feats, const uint8_t* __restrict__ mask,
                 const int64_t* __restrict__ node_ptr, int npg, int max_nodes, const int32_t* __restrict__ row_ptr,
                 const int32_t* __restrict__ col, const float* __restrict__ val, const int64_t* __restrict__ gidx,
                 int64_t B, int D, float* __restrict__ u_out, float* __restrict__ z_out) {
  extern __shared__ __align__(16) float sm[];
  float* A = sm;
  float* Bf = A + max_nodes * D;
  float* h0 = Bf + max_nodes * D;
  float* h1 = h0 + 2 * KT_MAX_DIM;
  const int dl = dims.gcn[dims.n_gcn];
  const CtaGroup G{static_cast<int>(threadIdx.x), CTA_THREADS};
  for (int64_t g = blockIdx.x; g < B; g += gridDim.x) {
    const GraphView v = graph_view(gidx ? gidx[g] : g, node_ptr, npg, row_ptr, col, val, mask);
    load_features(G, v, feats, dims.F, fmean, fstd, A, D);
    G.sync();
    for (int l = 0; l < dims.n_gcn; ++l) {
      csr_aggregate(G, v, A, Bf, dims.gcn[l], D);
      G.sync();
      dense(G, Bf, params + dims.off_gcn[l], A, v.n, dims.gcn[l], dims.gcn[l + 1], D, true);
      G.sync();
    }
    readout(G, A, v.n, dl, D, params + dims.off_agg, h0, static_cast<int*>(nullptr));
    G.sync();
    for (int c = G.r; c < 2 * dl; c += G.n) u_out[g * 2 * dl + c] = h0[c];
    if (z_out) {
      const float z = head_row(G, dims, params, h0, h1);
      if (G.r == 0) z_out[g] = z;
    }
    G.sync();
  }
}

__global__ void __launch_bounds__(WARPS * 32)
head_kernel(kt_dims dims, const float* __restrict__ params, const float* __restrict__ u, int64_t B,
            float* __restrict__ z_out) {
  __shared__ float buf[WARPS][2][KT_MAX_DIM * 2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int d0 = dims.head[0];
  for (int64_t g = static_cast<int64_t>(blockIdx.x) * WARPS + warp; g < B;
       g += static_cast<int64_t>(gridDim.x) * WARPS) {
    for (int c = lane; c < d0; c += 32) buf[warp][0][c] = u[g * d0 + c];
    __syncwarp();
    const float z = head_row(WarpGroup{lane}, dims, params, buf[warp][0], buf[warp][1]);
    if (lane == 0) z_out[g] = z;
    __syncwarp();
  }
}

}  // namespace fwd

int check_dims(const kt_dims& d) {
  KT_REQUIRE(d.n_gcn >= 1 && d.n_gcn <= KT_MAX_LAYERS && d.n_head >= 1 && d.n_head <= KT_MAX_LAYERS + 1,
             KT_E_UNSUPPORTED, "model depth beyond compiled limits");
  for (int i = 0; i <= d.n_gcn; ++i)
    KT_REQUIRE(d.gcn[i] >= 1 && d.gcn[i] <= KT_MAX_DIM, KT_E_UNSUPPORTED, "GCN width %d beyond %d", d.gcn[i],
               KT_MAX_DIM);
  for (int i = 0; i <= d.n_head; ++i)
    KT_REQUIRE(d.head[i] >= 1 && d.head[i] <= 2 * KT_MAX_DIM, KT_E_UNSUPPORTED, "head width %d beyond %d",
               d.head[i], 2 * KT_MAX_DIM);
  KT_REQUIRE(d.head[d.n_head] == 1, KT_E_SHAPE, "head must end in one output");
  return KT_OK;
}

}  // namespace kt

extern "C" {

int kt_embed_csr(const kt_dims* dims, const float* params, const double* fmean, const double* fstd,
                 const double* feats, const uint8_t* mask, const int64_t* node_ptr, int32_t nodes_per_graph,
                 int32_t max_nodes, const int32_t* row_ptr, const int32_t* col, const float* val,
                 const int64_t* graph_idx, int64_t B, float* u_out, float* z_out, void* stream) {
  using namespace kt;
  KT_REQUIRE(dims && params && fmean && fstd && feats && mask && row_ptr && col && val && u_out, KT_E_ARG,
             "kt_embed_csr: null pointer");
  KT_REQUIRE(B > 0, KT_E_EMPTY, "kt_embed_csr: empty batch");
  KT_REQUIRE(nodes_per_graph > 0 || node_ptr, KT_E_ARG, "kt_embed_csr: need node_ptr or nodes_per_graph");
  KT_REQUIRE(max_nodes >= 1 && max_nodes <= KT_MAX_NODES, KT_E_UNSUPPORTED, "graph of %d nodes beyond %d",
             max_nodes, KT_MAX_NODES);
  int rc = check_dims(*dims);
  if (rc) return rc;
  int D = dims->F;
  for (int i = 1; i <= dims->n_gcn; ++i) D = D > dims->gcn[i] ? D : dims->gcn[i];
  D = (D + 3) & ~3;
  if (D % 32 == 0) D += 4;  // (bank spread for the 4-wide dense, as kt_grad's row_stride)
  if (B <= kNumSMs) {
    const size_t smem1 = sizeof(float) * (2 * max_nodes * D + 4 * KT_MAX_DIM);
    static SmemAttr attr1;
    attr1.ensure(fwd::embed_cta_kernel, smem1);
    fwd::embed_cta_kernel<<<(int)B, fwd::CTA_THREADS, smem1, as_stream(stream)>>>(
        *dims, params, fmean, fstd, feats, mask, node_ptr, nodes_per_graph, max_nodes, row_ptr, col, val, graph_idx,
        B, D, u_out, z_out);
    note_launches(1);
    return check_launch("kt_embed_csr");
  }
  const size_t smem = sizeof(float) * fwd::WARPS * (2 * max_nodes * D + 4 * KT_MAX_DIM);
  static SmemAttr attr;
  attr.ensure(fwd::embed_kernel, smem);
#ifndef KT_EMB_BPS
#define KT_EMB_BPS 64  // grid-stride CTAs per SM (8: 12.5 ms per 1M graphs, 64: 10.0 ms)
#endif
  int64_t blocks = (B + fwd::WARPS - 1) / fwd::WARPS;
  if (blocks > kNumSMs * KT_EMB_BPS) blocks = kNumSMs * KT_EMB_BPS;
  fwd::embed_kernel<<<(int)blocks, fwd::WARPS * 32, smem, as_stream(stream)>>>(
      *dims, params, fmean, fstd, feats, mask, node_ptr, nodes_per_graph, max_nodes, row_ptr, col, val, graph_idx,
      B, D, u_out, z_out);
  note_launches(1);
  return check_launch("kt_embed_csr");
}

int kt_head_forward(const kt_dims* dims, const float* params, const float* u, int64_t B, float* z_out,
                    void* stream) {
  using namespace kt;
  KT_REQUIRE(dims && params && u && z_out, KT_E_ARG, "kt_head_forward: null pointer");
  KT_REQUIRE(B > 0, KT_E_EMPTY, "kt_head_forward: empty batch");
  int rc = check_dims(*dims);
  if (rc) return rc;
#ifndef KT_HEADF_BPS
#define KT_HEADF_BPS 64  // (8: 4.2 ms per 1M rows, 64: 3.7 ms)
#endif
  int64_t blocks = (B + fwd::WARPS - 1) / fwd::WARPS;
  if (blocks > kNumSMs * KT_HEADF_BPS) blocks = kNumSMs * KT_HEADF_BPS;
  fwd::head_kernel<<<(int)blocks, fwd::WARPS * 32, 0, as_stream(stream)>>>(*dims, params, u, B, z_out);
  note_launches(1);
  return check_launch("kt_head_forward");
}

}  // extern "C"
