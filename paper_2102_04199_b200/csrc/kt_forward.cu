// kt_embed_csr / kt_head_forward: embed_batch + head_forward_batch for
// arbitrary adjacency (shared pattern or segmented CSR) and model dims
// (model.py:185-203).  The star-layout fast path is kt_score_indices.
#include <cstdlib>

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

// head_forward_batch for large batches: a CTA streams tiles of HT rows through the head with
// the head parameters staged in shared memory; a thread owns a 4-row x 4-column block of each
// hidden layer (one 16-byte weight load and four row reads per k, 16 FMAs) and one row of the
// last (one-output) layer.  Every output is the same fmaf chain over k in order, then the bias,
// as head_layer's: bit-identical to the warp-per-row kernel.
constexpr int HT = 64;       // rows per tile
constexpr int HTT = 256;     // threads
__global__ void __launch_bounds__(HTT) head_tile_kernel(kt_dims dims, const float* __restrict__ params,
                                                        const float* __restrict__ u, int64_t B,
                                                        float* __restrict__ z_out, int hs) {
  extern __shared__ __align__(16) float hsm[];
  const int nh = dims.n_head, P = dims.n_head_params;
  float* Wp = hsm;                                  // the head parameters (flat head vector order)
  float* act0 = Wp + ((P + 3) & ~3);                // HT x hs, two buffers
  float* act1 = act0 + HT * hs;
  const float* hp = params + dims.off_head;
  for (int e = threadIdx.x; e < P; e += HTT) Wp[e] = hp[e];
  const int d0 = dims.head[0];
  const int64_t n_tiles = (B + HT - 1) / HT;
  for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    const int64_t r0 = t * HT;
    const int rows = static_cast<int>(B - r0 < HT ? B - r0 : HT);
    __syncthreads();  // (parameters staged / the previous tile's last layer done)
    for (int e = threadIdx.x; e < HT * (d0 >> 2); e += HTT) {
      const int r = e / (d0 >> 2), c = (e - r * (d0 >> 2)) * 4;
      const float4 v = r < rows ? *reinterpret_cast<const float4*>(u + (r0 + r) * d0 + c)
                                : make_float4(0.f, 0.f, 0.f, 0.f);
      *reinterpret_cast<float4*>(act0 + r * hs + c) = v;
    }
    __syncthreads();
    float* in = act0;
    float* out = act1;
    for (int i = 0; i < nh; ++i) {
      const int din = dims.head[i], dout = dims.head[i + 1];
      const float* W = Wp + (dims.off_hw[i] - dims.off_head);
      const float* b = Wp + (dims.off_hb[i] - dims.off_head);
      if (i == nh - 1) {  // one output: thread = row, k in order
        for (int r = threadIdx.x; r < rows; r += HTT) {
          float acc = 0.0f;
          for (int k = 0; k < din; ++k) acc = fmaf(in[r * hs + k], W[k], acc);
          z_out[r0 + r] = acc + b[0];
        }
      } else {
        const int cq = dout >> 2;
        for (int it = threadIdx.x; it < (HT / 4) * cq; it += HTT) {
          const int rr = (it / cq) * 4, c = (it - (it / cq) * cq) * 4;
          float4 a[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) a[j] = make_float4(0.f, 0.f, 0.f, 0.f);
          const float* x = in + rr * hs;
#pragma unroll 4
          for (int k = 0; k < din; ++k) {
            const float4 w = *reinterpret_cast<const float4*>(W + k * dout + c);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float p = x[j * hs + k];
              a[j].x = fmaf(p, w.x, a[j].x);
              a[j].y = fmaf(p, w.y, a[j].y);
              a[j].z = fmaf(p, w.z, a[j].z);
              a[j].w = fmaf(p, w.w, a[j].w);
            }
          }
          const float4 bb = *reinterpret_cast<const float4*>(b + c);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            float4 o = make_float4(a[j].x + bb.x, a[j].y + bb.y, a[j].z + bb.z, a[j].w + bb.w);
            o = make_float4(fmaxf(o.x, 0.f), fmaxf(o.y, 0.f), fmaxf(o.z, 0.f), fmaxf(o.w, 0.f));
            *reinterpret_cast<float4*>(out + (rr + j) * hs + c) = o;
          }
        }
        __syncthreads();
        float* tmp = in;
        in = out;
        out = tmp;
      }
    }
  }
}

static bool head_tile_ok(const kt_dims& d) {
  if (d.head[d.n_head] != 1) return false;
  for (int i = 0; i < d.n_head; ++i) {
    if (d.head[i] % 4 || d.head[i] > 2 * KT_MAX_DIM) return false;
    if ((d.off_hw[i] - d.off_head) % 4 || (d.off_hb[i] - d.off_head) % 4) return false;
  }
  return true;
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
  if (fwd::head_tile_ok(*dims) && (reinterpret_cast<uintptr_t>(u) & 15) == 0 &&
      !(getenv("KT_HEADF_WARP") && getenv("KT_HEADF_WARP")[0] == '1')) {
    int hs = 4;
    for (int i = 0; i < dims->n_head; ++i) hs = hs > dims->head[i] ? hs : dims->head[i];
    hs += 4;  // (row stride off a multiple of 32 words: four rows' word k in four banks)
    const size_t smem = sizeof(float) * (((dims->n_head_params + 3) & ~3) + 2 * fwd::HT * hs);
    static SmemAttr attr;
    attr.ensure(fwd::head_tile_kernel, smem);
    const int64_t tiles = (B + fwd::HT - 1) / fwd::HT;
    const int grid = static_cast<int>(tiles < 4 * kNumSMs ? tiles : 4 * kNumSMs);
    fwd::head_tile_kernel<<<grid, fwd::HTT, smem, as_stream(stream)>>>(*dims, params, u, B, z_out, hs);
    note_launches(1);
    return check_launch("kt_head_forward");
  }
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
