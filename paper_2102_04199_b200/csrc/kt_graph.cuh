// Warp-per-graph building blocks for general (non-star) graphs and arbitrary
// model dims: normalisation, CSR aggregation, dense transform + ReLU, readout,
// head forward.  Shared by the general forward, training and MAML kernels.
//
// A warp owns one graph; its activations live in that warp's shared-memory
// slab with row stride D (>= every layer width).  Lanes stride over feature
// columns, so CSR neighbour gathers read whole rows conflict-free and weight
// reads (W[k][c], lanes on c) are coalesced and L1-resident.
#pragma once

#include "kt_common.cuh"

namespace kt {

struct GraphView {
  int n;                 // nodes in this graph
  int64_t node0;         // first global node id
  const int32_t* row_ptr;
  const int32_t* col;
  const float* val;
  int64_t rp_base;       // row_ptr index of local row 0
  int64_t col_base;      // node id subtracted from col entries
  const uint8_t* mask;   // mask of local row 0
};

__device__ __forceinline__ GraphView graph_view(int64_t g, const int64_t* node_ptr, int npg,
                                                const int32_t* row_ptr, const int32_t* col,
                                                const float* val, const uint8_t* mask) {
  GraphView v;
  if (npg > 0) {
    v.n = npg;
    v.node0 = g * npg;
    v.rp_base = 0;
    v.col_base = 0;
    v.mask = mask;
  } else {
    v.node0 = node_ptr[g];
    v.n = static_cast<int>(node_ptr[g + 1] - v.node0);
    v.rp_base = v.node0;
    v.col_base = v.node0;
    v.mask = mask + v.node0;
  }
  v.row_ptr = row_ptr;
  v.col = col;
  v.val = val;
  return v;
}

// X (n x F) <- normalised raw features of the graph's masked rows, zero elsewhere.
__device__ __forceinline__ void load_features(const GraphView& v, const double* feats, int F,
                                              const double* fmean, const double* fstd, float* X, int D,
                                              int lane) {
  for (int e = lane; e < v.n * F; e += 32) {
    const int r = e / F, f = e - (e / F) * F;
    float x = 0.0f;
    if (v.mask[r]) x = static_cast<float>((feats[(v.node0 + r) * F + f] - fmean[f]) / fstd[f]);
    X[r * D + f] = x;
  }
}

// T (n x din) <- A_hat H
__device__ __forceinline__ void csr_aggregate(const GraphView& v, const float* Hs, float* Ts, int din, int D,
                                              int lane) {
  for (int r = 0; r < v.n; ++r) {
    const int64_t b = v.row_ptr[v.rp_base + r], e = v.row_ptr[v.rp_base + r + 1];
    for (int c = lane; c < din; c += 32) {
      float acc = 0.0f;
      for (int64_t q = b; q < e; ++q) acc = fmaf(v.val[q], Hs[(v.col[q] - v.col_base) * D + c], acc);
      Ts[r * D + c] = acc;
    }
  }
}

// Out (n x dout) <- T W (+ optional ReLU); W row-major (din x dout) in global memory.
__device__ __forceinline__ void dense(const float* Ts, const float* __restrict__ W, float* Out, int n, int din,
                                      int dout, int D, bool relu_out, int lane) {
  for (int c = lane; c < dout; c += 32) {
    for (int r = 0; r < n; ++r) {
      float acc = 0.0f;
      for (int k = 0; k < din; ++k) acc = fmaf(Ts[r * D + k], __ldg(W + k * dout + c), acc);
      Out[r * D + c] = relu_out ? fmaxf(acc, 0.0f) : acc;
    }
  }
}

// u = [sum_n a_c H[n][c], max_n H[n][c]]  (model.py:136-141 / 192-194)
__device__ __forceinline__ void readout(const float* Hs, int n, int d, int D, const float* __restrict__ agg,
                                       float* u, int lane) {
  for (int c = lane; c < d; c += 32) {
    const float a = __ldg(agg + c);
    float s = 0.0f, m = -INFINITY;
    for (int r = 0; r < n; ++r) {
      const float h = Hs[r * D + c];
      s += h * a;
      m = fmaxf(m, h);
    }
    u[c] = s;
    u[d + c] = m;
  }
}

// Head forward of one row vector a (len dims.head[0]) using two ping-pong
// buffers of >= KT_MAX_DIM floats; returns the scalar output.
__device__ __forceinline__ float head_row(const kt_dims& dims, const float* __restrict__ params, float* a,
                                          float* tmp, int lane) {
  float* in = a;
  float* out = tmp;
  for (int i = 0; i < dims.n_head; ++i) {
    const int din = dims.head[i], dout = dims.head[i + 1];
    const float* W = params + dims.off_hw[i];
    const float* b = params + dims.off_hb[i];
    const bool last = i == dims.n_head - 1;
    __syncwarp();
    for (int c = lane; c < dout; c += 32) {
      float acc = 0.0f;
      for (int k = 0; k < din; ++k) acc = fmaf(in[k], __ldg(W + k * dout + c), acc);
      acc += __ldg(b + c);
      out[c] = last ? acc : fmaxf(acc, 0.0f);
    }
    __syncwarp();
    float* t = in; in = out; out = t;
  }
  return in[0];
}

}  // namespace kt
