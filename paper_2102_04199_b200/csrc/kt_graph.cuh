// Thread-group building blocks for general (non-star) graphs and arbitrary
// model dims: normalisation, CSR aggregation, dense transform + ReLU, readout,
// head forward, and the reverse-mode pieces of model.grad (model.py:218-285).
//
// A group (one warp, or a whole CTA for the sequential-SGD kernel) owns one
// graph; its activations live in the group's shared-memory slab with row
// stride D (>= every layer width).  Threads stride over feature columns, so CSR
// neighbour gathers read whole rows conflict-free and weight reads W[k][c]
// (threads on c) are coalesced and L1-resident.
#pragma once

#include "kt_common.cuh"

#ifndef KT_VEC_CSR
#define KT_VEC_CSR 1
#endif
#ifndef KT_VEC_DENSE
#define KT_VEC_DENSE 1
#endif
#ifndef KT_DPAD
#define KT_DPAD 1
#endif

namespace kt {

struct WarpGroup {
  int r;  // rank in group
  static constexpr int n = 32;
  __device__ __forceinline__ void sync() const { __syncwarp(); }
};

struct CtaGroup {
  int r, n;
  __device__ __forceinline__ void sync() const { __syncthreads(); }
};

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

// X (n x F) <- normalised raw features of the graph's masked rows, zero elsewhere (model.py:108-112).
template <class Grp>
__device__ __forceinline__ void load_features(const Grp& G, const GraphView& v, const double* feats, int F,
                                              const double* fmean, const double* fstd, float* X, int D) {
  for (int e = G.r; e < v.n * F; e += G.n) {
    const int r = e / F, f = e - (e / F) * F;
    float x = 0.0f;
    if (v.mask[r]) x = static_cast<float>((feats[(v.node0 + r) * F + f] - fmean[f]) / fstd[f]);
    X[r * D + f] = x;
  }
}

__device__ __forceinline__ bool aligned16(const void* a, const void* b) {
  return ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15) == 0;
}
__device__ __forceinline__ void fma4(float w, const float4& x, float4& acc) {
  acc.x = fmaf(w, x.x, acc.x);
  acc.y = fmaf(w, x.y, acc.y);
  acc.z = fmaf(w, x.z, acc.z);
  acc.w = fmaf(w, x.w, acc.w);
}

// T (n x din) <- A_hat H   (A_hat symmetric, so A_hat^T products use the same routine)
// Width a multiple of 4: a thread owns a channel quad (16-byte row pieces, the CSR entries
// read once per quad); the per-channel edge order is the same either way.
template <class Grp>
__device__ __forceinline__ void csr_aggregate(const Grp& G, const GraphView& v, const float* Hs, float* Ts,
                                              int din, int D) {
  if (KT_VEC_CSR && (din & 3) == 0 && (D & 3) == 0 && aligned16(Hs, Ts)) {
    const int q4 = din >> 2;
    for (int e = G.r; e < v.n * q4; e += G.n) {
      const int r = e / q4, c = 4 * (e - r * q4);
      const int64_t b = v.row_ptr[v.rp_base + r], end = v.row_ptr[v.rp_base + r + 1];
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int64_t q = b; q < end; ++q)
        fma4(v.val[q], *reinterpret_cast<const float4*>(Hs + (v.col[q] - v.col_base) * D + c), acc);
      *reinterpret_cast<float4*>(Ts + r * D + c) = acc;
    }
    return;
  }
  for (int e = G.r; e < v.n * din; e += G.n) {
    const int r = e / din, c = e - (e / din) * din;
    const int64_t b = v.row_ptr[v.rp_base + r], end = v.row_ptr[v.rp_base + r + 1];
    float acc = 0.0f;
    for (int64_t q = b; q < end; ++q) acc = fmaf(v.val[q], Hs[(v.col[q] - v.col_base) * D + c], acc);
    Ts[r * D + c] = acc;
  }
}

// Out (n x dout) <- T W (+ optional ReLU); W row-major (din x dout).  Width a multiple of 4:
// a thread owns four adjacent outputs of a row (one 16-byte W load per k, k order unchanged).
template <class Grp>
__device__ __forceinline__ void dense(const Grp& G, const float* Ts, const float* __restrict__ W, float* Out, int n,
                                      int din, int dout, int D, bool relu_out) {
  if (KT_VEC_DENSE && (dout & 3) == 0 && (D & 3) == 0 && aligned16(W, Out)) {
    const int q4 = dout >> 2;
    for (int e = G.r; e < n * q4; e += G.n) {
      const int r = e / q4, c = 4 * (e - r * q4);
      const float* t = Ts + r * D;
      const float* w = W + c;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int k = 0; k < din; ++k) fma4(t[k], *reinterpret_cast<const float4*>(w + k * dout), acc);
      if (relu_out) acc = make_float4(fmaxf(acc.x, 0.f), fmaxf(acc.y, 0.f), fmaxf(acc.z, 0.f), fmaxf(acc.w, 0.f));
      *reinterpret_cast<float4*>(Out + r * D + c) = acc;
    }
    return;
  }
  for (int e = G.r; e < n * dout; e += G.n) {
    const int r = e / dout, c = e - (e / dout) * dout;
    float acc = 0.0f;
    for (int k = 0; k < din; ++k) acc = fmaf(Ts[r * D + k], W[k * dout + c], acc);
    Out[r * D + c] = relu_out ? fmaxf(acc, 0.0f) : acc;
  }
}

// Out (n x din) <- dZ W^T   (W is din x dout).  Lanes of a warp own consecutive k, so a
// plain c loop would read W[k dout + c] with a stride of dout words -- one shared-memory
// bank for the whole warp when W sits in shared memory; each output instead starts its
// (fixed-order) sum at c = k mod dout, which spreads the lanes over the banks.
template <class Grp>
__device__ __forceinline__ void dense_t(const Grp& G, const float* dZ, const float* __restrict__ W, float* Out,
                                        int n, int din, int dout, int D) {
  for (int e = G.r; e < n * din; e += G.n) {
    const int r = e / din, k = e - (e / din) * din;
    float acc = 0.0f;
    int c = k % dout;
    for (int j = 0; j < dout; ++j) {
      acc = fmaf(dZ[r * D + c], W[k * dout + c], acc);
      if (++c == dout) c = 0;
    }
    Out[r * D + k] = acc;
  }
}

// u = [sum_n a_c H[n][c], max_n H[n][c]]  (model.py:136-141 / 192-194); arg[c] = first argmax
template <class Grp>
__device__ __forceinline__ void readout(const Grp& G, const float* Hs, int n, int d, int D,
                                       const float* __restrict__ agg, float* u, int* arg) {
  for (int c = G.r; c < d; c += G.n) {
    const float a = agg[c];
    float s = 0.0f, m = -INFINITY;
    int am = 0;
    for (int r = 0; r < n; ++r) {
      const float h = Hs[r * D + c];
      s += h * a;
      if (h > m) { m = h; am = r; }
    }
    u[c] = s;
    u[d + c] = m;
    if (arg) arg[c] = am;
  }
}

// One affine head layer: out = in W + b (+ReLU unless last); W (din x dout) at params+off_w.
template <class Grp>
__device__ __forceinline__ void head_layer(const Grp& G, const float* in, const float* __restrict__ W,
                                           const float* __restrict__ b, float* out, int din, int dout, bool relu_out) {
  for (int c = G.r; c < dout; c += G.n) {
    float acc = 0.0f;
    for (int k = 0; k < din; ++k) acc = fmaf(in[k], W[k * dout + c], acc);
    acc += b[c];
    out[c] = relu_out ? fmaxf(acc, 0.0f) : acc;
  }
}

// Head forward of one row vector a (len dims.head[0]) using two ping-pong
// buffers of >= 2*KT_MAX_DIM floats; returns the scalar output.
template <class Grp>
__device__ __forceinline__ float head_row(const Grp& G, const kt_dims& dims, const float* __restrict__ params,
                                          float* a, float* tmp) {
  float* in = a;
  float* out = tmp;
  for (int i = 0; i < dims.n_head; ++i) {
    G.sync();
    head_layer(G, in, params + dims.off_hw[i], params + dims.off_hb[i], out, dims.head[i], dims.head[i + 1],
               i != dims.n_head - 1);
    G.sync();
    float* t = in; in = out; out = t;
  }
  return in[0];
}

// Backwards compatible warp helpers (lane-based) used by the forward kernels.
__device__ __forceinline__ WarpGroup warp_group(int lane) { return WarpGroup{lane}; }

}  // namespace kt
