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
#include "kt_graph.cuh"

namespace kt {

int check_dims(const kt_dims& d);

namespace meta {

constexpr int NT = 256;
constexpr int RC = 8;               // rows per chunk
constexpr int HMAX = 2 * KT_MAX_DIM; // widest head vector (input 2 d_L)

struct Head {
  int nh;
  int dim[KT_MAX_LAYERS + 2];
  int ow[KT_MAX_LAYERS + 1], ob[KT_MAX_LAYERS + 1];  // offsets into the flat head vector
  int P;
};

__host__ __device__ inline Head head_of(const kt_dims& d) {
  Head h;
  h.nh = d.n_head;
  for (int i = 0; i <= d.n_head; ++i) h.dim[i] = d.head[i];
  for (int i = 0; i < d.n_head; ++i) {
    h.ow[i] = d.off_hw[i] - d.off_head;
    h.ob[i] = d.off_hb[i] - d.off_head;
  }
  h.P = d.n_head_params;
  return h;
}

// Row-chunk scratch: activations A[0..nh], pre-activations Z[0..nh-1], tangents,
// deltas -- each RC x HMAX.
struct Scratch {
  float* A[KT_MAX_LAYERS + 2];
  float* Z[KT_MAX_LAYERS + 1];
  float* TA[KT_MAX_LAYERS + 2];  // forward tangents (HVP only)
  float* D0;
  float* D1;
  float* TD0;
  float* TD1;
  float* red;  // NT floats for block reductions
};

__host__ __device__ inline int scratch_floats(int nh, bool hvp) {
  return ((nh + 1) + nh + (hvp ? nh + 1 : 0) + (hvp ? 4 : 2)) * RC * HMAX + NT;
}

__device__ inline Scratch carve(float* p, int nh, bool hvp) {
  Scratch s;
  for (int i = 0; i <= nh; ++i) { s.A[i] = p; p += RC * HMAX; }
  for (int i = 0; i < nh; ++i) { s.Z[i] = p; p += RC * HMAX; }
  if (hvp)
    for (int i = 0; i <= nh; ++i) { s.TA[i] = p; p += RC * HMAX; }
  s.D0 = p; p += RC * HMAX;
  s.D1 = p; p += RC * HMAX;
  if (hvp) {
    s.TD0 = p; p += RC * HMAX;
    s.TD1 = p; p += RC * HMAX;
  } else {
    s.TD0 = s.TD1 = nullptr;
  }
  s.red = p;
  return s;
}

__device__ __forceinline__ float block_sum(float v, float* red) {
  red[threadIdx.x] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    float s = 0.0f;
    for (int i = 0; i < NT; ++i) s += red[i];  // fixed order
    red[0] = s;
  }
  __syncthreads();
  const float s = red[0];
  __syncthreads();
  return s;
}

// Loads rows [r0, r0+nr) (gathered through ridx when given) into A[0].
__device__ __forceinline__ void load_rows(const Head& h, const float* u, const int64_t* ridx, int r0, int nr,
                                          float* A0) {
  const int d0 = h.dim[0];
  for (int e = threadIdx.x; e < nr * d0; e += NT) {
    const int r = e / d0, c = e - (e / d0) * d0;
    const int64_t row = ridx ? ridx[r0 + r] : r0 + r;
    A0[r * HMAX + c] = u[row * d0 + c];
  }
}

// grad (and mse) of the head MSE at theta over n rows; if v != nullptr computes
// the Hessian-vector product H(theta) v instead (forward-over-reverse, ReLU masks
// constant).  out (h.P floats, smem) is overwritten.  Returns the mse.
__device__ float head_pass(const Head& h, const float* th, const float* v, const float* u, const int64_t* ridx,
                           const float* y, const int64_t* yidx, int n, float* out, const Scratch& S) {
  const int nh = h.nh;
  const bool hvp = v != nullptr;
  for (int e = threadIdx.x; e < h.P; e += NT) out[e] = 0.0f;
  float sq_local = 0.0f;
  const float two_n = 2.0f / static_cast<float>(n);
  for (int r0 = 0; r0 < n; r0 += RC) {
    const int nr = n - r0 < RC ? n - r0 : RC;
    __syncthreads();
    load_rows(h, u, ridx, r0, nr, S.A[0]);
    if (hvp)
      for (int e = threadIdx.x; e < nr * h.dim[0]; e += NT) {
        const int r = e / h.dim[0], c = e - (e / h.dim[0]) * h.dim[0];
        S.TA[0][r * HMAX + c] = 0.0f;
      }
    __syncthreads();
    // forward
    for (int i = 0; i < nh; ++i) {
      const int din = h.dim[i], dout = h.dim[i + 1];
      const float* W = th + h.ow[i];
      const float* b = th + h.ob[i];
      const bool last = i == nh - 1;
      for (int e = threadIdx.x; e < nr * dout; e += NT) {
        const int r = e / dout, c = e - (e / dout) * dout;
        float acc = 0.0f;
        for (int k = 0; k < din; ++k) acc = fmaf(S.A[i][r * HMAX + k], W[k * dout + c], acc);
        acc += b[c];
        S.Z[i][r * HMAX + c] = acc;
        S.A[i + 1][r * HMAX + c] = last ? acc : fmaxf(acc, 0.0f);
        if (hvp) {
          const float* vW = v + h.ow[i];
          float t = v[h.ob[i] + c];
          for (int k = 0; k < din; ++k) {
            t = fmaf(S.TA[i][r * HMAX + k], W[k * dout + c], t);
            t = fmaf(S.A[i][r * HMAX + k], vW[k * dout + c], t);
          }
          S.TA[i + 1][r * HMAX + c] = (last || acc > 0.0f) ? t : 0.0f;
        }
      }
      __syncthreads();
    }
    // output deltas (model.py:382-383 / 422-423)
    for (int r = threadIdx.x; r < nr; r += NT) {
      const float yy = yidx ? y[yidx[r0 + r]] : y[r0 + r];
      const float resid = S.A[nh][r * HMAX] - yy;
      sq_local += resid * resid;
      S.D0[r * HMAX] = two_n * resid;
      if (hvp) S.TD0[r * HMAX] = two_n * S.TA[nh][r * HMAX];
    }
    __syncthreads();
    // backward
    float* da = S.D0;
    float* dn = S.D1;
    float* tda = S.TD0;
    float* tdn = S.TD1;
    for (int i = nh - 1; i >= 0; --i) {
      const int din = h.dim[i], dout = h.dim[i + 1];
      const bool last = i == nh - 1;
      // mask deltas in place: dz = da * (z > 0) (not on the linear output layer)
      if (!last) {
        for (int e = threadIdx.x; e < nr * dout; e += NT) {
          const int r = e / dout, c = e - (e / dout) * dout;
          if (!(S.Z[i][r * HMAX + c] > 0.0f)) {
            da[r * HMAX + c] = 0.0f;
            if (hvp) tda[r * HMAX + c] = 0.0f;
          }
        }
        __syncthreads();
      }
      // parameter gradient: out_w += A^T dz (grad) or TA^T dz + A^T tdz (hvp); out_b += sum dz / tdz
      float* gw = out + h.ow[i];
      for (int e = threadIdx.x; e < din * dout; e += NT) {
        const int k = e / dout, c = e - (e / dout) * dout;
        float acc = gw[e];
        for (int r = 0; r < nr; ++r) {
          if (hvp)
            acc = fmaf(S.TA[i][r * HMAX + k], da[r * HMAX + c], fmaf(S.A[i][r * HMAX + k], tda[r * HMAX + c], acc));
          else
            acc = fmaf(S.A[i][r * HMAX + k], da[r * HMAX + c], acc);
        }
        gw[e] = acc;
      }
      for (int c = threadIdx.x; c < dout; c += NT) {
        float acc = out[h.ob[i] + c];
        for (int r = 0; r < nr; ++r) acc += hvp ? tda[r * HMAX + c] : da[r * HMAX + c];
        out[h.ob[i] + c] = acc;
      }
      // propagate: da' = dz W^T ; tda' = tdz W^T + dz vW^T
      if (i > 0) {
        const float* W = th + h.ow[i];
        for (int e = threadIdx.x; e < nr * din; e += NT) {
          const int r = e / din, k = e - (e / din) * din;
          float acc = 0.0f, tacc = 0.0f;
          for (int c = 0; c < dout; ++c) {
            acc = fmaf(da[r * HMAX + c], W[k * dout + c], acc);
            if (hvp)
              tacc = fmaf(tda[r * HMAX + c], W[k * dout + c], fmaf(da[r * HMAX + c], v[h.ow[i] + k * dout + c], tacc));
          }
          dn[r * HMAX + k] = acc;
          if (hvp) tdn[r * HMAX + k] = tacc;
        }
      }
      __syncthreads();
      float* t = da; da = dn; dn = t;
      t = tda; tda = tdn; tdn = t;
    }
  }
  const float sq = block_sum(sq_local, S.red);
  return sq / static_cast<float>(n);
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
maml_task_kernel(kt_dims dims, const float* __restrict__ theta, TaskSet ts, int T, float alpha, int inner_steps,
                 int first_order, float* __restrict__ theta_ws, float* __restrict__ g_out,
                 float* __restrict__ loss_out) {
  extern __shared__ __align__(16) float sm[];
  const Head h = head_of(dims);
  const int P4 = (h.P + 3) & ~3;
  float* th = sm;             // current theta_k
  float* th1 = th + P4;       // next theta / theta_0 for HVP
  float* gb = th1 + P4;       // support gradient / HVP output
  float* vb = gb + P4;        // query gradient v
  const Scratch S = carve(vb + P4, h.nh, !first_order);
  const int t = blockIdx.x;
  if (t >= T) return;
  const int64_t s0 = ts.s_off[t], ns = ts.s_off[t + 1] - s0;
  const int64_t q0 = ts.q_off[t], nq = ts.q_off[t + 1] - q0;
  for (int e = threadIdx.x; e < h.P; e += NT) th[e] = theta[e];
  __syncthreads();
  float ls0 = 0.0f;
  float* cur = th;
  float* nxt = th1;
  for (int k = 0; k < inner_steps; ++k) {
    if (!first_order && inner_steps > 1)
      for (int e = threadIdx.x; e < h.P; e += NT) theta_ws[(static_cast<int64_t>(t) * inner_steps + k) * h.P + e] = cur[e];
    const float ls = head_pass(h, cur, nullptr, ts.u, ts.s_idx + s0, ts.y, ts.s_idx + s0, static_cast<int>(ns), gb, S);
    if (k == 0) ls0 = ls;
    __syncthreads();
    for (int e = threadIdx.x; e < h.P; e += NT) nxt[e] = cur[e] - alpha * gb[e];
    __syncthreads();
    float* tmp = cur; cur = nxt; nxt = tmp;
  }
  const float lq = head_pass(h, cur, nullptr, ts.u, ts.q_idx + q0, ts.y, ts.q_idx + q0, static_cast<int>(nq), vb, S);
  __syncthreads();
  if (!first_order) {
    for (int k = inner_steps - 1; k >= 0; --k) {
      // theta_k -> nxt
      for (int e = threadIdx.x; e < h.P; e += NT)
        nxt[e] = inner_steps > 1 ? theta_ws[(static_cast<int64_t>(t) * inner_steps + k) * h.P + e] : theta[e];
      __syncthreads();
      head_pass(h, nxt, vb, ts.u, ts.s_idx + s0, ts.y, ts.s_idx + s0, static_cast<int>(ns), gb, S);
      __syncthreads();
      for (int e = threadIdx.x; e < h.P; e += NT) vb[e] -= alpha * gb[e];
      __syncthreads();
    }
  }
  for (int e = threadIdx.x; e < h.P; e += NT) g_out[static_cast<int64_t>(t) * h.P + e] = vb[e];
  if (threadIdx.x == 0) {
    loss_out[2 * t] = ls0;
    loss_out[2 * t + 1] = lq;
  }
}

// sum_out[p] = sum_t g[t][p] (fixed order, fp64 accumulate); stats = (sum ls, sum lq)
__global__ void task_sum_kernel(const float* __restrict__ g, int T, int P, float* __restrict__ sum_out,
                                const float* __restrict__ losses, double* __restrict__ stats) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < P) {
    double s = 0.0;
    for (int t = 0; t < T; ++t) s += static_cast<double>(g[static_cast<int64_t>(t) * P + p]);
    sum_out[p] = static_cast<float>(s);
  }
  if (stats && blockIdx.x == 0 && threadIdx.x < 2) {
    double s = 0.0;
    for (int t = 0; t < T; ++t) s += static_cast<double>(losses[2 * t + threadIdx.x]);
    stats[threadIdx.x] = s;
  }
}

// head_loss_grad / head_hvp / fine-tune: one CTA on one theta.
__global__ void __launch_bounds__(NT)
head_kernel(kt_dims dims, const float* __restrict__ theta, const float* __restrict__ v, const float* __restrict__ u,
            const float* __restrict__ y, int n, int steps, float alpha, float* __restrict__ out,
            float* __restrict__ mse_out) {
  extern __shared__ __align__(16) float sm[];
  const Head h = head_of(dims);
  const int P4 = (h.P + 3) & ~3;
  float* th = sm;
  float* gb = th + P4;
  float* vb = gb + P4;
  const bool hvp = v != nullptr;
  const Scratch S = carve(vb + P4, h.nh, hvp);
  for (int e = threadIdx.x; e < h.P; e += NT) {
    th[e] = theta[e];
    if (hvp) vb[e] = v[e];
  }
  __syncthreads();
  if (steps <= 0) {  // single evaluation: grad (or hvp) -> out
    const float mse = head_pass(h, th, hvp ? vb : nullptr, u, nullptr, y, nullptr, n, gb, S);
    __syncthreads();
    for (int e = threadIdx.x; e < h.P; e += NT) out[e] = gb[e];
    if (threadIdx.x == 0 && mse_out) mse_out[0] = mse;
    return;
  }
  for (int s = 0; s < steps; ++s) {  // fine_tune_embedded: theta -= alpha * grad, `steps` times
    const float mse = head_pass(h, th, nullptr, u, nullptr, y, nullptr, n, gb, S);
    __syncthreads();
    for (int e = threadIdx.x; e < h.P; e += NT) th[e] -= alpha * gb[e];
    if (threadIdx.x == 0 && mse_out) mse_out[s] = mse;
    __syncthreads();
  }
  for (int e = threadIdx.x; e < h.P; e += NT) out[e] = th[e];
}

static size_t task_smem(const Head& h, bool so) { return sizeof(float) * (4 * ((h.P + 3) & ~3) + scratch_floats(h.nh, so)); }
static size_t head_smem(const Head& h, bool hvp) { return sizeof(float) * (3 * ((h.P + 3) & ~3) + scratch_floats(h.nh, hvp)); }

static int check_head(const kt_dims& d) {
  KT_REQUIRE(d.n_head >= 1 && d.n_head <= KT_MAX_LAYERS + 1, KT_E_UNSUPPORTED, "head depth beyond limits");
  for (int i = 0; i <= d.n_head; ++i)
    KT_REQUIRE(d.head[i] >= 1 && d.head[i] <= HMAX, KT_E_UNSUPPORTED, "head width %d beyond %d", d.head[i], HMAX);
  KT_REQUIRE(d.head[d.n_head] == 1, KT_E_SHAPE, "head must end in one output");
  return KT_OK;
}

template <class K>
static int set_smem(K kernel, size_t smem, size_t& cached) {
  KT_REQUIRE(smem <= 227 * 1024, KT_E_UNSUPPORTED, "head too large for shared memory (%zu bytes)", smem);
  if (smem > 48 * 1024 && smem > cached) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    cached = smem;
  }
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
  const meta::Head h = meta::head_of(*dims);
  static size_t cached = 0;
  const size_t smem = meta::head_smem(h, false);
  rc = meta::set_smem(meta::head_kernel, smem, cached);
  if (rc) return rc;
  meta::head_kernel<<<1, meta::NT, smem, as_stream(stream)>>>(*dims, theta, nullptr, u, y, (int)n, 0, 0.f, grad_out,
                                                               mse_out);
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
  const meta::Head h = meta::head_of(*dims);
  static size_t cached = 0;
  const size_t smem = meta::head_smem(h, true);
  rc = meta::set_smem(meta::head_kernel, smem, cached);
  if (rc) return rc;
  meta::head_kernel<<<1, meta::NT, smem, as_stream(stream)>>>(*dims, theta, v, u, y, (int)n, 0, 0.f, hvp_out, nullptr);
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
  const meta::Head h = meta::head_of(*dims);
  static size_t cached = 0;
  const size_t smem = meta::head_smem(h, false);
  rc = meta::set_smem(meta::head_kernel, smem, cached);
  if (rc) return rc;
  meta::head_kernel<<<1, meta::NT, smem, as_stream(stream)>>>(*dims, theta, nullptr, u, y, (int)n, steps, alpha,
                                                               theta_out, mse_out);
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
  const meta::Head h = meta::head_of(*dims);
  const bool so = !first_order;
  static size_t cached = 0;
  const size_t smem = meta::task_smem(h, so);
  rc = meta::set_smem(meta::maml_task_kernel, smem, cached);
  if (rc) return rc;
  float* g = static_cast<float*>(workspace);
  float* losses = g + (int64_t)T * h.P;
  float* thws = losses + 2 * T;
  meta::TaskSet ts{u, y, s_off, s_idx, q_off, q_idx};
  cudaStream_t st = as_stream(stream);
  meta::maml_task_kernel<<<T, meta::NT, smem, st>>>(*dims, theta, ts, T, alpha, inner_steps, first_order, thws, g,
                                                    losses);
  meta::task_sum_kernel<<<(h.P + 255) / 256, 256, 0, st>>>(g, T, h.P, g_sum, losses, stats);
  note_launches(2);
  return check_launch("kt_maml_tasks");
}

}  // extern "C"
