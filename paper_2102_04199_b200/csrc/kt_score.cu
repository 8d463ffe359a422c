// kt_score_indices: fused candidate scorer for star-layout schedule graphs.
//
// Replaces the predictor closure meta_scores (search.py:534-541):
//   encode_batch (graphs.py:305) -> embed_batch (model.py:185-194)
//   -> head_forward_batch (model.py:197-203)
// for the default model dims (F=12, GCN 12->32->32, head 64->64->64->1).
//
// Star-layout algebra (batch_layout graphs.py:278-302 always yields it: root
// -> for_i -> iterval_i, features only on iterval rows, A_hat = D^-1/2 (A+I) D^-1/2
// with deg(root) = P+1, deg(for) = 3, deg(iterval) = 2 for P (for, iterval) pairs):
//   layer 1:  (A X)[for_i] = x_i / sqrt(6),  (A X)[iter_i] = x_i / 2,  (A X)[root] = 0
//             => H1 rows are positive multiples of r_i = ReLU(x_i W1)
//   layer 2:  (A H1)[for_i]  = c_f r_i, c_f = 5 / (6 sqrt 6)
//             (A H1)[iter_i] = c_t r_i, c_t = 5 / 12
//             (A H1)[root]   = c_r sum_i r_i, c_r = 1 / sqrt(18 (P+1))
//             => with s_i = r_i W2:  H2[for_i] = c_f ReLU(s_i), H2[iter_i] = c_t ReLU(s_i),
//                H2[root] = ReLU(c_r sum_i s_i)
//   readout:  sum_c = a_c (H2[root]_c + (c_f + c_t) sum_i ReLU(s_ic))
//             max_c = max(H2[root]_c, c_t max_i ReLU(s_ic))        (c_t > c_f, H2 >= 0)
// Unfilled super-graph slots and padding rows have x_i = 0 => s_i = 0 and add
// nothing, so every graph is processed as 12 loop rows.  The per-graph work is
// 12*12*32 + 12*32*32 + 64*64 + 64*64 + 64 = 25,152 MACs (vs 47.5k for the
// dense 25-node evaluation).  Arithmetic is fp32 on the FMA pipe (FFMA2); per
// candidate it is deterministic and independent of batch position, so exact
// ties in the reference stay exact ties here.
//
// CTA = 256 threads, tile = 64 graphs, persistent over tiles (grid = 148).
//   A1  64 threads decode config indices -> choices (smem)
//   A2  (graph, loop) items -> normalised feature rows X^T (smem)
//   B   thread (g, 8-channel group): R = ReLU(X W1), 12x8 register tile
//   C   S = R W2, 12x8 register tile, readout in registers -> U^T (smem)
//   D/E head: thread (4 graphs x 4 channels) register tiles, final dot by shuffles
#include "kt_encode.cuh"

namespace kt {
namespace score {

constexpr int G = 64;
constexpr int NT = 256;
constexpr int XS = KT_F * 12 + 4;  // X^T stride per graph (f-major, 12 rows) -> conflict-free
constexpr int RS = 32 * 12 + 4;    // R^T stride per graph
constexpr int US = G + 4;          // U^T / Z1^T row stride
constexpr int H = 64;

struct Smem {
  float w1[KT_F * 32];
  float w2[32 * 32];
  float h0[H * H];
  float h1[H * H];
  float b0[H], b1[H], w3[H];
  float agg[32];
  float buf[G * RS];  // X^T, then R^T, then Z1^T
  float ut[H * US];   // U^T
  int ch[G][KT_MAX_KNOBS];
  int valid[G];
};

__device__ __forceinline__ float relu(float v) { return fmaxf(v, 0.0f); }

__global__ void __launch_bounds__(NT, 1)
score_star_kernel(const kt_spec_table* __restrict__ tab, kt_dims dims, const float* __restrict__ params,
                  const int64_t* __restrict__ idx, int64_t idx_base, int64_t B,
                  float* __restrict__ z_out, float* __restrict__ u_out, int32_t* __restrict__ err) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>(smem_raw);
  const kt_spec_table& T = *tab;
  const int tid = threadIdx.x;

  // weights -> smem (once per CTA)
  for (int i = tid; i < KT_F * 32; i += NT) S.w1[i] = params[dims.off_gcn[0] + i];
  for (int i = tid; i < 32 * 32; i += NT) S.w2[i] = params[dims.off_gcn[1] + i];
  for (int i = tid; i < H * H; i += NT) {
    S.h0[i] = params[dims.off_hw[0] + i];
    S.h1[i] = params[dims.off_hw[1] + i];
  }
  if (tid < H) {
    S.b0[tid] = params[dims.off_hb[0] + tid];
    S.b1[tid] = params[dims.off_hb[1] + tid];
    S.w3[tid] = params[dims.off_hw[2] + tid];
  }
  if (tid < 32) S.agg[tid] = params[dims.off_agg + tid];
  const float b3 = params[dims.off_hb[2]];
  const int n_loops = T.n_loops;
  const float c_f = static_cast<float>(5.0 / (6.0 * sqrt(6.0)));
  const float c_t = static_cast<float>(5.0 / 12.0);
  const float c_ft = static_cast<float>(5.0 / (6.0 * sqrt(6.0)) + 5.0 / 12.0);
  const float c_r = static_cast<float>(1.0 / sqrt(18.0 * (T.n_pairs + 1)));

  const int64_t n_tiles = (B + G - 1) / G;
  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int64_t g0 = tile * G;
    __syncthreads();  // previous tile fully consumed (and weights staged)

    // ---- A1: decode ------------------------------------------------------------
    if (tid < G) {
      const int64_t i = g0 + tid;
      int ch[KT_MAX_KNOBS];
      bool ok = false;
      if (i < B) {
        const int64_t v = idx ? idx[i] : idx_base + i;
        ok = decode_checked(T, v, ch);
        if (!ok) atomicOr(err, 1);
      } else {
        for (int j = 0; j < KT_MAX_KNOBS; ++j) ch[j] = 0;
      }
#pragma unroll
      for (int j = 0; j < KT_MAX_KNOBS; ++j) S.ch[tid][j] = ch[j];
      S.valid[tid] = ok;
    }
    __syncthreads();

    // ---- A2: feature rows -> X^T[g][f][k] -----------------------------------------
    for (int item = tid; item < G * 12; item += NT) {
      const int g = item / 12, k = item - (item / 12) * 12;
      float x[KT_F];
      if (k < n_loops && S.valid[g]) {
        norm_row(T, S.ch[g], k, x);
      } else {
#pragma unroll
        for (int f = 0; f < KT_F; ++f) x[f] = 0.0f;
      }
      float* dst = S.buf + g * XS + k;
#pragma unroll
      for (int f = 0; f < KT_F; ++f) dst[f * 12] = x[f];
    }
    __syncthreads();

    // ---- B: R = ReLU(X W1) ---------------------------------------------------------
    const int g = tid >> 2, cg = tid & 3;
    float2 acc[12][4];
#pragma unroll
    for (int k = 0; k < 12; ++k)
#pragma unroll
      for (int p = 0; p < 4; ++p) acc[k][p] = make_float2(0.f, 0.f);
    {
      const float* xg = S.buf + g * XS;
#pragma unroll
      for (int f = 0; f < KT_F; ++f) {
        float xv[12];
        *reinterpret_cast<float4*>(xv + 0) = *reinterpret_cast<const float4*>(xg + f * 12 + 0);
        *reinterpret_cast<float4*>(xv + 4) = *reinterpret_cast<const float4*>(xg + f * 12 + 4);
        *reinterpret_cast<float4*>(xv + 8) = *reinterpret_cast<const float4*>(xg + f * 12 + 8);
        const float4 wa = *reinterpret_cast<const float4*>(S.w1 + f * 32 + cg * 8);
        const float4 wb = *reinterpret_cast<const float4*>(S.w1 + f * 32 + cg * 8 + 4);
        const float2 w[4] = {make_float2(wa.x, wa.y), make_float2(wa.z, wa.w), make_float2(wb.x, wb.y),
                             make_float2(wb.z, wb.w)};
#pragma unroll
        for (int k = 0; k < 12; ++k)
#pragma unroll
          for (int p = 0; p < 4; ++p) acc[k][p] = ffma2s(xv[k], w[p], acc[k][p]);
      }
    }
    __syncthreads();  // all X^T reads done before R^T overwrites buf
    {
      float* rg = S.buf + g * RS;
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        float lo[12], hi[12];
#pragma unroll
        for (int k = 0; k < 12; ++k) {
          lo[k] = relu(acc[k][p].x);
          hi[k] = relu(acc[k][p].y);
        }
        float* dlo = rg + (cg * 8 + 2 * p) * 12;
        float* dhi = dlo + 12;
#pragma unroll
        for (int q = 0; q < 12; q += 4) {
          *reinterpret_cast<float4*>(dlo + q) = make_float4(lo[q], lo[q + 1], lo[q + 2], lo[q + 3]);
          *reinterpret_cast<float4*>(dhi + q) = make_float4(hi[q], hi[q + 1], hi[q + 2], hi[q + 3]);
        }
      }
    }
    __syncthreads();

    // ---- C: S = R W2, readout ------------------------------------------------------
#pragma unroll
    for (int k = 0; k < 12; ++k)
#pragma unroll
      for (int p = 0; p < 4; ++p) acc[k][p] = make_float2(0.f, 0.f);
    {
      const float* rg = S.buf + g * RS;
#pragma unroll 4
      for (int j = 0; j < 32; ++j) {
        float rv[12];
        *reinterpret_cast<float4*>(rv + 0) = *reinterpret_cast<const float4*>(rg + j * 12 + 0);
        *reinterpret_cast<float4*>(rv + 4) = *reinterpret_cast<const float4*>(rg + j * 12 + 4);
        *reinterpret_cast<float4*>(rv + 8) = *reinterpret_cast<const float4*>(rg + j * 12 + 8);
        const float4 wa = *reinterpret_cast<const float4*>(S.w2 + j * 32 + cg * 8);
        const float4 wb = *reinterpret_cast<const float4*>(S.w2 + j * 32 + cg * 8 + 4);
        const float2 w[4] = {make_float2(wa.x, wa.y), make_float2(wa.z, wa.w), make_float2(wb.x, wb.y),
                             make_float2(wb.z, wb.w)};
#pragma unroll
        for (int k = 0; k < 12; ++k)
#pragma unroll
          for (int p = 0; p < 4; ++p) acc[k][p] = ffma2s(rv[k], w[p], acc[k][p]);
      }
    }
    {
      const int64_t gi = g0 + g;
#pragma unroll
      for (int p = 0; p < 4; ++p) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          float tot = 0.f, rsum = 0.f, rmax = 0.f;
#pragma unroll
          for (int k = 0; k < 12; ++k) {
            const float s = h ? acc[k][p].y : acc[k][p].x;
            tot += s;
            rsum += relu(s);
            rmax = fmaxf(rmax, s);
          }
          const int c = cg * 8 + 2 * p + h;
          const float root = relu(c_r * tot);
          const float us = S.agg[c] * (root + c_ft * rsum);
          const float um = fmaxf(root, c_t * rmax);
          S.ut[c * US + g] = us;
          S.ut[(32 + c) * US + g] = um;
          if (u_out && gi < B) {
            u_out[gi * 64 + c] = us;
            u_out[gi * 64 + 32 + c] = um;
          }
        }
      }
    }
    __syncthreads();

    // ---- D: Z1 = ReLU(U H0 + b0) -> Z1^T (buf) --------------------------------------
    const int gq = tid >> 4, cq = tid & 15;
    {
      float2 a2[4][2];
#pragma unroll
      for (int i = 0; i < 4; ++i) a2[i][0] = a2[i][1] = make_float2(0.f, 0.f);
#pragma unroll 8
      for (int k = 0; k < H; ++k) {
        const float4 u4 = *reinterpret_cast<const float4*>(S.ut + k * US + gq * 4);
        const float4 w4 = *reinterpret_cast<const float4*>(S.h0 + k * H + cq * 4);
        const float uu[4] = {u4.x, u4.y, u4.z, u4.w};
        const float2 wl = make_float2(w4.x, w4.y), wh = make_float2(w4.z, w4.w);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          a2[i][0] = ffma2s(uu[i], wl, a2[i][0]);
          a2[i][1] = ffma2s(uu[i], wh, a2[i][1]);
        }
      }
      const float4 bb = *reinterpret_cast<const float4*>(S.b0 + cq * 4);
      float* zt = S.buf + (cq * 4) * US + gq * 4;
      *reinterpret_cast<float4*>(zt + 0 * US) = make_float4(
          relu(a2[0][0].x + bb.x), relu(a2[1][0].x + bb.x), relu(a2[2][0].x + bb.x), relu(a2[3][0].x + bb.x));
      *reinterpret_cast<float4*>(zt + 1 * US) = make_float4(
          relu(a2[0][0].y + bb.y), relu(a2[1][0].y + bb.y), relu(a2[2][0].y + bb.y), relu(a2[3][0].y + bb.y));
      *reinterpret_cast<float4*>(zt + 2 * US) = make_float4(
          relu(a2[0][1].x + bb.z), relu(a2[1][1].x + bb.z), relu(a2[2][1].x + bb.z), relu(a2[3][1].x + bb.z));
      *reinterpret_cast<float4*>(zt + 3 * US) = make_float4(
          relu(a2[0][1].y + bb.w), relu(a2[1][1].y + bb.w), relu(a2[2][1].y + bb.w), relu(a2[3][1].y + bb.w));
    }
    __syncthreads();

    // ---- E: Z2 = ReLU(Z1 H1 + b1); z = Z2 . w3 + b3 ----------------------------------
    {
      float2 a2[4][2];
#pragma unroll
      for (int i = 0; i < 4; ++i) a2[i][0] = a2[i][1] = make_float2(0.f, 0.f);
#pragma unroll 8
      for (int k = 0; k < H; ++k) {
        const float4 u4 = *reinterpret_cast<const float4*>(S.buf + k * US + gq * 4);
        const float4 w4 = *reinterpret_cast<const float4*>(S.h1 + k * H + cq * 4);
        const float uu[4] = {u4.x, u4.y, u4.z, u4.w};
        const float2 wl = make_float2(w4.x, w4.y), wh = make_float2(w4.z, w4.w);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          a2[i][0] = ffma2s(uu[i], wl, a2[i][0]);
          a2[i][1] = ffma2s(uu[i], wh, a2[i][1]);
        }
      }
      const float4 bb = *reinterpret_cast<const float4*>(S.b1 + cq * 4);
      const float4 w3 = *reinterpret_cast<const float4*>(S.w3 + cq * 4);
      float part[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        part[i] = relu(a2[i][0].x + bb.x) * w3.x;
        part[i] = fmaf(relu(a2[i][0].y + bb.y), w3.y, part[i]);
        part[i] = fmaf(relu(a2[i][1].x + bb.z), w3.z, part[i]);
        part[i] = fmaf(relu(a2[i][1].y + bb.w), w3.w, part[i]);
      }
      // reduce over the 16 lanes that share gq (fixed order -> deterministic)
#pragma unroll
      for (int off = 8; off >= 1; off >>= 1)
#pragma unroll
        for (int i = 0; i < 4; ++i) part[i] += __shfl_xor_sync(0xffffffffu, part[i], off);
      if (cq == 0) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int gl = gq * 4 + i;
          const int64_t gi = g0 + gl;
          if (gi < B) z_out[gi] = S.valid[gl] ? part[i] + b3 : __int_as_float(0x7fc00000);
        }
      }
    }
  }
}

}  // namespace score

static bool default_dims(const kt_dims& d) {
  return d.F == KT_F && d.n_gcn == 2 && d.gcn[1] == 32 && d.gcn[2] == 32 && d.n_head == 3 &&
         d.head[0] == 64 && d.head[1] == 64 && d.head[2] == 64 && d.head[3] == 1;
}

}  // namespace kt

extern "C" int kt_score_indices(const kt_spec_table* tab, const kt_dims* dims, const float* params,
                                const int64_t* idx, int64_t idx_base, int64_t B, float* z_out,
                                float* u_out, int32_t* err_flag, void* stream) {
  using namespace kt;
  KT_REQUIRE(tab && dims && params && z_out && err_flag, KT_E_ARG, "kt_score_indices: null pointer");
  KT_REQUIRE(B > 0, KT_E_EMPTY, "kt_score_indices: empty batch");
  KT_REQUIRE(default_dims(*dims), KT_E_UNSUPPORTED,
             "kt_score_indices: fused scorer needs F=12, gcn (32,32), head (64,64)");
  static bool attr_set = false;
  const int smem = static_cast<int>(sizeof(score::Smem));
  if (!attr_set) {
    cudaFuncSetAttribute(score::score_star_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr_set = true;
  }
  const int64_t n_tiles = (B + score::G - 1) / score::G;
  const int grid = static_cast<int>(n_tiles < kNumSMs ? n_tiles : kNumSMs);
  score::score_star_kernel<<<grid, score::NT, smem, as_stream(stream)>>>(tab, *dims, params, idx, idx_base,
                                                                         B, z_out, u_out, err_flag);
  note_launches(1);
  return check_launch("kt_score_indices");
}
