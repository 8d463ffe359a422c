// kt_score_indices_fp32: fused candidate scorer for star-layout schedule graphs on the
// FP32 FMA pipe (FFMA2).  kt_score_tc.cu holds the tensor-core version (kt_score_indices).
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
// nothing, so every graph is processed as 12 loop rows.  Per graph:
// 12*12*32 + 12*32*32 + 64*64 + 64*64 + 64 = 25,152 MACs (the dense 25-node
// evaluation is 47.5k).  fp32 on the FMA pipe via FFMA2; per candidate the
// arithmetic is fixed and independent of batch position, so the reference's
// exact ties stay exact ties.
//
// CTA = 128 threads, tile = 32 graphs, persistent over tiles, 2 CTAs / SM
// (~90 KB smem each) so one CTA's encode phase overlaps the other's GEMMs.
//   A1  one thread per graph: magic-number index decode, per-axis tile choice,
//       loop extents and their suffix products (touched, fp64) -> smem
//   A2  (graph, loop) items: normalised rows; choice-only slots come from the
//       smem-staged host tables, touched/arith slots use fp64 log2 + IEEE div
//   B   thread (graph, row-quarter kq): rows 3kq..3kq+2, all 32 channels in
//       registers: R = ReLU(X W1), then S = R W2 in four 8-channel passes,
//       readout partials combined across the 4 row-quarter lanes by shuffles
//   D/E head: thread (4 graphs x 4 channels) register tiles, final dot by shuffles
#include "kt_encode.cuh"

namespace kt {
namespace score {

constexpr int G = 32;                // graphs per tile
constexpr int NT = 128;              // threads per CTA
constexpr int H = 64;
constexpr int XF = 16;               // per-feature row group: 4 quarters x (3 rows + 1 pad)
constexpr int XS = KT_F * XF + 4;    // X^T stride per graph (196 -> conflict-free LDS.128)
constexpr int US = G + 4;            // U^T / Z1^T row stride
constexpr int TAB = 448;             // packed per-choice table entries (sum of tile cards <= 412)

struct Smem {
  float w1[KT_F * 32];
  float w2[32 * 32];
  float h0[H * H];
  float h1[H * H];
  float b0[H], b1[H], w3[H];
  float agg[32];
  float x[G * XS];          // X^T[g][f][quarter][3 rows + pad]; later Z1^T
  float ut[H * US];         // U^T
  // per-choice tables packed by axis (choice c of axis a at tab_off[a] + c)
  int2 oi[TAB];             // (outer extent, inner extent)
  float4 nrm_o[TAB];        // outer loop: (ext, log2 ext, stride slot, -)
  float2 nrm_i[TAB];        // inner loop: (ext, log2 ext)
  float nconst[KT_MAX_LOOPS][8];  // slots 2,3,4(off),4(on),5(inner),10,11 per loop
  int tab_off[KT_MAX_AXES];
  double touched[G][KT_MAX_LOOPS];
  unsigned char choice[G][KT_MAX_AXES];
  unsigned short unroll[G];  // bit a: inner loop of axis a unrolled
  int valid[G];
};

__device__ __forceinline__ float relu(float v) { return fmaxf(v, 0.0f); }

__device__ __forceinline__ uint32_t udiv(uint32_t v, uint32_t d, uint64_t magic) {
  return d == 1 ? v : static_cast<uint32_t>(__umul64hi(static_cast<uint64_t>(v), magic));
}

__global__ void __launch_bounds__(NT, 2)
score_star_kernel(const kt_spec_table* __restrict__ tab, kt_dims dims, const float* __restrict__ params,
                  const int64_t* __restrict__ idx, int64_t idx_base, int64_t B,
                  float* __restrict__ z_out, float* __restrict__ u_out, int32_t* __restrict__ err) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>(smem_raw);
  const kt_spec_table& T = *tab;
  const int tid = threadIdx.x;
  const int na = T.n_axes, n_loops = T.n_loops, n_knobs = T.n_knobs;

  // ---- once per CTA: weights and per-choice tables -> smem ------------------------
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
  if (tid == 0) {
    int off = 0;
    for (int a = 0; a < na; ++a) {
      S.tab_off[a] = off;
      off += T.axis_knob[a] >= 0 ? static_cast<int>(T.card[T.axis_knob[a]]) : 1;
    }
  }
  if (tid < KT_MAX_LOOPS) {
    const int k = tid;
    S.nconst[k][0] = T.nrm_const[k][2];
    S.nconst[k][1] = T.nrm_const[k][3];
    S.nconst[k][2] = T.nrm_const[k][4];
    S.nconst[k][3] = T.nrm_unroll1[k];
    S.nconst[k][4] = T.nrm_const[k][5];
    S.nconst[k][5] = T.nrm_const[k][10];
    S.nconst[k][6] = T.nrm_const[k][11];
    S.nconst[k][7] = 0.f;
  }
  __syncthreads();
  for (int a = 0; a < na; ++a) {
    const int n = T.axis_knob[a] >= 0 ? static_cast<int>(T.card[T.axis_knob[a]]) : 1;
    for (int c = tid; c < n; c += NT) {
      const int e = S.tab_off[a] + c;
      S.oi[e] = make_int2(T.outer[a][c], T.inner[a][c]);
      S.nrm_o[e] = make_float4(T.nrm_ext[a][c], T.nrm_log2ext[a][c], T.nrm_stride[a][c], 0.f);
      S.nrm_i[e] = make_float2(T.nrm_ext[na + a][c], T.nrm_log2ext[na + a][c]);
    }
  }
  const float b3 = params[dims.off_hb[2]];
  const float c_t = static_cast<float>(5.0 / 12.0);
  const float c_ft = static_cast<float>(5.0 / (6.0 * sqrt(6.0)) + 5.0 / 12.0);
  const float c_r = static_cast<float>(1.0 / sqrt(18.0 * (T.n_pairs + 1)));
  const double m6 = T.fmean[6], s6 = T.fstd[6], m7 = T.fmean[7], s7 = T.fstd[7];
  const double m8 = T.fmean[8], s8 = T.fstd[8], m9 = T.fmean[9], s9 = T.fstd[9];

  const int64_t n_tiles = (B + G - 1) / G;
  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int64_t g0 = tile * G;
    __syncthreads();  // previous tile consumed; tables staged

    // ---- A1: decode + extents + suffix products (one thread per graph) ------------
    if (tid < G) {
      const int g = tid;
      const int64_t i = g0 + g;
      bool ok = false;
      int ch[KT_MAX_KNOBS];
#pragma unroll
      for (int j = 0; j < KT_MAX_KNOBS; ++j) ch[j] = 0;
      if (i < B) {
        const int64_t v = idx ? idx[i] : idx_base + i;
        ok = v >= 0 && static_cast<uint64_t>(v) < T.space_size;
        if (ok) {
          uint32_t r = static_cast<uint32_t>(v);
#pragma unroll
          for (int j = KT_MAX_KNOBS - 1; j >= 0; --j) {
            if (j < n_knobs) {
              const uint32_t d = T.card[j];
              const uint32_t q = udiv(r, d, T.card_magic[j]);
              ch[j] = static_cast<int>(r - q * d);
              r = q;
            }
          }
        } else {
          atomicOr(err, 1);
        }
      }
      const int autov = T.auto_knob >= 0 ? T.auto_vals[ch[T.auto_knob]] : 0;
      const int expl = T.expl_knob >= 0 ? T.expl_vals[ch[T.expl_knob]] : 0;
      int eo[KT_MAX_AXES], ei[KT_MAX_AXES];
      unsigned unr = 0;
#pragma unroll
      for (int a = 0; a < KT_MAX_AXES; ++a) {
        eo[a] = ei[a] = 1;
        if (a < na) {
          const int c = T.axis_knob[a] >= 0 ? ch[T.axis_knob[a]] : 0;
          S.choice[g][a] = static_cast<unsigned char>(c);
          const int2 p = S.oi[S.tab_off[a] + c];
          eo[a] = p.x;
          ei[a] = p.y;
          if (expl != 0 && autov > 0 && p.y <= autov) unr |= 1u << a;
        }
      }
      // touched[k] = prod of the extents of loops k+1 .. n-1 (chain: outer axes, inner axes);
      // absent axes contribute 1, products are exact integers in fp64
      double t = 1.0;
#pragma unroll
      for (int a = KT_MAX_AXES - 1; a >= 0; --a) {
        if (a < na) S.touched[g][na + a] = t;
        t *= static_cast<double>(ei[a]);
      }
#pragma unroll
      for (int a = KT_MAX_AXES - 1; a >= 0; --a) {
        if (a < na) S.touched[g][a] = t;
        t *= static_cast<double>(eo[a]);
      }
      S.unroll[g] = static_cast<unsigned short>(unr);
      S.valid[g] = ok;
    }
    __syncthreads();

    // ---- A2: normalised feature rows -> X^T[g][f][4*(k/3) + k%3] ----------------------
    for (int item = tid; item < G * 12; item += NT) {
      const int g = item / 12, k = item - (item / 12) * 12;
      float x[KT_F];
      if (k < n_loops && S.valid[g]) {
        const int level = k >= na;
        const int a = level ? k - na : k;
        const int e = S.tab_off[a] + S.choice[g][a];
        if (level) {
          const float2 ni = S.nrm_i[e];
          x[0] = ni.x;
          x[1] = ni.y;
          x[5] = S.nconst[k][4];
        } else {
          const float4 no = S.nrm_o[e];
          x[0] = no.x;
          x[1] = no.y;
          x[5] = no.z;
        }
        x[2] = S.nconst[k][0];
        x[3] = S.nconst[k][1];
        x[4] = (level && ((S.unroll[g] >> a) & 1u)) ? S.nconst[k][3] : S.nconst[k][2];
        const double tch = S.touched[g][k];
        const double ar = 2.0 * tch;
        x[6] = static_cast<float>((tch - m6) / s6);
        x[7] = static_cast<float>((log2(tch) - m7) / s7);
        x[8] = static_cast<float>((ar - m8) / s8);
        x[9] = static_cast<float>((log2(ar) - m9) / s9);
        x[10] = S.nconst[k][5];
        x[11] = S.nconst[k][6];
      } else {
#pragma unroll
        for (int f = 0; f < KT_F; ++f) x[f] = 0.0f;
      }
      float* dst = S.x + g * XS + 4 * (k / 3) + (k - 3 * (k / 3));
#pragma unroll
      for (int f = 0; f < KT_F; ++f) dst[f * XF] = x[f];
    }
    __syncthreads();

    // ---- B/C: R = ReLU(X W1) (3 rows x 32 ch in registers), S = R W2, readout ---------
    {
      const int g = tid >> 2, kq = tid & 3;
      float2 r2[3][16];
#pragma unroll
      for (int q = 0; q < 3; ++q)
#pragma unroll
        for (int p = 0; p < 16; ++p) r2[q][p] = make_float2(0.f, 0.f);
      const float* xg = S.x + g * XS + 4 * kq;
#pragma unroll
      for (int f = 0; f < KT_F; ++f) {
        const float4 xv = *reinterpret_cast<const float4*>(xg + f * XF);
        const float4* wr = reinterpret_cast<const float4*>(S.w1 + f * 32);
#pragma unroll
        for (int p4 = 0; p4 < 8; ++p4) {
          const float4 w = wr[p4];
          const float2 wa = make_float2(w.x, w.y), wb = make_float2(w.z, w.w);
          r2[0][2 * p4] = ffma2s(xv.x, wa, r2[0][2 * p4]);
          r2[0][2 * p4 + 1] = ffma2s(xv.x, wb, r2[0][2 * p4 + 1]);
          r2[1][2 * p4] = ffma2s(xv.y, wa, r2[1][2 * p4]);
          r2[1][2 * p4 + 1] = ffma2s(xv.y, wb, r2[1][2 * p4 + 1]);
          r2[2][2 * p4] = ffma2s(xv.z, wa, r2[2][2 * p4]);
          r2[2][2 * p4 + 1] = ffma2s(xv.z, wb, r2[2][2 * p4 + 1]);
        }
      }
#pragma unroll
      for (int q = 0; q < 3; ++q)
#pragma unroll
        for (int p = 0; p < 16; ++p) r2[q][p] = make_float2(relu(r2[q][p].x), relu(r2[q][p].y));

#pragma unroll
      for (int pass = 0; pass < 4; ++pass) {  // output channels 8*pass .. 8*pass+7
        float2 s2[3][4];
#pragma unroll
        for (int q = 0; q < 3; ++q)
#pragma unroll
          for (int p = 0; p < 4; ++p) s2[q][p] = make_float2(0.f, 0.f);
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float4* wr = reinterpret_cast<const float4*>(S.w2 + j * 32 + pass * 8);
          const float r0 = (j & 1) ? r2[0][j >> 1].y : r2[0][j >> 1].x;
          const float r1 = (j & 1) ? r2[1][j >> 1].y : r2[1][j >> 1].x;
          const float rr2 = (j & 1) ? r2[2][j >> 1].y : r2[2][j >> 1].x;
#pragma unroll
          for (int p4 = 0; p4 < 2; ++p4) {
            const float4 w = wr[p4];
            const float2 wa = make_float2(w.x, w.y), wb = make_float2(w.z, w.w);
            s2[0][2 * p4] = ffma2s(r0, wa, s2[0][2 * p4]);
            s2[0][2 * p4 + 1] = ffma2s(r0, wb, s2[0][2 * p4 + 1]);
            s2[1][2 * p4] = ffma2s(r1, wa, s2[1][2 * p4]);
            s2[1][2 * p4 + 1] = ffma2s(r1, wb, s2[1][2 * p4 + 1]);
            s2[2][2 * p4] = ffma2s(rr2, wa, s2[2][2 * p4]);
            s2[2][2 * p4 + 1] = ffma2s(rr2, wb, s2[2][2 * p4 + 1]);
          }
        }
        // readout partials over this thread's 3 rows, then across the 4 row quarters
        float tot[8], rsum[8], rmax[8];
#pragma unroll
        for (int p = 0; p < 4; ++p) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const float a0 = h ? s2[0][p].y : s2[0][p].x;
            const float a1 = h ? s2[1][p].y : s2[1][p].x;
            const float a2 = h ? s2[2][p].y : s2[2][p].x;
            tot[2 * p + h] = a0 + a1 + a2;
            rsum[2 * p + h] = relu(a0) + relu(a1) + relu(a2);
            rmax[2 * p + h] = fmaxf(fmaxf(relu(a0), relu(a1)), relu(a2));
          }
        }
#pragma unroll
        for (int off = 1; off <= 2; off <<= 1) {
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            tot[c] += __shfl_xor_sync(0xffffffffu, tot[c], off);
            rsum[c] += __shfl_xor_sync(0xffffffffu, rsum[c], off);
            rmax[c] = fmaxf(rmax[c], __shfl_xor_sync(0xffffffffu, rmax[c], off));
          }
        }
        // quarter kq publishes channels 8*pass + 2kq, 8*pass + 2kq + 1
        const int64_t gi = g0 + g;
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          float t_ = tot[0], rs = rsum[0], rm = rmax[0];
#pragma unroll
          for (int c = 1; c < 8; ++c)
            if (c == 2 * kq + cc) { t_ = tot[c]; rs = rsum[c]; rm = rmax[c]; }
          const int c = pass * 8 + 2 * kq + cc;
          const float root = relu(c_r * t_);
          const float us = S.agg[c] * (root + c_ft * rs);
          const float um = fmaxf(root, c_t * rm);
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

    // ---- D: Z1 = ReLU(U H0 + b0) -> Z1^T (x region) -----------------------------------
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
      float* zt = S.x + (cq * 4) * US + gq * 4;
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

    // ---- E: Z2 = ReLU(Z1 H1 + b1); z = Z2 . w3 + b3 ------------------------------------
    {
      float2 a2[4][2];
#pragma unroll
      for (int i = 0; i < 4; ++i) a2[i][0] = a2[i][1] = make_float2(0.f, 0.f);
#pragma unroll 8
      for (int k = 0; k < H; ++k) {
        const float4 u4 = *reinterpret_cast<const float4*>(S.x + k * US + gq * 4);
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

extern "C" int kt_score_indices_fp32(const kt_spec_table* tab, const kt_dims* dims, const float* params,
                                const int64_t* idx, int64_t idx_base, int64_t B, float* z_out,
                                float* u_out, int32_t* err_flag, void* stream) {
  using namespace kt;
  KT_REQUIRE(tab && dims && params && z_out && err_flag, KT_E_ARG, "kt_score_indices_fp32: null pointer");
  KT_REQUIRE(B > 0, KT_E_EMPTY, "kt_score_indices: empty batch");
  KT_REQUIRE(default_dims(*dims), KT_E_UNSUPPORTED,
             "kt_score_indices: fused scorer needs F=12, gcn (32,32), head (64,64)");
  static PerDeviceInt grid_caps;
  int& grid_cap = grid_caps.get();
  const int smem = static_cast<int>(sizeof(score::Smem));
  if (!grid_cap) {
    cudaFuncSetAttribute(score::score_star_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, score::score_star_kernel, score::NT, smem);
    grid_cap = kNumSMs * (per_sm > 0 ? per_sm : 1);
  }
  const int64_t n_tiles = (B + score::G - 1) / score::G;
  const int grid = static_cast<int>(n_tiles < grid_cap ? n_tiles : grid_cap);
  score::score_star_kernel<<<grid, score::NT, smem, as_stream(stream)>>>(tab, *dims, params, idx, idx_base,
                                                                         B, z_out, u_out, err_flag);
  note_launches(1);
  return check_launch("kt_score_indices_fp32");
}
