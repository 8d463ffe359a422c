// kt_score_indices (tensor-core path): the fused candidate scorer with all four
// GEMMs on the 5th-generation tensor cores (tcgen05.mma kind::tf32, accumulators
// in TMEM) in 3xTF32 split precision (A*B ~= Ah*Bh + Ah*Bl + Al*Bh, fp32-level
// accuracy).  Same math and contract as the FFMA2 kernel in kt_score.cu
// (star-layout algebra documented there); replaces meta_scores
// (search.py:534-541) = encode_batch -> embed_batch -> head_forward_batch.
//
// Work unit: a tile of 120 graphs = 12 chunks x 10 graphs; a chunk is one
// 128-row MMA tile (graph g of the chunk owns rows 12g..12g+11, rows 120..127
// are padding).  Per chunk:
//   GEMM1  D1[128x32]  = X[128x16] * W1          (A = X in TMEM, 2 K-steps x 3)
//   GEMM2  D2[128x32]  = ReLU(D1) * W2           (A = R in TMEM, 4 K-steps x 3)
// then the star readout (sum / max over each graph's 12 rows) into U[120x64].
// Per tile:
//   GEMM3  D3[128x64]  = U * H0 + b0 -> ReLU     (A = U in smem, 8 K-steps x 3)
//   GEMM4  D4[128x64]  = Z1 * H1 + b1 -> ReLU -> . w3 + b3   (A = Z1 in TMEM)
//
// Warp specialisation (256 threads, 1 CTA / SM, 512 TMEM columns):
//   warps 4-7 (producer): encode feature rows of chunk q (index decode, fp64
//     touched/log2/z-norm, host tables for the rest), split hi/lo and tcgen05.st
//     them into the double-buffered TMEM A operand X[q % 2];  mbarrier x_full.
//   warps 0-3 (consumer): thread 0 issues the MMAs and tcgen05.commit's
//     (x_empty releases X buffers, bar_g1/g2/h signal accumulators); all four
//     warps run the epilogues -- each thread owns one TMEM lane = one row.
// The encode of chunk q+1 overlaps GEMM1/GEMM2 and the epilogues of chunk q.
#include "kt_encode.cuh"
#include "kt_tc.cuh"

namespace kt {
namespace tcs {

using namespace kt::tc;

constexpr int NT = 256;
constexpr int GPC = 10;             // graphs per chunk
constexpr int CPT = 12;             // chunks per tile
constexpr int GT = GPC * CPT;       // graphs per tile (head M = 128 rows, 120 used)
constexpr int H = 64;
constexpr int ULBO = 144;           // padded K-chunk stride of U (bank spread for column writes)
constexpr int UF = (128 / 8) * (H / 4) * ULBO / 4;  // floats per U plane
constexpr int SS = 33;              // readout staging row stride
constexpr int TAB = 448;

// TMEM column map (512 allocated)
constexpr uint32_t T_D1 = 0, T_RH = 32, T_RL = 64, T_D2 = 96, T_D3 = 128, T_ZH = 192, T_ZL = 256, T_D4 = 320,
                   T_X = 384;  // X[buf]: hi at T_X + 32 buf, lo at T_X + 32 buf + 16

struct __align__(16) Smem {
  float b1h[32 * 16], b1l[32 * 16];  // W1^T  (N=32, K=16; K 12..15 zero)
  float b2h[32 * 32], b2l[32 * 32];  // W2^T
  float b3h[H * H], b3l[H * H];      // H0^T
  float b4h[H * H], b4l[H * H];      // H1^T
  float uh[UF], ul[UF];              // U operand (head A), K-major with LBO 144
  float s[128 * SS];                 // D2 rows staged for the per-graph readout
  float bias0[H], bias1[H], w3[H], agg[32];
  int2 oi[TAB];
  float4 nrm_o[TAB];
  float2 nrm_i[TAB];
  float nconst[KT_MAX_LOOPS][8];
  int tab_off[KT_MAX_AXES];
  uint64_t x_full[2], x_empty[2], bar_g1, bar_g2, bar_h;
  uint32_t tmem_base;
};

__device__ __forceinline__ float relu(float v) { return fmaxf(v, 0.0f); }

__device__ __forceinline__ uint32_t udiv(uint32_t v, uint32_t d, uint64_t magic) {
  return d == 1 ? v : static_cast<uint32_t>(__umul64hi(static_cast<uint64_t>(v), magic));
}

// Normalised feature row of loop k of the graph with config index v (valid, < 2^32).
__device__ __forceinline__ void encode_row(const kt_spec_table& T, const Smem& S, uint32_t v, int k, float* x) {
  const int na = T.n_axes, n_loops = T.n_loops;
  int ch[KT_MAX_KNOBS];
#pragma unroll
  for (int j = KT_MAX_KNOBS - 1; j >= 0; --j) {
    ch[j] = 0;
    if (j < T.n_knobs) {
      const uint32_t d = T.card[j];
      const uint32_t q = udiv(v, d, T.card_magic[j]);
      ch[j] = static_cast<int>(v - q * d);
      v = q;
    }
  }
  const int autov = T.auto_knob >= 0 ? T.auto_vals[ch[T.auto_knob]] : 0;
  const int expl = T.expl_knob >= 0 ? T.expl_vals[ch[T.expl_knob]] : 0;
  // chain extents: outer loops of axes 0..na-1, then inner loops; touched = prod over loops > k
  double t = 1.0;
  int my_c = 0, my_e = 1, my_unr = 0;
#pragma unroll
  for (int lvl = 1; lvl >= 0; --lvl) {
#pragma unroll
    for (int a = KT_MAX_AXES - 1; a >= 0; --a) {
      if (a < na) {
        const int c = T.axis_knob[a] >= 0 ? ch[T.axis_knob[a]] : 0;
        const int2 p = S.oi[S.tab_off[a] + c];
        const int e = lvl ? p.y : p.x;
        const int j = lvl ? na + a : a;
        if (j == k) {
          my_c = S.tab_off[a] + c;
          my_e = e;
          my_unr = lvl && expl != 0 && autov > 0 && p.y <= autov;
        }
        if (j > k) t *= static_cast<double>(e);
      }
    }
  }
  (void)my_e;
  const bool level = k >= na;
  if (level) {
    const float2 ni = S.nrm_i[my_c];
    x[0] = ni.x;
    x[1] = ni.y;
    x[5] = S.nconst[k][4];
  } else {
    const float4 no = S.nrm_o[my_c];
    x[0] = no.x;
    x[1] = no.y;
    x[5] = no.z;
  }
  x[2] = S.nconst[k][0];
  x[3] = S.nconst[k][1];
  x[4] = my_unr ? S.nconst[k][3] : S.nconst[k][2];
  const double ar = 2.0 * t;
  x[6] = static_cast<float>((t - T.fmean[6]) / T.fstd[6]);
  x[7] = static_cast<float>((log2(t) - T.fmean[7]) / T.fstd[7]);
  x[8] = static_cast<float>((ar - T.fmean[8]) / T.fstd[8]);
  x[9] = static_cast<float>((log2(ar) - T.fmean[9]) / T.fstd[9]);
  x[10] = S.nconst[k][5];
  x[11] = S.nconst[k][6];
  (void)n_loops;
}

__device__ __forceinline__ void stage_operand(const float* W, int K_src, int N, int K, float* hi, float* lo, int tid) {
  // B operand = W^T (rows n, K-major) from row-major W[k][n]; K beyond K_src zero
  for (int e = tid; e < N * K; e += NT) {
    const int n = e / K, k = e - n * K;
    const float v = k < K_src ? W[k * N + n] : 0.0f;
    const float h = tf32_hi(v);
    const int off = kmajor_offset(n, k, K) >> 2;
    hi[off] = h;
    lo[off] = v - h;
  }
}

__global__ void __launch_bounds__(NT, 1)
score_tc_kernel(const kt_spec_table* __restrict__ tab, kt_dims dims, const float* __restrict__ params,
                const int64_t* __restrict__ idx, int64_t idx_base, int64_t B, float* __restrict__ z_out,
                float* __restrict__ u_out, int32_t* __restrict__ err) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>(smem_raw);
  const kt_spec_table& T = *tab;
  const int tid = threadIdx.x, warp = tid >> 5;

  // ---- setup: operands, tables, barriers, TMEM ------------------------------------------
  stage_operand(params + dims.off_gcn[0], KT_F, 32, 16, S.b1h, S.b1l, tid);
  stage_operand(params + dims.off_gcn[1], 32, 32, 32, S.b2h, S.b2l, tid);
  stage_operand(params + dims.off_hw[0], H, H, H, S.b3h, S.b3l, tid);
  stage_operand(params + dims.off_hw[1], H, H, H, S.b4h, S.b4l, tid);
  for (int i = tid; i < UF; i += NT) S.uh[i] = S.ul[i] = 0.0f;
  if (tid < H) {
    S.bias0[tid] = params[dims.off_hb[0] + tid];
    S.bias1[tid] = params[dims.off_hb[1] + tid];
    S.w3[tid] = params[dims.off_hw[2] + tid];
  }
  if (tid < 32) S.agg[tid] = params[dims.off_agg + tid];
  const int na = T.n_axes;
  if (tid == 0) {
    int off = 0;
    for (int a = 0; a < na; ++a) {
      S.tab_off[a] = off;
      off += T.axis_knob[a] >= 0 ? static_cast<int>(T.card[T.axis_knob[a]]) : 1;
    }
    mbar_init(&S.x_full[0], 128);
    mbar_init(&S.x_full[1], 128);
    mbar_init(&S.x_empty[0], 1);
    mbar_init(&S.x_empty[1], 1);
    mbar_init(&S.bar_g1, 1);
    mbar_init(&S.bar_g2, 1);
    mbar_init(&S.bar_h, 1);
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
  if (warp == 0) tmem_alloc(&S.tmem_base, 512);
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
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = S.tmem_base;
  const int64_t n_tiles = (B + GT - 1) / GT;
  const int64_t my_tiles = blockIdx.x < n_tiles ? (n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t n_chunks = my_tiles * CPT;
  const uint64_t size = T.space_size;

  if (warp >= 4) {
    // ===================== producer: encode rows into TMEM X[q % 2] =====================
    const int row = tid - 128;
    const uint32_t lane_addr = static_cast<uint32_t>((row & ~31) << 16);
    const int gl = row / 12, k = row - (row / 12) * 12;
    for (int64_t q = 0; q < n_chunks; ++q) {
      const int buf = static_cast<int>(q & 1);
      mbar_wait(&S.x_empty[buf], static_cast<uint32_t>(((q >> 1) & 1) ^ 1));
      tc_fence_after();
      const int64_t tile = blockIdx.x + (q / CPT) * gridDim.x;
      const int c = static_cast<int>(q % CPT);
      float x[16];
#pragma unroll
      for (int f = 0; f < 16; ++f) x[f] = 0.0f;
      if (row < GT / CPT * 12) {
        const int64_t gi = tile * GT + c * GPC + gl;
        if (gi < B) {
          const int64_t v = idx ? idx[gi] : idx_base + gi;
          const bool ok = v >= 0 && static_cast<uint64_t>(v) < size;
          if (!ok) {
            if (k == 0) atomicOr(err, 1);
          } else if (k < T.n_loops) {
            encode_row(T, S, static_cast<uint32_t>(v), k, x);
          }
        }
      }
      float hi[16], lo[16];
#pragma unroll
      for (int f = 0; f < 16; ++f) {
        hi[f] = tf32_hi(x[f]);
        lo[f] = x[f] - hi[f];
      }
      tmem_st16(tmem + lane_addr + T_X + 32 * buf, hi);
      tmem_st16(tmem + lane_addr + T_X + 32 * buf + 16, lo);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&S.x_full[buf]);
    }
  } else {
    // ===================== consumer: MMA issue + epilogues (thread = TMEM lane = row) =====
    const int t = tid;
    const uint32_t lane_addr = static_cast<uint32_t>((t & ~31) << 16);
    const bool issuer = t == 0;
    const uint32_t id32 = idesc_tf32(128, 32), id64 = idesc_tf32(128, 64);
    const float c_t = static_cast<float>(5.0 / 12.0);
    const float c_ft = static_cast<float>(5.0 / (6.0 * sqrt(6.0)) + 5.0 / 12.0);
    const float c_r = static_cast<float>(1.0 / sqrt(18.0 * (T.n_pairs + 1)));
    uint32_t ph_g1 = 0, ph_g2 = 0, ph_h = 0;

    auto issue_g1 = [&](int64_t q) {
      const int buf = static_cast<int>(q & 1);
      mbar_wait(&S.x_full[buf], static_cast<uint32_t>((q >> 1) & 1));
      tc_fence_after();
      const uint32_t xh = tmem + T_X + 32 * buf, xl = xh + 16;
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        mma_tf32_ts(tmem + T_D1, xh + 8 * kk, kdesc(S.b1h, 16, kk), id32, kk > 0);
        mma_tf32_ts(tmem + T_D1, xh + 8 * kk, kdesc(S.b1l, 16, kk), id32, 1);
        mma_tf32_ts(tmem + T_D1, xl + 8 * kk, kdesc(S.b1h, 16, kk), id32, 1);
      }
      mma_commit(&S.x_empty[buf]);
      mma_commit(&S.bar_g1);
    };

    if (issuer && n_chunks > 0) issue_g1(0);
    int64_t q = 0;
    for (int64_t ti = 0; ti < my_tiles; ++ti) {
      const int64_t tile = blockIdx.x + ti * gridDim.x;
      for (int c = 0; c < CPT; ++c, ++q) {
        // ---- epilogue 1: R = ReLU(D1) -> TMEM (hi, lo)
        mbar_wait(&S.bar_g1, ph_g1);
        ph_g1 ^= 1;
        tc_fence_after();
        {
          float v[32], lo[32];
          tmem_ld32(tmem + lane_addr + T_D1, v);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float r = relu(v[j]);
            v[j] = tf32_hi(r);
            lo[j] = r - v[j];
          }
          tmem_st32(tmem + lane_addr + T_RH, v);
          tmem_st32(tmem + lane_addr + T_RL, lo);
          tmem_wait_st();
        }
        tc_fence_before();
        named_sync(1, 128);
        tc_fence_after();
        if (issuer) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            mma_tf32_ts(tmem + T_D2, tmem + T_RH + 8 * kk, kdesc(S.b2h, 32, kk), id32, kk > 0);
            mma_tf32_ts(tmem + T_D2, tmem + T_RH + 8 * kk, kdesc(S.b2l, 32, kk), id32, 1);
            mma_tf32_ts(tmem + T_D2, tmem + T_RL + 8 * kk, kdesc(S.b2h, 32, kk), id32, 1);
          }
          mma_commit(&S.bar_g2);
          if (q + 1 < n_chunks) issue_g1(q + 1);
        }
        // ---- epilogue 2: D2 rows -> smem, per-graph readout -> U
        mbar_wait(&S.bar_g2, ph_g2);
        ph_g2 ^= 1;
        tc_fence_after();
        {
          float v[32];
          tmem_ld32(tmem + lane_addr + T_D2, v);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j) S.s[t * SS + j] = v[j];
        }
        tc_fence_before();
        named_sync(1, 128);
        for (int item = t; item < GPC * 32; item += 128) {
          const int g = item >> 5, chn = item & 31;
          const float* col = S.s + (g * 12) * SS + chn;
          float tot = 0.f, rsum = 0.f, rmax = 0.f;
#pragma unroll
          for (int k = 0; k < 12; ++k) {
            const float sv = col[k * SS];
            tot += sv;
            rsum += relu(sv);
            rmax = fmaxf(rmax, sv);
          }
          const float root = relu(c_r * tot);
          const float us = S.agg[chn] * (root + c_ft * rsum);
          const float um = fmaxf(root, c_t * rmax);
          const int ur = c * GPC + g;
          const int o1 = kmajor_offset_lbo(ur, chn, H, ULBO) >> 2;
          const int o2 = kmajor_offset_lbo(ur, 32 + chn, H, ULBO) >> 2;
          const float h1 = tf32_hi(us), h2 = tf32_hi(um);
          S.uh[o1] = h1;
          S.ul[o1] = us - h1;
          S.uh[o2] = h2;
          S.ul[o2] = um - h2;
          if (u_out) {
            const int64_t gi = tile * GT + ur;
            if (gi < B) {
              u_out[gi * 64 + chn] = us;
              u_out[gi * 64 + 32 + chn] = um;
            }
          }
        }
      }
      // ---- head: GEMM3 (U from smem) -> ReLU(+b0) -> Z1 (TMEM) -> GEMM4 -> ReLU(+b1) . w3 + b3
      fence_async_smem();
      tc_fence_before();
      named_sync(1, 128);
      tc_fence_after();
      if (issuer) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          mma_tf32(tmem + T_D3, kdesc_lbo(S.uh, H, kk, ULBO), kdesc(S.b3h, H, kk), id64, kk > 0);
          mma_tf32(tmem + T_D3, kdesc_lbo(S.uh, H, kk, ULBO), kdesc(S.b3l, H, kk), id64, 1);
          mma_tf32(tmem + T_D3, kdesc_lbo(S.ul, H, kk, ULBO), kdesc(S.b3h, H, kk), id64, 1);
        }
        mma_commit(&S.bar_h);
      }
      mbar_wait(&S.bar_h, ph_h);
      ph_h ^= 1;
      tc_fence_after();
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        float v[32], lo[32];
        tmem_ld32(tmem + lane_addr + T_D3 + 32 * half, v);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float z = relu(v[j] + S.bias0[32 * half + j]);
          v[j] = tf32_hi(z);
          lo[j] = z - v[j];
        }
        tmem_st32(tmem + lane_addr + T_ZH + 32 * half, v);
        tmem_st32(tmem + lane_addr + T_ZL + 32 * half, lo);
      }
      tmem_wait_st();
      tc_fence_before();
      named_sync(1, 128);
      tc_fence_after();
      if (issuer) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          mma_tf32_ts(tmem + T_D4, tmem + T_ZH + 8 * kk, kdesc(S.b4h, H, kk), id64, kk > 0);
          mma_tf32_ts(tmem + T_D4, tmem + T_ZH + 8 * kk, kdesc(S.b4l, H, kk), id64, 1);
          mma_tf32_ts(tmem + T_D4, tmem + T_ZL + 8 * kk, kdesc(S.b4h, H, kk), id64, 1);
        }
        mma_commit(&S.bar_h);
      }
      mbar_wait(&S.bar_h, ph_h);
      ph_h ^= 1;
      tc_fence_after();
      float acc = params[dims.off_hb[2]];
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        float v[32];
        tmem_ld32(tmem + lane_addr + T_D4 + 32 * half, v);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; ++j) acc = fmaf(relu(v[j] + S.bias1[32 * half + j]), S.w3[32 * half + j], acc);
      }
      const int64_t gi = tile * GT + t;
      if (t < GT && gi < B) {
        const int64_t v = idx ? idx[gi] : idx_base + gi;
        const bool ok = v >= 0 && static_cast<uint64_t>(v) < size;
        z_out[gi] = ok ? acc : __int_as_float(0x7fc00000);
      }
      tc_fence_before();
      named_sync(1, 128);  // all D3/D4 reads done before the next tile's head overwrites them
      tc_fence_after();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

}  // namespace tcs

static bool default_dims_tc(const kt_dims& d) {
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
  KT_REQUIRE(default_dims_tc(*dims), KT_E_UNSUPPORTED,
             "kt_score_indices: fused scorer needs F=12, gcn (32,32), head (64,64)");
  static bool attr = false;
  const int smem = static_cast<int>(sizeof(tcs::Smem));
  if (!attr) {
    cudaFuncSetAttribute(tcs::score_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  const int64_t n_tiles = (B + tcs::GT - 1) / tcs::GT;
  const int grid = static_cast<int>(n_tiles < kNumSMs ? n_tiles : kNumSMs);
  tcs::score_tc_kernel<<<grid, tcs::NT, smem, as_stream(stream)>>>(tab, *dims, params, idx, idx_base, B, z_out,
                                                                    u_out, err_flag);
  note_launches(1);
  return check_launch("kt_score_indices");
}
