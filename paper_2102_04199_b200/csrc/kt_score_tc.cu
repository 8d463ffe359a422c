// kt_score_indices (tensor-core path): the fused candidate scorer with all four
// GEMMs on the 5th-generation tensor cores (tcgen05.mma kind::tf32, accumulators
// in TMEM) in 3xTF32 split precision (A*B ~= Ah*Bh + Ah*Bl + Al*Bh, fp32-level
// accuracy).  Same math and contract as the FFMA2 kernel in kt_score.cu (the
// star-layout algebra is documented there); replaces meta_scores
// (search.py:534-541) = encode_batch -> embed_batch -> head_forward_batch.
//
// Loop-major tiling.  A tile is 128 graphs and TMEM lane g is graph g of the
// tile for every accumulator.  The tile is processed as n_loops chunks; chunk k
// holds loop row k of all 128 graphs:
//   GEMM1  D1[128x32] = X'_k[128x8] * B_k            (A = X'_k in TMEM, 1 K-step x 3)
//   GEMM2  D2[128x32] = ReLU(D1) * W2 = s_k          (A = R_k in TMEM, 4 K-steps x 3)
// so the star readout (sum_k s_k, sum_k ReLU(s_k), max_k s_k per channel) is a
// per-thread running reduction over chunks -- no cross-lane traffic at all.
// After the last chunk each readout thread owns its graph's readout row u:
//   GEMM3  D3[128x64] = U * H0                        (A = U in smem, 8 K-steps x 3)
//   GEMM4  D4[128x64] = ReLU(D3 + b0) * H1            (A = Z1 in TMEM, 8 K-steps x 3)
//   z = ReLU(D4 + b1) . w3 + b3
//
// Folded layer-1 operand.  Of the 12 feature slots of a loop row (model.py:108-112 on
// graphs.py:89-126) six are constants of the loop position k (slots 2, 3, 10, 11, the
// unroll slot 4 up to a 0/1 flag, slot 5 on inner loops), and the touched-derived pairs
// are affine in one another: x8 = a8 x6 + b8 (arith = 2 touched) and x9 = a9 x7 + b9
// (log2 arith = log2 touched + 1), a/b from the feature norm.  So
//   x_k W1 = X'_k B_k,  X' = [x0, x1, x5 (outer rows), x6, x7, unroll flag, 1, 0]
// with B_k (8 x 32) folded per loop row in the prologue (fp64 sums, one rounding):
// rows W1[0], W1[1], W1[5], W1[6] + a8 W1[8], W1[7] + a9 W1[9], the unroll step, and
// the loop row's constant bias.  Exact in real arithmetic; fp32-level in floating point;
// a deterministic function of the features, so equal features still score equal.  GEMM1
// is one K-step instead of two and an X slot is 16 TMEM columns instead of 32.
//
// Warp roles (896 threads = 7 warpgroups, 1 CTA / SM, 512 TMEM
// columns; registers rebalanced per warpgroup with setmaxnreg, which ptxas also takes as
// each region's compile-time budget):
//   WG 0 (warps 0-3)    head: thread = TMEM lane = graph; per tile ReLU(D3 + b0) -> Z1
//                       (TMEM, hi / lo), then ReLU(D4 + b1) . w3 + b3 -> score, top-k key
//   WG 1 (warps 4-7)    encode: thread = graph; per tile the axes' knob digits straight from
//                       the index (two magic-number divisions each); per row the table
//                       slots, the chained fp64 touched / log2 slots, hi/lo split,
//                       tcgen05.st into an X slot
//   WG 2-3 (8-15)       R: thread = TMEM lane = graph; ReLU(D1) split hi/lo into R (TMEM),
//                       one warpgroup per chunk parity
//   WG 4-5 (16-23)      readout, two warps per lane quadrant, 16 channels each: running
//                       sum / ReLU-sum / max over the chunks; at a tile's end U -> TMEM
//   WG 6 (warps 24-26)  MMA issue, one stream each: GEMM1s, GEMM2s, head GEMMs (one
//                       elected lane issues; each waits only on its own operand barriers)
// kt_sa_run runs the same kernel in annealing mode (one CTA, a tile per step; see SaArgs).
// The head warps run a tile's head while the readout warps stream the next tile, so no
// stage of the chunk pipeline ever waits for the head epilogue.
#include "kt_encode.cuh"
#include "kt_tc.cuh"

// Debug timeline (tools/tc_trace.py builds with -DKT_TC_TRACE): clock64 stamps of
// CTA 0's pipeline events.  Compiled out of the product library.
#ifdef KT_TC_TRACE
#define KT_TRACE_N 64
__device__ long long g_kt_trace[32][KT_TRACE_N];
#define TRACE(ev, i)                                              \
  do {                                                            \
    if (blockIdx.x == 0 && (i) < KT_TRACE_N) g_kt_trace[ev][i] = clock64(); \
  } while (0)
extern "C" int kt_debug_trace_read(void* host) {
  return static_cast<int>(cudaMemcpyFromSymbol(host, g_kt_trace, sizeof(g_kt_trace)));
}
#else
#define TRACE(ev, i) \
  do {               \
  } while (0)
#endif

namespace kt {
namespace tcs {

using namespace kt::tc;

constexpr int WG_R = 2, WG_RO = WG_R + 2, WG_MMA = WG_RO + 2;  // warpgroup of each role
constexpr int NWG = WG_MMA + 1;
constexpr int NT = 128 * NWG;  // (roles by warpgroup, see the header)
// per-warpgroup register budgets (setmaxnreg): the NWG warps of an SMSP share its 512
// registers per lane; the launch gives each REG_BASE, the roles rebalance them
constexpr int REG_BASE = (512 / NWG) & ~7;
#ifndef KT_REG_HEAD
#define KT_REG_HEAD 56
#endif
#ifndef KT_REG_ENC
#define KT_REG_ENC 72
#endif
#ifndef KT_REG_R
#define KT_REG_R 56
#endif
#ifndef KT_REG_RO
#define KT_REG_RO 104
#endif
#ifndef KT_REG_MMA
#define KT_REG_MMA 56
#endif
constexpr int REG_HEAD = KT_REG_HEAD, REG_ENC = KT_REG_ENC, REG_R = KT_REG_R, REG_RO = KT_REG_RO, REG_MMA = KT_REG_MMA;
static_assert(REG_HEAD + REG_ENC + 2 * REG_R + 2 * REG_RO + REG_MMA <= NWG * REG_BASE, "register budget");
constexpr int GT = 128;   // graphs per tile (one TMEM lane each)
constexpr int H = 64;
constexpr int XK = 8;     // folded layer-1 operand width (one tf32 K-step)
#ifndef KT_XS
#define KT_XS 4
#endif
constexpr int XS = KT_XS;  // X ring slots
constexpr int N1 = 2;     // D1 buffers
constexpr int NR = 2;     // R buffers
#ifndef KT_N2
#define KT_N2 2
#endif
constexpr int N2 = KT_N2;  // D2 buffers
constexpr int TAB = 448;
// per-role wait flavour: 0 = try_wait (hardware-suspended), N = probe + N ns sleeps
#ifndef KT_SLEEP_MMA
#define KT_SLEEP_MMA 0
#endif
#ifndef KT_SLEEP_R
#define KT_SLEEP_R 0
#endif
#ifndef KT_SLEEP_RO
#define KT_SLEEP_RO 0
#endif
#ifndef KT_SLEEP_ENC
#define KT_SLEEP_ENC 0
#endif
#ifndef KT_HEAD_SLEEP
#define KT_HEAD_SLEEP 64  // ns between probes of the head warpgroup's (long) waits (0: hardware wait)
#endif
#ifndef KT_HEAD_SLEEP_Z
#define KT_HEAD_SLEEP_Z 128  // the head MMA warp's wait for Z1
#endif

// TMEM column map (512 allocated)
constexpr uint32_t T_X = 0;                  // X[s]: hi at 16 s, lo at 16 s + 8
constexpr uint32_t T_D1 = T_X + 16 * XS;     // D1[b] at T_D1 + 32 b
constexpr uint32_t T_R = T_D1 + 32 * N1;     // R[b]: hi at T_R + 64 b, lo at +32
constexpr int D1_STRIDE = 32;
constexpr uint32_t T_D2 = T_R + 64 * NR;     // D2[b] at T_D2 + 32 b
constexpr uint32_t T_D34 = T_D2 + 32 * N2;   // head accumulator: D3, then D4 (64 columns)
constexpr uint32_t T_Z = T_D34 + 64;         // head A operand, U then Z1 = ReLU(D3 + b0): hi at T_Z, lo at +64
static_assert(T_Z + 128 <= 512, "TMEM budget: 512 columns");

// Annealing mode (kt_sa_run, sa_explore search.py:202-254): one CTA, tile t = the chains'
// configurations of step t (lane g = chain g).  The encode warps propose step t's
// neighbours (kt_sa_propose's rule) once the head has accepted step t-1, and the head
// applies the Metropolis test (kt_sa_accept's fp64 arithmetic) to each tile's scores: the
// whole exploration is one launch, the scorer's prologue paid once.  n_steps == 0: off.
struct SaArgs {
  int n_steps, n_chains, n_knobs;
  int cards[KT_MAX_KNOBS];
  long long mult[KT_MAX_KNOBS];
  const int32_t* knob;    // (n_steps, n_chains) draws, the reference's order (search.py:233-237)
  const uint8_t* nudge;
  const int32_t* delta;
  const int32_t* resample;
  const double* u;
  const double* temps;    // (n_steps,) temperature of each step
  const int32_t* cur0;    // (n_chains, n_knobs) starting choices
  int64_t* hist_idx;      // (n_steps + 1, n_chains): row 0 = the starts (input), then each step's proposals
  float* hist_z;          // (n_steps + 1, n_chains) scores
};

struct __align__(1024) Smem {
  float b1h[KT_MAX_LOOPS][32 * XK], b1l[KT_MAX_LOOPS][32 * XK];  // B_k^T (N=32, K=8) per loop row
  float b2h[32 * 32], b2l[32 * 32];  // W2^T
  float b3h[H * H], b3l[H * H];      // H0^T
  float b4h[H * H], b4l[H * H];      // H1^T
  float bias0[H], bias1[H], w3[H], agg[32];
  int2 oi[TAB];
  float4 nrm_o[TAB];
  float2 nrm_i[TAB];
  double2 l2[TAB];  // numpy log2 of (outer, inner) extent
  int tab_off[KT_MAX_AXES + 1];  // start of each axis' choices in the per-choice tables; [n_axes] = total
  // the graphs' config indices per tile (INT64_MIN: padding), tile ti in slot ti % 3, for
  // the head warps (score validity, top-k key); v_free[slot] hands a slot back to the encode
  int64_t vtile[4][GT];
  unsigned int khist[2048];       // first radix digit (key >> 53) of this CTA's top-k keys
  // digit extraction for slot d (axes 0..5, 6 = auto_unroll knob, 7 = explicit knob):
  // choice = (v / dmult[d]) % dcard[d], both divisions by magic multiply
  unsigned long long dm_magic[8], dc_magic[8];
  uint32_t dmult[8], dcard[8];
  int axis_knob[KT_MAX_AXES];
  int auto_vals[4], expl_vals[2];
  int auto_knob, expl_knob;
  uint64_t x_full[XS], x_empty[XS];
  uint64_t d1_full[N1], d1_empty[N1], r_full[NR], r_empty[NR], d2_full[N2], d2_empty[N2];
  uint64_t u_full, uz_empty, z_full, d3_full, d4_full, d4_empty, v_free[4];
  uint64_t acc_done;                            // annealing: the head has accepted a step
  int32_t sa_cur[GT][KT_MAX_KNOBS], sa_nxt[GT][KT_MAX_KNOBS];
  double sa_energy[GT];
  long long sa_mult[KT_MAX_KNOBS];
  int sa_cards[KT_MAX_KNOBS];
  uint32_t tmem_base;
};

__device__ __forceinline__ float relu(float v) { return fmaxf(v, 0.0f); }

// Position in an N-deep ring of buffers: slot i and the parity of its current phase
// (no 64-bit % or / per chunk: N = 3 rings would pay a 64-bit division each time).
template <int N>
struct Ring {
  int i = 0;
  uint32_t ph = 0;
  __device__ __forceinline__ void next() {
    if (++i == N) {
      i = 0;
      ph ^= 1u;
    }
  }
};

template <int NS>
__device__ __forceinline__ void role_wait(uint64_t* bar, uint32_t parity) {
  if constexpr (NS == 0)
    mbar_wait(bar, parity);
  else
    mbar_wait_sleep<NS>(bar, parity);
}

// Warpgroup register reallocation (all four warps of a warpgroup execute it).
template <int N>
__device__ __forceinline__ void setmaxnreg_inc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" : : "n"(N));
}
template <int N>
__device__ __forceinline__ void setmaxnreg_dec();
// to N registers from the launch's REG_BASE, in whichever direction
template <int N>
__device__ __forceinline__ void setmaxnreg() {
  if constexpr (N > REG_BASE) setmaxnreg_inc<N>();
  if constexpr (N < REG_BASE) setmaxnreg_dec<N>();
}
template <int N>
__device__ __forceinline__ void setmaxnreg_dec() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" : : "n"(N));
}

__device__ __forceinline__ uint32_t udiv(uint32_t v, uint32_t d, uint64_t magic) {
  return d == 1 ? v : static_cast<uint32_t>(__umul64hi(static_cast<uint64_t>(v), magic));
}

// B operand = W^T (rows n, K-major) from row-major W[k][n]; K beyond K_src zero.  Split
// into a load half and a store half so that a thread's loads for all operands are in
// flight together (the staging is on the critical path of every launch).
template <int N, int K>
struct OperandRegs {
  static constexpr int IT = (N * K + NT - 1) / NT;
  float v[IT];
};
template <int N, int K>
__device__ __forceinline__ void load_operand(OperandRegs<N, K>& r, const float* W, int K_src, int tid) {
#pragma unroll
  for (int i = 0; i < OperandRegs<N, K>::IT; ++i) {
    const int e = tid + i * NT, k = e / N, n = e - k * N;  // n fastest: coalesced rows of W
    r.v[i] = e < N * K && k < K_src ? __ldg(W + k * N + n) : 0.0f;
  }
}
__device__ __forceinline__ void store_split(float* hi, float* lo, int off, float v) {
  const float h = tf32_hi(v);
  hi[off] = h;
  lo[off] = v - h;
}
template <int N, int K>
__device__ __forceinline__ void store_operand(const OperandRegs<N, K>& r, float* hi, float* lo, int tid) {
  constexpr int IT = OperandRegs<N, K>::IT;
#pragma unroll
  for (int i = 0; i < IT; ++i) {
    const int e = tid + i * NT, k = e / N, n = e - k * N;
    if (e < N * K) store_split(hi, lo, kmajor_offset(n, k, K) >> 2, r.v[i]);
  }
}

// 16 values -> hi (truncated tf32) / lo (exact remainder) halves, packed fp32x2 subtractions
__device__ __forceinline__ void split16(const float* v, float* hi, float* lo) {
#pragma unroll
  for (int j = 0; j < 16; j += 2) {
    const float2 t = make_float2(tf32_trunc(v[j]), tf32_trunc(v[j + 1]));
    const float2 l = fsub2(make_float2(v[j], v[j + 1]), t);
    hi[j] = t.x;
    hi[j + 1] = t.y;
    lo[j] = l.x;
    lo[j + 1] = l.y;
  }
}

// knob digit d of a (32-bit) config index: (v / dmult[d]) % dcard[d] (kernels.py:278-286)
__device__ __forceinline__ int knob_digit(const Smem& S, uint32_t v, int d) {
  const uint32_t qd = udiv(v, S.dmult[d], S.dm_magic[d]);
  const uint32_t c = S.dcard[d];
  return static_cast<int>(qd - udiv(qd, c, S.dc_magic[d]) * c);
}

struct EncodeCtx {
  const int64_t* idx;
  const uint32_t* idx32;
  int64_t idx_base, B, my_tiles;
  uint64_t size;
  int32_t* err;
  uint32_t tmem, lane;
  int g;
  double m6, r6, m7, r7;  // touched-derived slots: fp64 (x - mean) * (1 / std)
  const SaArgs* sa;       // annealing mode (n_steps > 0), else unused
};

// Annealing mode: chain g's configuration for tile ti -- the start (ti = 0), else the
// neighbour of step ti - 1 proposed from the accepted chain state (kt_sa_propose's rule,
// search.py:232-241), recorded in the history.
__device__ __forceinline__ int64_t sa_propose(Smem& S, const EncodeCtx& X, int64_t ti) {
  const SaArgs& A = *X.sa;
  const int g = X.g, n = A.n_chains;
  // the step's draws are inputs: loaded before waiting for the previous step's acceptance
  const int64_t o = (ti - 1) * n + g;
  const bool mine = ti > 0 && g < n;
  const int kn = mine ? A.knob[o] : 0, dl = mine ? A.delta[o] : 0, rs = mine ? A.resample[o] : 0;
  const bool nd = mine && A.nudge[o];
  if (ti > 0) mbar_wait(&S.acc_done, static_cast<uint32_t>((ti - 1) & 1));
  if (g >= n) return INT64_MIN;
  if (ti == 0) return A.hist_idx[g];
  int64_t id = 0;
  for (int j = 0; j < A.n_knobs; ++j) {
    int v = S.sa_cur[g][j];
    if (j == kn) {
      const int stepped = min(max(v + dl, 0), S.sa_cards[j] - 1);
      v = nd ? stepped : rs;
    }
    S.sa_nxt[g][j] = v;
    id += static_cast<int64_t>(v) * S.sa_mult[j];
  }
  A.hist_idx[ti * n + g] = id;
  return id;
}

// A tile's per-graph encode state: the config index, the unroll knobs, the axes' table
// entries and extents, and the running touched / log2 touched.
template <int NA>
struct EncodeTile {
  float one;  // 1 for a valid config, 0 for padding / an invalid index (all-zero rows)
  bool unr_on;
  int autov;
  int e[NA];
  int2 oi[NA];
  double t, lt;
};

// The unroll knobs' values (used by the inner loops' rows) from a 32-bit config index.
template <int NA>
__device__ __forceinline__ void encode_knobs(Smem& S, uint32_t v, EncodeTile<NA>& st) {
  // branch-free: a slot without a knob has mult = card = 1 (host tables), so its digit is 0
  // and every digit's loads and multiplies are independent
  const int av = S.auto_vals[knob_digit(S, v, 6)], ev = S.expl_vals[knob_digit(S, v, 7)];
  st.autov = S.auto_knob >= 0 ? av : 0;
  const int expl = S.expl_knob >= 0 ? ev : 0;
  st.unr_on = expl != 0 && st.autov > 0;
}

// Axis a's choice entry and (outer, inner) extents.
template <int NA>
__device__ __forceinline__ void encode_axis(Smem& S, uint32_t v, EncodeTile<NA>& st, int a) {
  st.e[a] = S.tab_off[a] + knob_digit(S, v, a);
  st.oi[a] = S.oi[st.e[a]];
}

__device__ __forceinline__ bool index_ok(const EncodeCtx& X, int64_t v64) {
  return v64 >= 0 && static_cast<uint64_t>(v64) < X.size;
}

// Tile ti's per-graph state that does not need the digits: the index published for the
// head, the padding / invalid flag, the chain's start.
template <int NA>
__device__ __forceinline__ void encode_begin(Smem& S, const EncodeCtx& X, int64_t ti, int64_t v64, EncodeTile<NA>& st) {
  const bool ok = index_ok(X, v64);
  mbar_wait(&S.v_free[ti & 3], static_cast<uint32_t>(((ti >> 2) & 1) ^ 1));  // head of tile ti-4 read it
  if (X.g == 0) TRACE(25, ti);
  S.vtile[ti & 3][X.g] = v64;
  if (v64 != INT64_MIN && !ok) atomicOr(X.err, 1);
  st.one = ok ? 1.0f : 0.0f;
  st.t = 1.0;
  st.lt = 0.0;
}

template <int NA>
__device__ __forceinline__ void encode_prepare(Smem& S, const EncodeCtx& X, int64_t ti, int64_t v64,
                                               EncodeTile<NA>& st) {
  encode_begin<NA>(S, X, ti, v64, st);
  const uint32_t v = index_ok(X, v64) ? static_cast<uint32_t>(v64) : 0u;
  encode_knobs<NA>(S, v, st);
#pragma unroll
  for (int a = 0; a < NA; ++a) encode_axis<NA>(S, v, st, a);
  if (X.g == 0) TRACE(31, ti);
}

// Row c (loop k = 2 NA - 1 - c, innermost first) of a tile -> hi / lo split -> X slot of
// chunk q (tcgen05.st) -> GEMM1.  The row's table slots (normalised extent / log2 extent,
// stride for an outer loop, unroll flag for an inner one) are gathered by its choice entry
// e; the two chained slots come from the running touched / log2 touched.  touched -- the
// product of the extents of the loops inside loop k, multiplied innermost outward as
// np.cumprod(e[::-1]) does -- accumulates exactly in fp64, and log2(touched) as the sum of
// the numpy log2 of those extents (log2(arith) = log2(2 touched) = that + 1).  Both are
// functions of the extent vector only, so configs with equal features score identically.
// All of it is computed before the X-slot wait, so from the fifth row of a tile on it
// overlaps the wait for GEMM1 to free a slot instead of delaying the tile's first rows.
template <int NA>
__device__ __forceinline__ void encode_hand_over(Smem& S, const EncodeCtx& X, EncodeTile<NA>& st, int c,
                                                 int64_t q) {
  const int k = 2 * NA - 1 - c;
  const bool level = k >= NA;  // inner loop
  const int a = level ? k - NA : k;
  float x[XK];
  x[3] = static_cast<float>((st.t - X.m6) * X.r6);
  x[4] = static_cast<float>((st.lt - X.m7) * X.r7);
  st.t *= static_cast<double>(level ? st.oi[a].y : st.oi[a].x);
  st.lt += reinterpret_cast<const double*>(&S.l2[st.e[a]])[level ? 1 : 0];
  if (level) {
    const float2 ni = S.nrm_i[st.e[a]];
    x[0] = ni.x;
    x[1] = ni.y;
    x[2] = 0.0f;
    x[5] = st.unr_on && st.oi[a].y <= st.autov ? 1.0f : 0.0f;  // unroll flag
  } else {
    const float4 no = S.nrm_o[st.e[a]];
    x[0] = no.x;
    x[1] = no.y;
    x[2] = no.z;  // stride slot
    x[5] = 0.0f;
  }
#pragma unroll
  for (int f = 0; f < 6; ++f) x[f] *= st.one;  // padding / invalid rows: all zero
  x[6] = st.one;
  x[7] = 0.0f;
  float hl[16];
#pragma unroll
  for (int f = 0; f < XK; f += 2) {
    hl[f] = tf32_trunc(x[f]);
    hl[f + 1] = tf32_trunc(x[f + 1]);
    const float2 l = fsub2(make_float2(x[f], x[f + 1]), make_float2(hl[f], hl[f + 1]));
    hl[XK + f] = l.x;
    hl[XK + f + 1] = l.y;
  }
  const int s = static_cast<int>(q % XS);
  if (X.g == 0) TRACE(20, q);
  role_wait<KT_SLEEP_ENC>(&S.x_empty[s], static_cast<uint32_t>(((q / XS) & 1) ^ 1));
  __syncwarp();
  if (X.g == 0) TRACE(21, q);
  tc_fence_after();
  tmem_st16(X.tmem + X.lane + T_X + 16 * s, hl);
  tmem_wait_st();
  tc_fence_before();
  warp_arrive(&S.x_full[s]);
  if (X.g == 0) TRACE(0, q);
}

// The encode warps' loop, specialised on the axis count so every per-axis / per-row
// quantity lives in registers.  Per tile, the digits and table entries (prepare), then the
// rows, each computed and handed to GEMM1 one X slot at a time.
template <int NA>
__device__ __forceinline__ void encode_loop(Smem& S, const EncodeCtx& X) {
  constexpr int C = 2 * NA;
  auto index_of = [&](int64_t ti) -> int64_t {  // this thread's config index in tile ti
    const int64_t gi = (blockIdx.x + ti * gridDim.x) * GT + X.g;
    if (ti >= X.my_tiles || gi >= X.B) return INT64_MIN;  // padding row
    // idx32 may point at pinned host memory (zero-copy: the kernel's reads are the H2D transfer)
    return X.idx32 ? static_cast<int64_t>(X.idx32[gi]) : X.idx ? __ldcs(X.idx + gi) : X.idx_base + gi;
  };
  if (X.my_tiles <= 0) return;
  int64_t q = 0;
  const bool sa = X.sa->n_steps > 0;
  int64_t v_next = sa ? 0 : index_of(0);
  for (int64_t ti = 0; ti < X.my_tiles; ++ti) {
    EncodeTile<NA> st;
    if (X.g == 0) TRACE(24, ti);
    encode_prepare<NA>(S, X, ti, sa ? sa_propose(S, X, ti) : v_next, st);
    if (!sa) v_next = index_of(ti + 1);  // next tile's index load in flight during this tile
    if (X.g == 0) TRACE(26, ti);
#pragma unroll
    for (int c = 0; c < C; ++c, ++q) {
      if (X.g == 0) TRACE(19, q);
      encode_hand_over<NA>(S, X, st, c, q);
    }
  }
}

__global__ void __launch_bounds__(NT, 1)
score_tc_kernel(const kt_spec_table* __restrict__ tab, kt_dims dims, const float* __restrict__ params,
                const int64_t* __restrict__ idx, const uint32_t* __restrict__ idx32, int64_t idx_base, int64_t B,
                float* __restrict__ z_out, float* __restrict__ u_out, unsigned long long* __restrict__ keys_out,
                unsigned int* __restrict__ key_hist, int32_t* __restrict__ err, int flags,
                const __grid_constant__ SaArgs sa) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>(smem_raw);
  const kt_spec_table& T = *tab;
  if (threadIdx.x == 0) TRACE(27, 0);  // kernel entry
  const int tid = threadIdx.x, warp = tid >> 5;
  if (T.space_size > 0xffffffffull) {  // 32-bit digit arithmetic below; larger spaces use kt_embed_csr
    if (blockIdx.x == 0 && tid == 0) atomicOr(err, 2);
    return;
  }

  // ---- setup, part 1: constant tables, barriers, TMEM (overlaps the previous kernel) --
  const int na = T.n_axes, n_loops = T.n_loops;
  if (tid < KT_MAX_AXES) S.axis_knob[tid] = T.axis_knob[tid];
  if (tid < 4) S.auto_vals[tid] = T.auto_vals[tid];
  if (tid < 2) S.expl_vals[tid] = T.expl_vals[tid];
  if (tid < 8) {  // digit divisors, computed on the host (graphs.build_spec_table)
    S.dmult[tid] = T.digit_mult[tid];
    S.dcard[tid] = T.digit_card[tid];
    S.dm_magic[tid] = T.digit_mult_magic[tid];
    S.dc_magic[tid] = T.digit_card_magic[tid];
    S.tab_off[tid < KT_MAX_AXES + 1 ? tid : KT_MAX_AXES] = T.choice_off[tid < KT_MAX_AXES + 1 ? tid : KT_MAX_AXES];
    if (tid == 0) {
      S.auto_knob = T.auto_knob;
      S.expl_knob = T.expl_knob;
    }
  }
  if (tid == 0) {
    for (int s = 0; s < XS; ++s) {
      mbar_init(&S.x_full[s], 4);
      mbar_init(&S.x_empty[s], 1);
    }
    for (int b = 0; b < N1; ++b) {
      mbar_init(&S.d1_full[b], 1);
      mbar_init(&S.d1_empty[b], 4);
    }
    for (int b = 0; b < NR; ++b) {
      mbar_init(&S.r_full[b], 4);
      mbar_init(&S.r_empty[b], 1);
    }
    for (int b = 0; b < N2; ++b) {
      mbar_init(&S.d2_full[b], 1);
      mbar_init(&S.d2_empty[b], 8);
    }
    mbar_init(&S.u_full, 8);
    mbar_init(&S.uz_empty, 1);
    mbar_init(&S.z_full, 4);
    mbar_init(&S.d3_full, 1);
    mbar_init(&S.d4_full, 1);
    mbar_init(&S.d4_empty, 4);
    mbar_init(&S.acc_done, 4);
    for (int i = 0; i < 4; ++i) mbar_init(&S.v_free[i], 4);
  }
  if (warp == 4 * WG_MMA) tmem_alloc(&S.tmem_base, 512);
  if (key_hist)
    for (int i = tid; i < 2048; i += NT) S.khist[i] = 0;
  const bool sa_mode = sa.n_steps > 0;
  if (sa_mode) {
    if (tid < sa.n_knobs) {
      S.sa_cards[tid] = sa.cards[tid];
      S.sa_mult[tid] = sa.mult[tid];
    }
  }
  __syncthreads();
  // per-choice tables, one flat pass over every axis' entries (loads independent across threads)
  for (int e = tid; e < S.tab_off[na]; e += NT) {
    int a = 0;
    while (a + 1 < na && S.tab_off[a + 1] <= e) ++a;
    const int c = e - S.tab_off[a];
    S.oi[e] = make_int2(T.outer[a][c], T.inner[a][c]);
    S.nrm_o[e] = make_float4(T.nrm_ext[a][c], T.nrm_log2ext[a][c], T.nrm_stride[a][c], 0.f);
    S.nrm_i[e] = make_float2(T.nrm_ext[na + a][c], T.nrm_log2ext[na + a][c]);
    S.l2[e] = make_double2(T.raw_log2[0][a][c], T.raw_log2[1][a][c]);
  }
  if (threadIdx.x == 0) TRACE(28, 0);  // table prologue done
  // PDL: everything above reads only the constant spec table.  The parameters, indices,
  // outputs and key_hist belong to the stream order from here on (a predecessor may write
  // the parameters, e.g. kt_maml_step / kt_sgd in place) -- unless the caller vouches that
  // the preceding kernel leaves the parameters alone (KT_SCORE_PARAMS_STABLE): then the
  // operand staging below overlaps it too and only the indices wait.
  const bool params_stable = (flags & KT_SCORE_PARAMS_STABLE) != 0;
  if (!params_stable) {
    pdl_wait();
    pdl_launch_dependents();
  }

  // ---- setup, part 2: operands from the parameters --------------------------------
  {
    OperandRegs<32, 32> r2;
    OperandRegs<H, H> r3, r4;
    load_operand(r2, params + dims.off_gcn[1], 32, tid);
    load_operand(r3, params + dims.off_hw[0], H, tid);
    load_operand(r4, params + dims.off_hw[1], H, tid);
    // folded layer-1 operand B_k (see the header), thread = (loop row k, channel n)
    if (tid < n_loops * 32) {
      const int k = tid >> 5, n = tid & 31;
      const float* W1 = params + dims.off_gcn[0];
      double w[KT_F];
#pragma unroll
      for (int f = 0; f < KT_F; ++f) w[f] = static_cast<double>(__ldg(W1 + f * 32 + n));
      const bool inner = k >= na;
      const double a8 = 2.0 * T.fstd[6] / T.fstd[8], b8 = (2.0 * T.fmean[6] - T.fmean[8]) / T.fstd[8];
      const double a9 = T.fstd[7] / T.fstd[9], b9 = (T.fmean[7] + 1.0 - T.fmean[9]) / T.fstd[9];
      const double c4 = T.nrm_const[k][4];
      double bias = T.nrm_const[k][2] * w[2] + T.nrm_const[k][3] * w[3] + c4 * w[4] + T.nrm_const[k][10] * w[10] +
                    T.nrm_const[k][11] * w[11] + b8 * w[8] + b9 * w[9];
      if (inner) bias += T.nrm_const[k][5] * w[5];
      const double rows[XK] = {w[0], w[1], inner ? 0.0 : w[5], w[6] + a8 * w[8], w[7] + a9 * w[9],
                               inner ? (static_cast<double>(T.nrm_unroll1[k]) - c4) * w[4] : 0.0, bias, 0.0};
#pragma unroll
      for (int f = 0; f < XK; ++f)
        store_split(S.b1h[k], S.b1l[k], kmajor_offset(n, f, XK) >> 2, static_cast<float>(rows[f]));
    }
    store_operand(r2, S.b2h, S.b2l, tid);
    store_operand(r3, S.b3h, S.b3l, tid);
    store_operand(r4, S.b4h, S.b4l, tid);
  }
  if (tid < H) {
    S.bias0[tid] = params[dims.off_hb[0] + tid];
    S.bias1[tid] = params[dims.off_hb[1] + tid];
    S.w3[tid] = params[dims.off_hw[2] + tid];
  }
  if (tid < 32) S.agg[tid] = params[dims.off_agg + tid];
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (params_stable) {
    pdl_wait();
    pdl_launch_dependents();
  }
  if (sa_mode) {  // the starting choices, after the programmatic wait (a predecessor may write them)
    for (int e = tid; e < sa.n_chains * sa.n_knobs; e += NT) S.sa_cur[e / sa.n_knobs][e % sa.n_knobs] = sa.cur0[e];
    __syncthreads();
  }
  if (threadIdx.x == 0) TRACE(30, 0);  // operand prologue done
  const uint32_t tmem = S.tmem_base;
  const int64_t n_tiles = (B + GT - 1) / GT;
  const int64_t my_tiles = blockIdx.x < n_tiles ? (n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  // one tile per CTA (small batches) or annealing (every tile waits on the previous one's
  // head): the head's waits are on the critical path, no sleeping
  const bool one_tile = my_tiles <= 1 || sa_mode;
  const int C = n_loops;  // chunks per tile
  const int64_t n_chunks = my_tiles * C;
  const uint64_t size = T.space_size;

  const int wg = warp >> 2;  // 0 head, 1 encode, WG_R.. R, WG_RO.. readout, WG_MMA MMA issue
  if (wg == 1) {
    setmaxnreg<REG_ENC>();
    // ===================== encode: thread = graph; one folded operand row per chunk =========
    const int g = tid - 128;
    // touched-derived slots in fp64 with reciprocal scales: within 1 fp64 ulp of the
    // IEEE (x - mean) / std of model.py:108-112 before the single cast to fp32
    const double m6 = T.fmean[6], r6 = 1.0 / T.fstd[6], m7 = T.fmean[7], r7 = 1.0 / T.fstd[7];
    const EncodeCtx X{idx, idx32, idx_base, B, my_tiles, size, err, tmem,
                      static_cast<uint32_t>((g & ~31) << 16), g, m6, r6, m7, r7, &sa};
    switch (na) {  // (kernels.py: 4 axes for 1-D ops, 5 depthwise, 6 the 2-D ops)
      case 6: encode_loop<6>(S, X); break;
      case 5: encode_loop<5>(S, X); break;
      case 4: encode_loop<4>(S, X); break;
      case 3: encode_loop<3>(S, X); break;
      case 2: encode_loop<2>(S, X); break;
      default: encode_loop<1>(S, X); break;
    }
  } else if (wg == WG_MMA) {
    setmaxnreg<REG_MMA>();
    // ===================== MMA: fixed issue order, blocking waits, one elected lane issues =====
    // Each wait parks the warp in hardware until the phase completes (no polling: a
    // polling warp costs its SMSP neighbours issue slots).
    const uint32_t id32 = idesc_tf32(128, 32), id64 = idesc_tf32(128, 64);
    auto wait_bar = [&](uint64_t* bar, uint32_t parity) {
      role_wait<KT_SLEEP_MMA>(bar, parity);
      __syncwarp();
      tc_fence_after();
    };
    // Three independent issue streams, one warp each: tcgen05.commit tracks the MMAs of
    // the issuing thread only, so GEMM1s, GEMM2s and the head GEMMs need no common
    // program order -- their data dependencies all go through the ring barriers.
    if (warp == 4 * WG_MMA) {
      int c = 0;  // chunk within the tile -> loop row k = C - 1 - c (the encode order)
      Ring<XS> rx;
      Ring<N1> r1;
      for (int64_t q = 0; q < n_chunks; ++q, rx.next(), r1.next()) {
        const int s = rx.i, b = r1.i;
        if ((tid & 31) == 0) TRACE(22, q);
        wait_bar(&S.x_full[s], rx.ph);
        wait_bar(&S.d1_empty[b], r1.ph ^ 1);
        if ((tid & 31) == 0) TRACE(23, q);
        const uint32_t xh = tmem + T_X + 16 * s, xl = xh + XK, d = tmem + T_D1 + D1_STRIDE * b;
        const int k = C - 1 - c;
        if (elect_one()) {
          mma_tf32_ts(d, xh, kdesc(S.b1h[k], XK, 0), id32, 0);
          mma_tf32_ts(d, xh, kdesc(S.b1l[k], XK, 0), id32, 1);
          mma_tf32_ts(d, xl, kdesc(S.b1h[k], XK, 0), id32, 1);
          mma_commit(&S.x_empty[s]);
          mma_commit(&S.d1_full[b]);
          TRACE(1, q);
        }
        __syncwarp();
        if (++c == C) c = 0;
      }
    } else if (warp == 4 * WG_MMA + 1) {
      Ring<NR> rr;
      Ring<N2> r2;
      for (int64_t q = 0; q < n_chunks; ++q, rr.next(), r2.next()) {
        const int b = rr.i, b2 = r2.i;
        if ((tid & 31) == 0) TRACE(17, q);
        wait_bar(&S.r_full[b], rr.ph);
        wait_bar(&S.d2_empty[b2], r2.ph ^ 1);
        if ((tid & 31) == 0) TRACE(18, q);
        const uint32_t rh = tmem + T_R + 64 * b, rl = rh + 32, d = tmem + T_D2 + 32 * b2;
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            mma_tf32_ts(d, rh + 8 * kk, kdesc(S.b2h, 32, kk), id32, kk > 0);
            mma_tf32_ts(d, rh + 8 * kk, kdesc(S.b2l, 32, kk), id32, 1);
            mma_tf32_ts(d, rl + 8 * kk, kdesc(S.b2h, 32, kk), id32, 1);
          }
          mma_commit(&S.r_empty[b]);
          mma_commit(&S.d2_full[b2]);
          TRACE(2, q);
        }
        __syncwarp();
      }
    } else if (warp == 4 * WG_MMA + 2) {
      for (int64_t t = 0; t < my_tiles; ++t) {
        const uint32_t ph = static_cast<uint32_t>(t & 1);
        // GEMM3: U (TMEM) x H0 into the head accumulator, once the head warps have read
        // D4 of the previous tile out of it
        if (one_tile)
          mbar_wait(&S.u_full, ph);
        else
          role_wait<KT_HEAD_SLEEP>(&S.u_full, ph);
        wait_bar(&S.d4_empty, ph ^ 1);
        const uint32_t ah = tmem + T_Z, al = ah + 64;
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            mma_tf32_ts(tmem + T_D34, ah + 8 * kk, kdesc(S.b3h, H, kk), id64, kk > 0);
            mma_tf32_ts(tmem + T_D34, ah + 8 * kk, kdesc(S.b3l, H, kk), id64, 1);
            mma_tf32_ts(tmem + T_D34, al + 8 * kk, kdesc(S.b3h, H, kk), id64, 1);
          }
          mma_commit(&S.d3_full);
          TRACE(3, t);
        }
        __syncwarp();
        // GEMM4: Z1 (TMEM, written over U) x H1, same accumulator (the head warps have read D3)
        if (one_tile)
          mbar_wait(&S.z_full, ph);
        else
          role_wait<KT_HEAD_SLEEP_Z>(&S.z_full, ph);
        __syncwarp();
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            mma_tf32_ts(tmem + T_D34, ah + 8 * kk, kdesc(S.b4h, H, kk), id64, kk > 0);
            mma_tf32_ts(tmem + T_D34, ah + 8 * kk, kdesc(S.b4l, H, kk), id64, 1);
            mma_tf32_ts(tmem + T_D34, al + 8 * kk, kdesc(S.b4h, H, kk), id64, 1);
          }
          mma_commit(&S.d4_full);
          mma_commit(&S.uz_empty);  // the readout may write the next tile's U
          TRACE(4, t);
        }
        __syncwarp();
      }
    }
  } else if (wg >= WG_R && wg < WG_RO) {
    setmaxnreg<REG_R>();
    // ===================== R: ReLU(D1) -> R (hi, lo) in TMEM; thread = lane = graph ===============
    const int quad = warp & 3;
    const int g = 32 * quad + (tid & 31);
    const uint32_t lane = static_cast<uint32_t>((32 * quad) << 16);
    // two R warpgroups, chunks of parity wg - WG_R each: buffer (q % 2) is theirs alone
    static_assert(N1 == 2 && NR == 2, "R parity split needs 2-deep D1 / R rings");
    Ring<1> r1, rr;
    r1.i = rr.i = wg - WG_R;
    for (int64_t q = wg - WG_R; q < n_chunks; q += 2, r1.ph ^= 1u, rr.ph ^= 1u) {
      const int b1 = r1.i, b = rr.i;
      role_wait<KT_SLEEP_R>(&S.d1_full[b1], r1.ph);
      __syncwarp();
      if (g == 0) TRACE(5, q);
      tc_fence_after();
      float v[32];
      tmem_ld16(tmem + lane + T_D1 + D1_STRIDE * b1, v);
      tmem_ld16(tmem + lane + T_D1 + D1_STRIDE * b1 + 16, v + 16);
      tmem_wait_ld();
      if (g == 0) TRACE(13, q);
      tc_fence_before();
      warp_arrive(&S.d1_empty[b1]);
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = relu(v[j]);
      role_wait<KT_SLEEP_R>(&S.r_empty[b], rr.ph ^ 1);  // GEMM2 of q-NR read R[b]
      __syncwarp();
      if (g == 0) TRACE(14, q);
      tc_fence_after();
#pragma unroll
      for (int h = 0; h < 4; ++h) {  // hi in place (v), lo alongside: 40 live values
        float lo[8];
#pragma unroll
        for (int j = 0; j < 8; j += 2) {
          const float2 t = make_float2(tf32_trunc(v[8 * h + j]), tf32_trunc(v[8 * h + j + 1]));
          const float2 l = fsub2(make_float2(v[8 * h + j], v[8 * h + j + 1]), t);
          v[8 * h + j] = t.x;
          v[8 * h + j + 1] = t.y;
          lo[j] = l.x;
          lo[j + 1] = l.y;
        }
        tmem_st8(tmem + lane + T_R + 64 * b + 8 * h, v + 8 * h);
        tmem_st8(tmem + lane + T_R + 64 * b + 32 + 8 * h, lo);
      }
      if (g == 0) TRACE(15, q);
      tmem_wait_st();
      if (g == 0) TRACE(16, q);
      tc_fence_before();
      warp_arrive(&S.r_full[b]);
      if (g == 0) TRACE(6, q);
    }
  } else if (wg >= WG_RO && wg < WG_MMA) {
    setmaxnreg<REG_RO>();
    // ===================== readout: thread = lane = graph, 16 channels =========================
    const int quad = warp & 3, eh = wg - WG_RO;

    const int g = 32 * quad + (tid & 31);
    const uint32_t lane = static_cast<uint32_t>((32 * quad) << 16);
    const float c_t = static_cast<float>(5.0 / 12.0);
    const float c_ft = static_cast<float>(5.0 / (6.0 * sqrt(6.0)) + 5.0 / 12.0);
    const float c_r = static_cast<float>(1.0 / sqrt(18.0 * (T.n_pairs + 1)));
    const bool tr = g == 0 && eh == 0;
    float2 tot[8], rs[8];  // per channel: sum of s, sum of |s| (sum relu(s) = (sum s + sum |s|) / 2)
    float mx[16];
    int kc = 0;       // chunk index within the current tile (no 64-bit % / on this path)
    int64_t ti = 0;   // local tile index
    for (int64_t p = 0; p < n_chunks; ++p) {
      const int b = static_cast<int>(p % N2);
      if (kc == 0) {
#pragma unroll
        for (int j = 0; j < 8; ++j) tot[j] = rs[j] = make_float2(0.0f, 0.0f);
#pragma unroll
        for (int j = 0; j < 16; ++j) mx[j] = 0.0f;  // max_k ReLU(s_k) = max(0, max_k s_k)
      }
      role_wait<KT_SLEEP_RO>(&S.d2_full[b], static_cast<uint32_t>((p / N2) & 1));
      __syncwarp();
      if (tr) TRACE(7, p);
      tc_fence_after();
      {
        float v[16];
        tmem_ld16(tmem + lane + T_D2 + 32 * b + 16 * eh, v);
        tmem_wait_ld();
        tc_fence_before();
        warp_arrive(&S.d2_empty[b]);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float2 s2 = make_float2(v[2 * i], v[2 * i + 1]);
          tot[i] = fadd2(tot[i], s2);
          rs[i].x += fabsf(s2.x);  // sum |s| (FADD with the |.| operand modifier); sum relu = (sum s + sum |s|) / 2
          rs[i].y += fabsf(s2.y);
          mx[2 * i] = fmaxf(mx[2 * i], s2.x);
          mx[2 * i + 1] = fmaxf(mx[2 * i + 1], s2.y);
        }
      }
      if (tr) TRACE(8, p);
      if (++kc < C) continue;
      kc = 0;
      // ---- tile ti done: readout row U -> TMEM (the head GEMM's A operand), this warp's
      // 16 sum and 16 max channels ----
      const int64_t gi = (blockIdx.x + ti * gridDim.x) * GT + g;
      // (ordered so that the accumulators die early: sum part first, then max part)
      float4* urow = u_out && gi < B ? reinterpret_cast<float4*>(u_out + gi * H) : nullptr;
      mbar_wait(&S.uz_empty, static_cast<uint32_t>((ti & 1) ^ 1));  // GEMM4 of tile ti-1 read Z1
      __syncwarp();
      tc_fence_after();
      {
        float u[16], lo[16];
#pragma unroll
        for (int jl = 0; jl < 16; ++jl) {
          const float tj = (jl & 1) ? tot[jl >> 1].y : tot[jl >> 1].x;
          const float rj = 0.5f * (((jl & 1) ? rs[jl >> 1].y : rs[jl >> 1].x) + tj);
          u[jl] = S.agg[16 * eh + jl] * (relu(c_r * tj) + c_ft * rj);
        }
        if (urow)
#pragma unroll
          for (int jq = 0; jq < 4; ++jq) urow[4 * eh + jq] = make_float4(u[4 * jq], u[4 * jq + 1], u[4 * jq + 2], u[4 * jq + 3]);
#pragma unroll
        for (int j = 0; j < 16; ++j) {  // in-place split: u -> hi, lo
          const float h = tf32_trunc(u[j]);
          lo[j] = u[j] - h;
          u[j] = h;
        }
        tmem_st16(tmem + lane + T_Z + 16 * eh, u);
        tmem_st16(tmem + lane + T_Z + 64 + 16 * eh, lo);
      }
      {
        float u[16], lo[16];
#pragma unroll
        for (int jl = 0; jl < 16; ++jl)
          u[jl] = fmaxf(relu(c_r * ((jl & 1) ? tot[jl >> 1].y : tot[jl >> 1].x)), c_t * mx[jl]);
        if (urow)
#pragma unroll
          for (int jq = 0; jq < 4; ++jq)
            urow[8 + 4 * eh + jq] = make_float4(u[4 * jq], u[4 * jq + 1], u[4 * jq + 2], u[4 * jq + 3]);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float h = tf32_trunc(u[j]);
          lo[j] = u[j] - h;
          u[j] = h;
        }
        tmem_st16(tmem + lane + T_Z + 32 + 16 * eh, u);
        tmem_st16(tmem + lane + T_Z + 96 + 16 * eh, lo);
      }
      tmem_wait_st();
      tc_fence_before();
      warp_arrive(&S.u_full);
      if (tr) TRACE(9, ti);
      ++ti;
    }
  } else {
    setmaxnreg<REG_HEAD>();
    // ===================== head: thread = lane = graph, all 64 channels ===========================
    const int quad = warp;
    const int g = 32 * quad + (tid & 31);
    const uint32_t lane = static_cast<uint32_t>((32 * quad) << 16);
    const float b3 = params[dims.off_hb[2]];
    const bool tr = g == 0;
    for (int64_t ti = 0; ti < my_tiles; ++ti) {
      const uint32_t ph = static_cast<uint32_t>(ti & 1);
      // annealing: this step's uniform and temperature, loaded ahead of the scores
      double sa_u = 0.0, sa_t = 1.0;
      if (sa_mode && ti > 0 && g < sa.n_chains) {
        sa_u = sa.u[(ti - 1) * sa.n_chains + g];
        sa_t = sa.temps[ti - 1];
      }
      if (one_tile)
        mbar_wait(&S.d3_full, ph);
      else
        role_wait<KT_HEAD_SLEEP>(&S.d3_full, ph);
      __syncwarp();
      if (tr) TRACE(10, ti);
      tc_fence_after();
      const int64_t v = S.vtile[ti & 3][g];  // this tile's indices; the slot goes back to the encode
      warp_arrive(&S.v_free[ti & 3]);
#pragma unroll
      for (int h = 0; h < 4; ++h) {  // D3 columns 16 h .. 16 h + 15 -> Z1 = ReLU(D3 + b0), hi / lo
        float z[16], hi[16], lo[16];
        tmem_ld16(tmem + lane + T_D34 + 16 * h, z);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 16; ++i) z[i] = relu(z[i] + S.bias0[16 * h + i]);
        split16(z, hi, lo);
        tmem_st16(tmem + lane + T_Z + 16 * h, hi);
        tmem_st16(tmem + lane + T_Z + 64 + 16 * h, lo);
      }
      tmem_wait_st();
      tc_fence_before();
      warp_arrive(&S.z_full);
      if (one_tile)
        mbar_wait(&S.d4_full, ph);
      else
        role_wait<KT_HEAD_SLEEP>(&S.d4_full, ph);
      __syncwarp();
      if (tr) TRACE(11, ti);
      tc_fence_after();
      float acc0 = 0.0f, acc1 = 0.0f;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float v[32];
        tmem_ld16(tmem + lane + T_D34 + 32 * h, v);
        tmem_ld16(tmem + lane + T_D34 + 32 * h + 16, v + 16);
        tmem_wait_ld();
        float acc = 0.0f;
#pragma unroll
        for (int j = 0; j < 32; ++j) acc = fmaf(relu(v[j] + S.bias1[32 * h + j]), S.w3[32 * h + j], acc);
        if (h == 0) acc0 = acc; else acc1 = acc;
      }
      tc_fence_before();
      warp_arrive(&S.d4_empty);
      if (sa_mode) {  // history, then the Metropolis test of step ti - 1 (kt_sa_accept, search.py:246-251)
        const int n = sa.n_chains;
        if (g < n) {
          const bool ok = v >= 0 && static_cast<uint64_t>(v) < size;
          const float zf = ok ? (b3 + acc0) + acc1 : __int_as_float(0x7fc00000);
          sa.hist_z[ti * n + g] = zf;
          const double en = static_cast<double>(zf);
          if (ti == 0) {
            S.sa_energy[g] = en;
          } else {
            const double eo = S.sa_energy[g];
            const double pr = exp(fmin((en - eo) / sa_t, 0.0));
            if ((en >= eo) || (sa_u < pr)) {
              for (int j = 0; j < sa.n_knobs; ++j) S.sa_cur[g][j] = S.sa_nxt[g][j];
              S.sa_energy[g] = en;
            }
          }
        }
        warp_arrive(&S.acc_done);
        if (tr) TRACE(12, ti);
        continue;
      }
      const int64_t gi = (blockIdx.x + ti * gridDim.x) * GT + g;
      if (gi < B) {
        const bool ok = v >= 0 && static_cast<uint64_t>(v) < size;
        const float zv = (b3 + acc0) + acc1;
        z_out[gi] = ok ? zv : __int_as_float(0x7fc00000);
        if (keys_out) {  // rank_history key for kt_topk_keys: (descending score code, index)
          const uint32_t bb = __float_as_uint(zv);
          const uint32_t asc = (bb & 0x80000000u) ? ~bb : (bb | 0x80000000u);
          const unsigned long long key =
              ok && zv == zv ? (static_cast<unsigned long long>(~asc) << 32) | static_cast<uint32_t>(v) : ~0ull;
          keys_out[gi] = key;
          if (key_hist) atomicAdd(&S.khist[static_cast<int>(key >> 53)], 1u);  // kt_topk_keys' first digit
        }
      }
      if (tr) TRACE(12, ti);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 4 * WG_MMA) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
  if (key_hist)
    for (int i = tid; i < 2048; i += NT)
      if (S.khist[i]) atomicAdd(&key_hist[i], S.khist[i]);
  if (threadIdx.x == 0) TRACE(29, 0);  // kernel exit
}

}  // namespace tcs

static bool default_dims_tc(const kt_dims& d) {
  return d.F == KT_F && d.n_gcn == 2 && d.gcn[1] == 32 && d.gcn[2] == 32 && d.n_head == 3 &&
         d.head[0] == 64 && d.head[1] == 64 && d.head[2] == 64 && d.head[3] == 1;
}

}  // namespace kt

extern "C" int kt_score_indices_flags(const kt_spec_table* tab, const kt_dims* dims, const float* params,
                                      const int64_t* idx, const uint32_t* idx32, int64_t idx_base, int64_t B,
                                      float* z_out, float* u_out, uint64_t* keys_out, uint32_t* key_hist,
                                      int32_t* err_flag, int32_t flags, void* stream) {
  using namespace kt;
  KT_REQUIRE(tab && dims && params && z_out && err_flag, KT_E_ARG, "kt_score_indices: null pointer");
  KT_REQUIRE(B > 0, KT_E_EMPTY, "kt_score_indices: empty batch");
  KT_REQUIRE(default_dims_tc(*dims), KT_E_UNSUPPORTED,
             "kt_score_indices: fused scorer needs F=12, gcn (32,32), head (64,64)");
  static SmemAttr attr;
  const int smem = static_cast<int>(sizeof(tcs::Smem));
  attr.ensure(tcs::score_tc_kernel, static_cast<size_t>(smem));
  const int64_t n_tiles = (B + tcs::GT - 1) / tcs::GT;
  const int grid = static_cast<int>(n_tiles < kNumSMs ? n_tiles : kNumSMs);
  const cudaError_t e =
      launch_pdl(tcs::score_tc_kernel, dim3(grid), dim3(tcs::NT), static_cast<size_t>(smem), as_stream(stream), tab,
                 *dims, params, idx, idx32, idx_base, B, z_out, u_out,
                 reinterpret_cast<unsigned long long*>(keys_out), keys_out ? key_hist : nullptr, err_flag,
                 static_cast<int>(flags), tcs::SaArgs{});
  KT_REQUIRE(e == cudaSuccess, KT_E_CUDA, "kt_score_indices: %s", cudaGetErrorString(e));
  note_launches(1);
  return check_launch("kt_score_indices");
}

extern "C" int kt_score_indices_ex(const kt_spec_table* tab, const kt_dims* dims, const float* params,
                                   const int64_t* idx, const uint32_t* idx32, int64_t idx_base, int64_t B,
                                   float* z_out, float* u_out, uint64_t* keys_out, uint32_t* key_hist,
                                   int32_t* err_flag, void* stream) {
  return kt_score_indices_flags(tab, dims, params, idx, idx32, idx_base, B, z_out, u_out, keys_out, key_hist,
                                err_flag, 0, stream);
}

extern "C" int kt_score_indices(const kt_spec_table* tab, const kt_dims* dims, const float* params,
                                const int64_t* idx, int64_t idx_base, int64_t B, float* z_out,
                                float* u_out, int32_t* err_flag, void* stream) {
  return kt_score_indices_ex(tab, dims, params, idx, nullptr, idx_base, B, z_out, u_out, nullptr, nullptr, err_flag,
                             stream);
}

extern "C" int kt_sa_run(const kt_spec_table* tab, const kt_dims* dims, const float* params, int32_t n_chains,
                         int32_t n_knobs, const int32_t* cards, const int64_t* mult, int32_t n_steps,
                         const int32_t* knob, const uint8_t* nudge, const int32_t* delta, const int32_t* resample,
                         const double* u, const double* temps, const int32_t* cur0, int64_t* hist_idx,
                         float* hist_z, int32_t* err_flag, void* stream) {
  using namespace kt;
  KT_REQUIRE(tab && dims && params && cards && mult && knob && nudge && delta && resample && u && temps && cur0 &&
                 hist_idx && hist_z && err_flag,
             KT_E_ARG, "kt_sa_run: null pointer");
  KT_REQUIRE(n_chains >= 1 && n_chains <= tcs::GT, KT_E_SHAPE, "kt_sa_run: 1..%d chains", tcs::GT);
  KT_REQUIRE(n_knobs >= 1 && n_knobs <= KT_MAX_KNOBS, KT_E_SHAPE, "kt_sa_run: 1..%d knobs", KT_MAX_KNOBS);
  KT_REQUIRE(n_steps >= 1, KT_E_EMPTY, "kt_sa_run: no steps");
  KT_REQUIRE(default_dims_tc(*dims), KT_E_UNSUPPORTED, "kt_sa_run: fused scorer needs the default dims");
  tcs::SaArgs a{};
  a.n_steps = n_steps;
  a.n_chains = n_chains;
  a.n_knobs = n_knobs;
  for (int j = 0; j < n_knobs; ++j) {
    KT_REQUIRE(cards[j] >= 1, KT_E_RANGE, "kt_sa_run: empty knob %d", j);
    a.cards[j] = cards[j];
    a.mult[j] = static_cast<long long>(mult[j]);
  }
  a.knob = knob;
  a.nudge = nudge;
  a.delta = delta;
  a.resample = resample;
  a.u = u;
  a.temps = temps;
  a.cur0 = cur0;
  a.hist_idx = hist_idx;
  a.hist_z = hist_z;
  static SmemAttr attr;
  const int smem = static_cast<int>(sizeof(tcs::Smem));
  attr.ensure(tcs::score_tc_kernel, static_cast<size_t>(smem));
  const int64_t B = static_cast<int64_t>(n_steps + 1) * tcs::GT;  // one tile per step, one CTA
  const cudaError_t e =
      launch_pdl(tcs::score_tc_kernel, dim3(1), dim3(tcs::NT), static_cast<size_t>(smem), as_stream(stream), tab,
                 *dims, params, static_cast<const int64_t*>(nullptr), static_cast<const uint32_t*>(nullptr),
                 int64_t{0}, B, hist_z, static_cast<float*>(nullptr), static_cast<unsigned long long*>(nullptr),
                 static_cast<unsigned int*>(nullptr), err_flag, 0, a);
  KT_REQUIRE(e == cudaSuccess, KT_E_CUDA, "kt_sa_run: %s", cudaGetErrorString(e));
  note_launches(1);
  return check_launch("kt_sa_run");
}
