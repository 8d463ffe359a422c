/*
 * kerntune_b200.h -- C-ABI of the B200 (sm_100a) MetaTune cost-model library.
 *
 * The reference (arXiv 2102.04199, package `kerntune`, pure Python/numpy) has
 * no native FFI; its hot path is a set of Python functions.  Each entry point
 * below is the device replacement of one of them and cites the reference
 * function it stands in for (path relative to /root/reference/pkg/src/kerntune).
 * The Python package `paper_2102_04199_b200` binds these with ctypes
 * (`_lib.py`) and keeps the reference's Python names and signatures.
 *
 * Conventions
 *   - every pointer argument is a DEVICE pointer unless named `host_*`;
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream);
 *   - no entry point allocates memory; scratch comes from the caller
 *     (`*_workspace_bytes` queries give the size);
 *   - all launches are stream-ordered and asynchronous; nothing synchronises
 *     the host except kt_sync_check;
 *   - return 0 (KT_OK) or a KT_E_* code; kt_last_error() describes the last
 *     failure on the calling thread.  The Python layer maps KT_E_SHAPE /
 *     KT_E_EMPTY / KT_E_RANGE / KT_E_UNSUPPORTED to DomainError and
 *     KT_E_CUDA / KT_E_NUMERIC to NumericError (reference errors.py:10-19).
 *
 * Flat parameter vector (fp32, device), layout described by kt_dims:
 *   [ gcn W_0 (F x d_1), ..., gcn W_{L-1}, agg (d_L),
 *     head W_0 (2 d_L x h_1), b_0, W_1, b_1, ..., W_H (h_H x 1), b_H ]
 * i.e. the GCN layers, the aggregation weights, then exactly the reference's
 * flat head vector head_to_vec() order (model.py:328-333).
 */
#ifndef KERNTUNE_B200_H
#define KERNTUNE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KT_OK 0
#define KT_E_SHAPE 1       /* shape / length mismatch           -> DomainError */
#define KT_E_EMPTY 2       /* empty batch                       -> DomainError */
#define KT_E_RANGE 3       /* config index out of space         -> DomainError */
#define KT_E_UNSUPPORTED 4 /* dims beyond the compiled limits   -> DomainError */
#define KT_E_CUDA 5        /* CUDA launch / runtime failure     -> NumericError */
#define KT_E_NUMERIC 6     /* non-finite result                 -> NumericError */
#define KT_E_ARG 7         /* null pointer / bad argument       -> DomainError */

#define KT_F 12            /* FEATURE_DIM (graphs.py:30-44) */
#define KT_MAX_KNOBS 8
#define KT_MAX_AXES 6
#define KT_MAX_LOOPS 12
#define KT_MAX_CARD 160
#define KT_MAX_LAYERS 4    /* GCN layers and head layers, each */
#define KT_MAX_DIM 64      /* widest GCN / head layer the general kernels take */
#define KT_MAX_NODES 64    /* largest graph the general kernels take */

/* Per-spec encode table (built on the host by graphs.EncodeTables, uploaded
 * once per (spec, layout, feature norm)).  Replaces the per-call Python work
 * of encode_batch (graphs.py:305-351) + index_config (kernels.py:278-286). */
typedef struct kt_spec_table {
  int32_t n_knobs, n_axes, n_loops, n_nodes;
  int32_t n_pairs;                       /* (for, iterval) pairs in the layout */
  int32_t auto_knob, expl_knob;          /* knob index or -1 */
  int32_t pad0;
  uint64_t space_size;
  uint32_t card[KT_MAX_KNOBS];           /* cardinalities, knob 0 most significant */
  int32_t axis_knob[KT_MAX_AXES];        /* knob index of tile_<axis> or -1 */
  int32_t axis_reduce[KT_MAX_AXES];
  int32_t loop_row[KT_MAX_LOOPS];        /* iterval node row of loop k */
  int32_t auto_vals[4];
  int32_t expl_vals[2];
  int32_t pad1[2];
  int32_t outer[KT_MAX_AXES][KT_MAX_CARD];  /* ceil(e / clamp(t)) per tile choice */
  int32_t inner[KT_MAX_AXES][KT_MAX_CARD];  /* clamp(t, 1, e) per tile choice */
  double raw_log2[2][KT_MAX_AXES][KT_MAX_CARD]; /* numpy log2 of outer/inner extents */
  /* normalised (fp64 (x-mean)/std cast to fp32, computed by numpy on the host) */
  float nrm_ext[KT_MAX_LOOPS][KT_MAX_CARD];      /* slot 0 per loop and choice */
  float nrm_log2ext[KT_MAX_LOOPS][KT_MAX_CARD];  /* slot 1 */
  float nrm_stride[KT_MAX_LOOPS][KT_MAX_CARD];   /* slot 5 (outer loops: t) */
  float nrm_const[KT_MAX_LOOPS][KT_F];           /* slots 2,3,5(inner),10,11 (+4 when 0) */
  float nrm_unroll1[KT_MAX_LOOPS];               /* slot 4 when unrolled */
  double fmean[KT_F], fstd[KT_F];
  uint64_t card_magic[KT_MAX_KNOBS];    /* floor(2^64 / card) + 1 (card >= 2): exact u32 division */
  /* knob digits the fused scorer extracts per row, d = 0..5 the axes' tile knobs, 6 the
   * auto-unroll knob, 7 the explicit-unroll knob: digit = (v / mult) % card (exact u32
   * magic-number divisions; mult / card 1 and magic 0 for an absent knob) */
  uint32_t digit_mult[8];
  uint32_t digit_card[8];
  uint64_t digit_mult_magic[8];
  uint64_t digit_card_magic[8];
  int32_t choice_off[KT_MAX_AXES + 1];  /* axis a's first entry in the concatenated per-choice tables */
  int32_t pad2;
} kt_spec_table;

/* Model dimensions and flat-vector offsets (in floats). */
typedef struct kt_dims {
  int32_t F;
  int32_t n_gcn;
  int32_t gcn[KT_MAX_LAYERS + 1];   /* gcn[0] = F, gcn[i+1] = d_{i+1} */
  int32_t n_head;                   /* number of affine head layers (>= 1) */
  int32_t head[KT_MAX_LAYERS + 2];  /* head[0] = 2 d_L, ..., head[n_head] = 1 */
  int32_t off_gcn[KT_MAX_LAYERS];
  int32_t off_agg;
  int32_t off_hw[KT_MAX_LAYERS + 1];
  int32_t off_hb[KT_MAX_LAYERS + 1];
  int32_t off_head;                 /* start of the head part (= off_hw[0]) */
  int32_t n_head_params;
  int32_t n_params;
} kt_dims;

/* ---- library ---------------------------------------------------------------- */
int kt_version(void);
const char* kt_last_error(void);
/* Number of kernels this library has launched in the process (bench evidence). */
int64_t kt_launch_count(void);
/* Synchronise `stream` and report any sticky device error. */
int kt_sync_check(void* stream);

/* ---- encoding ---------------------------------------------------------------- */
/* encode_batch (graphs.py:305-351) from config indices (index_config decode on
 * device): raw fp64 features (B, n_nodes, 12), zeros off the iterval rows.
 * Indices outside [0, space_size) set *err_flag = 1 and write zero rows. */
int kt_encode_raw(const kt_spec_table* tab, const int64_t* idx, int64_t B,
                  double* feats_out, int32_t* err_flag, void* stream);
/* Same from a choice matrix (B, n_knobs) int64 (the list[KnobConfig] form). */
int kt_encode_raw_choices(const kt_spec_table* tab, const int64_t* choices, int64_t B,
                          double* feats_out, int32_t* err_flag, void* stream);

/* ---- candidate scoring (the predictor of search.py:534-541) ------------------------ */
/* Fused encode -> GCN(12->32->32) -> weighted-sum+max readout -> head(64->64->64->1),
 * for knob spaces below 2^32 configs (larger spaces set *err_flag = 2 and score nothing),
 * all four GEMMs on tcgen05 tensor cores in 3xTF32 (fp32-accurate),
 * for graphs on the star layouts batch_layout (graphs.py:278) produces; equals
 * head_forward_batch(embed_batch(encode_batch(...))) (model.py:185-203).
 * Requires the default dims (F=12, gcn (32,32), head (64,64)).  `idx` may be NULL:
 * then candidate i is config index idx_base + i (a contiguous sweep shard).
 * If u_out != NULL the (B, 64) embeddings are written too (fine-tune rows). */
int kt_score_indices(const kt_spec_table* tab, const kt_dims* dims, const float* params,
                     const int64_t* idx, int64_t idx_base, int64_t B,
                     float* z_out, float* u_out, int32_t* err_flag, void* stream);
/* kt_score_indices with more inputs / outputs: indices as int64 (idx), as uint32
 * (idx32, may point at pinned host memory: zero-copy) or idx_base + i; optional
 * keys_out (B x uint64) receives rank_history keys, (descending-order score code) << 32
 * | index, EMPTY (all ones) for invalid indices, for kt_topk_keys; optional key_hist
 * (2048 uint32 bins, e.g. kt_topk_key_hist(workspace)) accumulates the keys' first
 * radix digit (key >> 53) so that kt_topk_keys(..., hist_ready = 1) can skip that pass. */
int kt_score_indices_ex(const kt_spec_table* tab, const kt_dims* dims, const float* params,
                        const int64_t* idx, const uint32_t* idx32, int64_t idx_base, int64_t B,
                        float* z_out, float* u_out, uint64_t* keys_out, uint32_t* key_hist,
                        int32_t* err_flag, void* stream);
/* kt_score_indices_ex with launch flags.  KT_SCORE_PARAMS_STABLE: the caller guarantees
 * that the kernel immediately before this launch on the stream does not write params
 * (e.g. the annealing steps after the first in one CUDA graph), so the operand staging
 * may overlap that kernel under programmatic dependent launch; indices, outputs and the
 * rest still wait for it. */
#define KT_SCORE_PARAMS_STABLE 1
int kt_score_indices_flags(const kt_spec_table* tab, const kt_dims* dims, const float* params,
                           const int64_t* idx, const uint32_t* idx32, int64_t idx_base, int64_t B,
                           float* z_out, float* u_out, uint64_t* keys_out, uint32_t* key_hist,
                           int32_t* err_flag, int32_t flags, void* stream);
/* Same contract as kt_score_indices on the FP32 FMA pipe (FFMA2 register tiles) instead
 * of tcgen05 3xTF32 tensor cores; kept as the second, independent implementation the
 * parity tests hold the tensor-core kernel against. */
int kt_score_indices_fp32(const kt_spec_table* tab, const kt_dims* dims, const float* params,
                          const int64_t* idx, int64_t idx_base, int64_t B,
                          float* z_out, float* u_out, int32_t* err_flag, void* stream);

/* ---- general forward (arbitrary adjacency, segmented batches) ------------------------ */
/* embed_batch (model.py:185-194) generalised to CSR batches.
 * Shared pattern (nodes_per_graph > 0, node_ptr NULL): every graph has the same
 *   n = nodes_per_graph nodes and adjacency; row_ptr (n+1) / col (local ids) /
 *   val describe it once and mask is (n,).
 * Segmented (nodes_per_graph == 0): graph g owns nodes [node_ptr[g], node_ptr[g+1]);
 *   row_ptr is indexed by global node, col holds global node ids, mask is per node.
 * feats: (total nodes, F) fp64 RAW features (normalised on device, model.py:108-112);
 * val: fp32 entries of the fp64 normalised adjacency; max_nodes bounds any graph.
 * graph_idx (optional, B entries) gathers graphs of a resident dataset (row b of
 * the output is graph graph_idx[b]).
 * Writes u (B, 2 d_L); if z_out != NULL also head_forward_batch (model.py:197-203). */
int kt_embed_csr(const kt_dims* dims, const float* params, const double* fmean, const double* fstd,
                 const double* feats, const uint8_t* mask, const int64_t* node_ptr,
                 int32_t nodes_per_graph, int32_t max_nodes,
                 const int32_t* row_ptr, const int32_t* col, const float* val,
                 const int64_t* graph_idx, int64_t B, float* u_out, float* z_out, void* stream);
/* ---- streaming aggregation (HBM-bound layer-by-layer form of embed_batch) ------------------ */
/* One GCN layer, out = ReLU(A_hat . in . W) per graph (gcn_forward model.py:127-133,
 * the einsum of embed_batch model.py:189-191), rows of all graphs contiguous.
 * in: (rows, d_in) fp32, or (in_f64 != 0) the raw fp64 features, z-normalised on the
 *   fly with fmean / fstd on nodes whose pattern mask is 1 and zero elsewhere
 *   (model.py:108-112).  W: (d_in, d_out) row-major.  out: (rows, d_out) fp32.
 * Rows: nodes_per_graph > 0 -> graph g owns rows [g n, (g+1) n) (node_ptr ignored);
 *   else [node_ptr[g], node_ptr[g+1]).
 * Adjacency: n_pat (<= 8) local CSR patterns (pat_n nodes each; pat_rp (n+1) per
 *   pattern, concatenated; pat_col / pat_val concatenated, pat_nnz in total <= 1024;
 *   pat_mask one byte per pattern node); graph g uses pattern pat_id ? pat_id[g] : 0.
 * Bulk (1D TMA) copies move each tile in / out when rows are 16-byte multiples. */
int kt_gcn_layer(const void* in, int32_t in_f64, const double* fmean, const double* fstd,
                 const float* W, int32_t d_in, int32_t d_out, int32_t relu, int64_t B,
                 int32_t nodes_per_graph, const int64_t* node_ptr, const int32_t* pat_id,
                 int32_t n_pat, const int32_t* pat_n, const int32_t* pat_rp, const int32_t* pat_col,
                 const float* pat_val, const uint8_t* pat_mask, int32_t pat_nnz, int32_t max_nodes,
                 float* out, void* stream);
/* aggregate (model.py:136-141) per graph: u[g] = [sum_n agg_w * h_n, max_n h_n],
 * h (rows, d) fp32 with graph rows as in kt_gcn_layer; u (B, 2 d). */
int kt_readout(const float* h, int32_t d, int64_t B, int32_t nodes_per_graph, const int64_t* node_ptr,
               const float* agg_w, float* u_out, void* stream);
/* head_forward_batch (model.py:197-203): u (B, head[0]) -> z (B). */
int kt_head_forward(const kt_dims* dims, const float* params, const float* u, int64_t B,
                    float* z_out, void* stream);

/* ---- end-to-end sweep step from host memory (the predictor seam, search.py:9-10) ---------- */
/* Pinned host indices (int64 or uint32: idx_bytes 8 / 4) are read in place by the
 * scorer and the scores written in place to pinned z_host (zero-copy both ways: the
 * host<->device transfer happens inside the kernel); the scorer's (score, index) keys
 * (keys_dev, B entries) are ranked by kt_topk_keys and the top-k copied to the host.
 * Asynchronous on `stream` (synchronise it before reading z_host / top_*_host). */
int kt_sweep_host(const kt_spec_table* tab, const kt_dims* dims, const float* params,
                  const void* idx_host, int32_t idx_bytes, int64_t B, uint64_t* keys_dev, float* z_host,
                  int32_t k, int64_t* top_idx_dev, float* top_score_dev, int64_t* top_idx_host,
                  float* top_score_host, void* topk_ws, int64_t topk_ws_bytes, int32_t* err_dev, void* stream);

/* ---- GP surrogate + batch UCB of the meta-BO proposer (search.py:39-159, 284-340) ---------- */
/* All fp64, device pointers.  Coordinates are (points x d) row-major, d <= 16.
 * gp_kernel (search.py:72-76): out (n1 x n2) = exp(-0.5 max(|a|^2 + |b|^2 - 2 a.b, 0)), a = x/ls. */
int kt_gp_gram(const double* x1, int32_t n1, const double* x2, int32_t n2, int32_t d, const double* ls, double* out,
               void* stream);
/* gp_fit's per-lengthscale work (search.py:79-121) for n_cand lengthscale vectors at once
 * (ls: n_cand x d): L (n_cand x n x n, the lower Cholesky factor of K + nv I stored
 * COLUMN-major) with nv escalated tenfold from `noise` until the factorisation succeeds
 * or nv >= max_jitter; alpha (n_cand x n) = K^-1 y; info (n_cand x 3) = {fitted nv,
 * marginal log likelihood, status (0 ok, 1 not positive definite at max_jitter)}. n <= 1024. */
int kt_gp_factor(const double* x, int32_t n, int32_t d, const double* ls, int32_t n_cand, const double* y,
                 double noise, double max_jitter, double* L, double* alpha, double* info, void* stream);
/* gp_predict_many (search.py:129-139) at P points xp: mean, var = max(1 - |L^-1 k(x,xp)|^2, 0);
 * if cov != NULL also _gp_posterior_cov (search.py:152-157): cov (P x P) = k(xp,xp) - v^T v
 * (needs kt_gp_workspace_bytes(n, P, 0)).  L as written by kt_gp_factor. */
int64_t kt_gp_workspace_bytes(int32_t n, int32_t P, int32_t take);
int kt_gp_posterior(const double* x, int32_t n, int32_t d, const double* ls, const double* L, const double* alpha,
                    const double* xp, int32_t P, double* mean, double* var, double* cov, void* workspace,
                    int64_t workspace_bytes, void* stream);
/* bo_propose_batch's sequential UCB with hallucinated downdates (search.py:324-340):
 * picks (take) = positions into the pool, in pick order.  P <= 4096, take <= 64;
 * workspace >= take * P * 8 bytes. */
int kt_gp_ucb(const double* mean, const double* cov, int32_t P, double noise, double beta, int32_t take,
              int32_t* picks, void* workspace, int64_t workspace_bytes, void* stream);

/* ---- simulated-annealing exploration (sa_explore, search.py:202-254) ----------------------- */
/* One proposal step for n_chains chains from pre-drawn randoms (the host draws them
 * from the caller's numpy Generator in the reference's order): the chosen knob of
 * chain c is nudged by delta[c] (clipped to [0, card-1]) if nudge[c], else set to
 * resample[c] (search.py:232-241).  cur / nxt: (n_chains, n_knobs) int32 choices;
 * nxt_idx: the neighbours' config indices, sum_j nxt[c][j] mult[j]. */
int kt_sa_propose(const int32_t* cur, int32_t n_chains, int32_t n_knobs, const int32_t* cards,
                  const int64_t* mult, const int32_t* knob, const uint8_t* nudge, const int32_t* delta,
                  const int32_t* resample, int32_t* nxt, int64_t* nxt_idx, void* stream);
/* The per-step random draws of sa_explore (search.py:233-237: integers(0, n_knobs),
 * random() < 0.5, integers(0, 2) * 2 - 1, integers(0, cards[knob]), random(), each of
 * size n_chains) for n_steps steps, reproducing numpy's Generator(PCG64) stream bit for
 * bit (dependency: numpy's PCG64 + bounded-integer algorithms).  pcg = {state_hi,
 * state_lo, inc_hi, inc_lo} of bit_generator.state; pcg / has_uint32 / uinteger are
 * advanced in place to the state numpy would hold after the same calls.  Host memory;
 * outputs (n_steps, n_chains) row-major.  Host-side: no GPU work. */
int kt_sa_draws(uint64_t* pcg, int32_t* has_uint32, uint32_t* uinteger, int32_t n_steps, int32_t n_chains,
                int32_t n_knobs, const int32_t* cards, int32_t* knob, uint8_t* nudge, int32_t* delta,
                int32_t* resample, double* u);
/* The whole of sa_explore's annealing loop (search.py:228-252) in one launch of the fused
 * scorer on one CTA: tile t holds the n_chains (<= 128) configurations of step t; the
 * encode warps propose step t's neighbours from the accepted chain state with
 * kt_sa_propose's rule once the head has run kt_sa_accept's Metropolis test on step
 * t - 1's scores.  Draws (n_steps, n_chains) and temps (n_steps) as kt_sa_draws / the
 * schedule give them; cur0 (n_chains, n_knobs) the starting choices; hist_idx row 0 holds
 * the starts on input; hist_idx / hist_z ((n_steps + 1) x n_chains) receive every
 * evaluated configuration and score, the trajectory the per-step kernels produce.
 * cards / mult are host arrays; the rest device memory.  Default dims only. */
int kt_sa_run(const kt_spec_table* tab, const kt_dims* dims, const float* params, int32_t n_chains,
              int32_t n_knobs, const int32_t* cards, const int64_t* mult, int32_t n_steps,
              const int32_t* knob, const uint8_t* nudge, const int32_t* delta, const int32_t* resample,
              const double* u, const double* temps, const int32_t* cur0, int64_t* hist_idx, float* hist_z,
              int32_t* err_flag, void* stream);
/* Metropolis acceptance (search.py:246-251) in fp64: accept if e_new >= energy or
 * u < exp(min((e_new - energy) / temp, 0)); accepted chains copy nxt into cur and
 * e_new into energy. */
int kt_sa_accept(int32_t n_chains, int32_t n_knobs, const float* e_new, const double* u, double temp,
                 const int32_t* nxt, int32_t* cur, double* energy, void* stream);

/* ---- training (model.py:218-310, meta.py:104-123) ----------------------------------------- */
/* grad(m, batch, scope) (model.py:218-285) over a CSR batch laid out as for
 * kt_embed_csr.  graph_idx (optional, B entries) gathers graphs of a resident
 * dataset.  Batch item b uses graph graph_idx ? graph_idx[b] : b and the
 * z-normalised label y[b] (model.py:99-101).
 * Writes the batch-mean gradient (flat layout) to grad_out (may be NULL) and the
 * MSE to *loss_out (fp64, may be NULL); if new_params != NULL also writes
 * params - lr * grad (sgd_step, model.py:288-310) there.  head_only != 0 is
 * scope "head_only" (gcn/agg gradients exactly zero).  The per-graph gradient
 * rows are summed in a fixed order in fp64: results are run-to-run identical. */
int64_t kt_grad_workspace_bytes(const kt_dims* dims, int64_t B);
int kt_grad(const kt_dims* dims, const float* params, const double* fmean, const double* fstd,
            const double* feats, const uint8_t* mask, const int64_t* node_ptr,
            int32_t nodes_per_graph, int32_t max_nodes, const int32_t* row_ptr, const int32_t* col,
            const float* val, const int64_t* graph_idx, const float* y, int64_t B, int32_t head_only,
            float* grad_out, double* loss_out, float lr, float* new_params,
            void* workspace, int64_t workspace_bytes, void* stream);
/* sgd_step on flat vectors: out = params - lr * grad (out may alias params). */
int kt_sgd(const float* params, const float* grad, float lr, int64_t n, float* out, void* stream);
/* The batch-1 SGD loop of pretrain (meta.py:117-122): for s in 0..n_steps-1,
 * params -= gamma * grad(params, [dataset graph order[s]], "all"); y is indexed
 * by dataset graph.  One CTA, parameters resident in shared memory; params is
 * updated in place. */
int kt_pretrain_sgd(const kt_dims* dims, float* params, const double* fmean, const double* fstd,
                    const double* feats, const uint8_t* mask, const int64_t* node_ptr,
                    int32_t nodes_per_graph, int32_t max_nodes, const int32_t* row_ptr,
                    const int32_t* col, const float* val, const int64_t* order, const float* y,
                    int64_t n_steps, float gamma, void* stream);

/* ---- head engine, MAML, fine-tune (model.py:358-432, meta.py:167-297) ---------------------- */
/* Flat head vectors (head_to_vec order) of n_head_params floats; dims supplies the
 * head shapes (only the head fields and n_head_params are read).  u: (n, head[0])
 * fp32 rows, y: (n,) normalised labels. */
/* head_loss_grad (model.py:358-389): grad_out (flat), *mse_out (may be NULL). */
int kt_head_loss_grad(const kt_dims* dims, const float* theta, const float* u, const float* y, int64_t n,
                      float* grad_out, float* mse_out, void* stream);
/* head_hvp (model.py:392-432): Hessian-vector product H(theta) v. */
int kt_head_hvp(const kt_dims* dims, const float* theta, const float* u, const float* y, const float* v,
                int64_t n, float* hvp_out, void* stream);
/* fine_tune_embedded (meta.py:274-282): `steps` full-batch head SGD steps of rate
 * alpha; theta_out may alias theta; mse_out (steps floats, may be NULL) gets the
 * loss before each step. */
int kt_fine_tune(const kt_dims* dims, const float* theta, const float* u, const float* y, int64_t n,
                 float alpha, int32_t steps, float* theta_out, float* mse_out, void* stream);
/* One CTA per task: maml_outer_grad (meta.py:167-196) for T tasks whose support
 * / query rows are u[s_idx[s_off[t] .. s_off[t+1])] / u[q_idx[...]] (labels y
 * indexed the same way).  Writes g_sum = sum_t g_t (fixed order, fp64 accumulate)
 * and stats = (sum_t support_loss_t, sum_t query_loss_t) (fp64, may be NULL).
 * meta_step's update is then theta - beta * g_sum (kt_sgd), after an all-reduce
 * of g_sum when tasks are sharded over ranks. */
int64_t kt_maml_workspace_bytes(const kt_dims* dims, int32_t T, int32_t inner_steps, int32_t first_order);
int kt_maml_tasks(const kt_dims* dims, const float* theta, const float* u, const float* y,
                  const int64_t* s_off, const int64_t* s_idx, const int64_t* q_off, const int64_t* q_idx,
                  int32_t T, float alpha, int32_t inner_steps, int32_t first_order, float* g_sum,
                  double* stats, void* workspace, int64_t workspace_bytes, void* stream);
/* meta_step on one GPU (meta.py:223-257): kt_maml_tasks with the outer update
 * theta <- theta - beta * g_sum (in place) folded into the task-sum pass (two launches
 * instead of three). */
int kt_maml_step(const kt_dims* dims, float* theta, const float* u, const float* y, const int64_t* s_off,
                 const int64_t* s_idx, const int64_t* q_off, const int64_t* q_idx, int32_t T, float alpha,
                 int32_t inner_steps, int32_t first_order, float beta, float* g_sum, double* stats,
                 void* workspace, int64_t workspace_bytes, void* stream);
/* Data-parallel meta_step, bit-identical to kt_maml_step: kt_maml_task_grads
 * writes the per-task outer gradients g_i (maml_outer_grad, meta.py:167-196) of this rank's
 * contiguous task share as rows g_rows (T x n_head_params) and per-task (support, query)
 * losses (T x 2), no reduction; after an all-gather of the rows in task order,
 * kt_task_sum_update sums all T rows in task order in fp64 into g_sum (and the losses into
 * stats) and, if theta != NULL, applies theta -= beta * g_sum with kt_maml_step's
 * arithmetic (meta.py:249-252: sum, not mean). */
int kt_maml_task_grads(const kt_dims* dims, const float* theta, const float* u, const float* y,
                       const int64_t* s_off, const int64_t* s_idx, const int64_t* q_off, const int64_t* q_idx,
                       int32_t T, float alpha, int32_t inner_steps, int32_t first_order, float* g_rows,
                       float* losses, void* workspace, int64_t workspace_bytes, void* stream);
int kt_task_sum_update(const kt_dims* dims, const float* g_rows, const float* losses, int32_t T, float beta,
                       float* theta, float* g_sum, double* stats, void* stream);

/* ---- ranking (search.py:257-264) ------------------------------------------------------ */
/* Top-k of (score desc, index asc) over B candidates; `visited` (sorted int64,
 * n_visited entries, may be NULL) are excluded.  Outputs k indices and scores
 * (fewer valid entries are padded with index -1).  idx == NULL means idx_base + i. */
int64_t kt_topk_workspace_bytes(int64_t B, int32_t k);
int kt_topk(const float* scores, const int64_t* idx, int64_t idx_base, int64_t B,
            const int64_t* visited, int64_t n_visited, int32_t k,
            int64_t* top_idx, float* top_score, void* workspace, int64_t workspace_bytes,
            void* stream);
/* Top-k of precomputed keys (kt_score_indices_ex keys_out): ascending key order.
 * hist_ready != 0: the workspace's first-digit histogram (kt_topk_key_hist) already
 * holds these keys' counts (filled by the scorer).  Every kt_topk* call leaves that
 * histogram zeroed; a fresh workspace must be zeroed once before a scorer fills it.
 * One cooperative launch (radix select, gather, sort); k <= 1024. */
int kt_topk_keys(const uint64_t* keys, int64_t B, int32_t k, int32_t hist_ready, int64_t* top_idx,
                 float* top_score, void* workspace, int64_t workspace_bytes, void* stream);
uint32_t* kt_topk_key_hist(void* workspace);
/* Merge world x k (score, index) candidate lists (the all-gathered per-rank top-k). */
int kt_topk_merge(const float* scores, const int64_t* idx, int64_t n, int32_t k,
                  int64_t* top_idx, float* top_score, void* workspace, int64_t workspace_bytes,
                  void* stream);

#ifdef __cplusplus
}
#endif
#endif /* KERNTUNE_B200_H */
