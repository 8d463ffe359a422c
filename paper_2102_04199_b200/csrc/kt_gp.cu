// GP surrogate + batch UCB of the meta-BO proposer (search.py:39-159, 284-340), fp64.
//
// The reference fits an exact GP on up to gp_obs_window (512) observations in knob
// coordinates every tuning round (gp_fit: one Cholesky per lengthscale of a 4-point
// grid, tenfold jitter escalation, marginal-likelihood selection) and proposes a batch
// by sequential UCB over a 512-candidate pool with hallucinated variance downdates
// (bo_propose_batch).  Here:
//   factor_kernel     one CTA per lengthscale candidate: Gram entries on the fly from
//                     the scaled coordinates (smem), blocked left-looking Cholesky into a
//                     column-major factor (thread = row, 16-column panels in registers), jitter
//                     escalation inside the kernel, forward / backward solves for alpha,
//                     and the marginal likelihood -- no host round trips;
//   posterior_kernel  16 pool points per CTA: k(x, xp) into shared memory, mean, the
//                     blocked triangular solve v = L^-1 k(x, xp) for the 16 right-hand
//                     sides (diagonal blocks by one warp, trailing rows by the CTA),
//                     var = 1 - |v|^2;
//   cov_kernel        k(xp, xp) - v^T v (64 x 64 output tiles, fp64 FMA);
//   ucb_kernel        one CTA: the sequential UCB loop.  Only the picked columns of the
//                     downdated covariance are ever needed, so column t is rebuilt from
//                     the original matrix and the earlier columns with the reference's
//                     operation order, ((cov - c0 c0[z]/d0) - c1 c1[z]/d1) ..., which is
//                     bit-identical to its dense downdates at O(P t) instead of O(P^2).
// Gram entries follow search.py:72-76 term by term: a = x / ls, d2 = (|a|^2 + |b|^2) - 2 a.b,
// exp(-0.5 max(d2, 0)).
#include "kt_common.cuh"

namespace kt {
namespace gp {

constexpr int MAXD = 16;     // knob coordinates per point
constexpr int MAXN = 1024;   // observations (gp_obs_window is 512)
constexpr int PC = 16;       // pool points per posterior CTA
constexpr int PT = 256;      // posterior kernel threads
constexpr int UT = 1024;     // ucb kernel threads
constexpr int MAXP = 4096;   // candidate pool
constexpr int PW = 16;       // Cholesky / triangular-solve panel width

__device__ __forceinline__ double gram(const double* a, double aa, const double* b, double bb, int d) {
  double ab = 0.0;
  for (int k = 0; k < d; ++k) ab = fma(a[k], b[k], ab);
  const double d2 = (aa + bb) - 2.0 * ab;
  return exp(-0.5 * fmax(d2, 0.0));
}

__device__ __forceinline__ double sq_norm(const double* a, int d) {
  double s = 0.0;
  for (int k = 0; k < d; ++k) s += a[k] * a[k];  // (a * a).sum(axis=1): products, then the sum
  return s;
}

template <int NT>
__device__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
  for (int i = 0; i < NT / 32; ++i) t += red[i];  // fixed order: deterministic
  return t;
}

// grid = candidates; x (n x d), ls (cand x d), L (cand x n x n, column-major lower factor),
// alpha (cand x n), info (cand x 3: fitted noise, mll, status 0 ok / 1 not PD at max jitter)
template <int FT>
__global__ void __launch_bounds__(FT) factor_kernel(const double* __restrict__ x, int n, int d,
                                                    const double* __restrict__ ls_all, const double* __restrict__ y,
                                                    double noise, double max_jitter, double* __restrict__ L_all,
                                                    double* __restrict__ alpha_all, double* __restrict__ info) {
  extern __shared__ double sm[];
  double* A = sm;              // n x d scaled coordinates
  double* AA = A + n * d;      // n squared norms
  double* R = AA + n;          // n: solve right-hand side
  __shared__ double red[FT / 32];
  __shared__ int s_fail;
  const int c = blockIdx.x, tid = threadIdx.x;
  const double* ls = ls_all + c * d;
  double* L = L_all + static_cast<size_t>(c) * n * n;
  double* alpha = alpha_all + static_cast<size_t>(c) * n;
  for (int e = tid; e < n * d; e += FT) A[e] = x[e] / ls[e % d];
  __syncthreads();
  for (int i = tid; i < n; i += FT) AA[i] = sq_norm(A + i * d, d);
  __syncthreads();

  // Blocked left-looking Cholesky, thread = row, panels of PW columns held in registers:
  //   1. acc[c] = K[i][j0 + c] - sum_{k < j0} L[i][k] L[j0 + c][k]: the earlier columns are
  //      read once per panel (column-major L: coalesced in i), the panel rows' values are
  //      staged through shared memory 16 columns at a time;
  //   2. the panel is factored right-looking in registers, the pivot row's entries
  //      broadcast through shared memory;
  //   3. the panel's columns are written out.
  constexpr int KC = 4 * PW;
  __shared__ double S[KC][PW], Pd[PW][PW + 1];
  double nv = noise;
  int status = 0;
  const int i = tid;
  for (;;) {
    if (tid == 0) s_fail = 0;
    __syncthreads();
    for (int j0 = 0; j0 < n && !s_fail; j0 += PW) {
      const int nb = n - j0 < PW ? n - j0 : PW;
      const bool mine = i >= j0 && i < n;
      double acc[PW];
#pragma unroll
      for (int c = 0; c < PW; ++c) {
        acc[c] = 0.0;
        if (mine && c < nb && i >= j0 + c) {
          acc[c] = gram(A + i * d, AA[i], A + (j0 + c) * d, AA[j0 + c], d);
          if (i == j0 + c) acc[c] += nv;
        }
      }
      for (int k0 = 0; k0 < j0; k0 += KC) {  // KC earlier columns staged per barrier pair
        const int kc = j0 - k0 < KC ? j0 - k0 : KC;  // (a multiple of PW)
        for (int e = tid; e < KC * PW; e += FT) {
          const int kk = e / PW, c = e % PW;
          S[kk][c] = kk < kc && c < nb ? L[static_cast<size_t>(k0 + kk) * n + j0 + c] : 0.0;
        }
        __syncthreads();
        if (mine) {
          for (int kb = 0; kb < kc; kb += PW) {
            double li[PW];  // the row's factor entries: all loads in flight before the FMAs
#pragma unroll
            for (int kk = 0; kk < PW; ++kk) li[kk] = L[static_cast<size_t>(k0 + kb + kk) * n + i];
#pragma unroll
            for (int kk = 0; kk < PW; ++kk) {
#pragma unroll
              for (int c = 0; c < PW; ++c) acc[c] = fma(-li[kk], S[kb + kk][c], acc[c]);
            }
          }
        }
        __syncthreads();
      }
      // diagonal block: the panel rows hand their sums to warp 0, which factors the
      // nb x nb block alone (lane = row, warp barriers only); every row below then solves
      // its nb panel entries against it -- one CTA barrier per panel instead of two per column
      if (i >= j0 && i < j0 + nb) {
#pragma unroll
        for (int c = 0; c < PW; ++c) Pd[i - j0][c] = acc[c];
      }
      __syncthreads();
      if (tid < 32) {
        const int r = tid;
        for (int c = 0; c < nb; ++c) {
          if (r == c) {
            const double sdiag = Pd[c][c];
            if (!(sdiag > 0.0)) s_fail = 1;
            Pd[c][c] = sqrt(sdiag);
          }
          __syncwarp();
          if (r > c && r < nb) Pd[r][c] /= Pd[c][c];
          __syncwarp();
          if (r > c && r < nb)
            for (int c2 = c + 1; c2 <= r; ++c2) Pd[r][c2] = fma(-Pd[r][c], Pd[c2][c], Pd[r][c2]);
          __syncwarp();
        }
      }
      __syncthreads();
      if (s_fail) break;
      if (i >= j0 + nb && i < n) {  // rows below: acc <- acc L_d^-T (forward substitution over the panel)
#pragma unroll
        for (int c = 0; c < PW; ++c) {
          if (c < nb) {
            double v = acc[c];
#pragma unroll
            for (int c2 = 0; c2 < c; ++c2) v = fma(-acc[c2], Pd[c][c2], v);
            acc[c] = v / Pd[c][c];
          }
        }
      } else if (mine) {
#pragma unroll
        for (int c = 0; c < PW; ++c) acc[c] = Pd[i - j0][c];
      }
      if (s_fail) break;
#pragma unroll
      for (int c = 0; c < PW; ++c)
        if (c < nb && mine && i >= j0 + c) L[static_cast<size_t>(j0 + c) * n + i] = acc[c];
      __syncthreads();
    }
    __syncthreads();
    if (!s_fail) break;
    if (nv >= max_jitter) {
      status = 1;
      break;
    }
    nv *= 10.0;
    __syncthreads();
  }
  if (status) {
    if (tid == 0) {
      info[3 * c] = nv;
      info[3 * c + 1] = -INFINITY;
      info[3 * c + 2] = 1.0;
    }
    return;
  }
  // zero the strict upper triangle (column-major: rows above the diagonal)
  for (size_t e = tid; e < static_cast<size_t>(n) * n; e += FT) {
    const int col = static_cast<int>(e / n), row = static_cast<int>(e % n);
    if (row < col) L[e] = 0.0;
  }
  // cho_solve, blocked by panels of PW rows: L z = y forward, then L^T alpha = z backward.
  // Warp 0 solves each PW x PW diagonal block (warp barriers only); the CTA then updates
  // every remaining row with the panel's solved values (two CTA barriers per panel).
  for (int i = tid; i < n; i += FT) R[i] = y[i];
  __syncthreads();
  for (int j0 = 0; j0 < n; j0 += PW) {
    const int nb = n - j0 < PW ? n - j0 : PW;
    if (tid < 32) {
      for (int c = 0; c < nb; ++c) {
        const int j = j0 + c;
        const double zj = R[j] / L[static_cast<size_t>(j) * n + j];
        __syncwarp();
        if (tid == 0) R[j] = zj;
        if (tid > c && tid < nb) R[j0 + tid] = fma(-L[static_cast<size_t>(j) * n + j0 + tid], zj, R[j0 + tid]);
        __syncwarp();
      }
    }
    __syncthreads();
    for (int i = j0 + nb + tid; i < n; i += FT) {
      double v = R[i];
#pragma unroll
      for (int c = 0; c < PW; ++c)
        if (c < nb) v = fma(-L[static_cast<size_t>(j0 + c) * n + i], R[j0 + c], v);
      R[i] = v;
    }
    __syncthreads();
  }
  for (int j1 = n; j1 > 0; j1 -= PW) {  // panel [j0, j1), last panel first
    const int j0 = j1 - PW > 0 ? j1 - PW : 0;
    const int nb = j1 - j0;
    if (tid < 32) {
      for (int c = nb - 1; c >= 0; --c) {
        const int j = j0 + c;
        const double aj = R[j] / L[static_cast<size_t>(j) * n + j];
        __syncwarp();
        if (tid == 0) R[j] = aj;
        if (tid < c) R[j0 + tid] = fma(-L[static_cast<size_t>(j0 + tid) * n + j], aj, R[j0 + tid]);
        __syncwarp();
      }
    }
    __syncthreads();
    for (int i = tid; i < j0; i += FT) {  // R[i] -= sum_c L[j0 + c][i] alpha[j0 + c]
      const double* row = L + static_cast<size_t>(i) * n + j0;  // column i of L, rows j0..: contiguous
      double v = R[i];
#pragma unroll
      for (int c = 0; c < PW; ++c)
        if (c < nb) v = fma(-row[c], R[j0 + c], v);
      R[i] = v;
    }
    __syncthreads();
  }
  double ya = 0.0, ld = 0.0;
  for (int i = tid; i < n; i += FT) {
    alpha[i] = R[i];
    ya = fma(y[i], R[i], ya);
    ld += log(L[static_cast<size_t>(i) * n + i]);
  }
  ya = block_sum<FT>(ya, red);
  ld = block_sum<FT>(ld, red);
  if (tid == 0) {
    info[3 * c] = nv;
    info[3 * c + 1] = -0.5 * ya - ld - 0.5 * n * log(2.0 * 3.14159265358979323846);
    info[3 * c + 2] = 0.0;
  }
}

// blockIdx.x: pool points [PC b, PC b + PC); V (n x P) row-major out
__global__ void __launch_bounds__(PT) posterior_kernel(const double* __restrict__ x, int n, int d,
                                                       const double* __restrict__ ls, const double* __restrict__ L,
                                                       const double* __restrict__ alpha, const double* __restrict__ xp,
                                                       int P, double* __restrict__ mean, double* __restrict__ var,
                                                       double* __restrict__ V) {
  extern __shared__ double sm[];
  double* Rv = sm;                 // n x PC right-hand sides -> v
  double* A = Rv + n * PC;         // n x d
  double* AA = A + n * d;          // n
  __shared__ double Bp[PC][MAXD + 1], BB[PC];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int p0 = blockIdx.x * PC;
  for (int e = tid; e < n * d; e += PT) A[e] = x[e] / ls[e % d];
  for (int e = tid; e < PC * d; e += PT) {
    const int p = e / d, k = e % d;
    Bp[p][k] = p0 + p < P ? xp[(p0 + p) * d + k] / ls[k] : 0.0;
  }
  __syncthreads();
  for (int i = tid; i < n; i += PT) AA[i] = sq_norm(A + i * d, d);
  if (tid < PC) BB[tid] = sq_norm(Bp[tid], d);
  __syncthreads();
  for (int e = tid; e < n * PC; e += PT) {
    const int i = e / PC, p = e % PC;
    Rv[e] = gram(A + i * d, AA[i], Bp[p], BB[p], d);
  }
  __syncthreads();
  if (w == 0 && lane < PC && p0 + lane < P) {  // mean = k(x, xp)^T alpha (sequential in i)
    double m = 0.0;
    for (int i = 0; i < n; ++i) m = fma(Rv[i * PC + lane], alpha[i], m);
    mean[p0 + lane] = m;
  }
  // blocked forward substitution for the PC columns, panels of PW rows:
  //   (a) the PW x PW diagonal block of L is staged in shared memory and warp 0
  //       (lane = column) solves the panel rows;
  //   (b) every later row loses sum_c L[i][j0 + c] v[j0 + c] (thread = row x 4 columns).
  __shared__ double Ld[PW][PW];
  constexpr int QPR = PC / 4;  // column quads per row
  const int rq = tid / QPR, cq = (tid % QPR) * 4;
  for (int j0 = 0; j0 < n; j0 += PW) {
    const int nb = n - j0 < PW ? n - j0 : PW;
    if (tid < PW * PW) {
      const int r = tid / PW, c = tid % PW;
      Ld[r][c] = r < nb && c <= r ? L[static_cast<size_t>(j0 + c) * n + j0 + r] : 0.0;
    }
    __syncthreads();
    if (w == 0 && lane < PC) {
      for (int c = 0; c < nb; ++c) {
        const double vj = Rv[(j0 + c) * PC + lane] / Ld[c][c];
        Rv[(j0 + c) * PC + lane] = vj;
        for (int r = c + 1; r < nb; ++r) Rv[(j0 + r) * PC + lane] = fma(-Ld[r][c], vj, Rv[(j0 + r) * PC + lane]);
      }
    }
    __syncthreads();
    for (int i = j0 + nb + rq; i < n; i += PT / QPR) {
      double li[PW];  // the row's panel entries of L: all loads in flight before the FMAs
#pragma unroll
      for (int c = 0; c < PW; ++c) li[c] = c < nb ? L[static_cast<size_t>(j0 + c) * n + i] : 0.0;
      double r0 = Rv[i * PC + cq], r1 = Rv[i * PC + cq + 1], r2 = Rv[i * PC + cq + 2], r3 = Rv[i * PC + cq + 3];
#pragma unroll
      for (int c = 0; c < PW; ++c) {
        if (c >= nb) break;
        const double l = li[c];
        const double* vr = Rv + (j0 + c) * PC + cq;
        r0 = fma(-l, vr[0], r0);
        r1 = fma(-l, vr[1], r1);
        r2 = fma(-l, vr[2], r2);
        r3 = fma(-l, vr[3], r3);
      }
      Rv[i * PC + cq] = r0;
      Rv[i * PC + cq + 1] = r1;
      Rv[i * PC + cq + 2] = r2;
      Rv[i * PC + cq + 3] = r3;
    }
    __syncthreads();
  }
  if (w == 0 && lane < PC && p0 + lane < P) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += Rv[i * PC + lane] * Rv[i * PC + lane];  // (v * v).sum(axis=0)
    var[p0 + lane] = fmax(1.0 - s, 0.0);
  }
  if (V)
    for (int e = tid; e < n * PC; e += PT) {
      const int i = e / PC, p = e % PC;
      if (p0 + p < P) V[static_cast<size_t>(i) * P + p0 + p] = Rv[e];
    }
}

// cov (P x P) = k(xp, xp) - V^T V; 64 x 64 tile per CTA, 4 x 4 per thread
__global__ void __launch_bounds__(256) cov_kernel(const double* __restrict__ xp, int d, const double* __restrict__ ls,
                                                  const double* __restrict__ V, int n, int P,
                                                  double* __restrict__ cov) {
  __shared__ double Vp[16][64], Vq[16][64];
  __shared__ double Bp[64][MAXD + 1], Bq[64][MAXD + 1], BBp[64], BBq[64];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int p0 = blockIdx.y * 64, q0 = blockIdx.x * 64;
  for (int e = tid; e < 64 * d; e += 256) {
    const int r = e / d, k = e % d;
    Bp[r][k] = p0 + r < P ? xp[(p0 + r) * d + k] / ls[k] : 0.0;
    Bq[r][k] = q0 + r < P ? xp[(q0 + r) * d + k] / ls[k] : 0.0;
  }
  __syncthreads();
  if (tid < 64) BBp[tid] = sq_norm(Bp[tid], d);
  else if (tid < 128) BBq[tid - 64] = sq_norm(Bq[tid - 64], d);
  double acc[4][4] = {};
  for (int k0 = 0; k0 < n; k0 += 16) {
    __syncthreads();
    for (int e = tid; e < 16 * 64; e += 256) {
      const int kk = e / 64, c = e % 64;
      const bool in = k0 + kk < n;
      Vp[kk][c] = in && p0 + c < P ? V[static_cast<size_t>(k0 + kk) * P + p0 + c] : 0.0;
      Vq[kk][c] = in && q0 + c < P ? V[static_cast<size_t>(k0 + kk) * P + q0 + c] : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < 16; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        a[r] = Vp[kk][ty + 16 * r];
        b[r] = Vq[kk][tx + 16 * r];
      }
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int s = 0; s < 4; ++s) acc[r][s] = fma(a[r], b[s], acc[r][s]);
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const int p = p0 + ty + 16 * r, q = q0 + tx + 16 * s;
      if (p < P && q < P)
        cov[static_cast<size_t>(p) * P + q] =
            gram(Bp[ty + 16 * r], BBp[ty + 16 * r], Bq[tx + 16 * s], BBq[tx + 16 * s], d) - acc[r][s];
    }
}

// gp_kernel: out (n1 x n2) row-major
__global__ void gram_kernel(const double* __restrict__ x1, int n1, const double* __restrict__ x2, int n2, int d,
                            const double* __restrict__ ls, double* __restrict__ out) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= static_cast<int64_t>(n1) * n2) return;
  const int i = static_cast<int>(e / n2), j = static_cast<int>(e % n2);
  double a[MAXD], b[MAXD];
  for (int k = 0; k < d; ++k) {
    a[k] = x1[i * d + k] / ls[k];
    b[k] = x2[j * d + k] / ls[k];
  }
  out[e] = gram(a, sq_norm(a, d), b, sq_norm(b, d), d);
}

// sequential UCB over P candidates; cols: take x P workspace (downdate columns)
__global__ void __launch_bounds__(UT) ucb_kernel(const double* __restrict__ mean, const double* __restrict__ cov, int P,
                                                 double noise, double sqrt_beta, int take, int* __restrict__ picks,
                                                 double* __restrict__ cols) {
  __shared__ double s_var[MAXP];
  __shared__ unsigned char s_act[MAXP];
  __shared__ double red_v[UT / 32];
  __shared__ int red_i[UT / 32];
  __shared__ double s_den[64];
  __shared__ int s_pick;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (int i = tid; i < P; i += UT) {
    s_var[i] = fmax(cov[static_cast<size_t>(i) * P + i], 0.0);
    s_act[i] = 1;
  }
  __syncthreads();
  for (int t = 0; t < take; ++t) {
    // argmax of ucb, first index on ties (np.argmax)
    double best = -INFINITY;
    int bi = P;
    for (int i = tid; i < P; i += UT) {
      const double u = s_act[i] ? mean[i] + sqrt_beta * sqrt(fmax(s_var[i], 0.0)) : -INFINITY;
      if (u > best || (u == best && i < bi)) {
        best = u;
        bi = i;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > best || (ov == best && oi < bi)) {
        best = ov;
        bi = oi;
      }
    }
    if (lane == 0) {
      red_v[w] = best;
      red_i[w] = bi;
    }
    __syncthreads();
    if (tid == 0) {
      double bv = red_v[0];
      int b = red_i[0];
      for (int k = 1; k < UT / 32; ++k)
        if (red_v[k] > bv || (red_v[k] == bv && red_i[k] < b)) {
          bv = red_v[k];
          b = red_i[k];
        }
      if (b >= P) b = 0;  // every ucb is -inf: np.argmax returns 0
      s_pick = b;
      picks[t] = b;
      s_act[b] = 0;
      s_den[t] = s_var[b] + noise;
    }
    __syncthreads();
    const int z = s_pick;
    const double den = s_den[t];
    if (den > 0.0) {
      double* ct = cols + static_cast<size_t>(t) * P;
      for (int i = tid; i < P; i += UT) {
        double c = cov[static_cast<size_t>(z) * P + i];  // column z (symmetric) = row z
        for (int s = 0; s < t; ++s) {
          if (!(s_den[s] > 0.0)) continue;
          const double* cs = cols + static_cast<size_t>(s) * P;
          c = c - (cs[i] * cs[z]) / s_den[s];
        }
        ct[i] = c;
      }
      __syncthreads();  // column t complete (ct[z] is read below by every thread)
      for (int i = tid; i < P; i += UT) {
        const double c = ct[i];
        s_var[i] = fmax(s_var[i] - (c * c) / den, 0.0);
      }
    }
    __syncthreads();
  }
}

}  // namespace gp
}  // namespace kt

using namespace kt;

extern "C" {

int64_t kt_gp_workspace_bytes(int32_t n, int32_t P, int32_t take) {
  // V (n x P) for the posterior covariance, downdate columns (take x P)
  return (static_cast<int64_t>(n) * P + static_cast<int64_t>(take > 0 ? take : 1) * P) * 8 + 256;
}

int kt_gp_gram(const double* x1, int32_t n1, const double* x2, int32_t n2, int32_t d, const double* ls, double* out,
               void* stream) {
  KT_REQUIRE(x1 && x2 && ls && out, KT_E_ARG, "kt_gp_gram: null pointer");
  KT_REQUIRE(n1 > 0 && n2 > 0, KT_E_EMPTY, "kt_gp_gram: empty inputs");
  KT_REQUIRE(d > 0 && d <= gp::MAXD, KT_E_UNSUPPORTED, "kt_gp_gram: 1..%d coordinates", gp::MAXD);
  const int64_t total = static_cast<int64_t>(n1) * n2;
  gp::gram_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, as_stream(stream)>>>(x1, n1, x2, n2, d, ls,
                                                                                             out);
  note_launches(1);
  return check_launch("kt_gp_gram");
}

int kt_gp_factor(const double* x, int32_t n, int32_t d, const double* ls, int32_t n_cand, const double* y,
                 double noise, double max_jitter, double* L, double* alpha, double* info, void* stream) {
  KT_REQUIRE(x && ls && y && L && alpha && info, KT_E_ARG, "kt_gp_factor: null pointer");
  KT_REQUIRE(n > 0, KT_E_EMPTY, "kt_gp_factor: no observations");
  KT_REQUIRE(n <= gp::MAXN && d > 0 && d <= gp::MAXD && n_cand > 0, KT_E_UNSUPPORTED,
             "kt_gp_factor: n <= %d observations, 1..%d coordinates", gp::MAXN, gp::MAXD);
  KT_REQUIRE(noise > 0.0, KT_E_ARG, "kt_gp_factor: noise must be positive (jitter escalates tenfold)");
  const size_t smem = (static_cast<size_t>(n) * d + 2 * n) * 8;
  KT_REQUIRE(smem <= 200 * 1024, KT_E_UNSUPPORTED, "kt_gp_factor: coordinates do not fit shared memory");
  // thread = row: 512 threads (128 registers each) up to the default observation window
  if (n <= 512) {
    cudaFuncSetAttribute(gp::factor_kernel<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    gp::factor_kernel<512><<<n_cand, 512, smem, as_stream(stream)>>>(x, n, d, ls, y, noise, max_jitter, L, alpha, info);
  } else {
    cudaFuncSetAttribute(gp::factor_kernel<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    gp::factor_kernel<1024><<<n_cand, 1024, smem, as_stream(stream)>>>(x, n, d, ls, y, noise, max_jitter, L, alpha,
                                                                      info);
  }
  note_launches(1);
  return check_launch("kt_gp_factor");
}

int kt_gp_posterior(const double* x, int32_t n, int32_t d, const double* ls, const double* L, const double* alpha,
                    const double* xp, int32_t P, double* mean, double* var, double* cov, void* workspace,
                    int64_t workspace_bytes, void* stream) {
  KT_REQUIRE(x && ls && L && alpha && xp && mean && var, KT_E_ARG, "kt_gp_posterior: null pointer");
  KT_REQUIRE(n > 0 && P > 0, KT_E_EMPTY, "kt_gp_posterior: empty inputs");
  KT_REQUIRE(n <= gp::MAXN && d > 0 && d <= gp::MAXD, KT_E_UNSUPPORTED, "kt_gp_posterior: n <= %d, d <= %d",
             gp::MAXN, gp::MAXD);
  KT_REQUIRE(!cov || (workspace && workspace_bytes >= kt_gp_workspace_bytes(n, P, 0)), KT_E_ARG,
             "kt_gp_posterior: covariance needs the workspace");
  const size_t smem = (static_cast<size_t>(n) * gp::PC + static_cast<size_t>(n) * d + n) * 8;
  KT_REQUIRE(smem <= 220 * 1024, KT_E_UNSUPPORTED, "kt_gp_posterior: %d observations do not fit shared memory", n);
  double* V = cov ? static_cast<double*>(workspace) : nullptr;
  cudaFuncSetAttribute(gp::posterior_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  gp::posterior_kernel<<<(P + gp::PC - 1) / gp::PC, gp::PT, smem, as_stream(stream)>>>(x, n, d, ls, L, alpha, xp, P,
                                                                                       mean, var, V);
  note_launches(1);
  if (cov) {
    const dim3 grid((P + 63) / 64, (P + 63) / 64);
    gp::cov_kernel<<<grid, 256, 0, as_stream(stream)>>>(xp, d, ls, V, n, P, cov);
    note_launches(1);
  }
  return check_launch("kt_gp_posterior");
}

int kt_gp_ucb(const double* mean, const double* cov, int32_t P, double noise, double beta, int32_t take,
              int32_t* picks, void* workspace, int64_t workspace_bytes, void* stream) {
  KT_REQUIRE(mean && cov && picks && workspace, KT_E_ARG, "kt_gp_ucb: null pointer");
  KT_REQUIRE(P > 0 && take > 0, KT_E_EMPTY, "kt_gp_ucb: empty pool or batch");
  KT_REQUIRE(P <= gp::MAXP && take <= 64 && take <= P, KT_E_UNSUPPORTED, "kt_gp_ucb: pool <= %d, batch <= 64",
             gp::MAXP);
  KT_REQUIRE(workspace_bytes >= static_cast<int64_t>(take) * P * 8, KT_E_ARG, "kt_gp_ucb: workspace too small");
  gp::ucb_kernel<<<1, gp::UT, 0, as_stream(stream)>>>(mean, cov, P, noise, sqrt(beta), take, picks,
                                                     static_cast<double*>(workspace));
  note_launches(1);
  return check_launch("kt_gp_ucb");
}

}  // extern "C"
