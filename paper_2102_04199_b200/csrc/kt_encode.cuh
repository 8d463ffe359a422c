// Device encoder: config choices -> loop feature rows (graphs.py:89-126, 305-351).
//
// Loop k of the lowered chain is the outer loop of axis k (k < n_axes) or the
// inner loop of axis k - n_axes.  Everything that depends on one axis choice
// only (extents, log2 extents, stride hints) and the per-position constants
// come precomputed from the host table (numpy fp64 -> bit-exact); the device
// computes touched = prod of inner extents, arith = 2*touched and their log2
// in fp64 and z-normalises them with IEEE fp64 (x - mean) / std, then casts
// once to fp32.  This TU family must not be compiled with fast-math.
#pragma once

#include "kt_common.cuh"

namespace kt {

struct LoopRow {
  int axis, level, choice, extent, unrolled;
  double touched;
};

__device__ __forceinline__ int axis_choice(const kt_spec_table& T, const int* ch, int a) {
  const int kn = T.axis_knob[a];
  return kn >= 0 ? ch[kn] : 0;
}

__device__ __forceinline__ int loop_extent(const kt_spec_table& T, const int* ch, int j) {
  const int na = T.n_axes;
  const int b = j >= na ? j - na : j;
  const int c = axis_choice(T, ch, b);
  return j >= na ? T.inner[b][c] : T.outer[b][c];
}

__device__ __forceinline__ LoopRow loop_row(const kt_spec_table& T, const int* ch, int k) {
  LoopRow r;
  const int na = T.n_axes;
  r.level = k >= na;
  r.axis = r.level ? k - na : k;
  r.choice = axis_choice(T, ch, r.axis);
  r.extent = r.level ? T.inner[r.axis][r.choice] : T.outer[r.axis][r.choice];
  // touched = product of extents strictly inside loop k, multiplied innermost
  // outward like np.cumprod(e[::-1]) (exact: integers < 2^53)
  double t = 1.0;
  for (int j = T.n_loops - 1; j > k; --j) t *= static_cast<double>(loop_extent(T, ch, j));
  r.touched = t;
  r.unrolled = 0;
  if (r.level) {
    const int autov = T.auto_knob >= 0 ? T.auto_vals[ch[T.auto_knob]] : 0;
    const int expl = T.expl_knob >= 0 ? T.expl_vals[ch[T.expl_knob]] : 0;
    r.unrolled = (expl != 0) && (autov > 0) && (r.extent <= autov);
  }
  return r;
}

// Raw fp64 feature row of loop k (the values encode_batch puts in the iterval row).
__device__ __forceinline__ void raw_row(const kt_spec_table& T, const int* ch, int k, double* out) {
  const LoopRow r = loop_row(T, ch, k);
  const double t = r.touched;
  const double ar = 2.0 * t;
  const int n = T.n_loops;
  out[0] = static_cast<double>(r.extent);
  out[1] = T.raw_log2[r.level][r.axis][r.choice];
  out[2] = static_cast<double>(r.level);
  out[3] = static_cast<double>(T.axis_reduce[r.axis]);
  out[4] = static_cast<double>(r.unrolled);
  out[5] = r.level ? 1.0 : static_cast<double>(T.inner[r.axis][r.choice]);
  out[6] = t;
  out[7] = log2(t);  // t >= 1, so log2(max(t, 1)) == log2(t)
  out[8] = ar;
  out[9] = log2(ar);
  out[10] = static_cast<double>(k + 1);
  out[11] = static_cast<double>(k) / static_cast<double>(n - 1 > 1 ? n - 1 : 1);
}

__device__ __forceinline__ float znorm(const kt_spec_table& T, int slot, double x) {
  return static_cast<float>((x - T.fmean[slot]) / T.fstd[slot]);
}

// Normalised fp32 feature row of loop k (model.py:108-112 applied to raw_row).
__device__ __forceinline__ void norm_row(const kt_spec_table& T, const int* ch, int k, float* out) {
  const LoopRow r = loop_row(T, ch, k);
  const double t = r.touched;
  const double ar = 2.0 * t;
  out[0] = T.nrm_ext[k][r.choice];
  out[1] = T.nrm_log2ext[k][r.choice];
  out[2] = T.nrm_const[k][2];
  out[3] = T.nrm_const[k][3];
  out[4] = r.unrolled ? T.nrm_unroll1[k] : T.nrm_const[k][4];
  out[5] = r.level ? T.nrm_const[k][5] : T.nrm_stride[k][r.choice];
  out[6] = znorm(T, 6, t);
  out[7] = znorm(T, 7, log2(t));
  out[8] = znorm(T, 8, ar);
  out[9] = znorm(T, 9, log2(ar));
  out[10] = T.nrm_const[k][10];
  out[11] = T.nrm_const[k][11];
}

// Validates a config index and decodes it; returns false (choices zeroed) if out of range.
__device__ __forceinline__ bool decode_checked(const kt_spec_table& T, int64_t idx, int* ch) {
  if (idx < 0 || static_cast<uint64_t>(idx) >= T.space_size) {
    for (int j = 0; j < KT_MAX_KNOBS; ++j) ch[j] = 0;
    return false;
  }
  decode_choices(T, static_cast<uint64_t>(idx), ch);
  return true;
}

}  // namespace kt
