// kt_encode_raw*: encode_batch (graphs.py:305-351) on device, raw fp64 output.
//
// One thread per (graph, node row): threads of a warp write consecutive
// 96-byte rows, so the (B, N, 12) fp64 output is written fully coalesced.
// Rows that are not iterval rows of the layout stay exactly zero.
#include "kt_encode.cuh"

namespace kt {

template <bool FROM_CHOICES>
__global__ void __launch_bounds__(256) encode_raw_kernel(const kt_spec_table* __restrict__ tab,
                                                         const int64_t* __restrict__ src, int64_t B,
                                                         double* __restrict__ out,
                                                         int32_t* __restrict__ err) {
  __shared__ int s_row_loop[64];  // node row -> loop index or -1
  // a block's rows are consecutive in the output: staged here, then written as one contiguous
  // run of 16-byte pieces (a thread's own row is 96 bytes: direct stores would leave every
  // warp store instruction scattered over 3 KB)
  __shared__ double2 s_out[256 * KT_F / 2];
  const kt_spec_table& T = *tab;
  const int N = T.n_nodes;
  for (int i = threadIdx.x; i < N && i < 64; i += blockDim.x) s_row_loop[i] = -1;
  __syncthreads();
  if (threadIdx.x < T.n_loops) s_row_loop[T.loop_row[threadIdx.x]] = threadIdx.x;
  __syncthreads();

  const int64_t total = B * N;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < total; base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t item = base + threadIdx.x;
    const int64_t g = item / N;
    const int row = static_cast<int>(item - g * N);
    double feat[KT_F];
#pragma unroll
    for (int f = 0; f < KT_F; ++f) feat[f] = 0.0;
    const int k = item < total ? s_row_loop[row] : -1;
    if (k >= 0) {
      int ch[KT_MAX_KNOBS];
      bool ok = true;
      if (FROM_CHOICES) {
        for (int j = 0; j < T.n_knobs; ++j) {
          const int64_t c = src[g * T.n_knobs + j];
          ok = ok && c >= 0 && c < static_cast<int64_t>(T.card[j]);
          ch[j] = ok ? static_cast<int>(c) : 0;
        }
        for (int j = T.n_knobs; j < KT_MAX_KNOBS; ++j) ch[j] = 0;
      } else {
        ok = decode_checked(T, src[g], ch);
      }
      if (ok) {
        raw_row(T, ch, k, feat);
      } else if (k == 0) {
        atomicOr(err, 1);
      }
    }
    if (item < total) {
#pragma unroll
      for (int f = 0; f < KT_F; f += 2) s_out[threadIdx.x * (KT_F / 2) + f / 2] = make_double2(feat[f], feat[f + 1]);
    }
    __syncthreads();
    const int64_t n_items = total - base < blockDim.x ? total - base : blockDim.x;
    double2* o = reinterpret_cast<double2*>(out + base * KT_F);
    for (int e = threadIdx.x; e < n_items * (KT_F / 2); e += blockDim.x) o[e] = s_out[e];
    __syncthreads();
  }
}

static int launch_encode(const kt_spec_table* tab, const int64_t* src, int64_t B, double* out,
                         int32_t* err, void* stream, bool choices) {
  KT_REQUIRE(tab && src && out && err, KT_E_ARG, "kt_encode: null pointer");
  KT_REQUIRE(B > 0, KT_E_EMPTY, "kt_encode: empty batch");
  const int threads = 256;
  int64_t blocks = (B * KT_MAX_NODES + threads - 1) / threads;
#ifndef KT_ENC_BPS
#define KT_ENC_BPS 64
#endif
  if (blocks > kNumSMs * KT_ENC_BPS) blocks = kNumSMs * KT_ENC_BPS;
  if (choices)
    encode_raw_kernel<true><<<(int)blocks, threads, 0, as_stream(stream)>>>(tab, src, B, out, err);
  else
    encode_raw_kernel<false><<<(int)blocks, threads, 0, as_stream(stream)>>>(tab, src, B, out, err);
  note_launches(1);
  return check_launch("kt_encode_raw");
}

}  // namespace kt

extern "C" {

int kt_encode_raw(const kt_spec_table* tab, const int64_t* idx, int64_t B, double* feats_out,
                  int32_t* err_flag, void* stream) {
  return kt::launch_encode(tab, idx, B, feats_out, err_flag, stream, false);
}

int kt_encode_raw_choices(const kt_spec_table* tab, const int64_t* choices, int64_t B,
                          double* feats_out, int32_t* err_flag, void* stream) {
  return kt::launch_encode(tab, choices, B, feats_out, err_flag, stream, true);
}

}  // extern "C"
