// kt_topk / kt_topk_merge: rank_history ordering (search.py:257-264) on device.
//
// Candidates are packed into one 64-bit key per candidate,
//   key = (descending-order code of the fp32 score) << 32 | (uint32 config index)
// so that ascending key order is exactly sorted((-score, index)) -- the
// reference's tie-break toward the lower index falls out of the low word.
// Visited indices (sorted int64) are excluded by binary search.  Selection is
// a chunked reduction: each CTA bitonic-sorts a 4096-key chunk in shared
// memory and keeps its k smallest; rounds repeat over the survivors until one
// chunk remains.  Deterministic (no atomics, no data-dependent launch order).
#include "kt_common.cuh"

namespace kt {
namespace topk {

constexpr int CHUNK = 4096;
constexpr int NT = 512;
constexpr unsigned long long EMPTY = ~0ull;

__device__ __forceinline__ uint32_t desc_code(float s) {
  uint32_t b = __float_as_uint(s);
  if (s != s) return 0xffffffffu;                      // NaN ranks last
  const uint32_t asc = (b & 0x80000000u) ? ~b : (b | 0x80000000u);  // ascending code
  return ~asc;                                         // descending
}

__device__ __forceinline__ float score_of(unsigned long long key) {
  const uint32_t asc = ~static_cast<uint32_t>(key >> 32);
  const uint32_t b = (asc & 0x80000000u) ? (asc & 0x7fffffffu) : ~asc;
  return __uint_as_float(b);
}

__device__ __forceinline__ bool is_visited(const int64_t* v, int64_t n, int64_t x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (v[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo < n && v[lo] == x;
}

__device__ void bitonic_sort(unsigned long long* s) {
  for (int size = 2; size <= CHUNK; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int t = threadIdx.x; t < CHUNK / 2; t += NT) {
        const int i = 2 * t - (t & (stride - 1));
        const int j = i + stride;
        const bool up = (i & size) == 0;
        const unsigned long long a = s[i], b = s[j];
        if ((a > b) == up) { s[i] = b; s[j] = a; }
      }
    }
  }
  __syncthreads();
}

// Round 0: build keys from (scores, idx or base) and reduce each chunk to k keys.
__global__ void __launch_bounds__(NT) first_round(const float* __restrict__ scores,
                                                  const int64_t* __restrict__ idx, int64_t base, int64_t B,
                                                  const int64_t* __restrict__ visited, int64_t n_visited,
                                                  int k, unsigned long long* __restrict__ out) {
  __shared__ unsigned long long s[CHUNK];
  const int64_t c0 = static_cast<int64_t>(blockIdx.x) * CHUNK;
  for (int t = threadIdx.x; t < CHUNK; t += NT) {
    const int64_t i = c0 + t;
    unsigned long long key = EMPTY;
    if (i < B) {
      const int64_t id = idx ? idx[i] : base + i;
      if (!(n_visited > 0 && is_visited(visited, n_visited, id)))
        key = (static_cast<unsigned long long>(desc_code(scores[i])) << 32) | static_cast<uint32_t>(id);
    }
    s[t] = key;
  }
  bitonic_sort(s);
  for (int t = threadIdx.x; t < k; t += NT) out[static_cast<int64_t>(blockIdx.x) * k + t] = s[t];
}

__global__ void __launch_bounds__(NT) next_round(const unsigned long long* __restrict__ in, int64_t n, int k,
                                                 unsigned long long* __restrict__ out) {
  __shared__ unsigned long long s[CHUNK];
  const int64_t c0 = static_cast<int64_t>(blockIdx.x) * CHUNK;
  for (int t = threadIdx.x; t < CHUNK; t += NT) {
    const int64_t i = c0 + t;
    s[t] = i < n ? in[i] : EMPTY;
  }
  bitonic_sort(s);
  for (int t = threadIdx.x; t < k; t += NT) out[static_cast<int64_t>(blockIdx.x) * k + t] = s[t];
}

__global__ void unpack(const unsigned long long* __restrict__ keys, int k, int64_t* __restrict__ top_idx,
                       float* __restrict__ top_score) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= k) return;
  const unsigned long long key = keys[t];
  if (key == EMPTY) {
    top_idx[t] = -1;
    top_score[t] = __int_as_float(0x7fc00000);
  } else {
    top_idx[t] = static_cast<int64_t>(static_cast<uint32_t>(key));
    top_score[t] = score_of(key);
  }
}

static int64_t n_chunks(int64_t n) { return (n + CHUNK - 1) / CHUNK; }

static int run(const float* scores, const int64_t* idx, int64_t base, int64_t B, const int64_t* visited,
               int64_t n_visited, int k, int64_t* top_idx, float* top_score, void* ws, int64_t ws_bytes,
               cudaStream_t st) {
  KT_REQUIRE(scores && top_idx && top_score && ws, KT_E_ARG, "kt_topk: null pointer");
  KT_REQUIRE(B > 0, KT_E_EMPTY, "kt_topk: empty candidate set");
  KT_REQUIRE(k >= 1 && k <= CHUNK / 4, KT_E_UNSUPPORTED, "kt_topk: k must be in [1, %d]", CHUNK / 4);
  KT_REQUIRE(ws_bytes >= kt_topk_workspace_bytes(B, k), KT_E_ARG, "kt_topk: workspace too small");
  unsigned long long* a = static_cast<unsigned long long*>(ws);
  unsigned long long* b = a + n_chunks(B) * k;
  int64_t chunks = n_chunks(B);
  first_round<<<static_cast<int>(chunks), NT, 0, st>>>(scores, idx, base, B, visited, n_visited, k, a);
  int launches = 2;
  int64_t n = chunks * k;
  while (n > k) {
    const int64_t c = n_chunks(n);
    next_round<<<static_cast<int>(c), NT, 0, st>>>(a, n, k, b);
    ++launches;
    unsigned long long* t = a; a = b; b = t;
    n = c * k;
    if (c == 1) break;
  }
  unpack<<<(k + 255) / 256, 256, 0, st>>>(a, k, top_idx, top_score);
  note_launches(launches);
  return check_launch("kt_topk");
}

}  // namespace topk
}  // namespace kt

extern "C" {

int64_t kt_topk_workspace_bytes(int64_t B, int32_t k) {
  const int64_t first = kt::topk::n_chunks(B) * k;
  return (first + kt::topk::n_chunks(first) * k + 2 * k) * 8;
}

int kt_topk(const float* scores, const int64_t* idx, int64_t idx_base, int64_t B, const int64_t* visited,
            int64_t n_visited, int32_t k, int64_t* top_idx, float* top_score, void* workspace,
            int64_t workspace_bytes, void* stream) {
  return kt::topk::run(scores, idx, idx_base, B, visited, n_visited, k, top_idx, top_score, workspace,
                       workspace_bytes, kt::as_stream(stream));
}

int kt_topk_merge(const float* scores, const int64_t* idx, int64_t n, int32_t k, int64_t* top_idx,
                  float* top_score, void* workspace, int64_t workspace_bytes, void* stream) {
  return kt::topk::run(scores, idx, 0, n, nullptr, 0, k, top_idx, top_score, workspace, workspace_bytes,
                       kt::as_stream(stream));
}

}  // extern "C"
