// kt_topk / kt_topk_merge: rank_history ordering (search.py:257-264) on device.
//
// Candidates are packed into one 64-bit key per candidate,
//   key = (descending-order code of the fp32 score) << 32 | (uint32 config index)
// so that ascending key order is exactly sorted((-score, index)) -- the
// reference's tie-break toward the lower index falls out of the low word, and
// keys are unique.  Visited indices (sorted int64) are excluded by binary search
// (their key becomes EMPTY, which sorts last).
//
// Selection is a radix select for the k-th smallest key T, most significant
// digit first (digits of 11/11/10 bits over the score code, then over the index):
//   pass p   every CTA histograms the digit of the keys that match the prefix
//            fixed so far (shared-memory bins, merged into global bins); the last
//            CTA to finish scans the bins, extends the prefix by the digit that
//            holds rank `need`, and stops the passes early once that bucket holds
//            exactly the keys still needed.
//   gather   keys below the prefix, plus keys equal to it, are appended to a
//            k-slot buffer (arrival order varies, the set does not);
//   sort     one CTA bitonic-sorts the k keys: the output is deterministic.
// Each pass streams the 4-byte scores once (1M candidates: 4 MB).
#include "kt_common.cuh"

namespace kt {
namespace topk {

constexpr int NT = 512;
constexpr int MAXK = 1024;
constexpr int NB = 2048;  // bins per pass (11-bit digits)
constexpr int PASSES = 6;
constexpr unsigned long long EMPTY = ~0ull;

struct State {
  unsigned long long prefix;  // digits fixed so far (right-aligned)
  int nbits;                  // bits fixed so far (0..64)
  int need;                   // rank still to find among keys matching the prefix
  int done;                   // bucket holds exactly `need` keys: stop
  int pass;
  unsigned int blocks_done;   // last-block detection
  unsigned int taken;         // gather slots used
  unsigned int taken_eq;      // gather slots used by keys equal to the prefix
  int pad;
};

__host__ __device__ constexpr int digit_bits(int pass) { return (pass % 3 == 2) ? 10 : 11; }

__device__ __forceinline__ uint32_t desc_code(float s) {
  uint32_t b = __float_as_uint(s);
  if (s != s) return 0xffffffffu;                                   // NaN ranks last
  const uint32_t asc = (b & 0x80000000u) ? ~b : (b | 0x80000000u);  // ascending code
  return ~asc;                                                      // descending
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

struct Src {
  const float* scores;
  const int64_t* idx;
  int64_t base, B;
  const int64_t* visited;
  int64_t n_visited;
  const unsigned long long* keys;  // merge mode: ready-made keys via (scores, idx) instead
};

__device__ __forceinline__ unsigned long long key_at(const Src& s, int64_t i) {
  if (s.keys) return s.keys[i];  // keys built by the scorer's epilogue (kt_score_indices_ex)
  const int64_t id = s.idx ? s.idx[i] : s.base + i;
  if (s.n_visited > 0 && is_visited(s.visited, s.n_visited, id)) return EMPTY;
  return (static_cast<unsigned long long>(desc_code(s.scores[i])) << 32) | static_cast<uint32_t>(id);
}

__global__ void init_state(State* st, unsigned int* hist, int k, int all) {
  for (int i = threadIdx.x; i < NB; i += blockDim.x) hist[i] = 0;
  if (threadIdx.x == 0) {
    st->prefix = 0;
    st->nbits = 0;
    st->need = k;
    st->done = all;  // B <= k: every candidate is selected
    st->pass = 0;
    st->blocks_done = 0;
    st->taken = 0;
    st->taken_eq = 0;
  }
}

// One radix pass: histogram + (last block) scan and prefix extension.
__global__ void __launch_bounds__(NT) hist_pass(Src src, State* st, unsigned int* __restrict__ hist) {
  __shared__ unsigned int h[NB];
  __shared__ int s_done;
  __shared__ unsigned long long s_prefix;
  __shared__ int s_nbits;
  __shared__ bool last;
  if (threadIdx.x == 0) {
    s_done = st->done;
    s_prefix = st->prefix;
    s_nbits = st->nbits;
  }
  for (int i = threadIdx.x; i < NB; i += NT) h[i] = 0;
  __syncthreads();
  if (s_done) return;
  const int nbits = s_nbits, db = digit_bits(st->pass);
  const int shift = 64 - nbits - db;
  const unsigned long long prefix = s_prefix;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * NT;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * NT + threadIdx.x; i < src.B; i += stride) {
    const unsigned long long key = key_at(src, i);
    if (nbits == 0 || (key >> (64 - nbits)) == prefix)
      atomicAdd(&h[static_cast<int>((key >> shift) & ((1u << db) - 1))], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < (1 << db); i += NT)
    if (h[i]) atomicAdd(&hist[i], h[i]);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&st->blocks_done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  // ---- last block: find the bucket holding rank `need` -------------------------------------
  __threadfence();
  __shared__ unsigned int cum[NT + 1];
  __shared__ unsigned int wsum[NT / 32];
  const int per = (1 << db) / NT;  // 4 or 2 bins per thread
  unsigned int mine = 0;
  for (int j = 0; j < per; ++j) mine += __ldcg(&hist[threadIdx.x * per + j]);
  // block-wide inclusive scan of the per-thread bin sums (warp shuffles, then warp totals)
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned int x = mine;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const unsigned int y = __shfl_up_sync(0xffffffffu, x, off);
    if (lane >= off) x += y;
  }
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  if (w == 0) {
    unsigned int t = lane < NT / 32 ? wsum[lane] : 0u;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const unsigned int y = __shfl_up_sync(0xffffffffu, t, off);
      if (lane >= off) t += y;
    }
    if (lane < NT / 32) wsum[lane] = t;
  }
  __syncthreads();
  cum[threadIdx.x + 1] = x + (w > 0 ? wsum[w - 1] : 0u);
  if (threadIdx.x == 0) cum[0] = 0;
  __syncthreads();
  const unsigned int need = static_cast<unsigned int>(st->need);
  if (cum[threadIdx.x] < need && need <= cum[threadIdx.x + 1]) {
    unsigned int before = cum[threadIdx.x];
    for (int j = 0; j < per; ++j) {
      const int b = threadIdx.x * per + j;
      const unsigned int c = __ldcg(&hist[b]);
      if (before + c >= need) {
        st->prefix = (prefix << db) | static_cast<unsigned long long>(b);
        st->nbits = nbits + db;
        st->need = static_cast<int>(need - before);
        st->done = (c == need - before) || (nbits + db == 64);
        break;
      }
      before += c;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < NB; i += NT) hist[i] = 0;
  if (threadIdx.x == 0) {
    st->pass += 1;
    st->blocks_done = 0;
  }
}

// Append every key below the prefix and (up to `need`) keys equal to it.
__global__ void __launch_bounds__(NT) gather(Src src, State* st, int k, unsigned long long* __restrict__ out) {
  const int nbits = st->nbits;
  const unsigned long long prefix = st->prefix;
  const unsigned int need = static_cast<unsigned int>(st->need);
  const int64_t stride = static_cast<int64_t>(gridDim.x) * NT;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * NT + threadIdx.x; i < src.B; i += stride) {
    const unsigned long long key = key_at(src, i);
    const unsigned long long kp = nbits == 0 ? 0ull : key >> (64 - nbits);
    if (kp < prefix) {
      const unsigned int slot = atomicAdd(&st->taken, 1u);
      if (slot < static_cast<unsigned int>(k)) out[slot] = key;
    } else if (kp == prefix) {
      if (atomicAdd(&st->taken_eq, 1u) < need) {
        const unsigned int slot = atomicAdd(&st->taken, 1u);
        if (slot < static_cast<unsigned int>(k)) out[slot] = key;
      }
    }
  }
}

// One CTA: sort the k gathered keys (EMPTY-padded) and unpack index / score.
__global__ void __launch_bounds__(NT) sort_unpack(const unsigned long long* __restrict__ keys, const State* st,
                                                  int k, int64_t* __restrict__ top_idx,
                                                  float* __restrict__ top_score) {
  __shared__ unsigned long long s[MAXK];
  int n = 1;
  while (n < k) n <<= 1;
  const unsigned int taken = st->taken < static_cast<unsigned int>(k) ? st->taken : static_cast<unsigned int>(k);
  for (int t = threadIdx.x; t < n; t += NT) s[t] = t < static_cast<int>(taken) ? keys[t] : EMPTY;
  for (int size = 2; size <= n; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int t = threadIdx.x; t < n / 2; t += NT) {
        const int i = 2 * t - (t & (stride - 1));
        const int j = i + stride;
        const bool up = (i & size) == 0;
        const unsigned long long a = s[i], b = s[j];
        if ((a > b) == up) {
          s[i] = b;
          s[j] = a;
        }
      }
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < k; t += NT) {
    const unsigned long long key = s[t];
    if (key == EMPTY) {
      top_idx[t] = -1;
      top_score[t] = __int_as_float(0x7fc00000);
    } else {
      top_idx[t] = static_cast<int64_t>(static_cast<uint32_t>(key));
      top_score[t] = score_of(key);
    }
  }
}

static int run(const float* scores, const int64_t* idx, int64_t base, int64_t B, const int64_t* visited,
               int64_t n_visited, int k, int64_t* top_idx, float* top_score, void* ws, int64_t ws_bytes,
               cudaStream_t stream, const unsigned long long* keys = nullptr) {
  KT_REQUIRE((scores || keys) && top_idx && top_score && ws, KT_E_ARG, "kt_topk: null pointer");
  KT_REQUIRE(B > 0, KT_E_EMPTY, "kt_topk: empty candidate set");
  KT_REQUIRE(k >= 1 && k <= MAXK, KT_E_UNSUPPORTED, "kt_topk: k must be in [1, %d]", MAXK);
  KT_REQUIRE(ws_bytes >= kt_topk_workspace_bytes(B, k), KT_E_ARG, "kt_topk: workspace too small");
  State* st = static_cast<State*>(ws);
  unsigned int* hist = reinterpret_cast<unsigned int*>(static_cast<char*>(ws) + 64);
  unsigned long long* buf = reinterpret_cast<unsigned long long*>(static_cast<char*>(ws) + 64 + NB * 4);
  Src src{scores, idx, base, B, visited, n_visited, keys};
  const int64_t want = (B + NT - 1) / NT;
  const int grid = static_cast<int>(want < 2 * kNumSMs ? want : 2 * kNumSMs);
  init_state<<<1, 256, 0, stream>>>(st, hist, k, B <= k ? 1 : 0);
  for (int p = 0; p < PASSES; ++p) hist_pass<<<grid, NT, 0, stream>>>(src, st, hist);
  gather<<<grid, NT, 0, stream>>>(src, st, k, buf);
  sort_unpack<<<1, NT, 0, stream>>>(buf, st, k, top_idx, top_score);
  note_launches(PASSES + 3);
  return check_launch("kt_topk");
}

}  // namespace topk
}  // namespace kt

extern "C" {

int64_t kt_topk_workspace_bytes(int64_t B, int32_t k) {
  (void)B;
  return 64 + kt::topk::NB * 4 + static_cast<int64_t>(k < 1 ? 1 : k) * 8;
}

int kt_topk(const float* scores, const int64_t* idx, int64_t idx_base, int64_t B, const int64_t* visited,
            int64_t n_visited, int32_t k, int64_t* top_idx, float* top_score, void* workspace,
            int64_t workspace_bytes, void* stream) {
  return kt::topk::run(scores, idx, idx_base, B, visited, n_visited, k, top_idx, top_score, workspace,
                       workspace_bytes, kt::as_stream(stream));
}

int kt_topk_keys(const uint64_t* keys, int64_t B, int32_t k, int64_t* top_idx, float* top_score, void* workspace,
                 int64_t workspace_bytes, void* stream) {
  return kt::topk::run(nullptr, nullptr, 0, B, nullptr, 0, k, top_idx, top_score, workspace, workspace_bytes,
                       kt::as_stream(stream), reinterpret_cast<const unsigned long long*>(keys));
}

int kt_topk_merge(const float* scores, const int64_t* idx, int64_t n, int32_t k, int64_t* top_idx,
                  float* top_score, void* workspace, int64_t workspace_bytes, void* stream) {
  return kt::topk::run(scores, idx, 0, n, nullptr, 0, k, top_idx, top_score, workspace, workspace_bytes,
                       kt::as_stream(stream));
}

}  // extern "C"
