// kt_topk / kt_topk_keys / kt_topk_merge: rank_history ordering (search.py:257-264) on device.
//
// Candidates are packed into one 64-bit key per candidate,
//   key = (descending-order code of the fp32 score) << 32 | (uint32 config index)
// so that ascending key order is exactly sorted((-score, index)) -- the reference's
// tie-break toward the lower index falls out of the low word, and keys are unique.
// Visited indices (sorted int64) are excluded by binary search (their key becomes
// EMPTY, which sorts last).
//
// Selection is a radix select, most significant digit first (11/11/10-bit digits over
// the score code, then over the index), in ONE cooperative kernel:
//   pass p   every CTA histograms the digit of the keys that match the prefix fixed so
//            far (shared-memory bins merged into global bins, three bin sets in rotation);
//            after one grid barrier every CTA scans the same bins and extends its copy of
//            the prefix by the digit that holds rank `need`.  Selection stops as soon as
//            every key at or below the prefix fits the CAP-key buffer (typically after
//            the second digit);
//   gather   every key at or below the prefix is appended to the buffer;
//   sort     the last CTA to finish gathering bitonic-sorts the buffer in shared memory
//            and emits the k smallest (arrival order varies, the set does not: the output
//            is deterministic).
// The sweep's scorer builds the keys and the first digit's histogram in its epilogue
// (kt_score_indices_ex keys_out / key_hist), so a sweep step reads its keys once for
// the second digit and once for the gather.
#include <cooperative_groups.h>

#include "kt_common.cuh"

namespace cg = cooperative_groups;

namespace kt {
namespace topk {

constexpr int NT = 512;
constexpr int MAXK = 1024;
constexpr int CAP = 4096;  // selection buffer (keys at or below the final prefix)
constexpr int NB = 2048;   // bins per pass (11-bit digits)
constexpr int PASSES = 6;
constexpr int KB = 4;  // keys per thread per batch of loads
constexpr unsigned long long EMPTY = ~0ull;

// Workspace: [counters 64 B][3 x NB bins][CAP keys].  All bins and counters are zero
// between calls (a call leaves them so); bins 0 may arrive pre-filled by the scorer.
struct Counters {
  unsigned int taken;   // gather slots used
  unsigned int arrive;  // CTAs done gathering (last one sorts)
  unsigned int pad[14];
};
static_assert(sizeof(Counters) == 64, "counter header is 64 bytes");

// per-CTA copy of the selection state (every CTA derives it from the same global bins)
struct Sel {
  unsigned long long prefix;  // digits fixed so far (right-aligned)
  int nbits;                  // bits fixed so far (0..64)
  int need;                   // rank still to find among keys matching the prefix
  int below;                  // keys strictly below the prefix
  int done;                   // every key at or below the prefix fits the buffer
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
  const unsigned long long* keys;  // ready-made keys (kt_score_indices_ex) instead of (scores, idx)
};

__device__ __forceinline__ unsigned long long key_at(const Src& s, int64_t i) {
  if (s.keys) return s.keys[i];
  const int64_t id = s.idx ? s.idx[i] : s.base + i;
  if (s.n_visited > 0 && is_visited(s.visited, s.n_visited, id)) return EMPTY;
  return (static_cast<unsigned long long>(desc_code(s.scores[i])) << 32) | static_cast<uint32_t>(id);
}

// Every CTA: find the bucket of the current digit that holds rank `need` and extend its
// copy of the prefix (the bins are global, so all CTAs reach the same decision).
__device__ void scan_bins(Sel& sel, const unsigned int* hist, int pass, unsigned int* cum, unsigned int* wsum) {
  const int db = digit_bits(pass);
  const int per = (1 << db) / NT;  // 4 or 2 bins per thread
  unsigned int mine = 0;
  for (int j = 0; j < per; ++j) mine += __ldcg(&hist[threadIdx.x * per + j]);
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
  const unsigned int need = static_cast<unsigned int>(sel.need);
  if (cum[threadIdx.x] < need && need <= cum[threadIdx.x + 1]) {
    unsigned int before = cum[threadIdx.x];
    for (int j = 0; j < per; ++j) {
      const int b = threadIdx.x * per + j;
      const unsigned int c = __ldcg(&hist[b]);
      if (before + c >= need) {
        sel.prefix = (sel.prefix << db) | static_cast<unsigned long long>(b);
        sel.nbits += db;
        sel.need = static_cast<int>(need - before);
        sel.below += static_cast<int>(before);
        sel.done = static_cast<unsigned int>(sel.below) + c <= static_cast<unsigned int>(CAP) || sel.nbits == 64;
        break;
      }
      before += c;
    }
  }
  __syncthreads();
}

__device__ void histogram(const Src& src, const Sel& sel, unsigned int* hist, unsigned int* h, int pass) {
  for (int i = threadIdx.x; i < NB; i += NT) h[i] = 0;
  __syncthreads();
  const int nbits = sel.nbits;
  const unsigned long long prefix = sel.prefix;
  const int db = digit_bits(pass);
  const int shift = 64 - nbits - db;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * NT;
  // KB keys per thread in flight (one HBM round trip per KB keys, not per key)
  for (int64_t i0 = static_cast<int64_t>(blockIdx.x) * NT + threadIdx.x; i0 < src.B; i0 += KB * stride) {
    unsigned long long kk[KB];
#pragma unroll
    for (int j = 0; j < KB; ++j) kk[j] = i0 + j * stride < src.B ? key_at(src, i0 + j * stride) : 0ull;
#pragma unroll
    for (int j = 0; j < KB; ++j) {
      const unsigned long long key = kk[j];
      if (i0 + j * stride < src.B && (nbits == 0 || (key >> (64 - nbits)) == prefix))
        atomicAdd(&h[static_cast<int>((key >> shift) & ((1u << db) - 1))], 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < (1 << db); i += NT)
    if (h[i]) atomicAdd(&hist[i], h[i]);
}

__global__ void __launch_bounds__(NT) select_kernel(Src src, Counters* ctr, unsigned int* hist3, int k,
                                                    int hist_ready, unsigned long long* buf, int64_t* top_idx,
                                                    float* top_score) {
  cg::grid_group grid = cg::this_grid();
  __shared__ unsigned int h[NB];
  __shared__ unsigned int cum[NT + 1];
  __shared__ unsigned int wsum[NT / 32];
  __shared__ Sel sel;
  __shared__ bool last;
  extern __shared__ unsigned long long sk[];  // last CTA: the sort buffer
  if (!hist_ready) {  // the caller's bins may be stale: clear, then count the first digit here
    const int64_t stride = static_cast<int64_t>(gridDim.x) * NT;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * NT + threadIdx.x; i < 3 * NB; i += stride) hist3[i] = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      ctr->taken = 0;
      ctr->arrive = 0;
    }
    if (threadIdx.x == 0) sel = Sel{0ull, 0, k, 0, 0};
    grid.sync();
    histogram(src, sel, hist3, h, 0);
    grid.sync();
  }
  if (threadIdx.x == 0) sel = Sel{0ull, 0, k, 0, src.B <= k ? 1 : 0};
  __syncthreads();
  if (!sel.done) scan_bins(sel, hist3, 0, cum, wsum);
  for (int pass = 1; pass < PASSES && !sel.done; ++pass) {
    unsigned int* bins = hist3 + (pass % 3) * NB;
    if (blockIdx.x == 0)  // bins of pass + 1 (last read two passes ago) start clean
      for (int i = threadIdx.x; i < NB; i += NT) hist3[((pass + 1) % 3) * NB + i] = 0;
    histogram(src, sel, bins, h, pass);
    grid.sync();
    scan_bins(sel, bins, pass, cum, wsum);
  }
  // gather every key at or below the prefix (<= CAP of them)
  {
    const int nbits = sel.nbits;
    const unsigned long long prefix = sel.prefix;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * NT;
    for (int64_t i0 = static_cast<int64_t>(blockIdx.x) * NT + threadIdx.x; i0 < src.B; i0 += KB * stride) {
      unsigned long long kk[KB];
#pragma unroll
      for (int j = 0; j < KB; ++j) kk[j] = i0 + j * stride < src.B ? key_at(src, i0 + j * stride) : 0ull;
#pragma unroll
      for (int j = 0; j < KB; ++j) {
        const unsigned long long key = kk[j];
        const unsigned long long kp = nbits == 0 ? 0ull : key >> (64 - nbits);
        if (i0 + j * stride < src.B && kp <= prefix) {
          const unsigned int slot = atomicAdd(&ctr->taken, 1u);
          if (slot < static_cast<unsigned int>(CAP)) buf[slot] = key;
        }
      }
    }
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&ctr->arrive, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  // ---- last CTA: sort the gathered keys, emit the k smallest, leave the workspace clean ------
  __threadfence();
  const unsigned int taken_all = __ldcg(&ctr->taken);
  const int taken = static_cast<int>(taken_all < static_cast<unsigned int>(CAP) ? taken_all : CAP);
  int n = 1;
  while (n < taken || n < k) n <<= 1;
  for (int t = threadIdx.x; t < n; t += NT) sk[t] = t < taken ? __ldcg(&buf[t]) : EMPTY;
  for (int i = threadIdx.x; i < 3 * NB; i += NT) hist3[i] = 0;
  if (threadIdx.x == 0) {
    ctr->taken = 0;
    ctr->arrive = 0;
  }
  for (int size = 2; size <= n; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int t = threadIdx.x; t < n / 2; t += NT) {
        const int i = 2 * t - (t & (stride - 1));
        const int j = i + stride;
        const bool up = (i & size) == 0;
        const unsigned long long a = sk[i], b = sk[j];
        if ((a > b) == up) {
          sk[i] = b;
          sk[j] = a;
        }
      }
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < k; t += NT) {
    const unsigned long long key = sk[t];
    if (key == EMPTY) {
      top_idx[t] = -1;
      top_score[t] = __int_as_float(0x7fc00000);
    } else {
      top_idx[t] = static_cast<int64_t>(static_cast<uint32_t>(key));
      top_score[t] = score_of(key);
    }
  }
}

static int run(const Src& src_in, int k, int hist_ready, int64_t* top_idx, float* top_score, void* ws,
               int64_t ws_bytes, cudaStream_t stream) {
  KT_REQUIRE((src_in.scores || src_in.keys) && top_idx && top_score && ws, KT_E_ARG, "kt_topk: null pointer");
  KT_REQUIRE(src_in.B > 0, KT_E_EMPTY, "kt_topk: empty candidate set");
  KT_REQUIRE(k >= 1 && k <= MAXK, KT_E_UNSUPPORTED, "kt_topk: k must be in [1, %d]", MAXK);
  KT_REQUIRE(ws_bytes >= kt_topk_workspace_bytes(src_in.B, k), KT_E_ARG, "kt_topk: workspace too small");
  Src src = src_in;
  Counters* ctr = static_cast<Counters*>(ws);
  unsigned int* hist3 = reinterpret_cast<unsigned int*>(static_cast<char*>(ws) + 64);
  unsigned long long* buf = reinterpret_cast<unsigned long long*>(static_cast<char*>(ws) + 64 + 3 * NB * 4);
  const size_t smem = static_cast<size_t>(CAP) * 8;
  static PerDeviceInt per_sms;
  int& per_sm = per_sms.get();
  if (!per_sm) {
    cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, select_kernel, NT, smem);
    if (per_sm < 1) per_sm = 1;
    if (per_sm > 2) per_sm = 2;
  }
  const int64_t want = (src.B + NT - 1) / NT;
  const int grid = static_cast<int>(want < per_sm * kNumSMs ? want : per_sm * kNumSMs);
  void* args[] = {&src, &ctr, &hist3, &k, &hist_ready, &buf, &top_idx, &top_score};
  const cudaError_t e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(select_kernel), dim3(grid), dim3(NT),
                                                    args, smem, stream);
  KT_REQUIRE(e == cudaSuccess, KT_E_CUDA, "kt_topk: cooperative launch failed (%s)", cudaGetErrorString(e));
  note_launches(1);
  return check_launch("kt_topk");
}

}  // namespace topk
}  // namespace kt

extern "C" {

int64_t kt_topk_workspace_bytes(int64_t B, int32_t k) {
  (void)B;
  (void)k;
  return 64 + 3 * kt::topk::NB * 4 + static_cast<int64_t>(kt::topk::CAP) * 8;
}

uint32_t* kt_topk_key_hist(void* workspace) {
  return workspace ? reinterpret_cast<uint32_t*>(static_cast<char*>(workspace) + 64) : nullptr;
}

int kt_topk(const float* scores, const int64_t* idx, int64_t idx_base, int64_t B, const int64_t* visited,
            int64_t n_visited, int32_t k, int64_t* top_idx, float* top_score, void* workspace,
            int64_t workspace_bytes, void* stream) {
  const kt::topk::Src src{scores, idx, idx_base, B, visited, n_visited, nullptr};
  return kt::topk::run(src, k, 0, top_idx, top_score, workspace, workspace_bytes, kt::as_stream(stream));
}

int kt_topk_keys(const uint64_t* keys, int64_t B, int32_t k, int32_t hist_ready, int64_t* top_idx,
                 float* top_score, void* workspace, int64_t workspace_bytes, void* stream) {
  const kt::topk::Src src{nullptr, nullptr, 0, B, nullptr, 0, reinterpret_cast<const unsigned long long*>(keys)};
  return kt::topk::run(src, k, hist_ready ? 1 : 0, top_idx, top_score, workspace, workspace_bytes,
                       kt::as_stream(stream));
}

int kt_topk_merge(const float* scores, const int64_t* idx, int64_t n, int32_t k, int64_t* top_idx,
                  float* top_score, void* workspace, int64_t workspace_bytes, void* stream) {
  const kt::topk::Src src{scores, idx, 0, n, nullptr, 0, nullptr};
  return kt::topk::run(src, k, 0, top_idx, top_score, workspace, workspace_bytes, kt::as_stream(stream));
}

}  // extern "C"
