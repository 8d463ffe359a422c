// Simulated-annealing exploration (sa_explore, search.py:202-254) on the device.
//
// The chains' random draws (knob, nudge, delta, resample, u per step and chain)
// do not depend on the predictions, so the host draws them from the caller's
// numpy Generator in the reference's order and uploads them once; the device then
// runs every step:  kt_sa_propose (the nudged / resampled neighbour and its config
// index, search.py:232-241), the fused scorer on the n_chains neighbours, and
// kt_sa_accept (Metropolis test in fp64, search.py:246-251).  With the same draws
// and the same predictor values the trajectory -- and so the exploration history
// -- is identical to the reference loop's.
#include "kt_common.cuh"

namespace kt {
namespace sa {
// Each step is propose -> scorer -> accept, all three launched as programmatic
// dependents: a kernel's launch (and the scorer's table prologue) overlaps the
// previous kernel, and pdl_wait() orders every global access after it.

__global__ void propose_kernel(const int32_t* __restrict__ cur, int n_chains, int n_knobs,
                               const int32_t* __restrict__ cards, const int64_t* __restrict__ mult,
                               const int32_t* __restrict__ knob, const uint8_t* __restrict__ nudge,
                               const int32_t* __restrict__ delta, const int32_t* __restrict__ resample,
                               int32_t* __restrict__ nxt, int64_t* __restrict__ nxt_idx) {
  pdl_launch_dependents();  // the scorer may start its prologue now
  pdl_wait();               // cur / nxt: the previous accept
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n_chains) return;
  const int kn = knob[c];
  int64_t id = 0;
  for (int j = 0; j < n_knobs; ++j) {
    int v = cur[c * n_knobs + j];
    if (j == kn) {
      // np.clip(cur + delta, 0, card - 1) if nudge else resample (search.py:239-241)
      const int stepped = min(max(v + delta[c], 0), cards[j] - 1);
      v = nudge[c] ? stepped : resample[c];
    }
    nxt[c * n_knobs + j] = v;
    id += static_cast<int64_t>(v) * mult[j];  // (mat * mult).sum(axis=1), search.py:220-221
  }
  nxt_idx[c] = id;
}

__global__ void accept_kernel(int n_chains, int n_knobs, const float* __restrict__ e_new,
                              const double* __restrict__ u, double temp, const int32_t* __restrict__ nxt,
                              int32_t* __restrict__ cur, double* __restrict__ energy) {
  pdl_launch_dependents();
  pdl_wait();  // e_new: the scorer
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n_chains) return;
  const double en = static_cast<double>(e_new[c]);
  const double eo = energy[c];
  // downhill_p = exp(min((e_new - energy) / temp, 0)); uphill always accepted (search.py:246-248)
  const double p = exp(fmin((en - eo) / temp, 0.0));
  const bool acc = (en >= eo) || (u[c] < p);
  if (acc) {
    for (int j = 0; j < n_knobs; ++j) cur[c * n_knobs + j] = nxt[c * n_knobs + j];
    energy[c] = en;
  }
}

// ---- numpy Generator(PCG64) stream, on the host -----------------------------------------
// The reference draws each step's randoms with five Generator calls (search.py:233-237);
// in Python that is ~2 us per call.  These are the same draws from the same bit-generator
// state (numpy's PCG64: 128-bit LCG, XSL-RR output; 32-bit draws take the low half of a
// 64-bit output and buffer the high half in the state; bounded integers by Lemire's
// multiply-shift with rejection; doubles as (next64 >> 11) * 2^-53), pinned bit for bit
// against numpy in tests/test_sa.py.
struct Pcg64 {
  unsigned __int128 state, inc;
  int has32;
  uint32_t buf32;
  uint64_t next64() {
    const unsigned __int128 mult =
        (static_cast<unsigned __int128>(0x2360ED051FC65DA4ULL) << 64) | 0x4385DF649FCCF645ULL;
    state = state * mult + inc;
    const uint64_t hi = static_cast<uint64_t>(state >> 64), lo = static_cast<uint64_t>(state);
    const unsigned rot = static_cast<unsigned>(state >> 122);
    const uint64_t x = hi ^ lo;
    return (x >> rot) | (x << ((64 - rot) & 63));
  }
  uint32_t next32() {
    if (has32) {
      has32 = 0;
      return buf32;
    }
    const uint64_t v = next64();
    has32 = 1;
    buf32 = static_cast<uint32_t>(v >> 32);
    return static_cast<uint32_t>(v);
  }
  double next_double() { return static_cast<double>(next64() >> 11) * (1.0 / 9007199254740992.0); }
  // integers(0, rng + 1): Lemire's bounded draw on 32-bit outputs (rng < 2^32 - 1)
  uint32_t bounded(uint32_t rng) {
    if (rng == 0) return 0;
    const uint32_t excl = rng + 1;
    uint64_t m = static_cast<uint64_t>(next32()) * excl;
    uint32_t left = static_cast<uint32_t>(m);
    if (left < excl) {
      const uint32_t threshold = (0xFFFFFFFFu - rng) % excl;
      while (left < threshold) {
        m = static_cast<uint64_t>(next32()) * excl;
        left = static_cast<uint32_t>(m);
      }
    }
    return static_cast<uint32_t>(m >> 32);
  }
};

}  // namespace sa
}  // namespace kt

extern "C" int kt_sa_draws(uint64_t* pcg, int32_t* has_uint32, uint32_t* uinteger, int32_t n_steps,
                           int32_t n_chains, int32_t n_knobs, const int32_t* cards, int32_t* knob, uint8_t* nudge,
                           int32_t* delta, int32_t* resample, double* u) {
  KT_REQUIRE(pcg && has_uint32 && uinteger && cards && knob && nudge && delta && resample && u, KT_E_ARG,
             "kt_sa_draws: null pointer");
  KT_REQUIRE(n_steps >= 0 && n_chains >= 0, KT_E_SHAPE, "kt_sa_draws: negative size");
  KT_REQUIRE(n_knobs > 0 && n_knobs <= KT_MAX_KNOBS, KT_E_SHAPE, "kt_sa_draws: 1..%d knobs", KT_MAX_KNOBS);
  for (int j = 0; j < n_knobs; ++j) KT_REQUIRE(cards[j] >= 1, KT_E_RANGE, "kt_sa_draws: empty knob %d", j);
  // PCG64's increment is odd (numpy's always is); an even one can cycle on a fixed point,
  // where the bounded draws' rejection loop would never end
  KT_REQUIRE((pcg[3] & 1u) == 1u, KT_E_ARG, "kt_sa_draws: not a PCG64 state (even increment)");
  kt::sa::Pcg64 g;
  g.state = (static_cast<unsigned __int128>(pcg[0]) << 64) | pcg[1];
  g.inc = (static_cast<unsigned __int128>(pcg[2]) << 64) | pcg[3];
  g.has32 = *has_uint32 != 0;
  g.buf32 = *uinteger;
  for (int64_t s = 0; s < n_steps; ++s) {
    const int64_t o = s * n_chains;
    for (int c = 0; c < n_chains; ++c) knob[o + c] = static_cast<int32_t>(g.bounded(n_knobs - 1));
    for (int c = 0; c < n_chains; ++c) nudge[o + c] = g.next_double() < 0.5;
    for (int c = 0; c < n_chains; ++c) delta[o + c] = static_cast<int32_t>(g.bounded(1)) * 2 - 1;
    for (int c = 0; c < n_chains; ++c) resample[o + c] = static_cast<int32_t>(g.bounded(cards[knob[o + c]] - 1));
    for (int c = 0; c < n_chains; ++c) u[o + c] = g.next_double();
  }
  pcg[0] = static_cast<uint64_t>(g.state >> 64);
  pcg[1] = static_cast<uint64_t>(g.state);
  *has_uint32 = g.has32;
  *uinteger = g.buf32;
  return KT_OK;
}

extern "C" int kt_sa_propose(const int32_t* cur, int32_t n_chains, int32_t n_knobs, const int32_t* cards,
                             const int64_t* mult, const int32_t* knob, const uint8_t* nudge, const int32_t* delta,
                             const int32_t* resample, int32_t* nxt, int64_t* nxt_idx, void* stream) {
  KT_REQUIRE(cur && cards && mult && knob && nudge && delta && resample && nxt && nxt_idx, KT_E_ARG,
             "kt_sa_propose: null pointer");
  KT_REQUIRE(n_chains > 0, KT_E_EMPTY, "kt_sa_propose: no chains");
  KT_REQUIRE(n_knobs > 0 && n_knobs <= KT_MAX_KNOBS, KT_E_SHAPE, "kt_sa_propose: 1..%d knobs", KT_MAX_KNOBS);
  const cudaError_t e = kt::launch_pdl(kt::sa::propose_kernel, dim3((n_chains + 127) / 128), dim3(128), 0,
                                       kt::as_stream(stream), cur, n_chains, n_knobs, cards, mult, knob, nudge,
                                       delta, resample, nxt, nxt_idx);
  KT_REQUIRE(e == cudaSuccess, KT_E_CUDA, "kt_sa_propose: %s", cudaGetErrorString(e));
  kt::note_launches(1);
  return kt::check_launch("kt_sa_propose");
}

extern "C" int kt_sa_accept(int32_t n_chains, int32_t n_knobs, const float* e_new, const double* u, double temp,
                            const int32_t* nxt, int32_t* cur, double* energy, void* stream) {
  KT_REQUIRE(e_new && u && nxt && cur && energy, KT_E_ARG, "kt_sa_accept: null pointer");
  KT_REQUIRE(n_chains > 0, KT_E_EMPTY, "kt_sa_accept: no chains");
  KT_REQUIRE(temp > 0.0, KT_E_RANGE, "kt_sa_accept: temperature must be positive");
  const cudaError_t e = kt::launch_pdl(kt::sa::accept_kernel, dim3((n_chains + 127) / 128), dim3(128), 0,
                                       kt::as_stream(stream), n_chains, n_knobs, e_new, u, temp, nxt, cur, energy);
  KT_REQUIRE(e == cudaSuccess, KT_E_CUDA, "kt_sa_accept: %s", cudaGetErrorString(e));
  kt::note_launches(1);
  return kt::check_launch("kt_sa_accept");
}
