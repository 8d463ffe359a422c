// kt_sweep_host: one end-to-end sweep step from host memory, orchestrated natively.
//
// The predictor seam hands the cost model host-side candidates and wants host-side
// scores (search.py:9-10, 534-541); for a large sweep this is the whole job:
// host indices -> device -> fused scorer -> rank_history top-k -> host.  The step is
// done as: the scorer reads the pinned host indices in place (zero-copy; its index
// loads run a tile ahead, so PCIe latency hides behind the tile in flight) and
// writes scores plus the 64-bit (score, index) keys; the scores go back D2H on a
// second stream while the radix top-k ranks the keys.  One native call per step
// (the Python orchestration it replaces spent ~0.2 ms per step on bookkeeping).
#include "kt_common.cuh"

extern "C" int kt_score_indices_ex(const kt_spec_table* tab, const kt_dims* dims, const float* params,
                                   const int64_t* idx, const uint32_t* idx32, int64_t idx_base, int64_t B,
                                   float* z_out, float* u_out, uint64_t* keys_out, int32_t* err_flag, void* stream);
extern "C" int kt_topk_keys(const uint64_t* keys, int64_t B, int32_t k, int64_t* top_idx, float* top_score,
                            void* workspace, int64_t workspace_bytes, void* stream);

namespace kt {
namespace sweep {

struct Events {
  cudaEvent_t scored, done;
  bool ok = false;
};

static Events& events() {  // created once per process (the sweep runs on one device per process)
  static Events ev;
  if (!ev.ok) {
    cudaEventCreateWithFlags(&ev.scored, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ev.done, cudaEventDisableTiming);
    ev.ok = true;
  }
  return ev;
}

}  // namespace sweep
}  // namespace kt

extern "C" int kt_sweep_host(const kt_spec_table* tab, const kt_dims* dims, const float* params,
                             const void* idx_host, int32_t idx_bytes, int64_t B, uint64_t* keys_dev, float* z_dev,
                             float* z_host, int32_t k, int64_t* top_idx_dev, float* top_score_dev,
                             int64_t* top_idx_host, float* top_score_host, void* topk_ws, int64_t topk_ws_bytes,
                             int32_t* err_dev, void* stream_compute, void* stream_d2h) {
  using namespace kt;
  KT_REQUIRE(tab && dims && params && idx_host && keys_dev && z_dev && z_host && top_idx_dev && top_score_dev &&
                 top_idx_host && top_score_host && topk_ws && err_dev,
             KT_E_ARG, "kt_sweep_host: null pointer");
  KT_REQUIRE(B > 0, KT_E_EMPTY, "kt_sweep_host: empty sweep");
  KT_REQUIRE(idx_bytes == 8 || idx_bytes == 4, KT_E_ARG, "kt_sweep_host: indices are int64 or uint32");
  cudaStream_t sc = as_stream(stream_compute), sd = as_stream(stream_d2h);
  sweep::Events& ev = sweep::events();
  // the scorer reads the pinned host indices directly (zero-copy over PCIe, prefetched a
  // tile ahead) and writes the scores plus the (score, index) keys the top-k ranks
  int rc = kt_score_indices_ex(tab, dims, params, idx_bytes == 8 ? static_cast<const int64_t*>(idx_host) : nullptr,
                               idx_bytes == 4 ? static_cast<const uint32_t*>(idx_host) : nullptr, 0, B, z_dev,
                               nullptr, keys_dev, err_dev, sc);
  if (rc) return rc;
  cudaEventRecord(ev.scored, sc);
  cudaStreamWaitEvent(sd, ev.scored, 0);
  cudaMemcpyAsync(z_host, z_dev, static_cast<size_t>(B) * 4, cudaMemcpyDeviceToHost, sd);  // overlaps the top-k
  rc = kt_topk_keys(keys_dev, B, k, top_idx_dev, top_score_dev, topk_ws, topk_ws_bytes, sc);
  if (rc) return rc;
  cudaMemcpyAsync(top_idx_host, top_idx_dev, static_cast<size_t>(k) * 8, cudaMemcpyDeviceToHost, sc);
  cudaMemcpyAsync(top_score_host, top_score_dev, static_cast<size_t>(k) * 4, cudaMemcpyDeviceToHost, sc);
  cudaEventRecord(ev.done, sd);
  cudaStreamWaitEvent(sc, ev.done, 0);  // the compute stream now covers the whole step
  return check_launch("kt_sweep_host");
}
