// kt_sweep_host: one end-to-end sweep step from host memory, orchestrated natively.
//
// The predictor seam hands the cost model host-side candidates and wants host-side
// scores (search.py:9-10, 534-541); for a large sweep this is the whole job:
// host indices -> device -> fused scorer -> rank_history top-k -> host.  The step is
// done as: the scorer reads the pinned host indices in place (zero-copy; its index
// loads run a tile ahead, so PCIe latency hides behind the tile in flight), writes
// the scores straight into pinned host memory (posted PCIe writes, 512 B per tile)
// and the 64-bit (score, index) keys into HBM; the radix top-k ranks the keys and
// only the k winners are copied back.  One native call per step.
#include "kt_common.cuh"

extern "C" int kt_score_indices_ex(const kt_spec_table* tab, const kt_dims* dims, const float* params,
                                   const int64_t* idx, const uint32_t* idx32, int64_t idx_base, int64_t B,
                                   float* z_out, float* u_out, uint64_t* keys_out, uint32_t* key_hist,
                                   int32_t* err_flag, void* stream);
extern "C" int kt_topk_keys(const uint64_t* keys, int64_t B, int32_t k, int32_t hist_ready, int64_t* top_idx,
                            float* top_score, void* workspace, int64_t workspace_bytes, void* stream);
extern "C" uint32_t* kt_topk_key_hist(void* workspace);

extern "C" int kt_sweep_host(const kt_spec_table* tab, const kt_dims* dims, const float* params,
                             const void* idx_host, int32_t idx_bytes, int64_t B, uint64_t* keys_dev, float* z_host,
                             int32_t k, int64_t* top_idx_dev, float* top_score_dev, int64_t* top_idx_host,
                             float* top_score_host, void* topk_ws, int64_t topk_ws_bytes, int32_t* err_dev,
                             void* stream) {
  using namespace kt;
  KT_REQUIRE(tab && dims && params && idx_host && keys_dev && z_host && top_idx_dev && top_score_dev &&
                 top_idx_host && top_score_host && topk_ws && err_dev,
             KT_E_ARG, "kt_sweep_host: null pointer");
  KT_REQUIRE(B > 0, KT_E_EMPTY, "kt_sweep_host: empty sweep");
  KT_REQUIRE(idx_bytes == 8 || idx_bytes == 4, KT_E_ARG, "kt_sweep_host: indices are int64 or uint32");
  cudaStream_t st = as_stream(stream);
  // the scorer reads the pinned host indices and writes the pinned host scores in place
  // (zero-copy both ways: the PCIe traffic rides under the kernel's tensor-core work)
  // plus the (score, index) keys in HBM; the radix top-k ranks the keys
  int rc = kt_score_indices_ex(tab, dims, params, idx_bytes == 8 ? static_cast<const int64_t*>(idx_host) : nullptr,
                               idx_bytes == 4 ? static_cast<const uint32_t*>(idx_host) : nullptr, 0, B, z_host,
                               nullptr, keys_dev, kt_topk_key_hist(topk_ws), err_dev, st);
  if (rc) return rc;
  rc = kt_topk_keys(keys_dev, B, k, 1, top_idx_dev, top_score_dev, topk_ws, topk_ws_bytes, st);
  if (rc) return rc;
  cudaMemcpyAsync(top_idx_host, top_idx_dev, static_cast<size_t>(k) * 8, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(top_score_host, top_score_dev, static_cast<size_t>(k) * 4, cudaMemcpyDeviceToHost, st);
  return check_launch("kt_sweep_host");
}
