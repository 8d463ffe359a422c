// Library plumbing: thread-local error text, launch checks, sync.
#include <atomic>
#include <cstdarg>
#include <cstdio>

#include <cstdlib>

#include "kt_common.cuh"

namespace kt {

static thread_local char g_err[512] = "";
static std::atomic<long long> g_launches{0};

void note_launches(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

bool pdl_enabled() {
  static const bool on = std::getenv("KT_NO_PDL") == nullptr;
  return on;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(KT_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return KT_OK;
}

}  // namespace kt

extern "C" {

int kt_version(void) { return 1; }

int64_t kt_launch_count(void) { return kt::g_launches.load(std::memory_order_relaxed); }

const char* kt_last_error(void) { return kt::g_err; }

int kt_sync_check(void* stream) {
  cudaError_t e = cudaStreamSynchronize(kt::as_stream(stream));
  if (e != cudaSuccess) return kt::fail(KT_E_CUDA, "stream sync: %s", cudaGetErrorString(e));
  e = cudaGetLastError();
  if (e != cudaSuccess) return kt::fail(KT_E_CUDA, "sticky error: %s", cudaGetErrorString(e));
  return KT_OK;
}

}  // extern "C"
