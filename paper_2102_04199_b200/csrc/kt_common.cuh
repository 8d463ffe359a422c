// Shared device/host helpers for the sm_100a MetaTune library.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "../../include/kerntune_b200.h"

namespace kt {

constexpr int kNumSMs = 148;

// ---- error reporting (thread-local; read back through kt_last_error) --------
void set_error(const char* fmt, ...);
int fail(int code, const char* fmt, ...);
int check_launch(const char* what);
void note_launches(int n);  // kernel launches issued (kt_launch_count)

#define KT_REQUIRE(cond, code, ...)          \
  do {                                       \
    if (!(cond)) return ::kt::fail((code), __VA_ARGS__); \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Kernel attributes are per-device state: launch sites cache "already set" per device,
// so a process that drives several GPUs (or switches devices) sets them on each.
constexpr int kMaxDevices = 64;
inline int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev >= 0 && dev < kMaxDevices ? dev : 0;
}
struct SmemAttr {
  bool done[kMaxDevices] = {};
  // lift the kernel's dynamic shared memory limit (once per device) to the sm_100 opt-in
  // maximum, never to just `bytes`: several entry points launch the same kernel with
  // their own SmemAttr, and a smaller limit set through one would fail another's launch
  template <class K>
  void ensure(K kernel, size_t bytes) {
    const int dev = current_device();
    if (bytes > 48 * 1024 && !done[dev]) {
      int optin = 227 * 1024;
      cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
      cudaFuncAttributes fa{};
      cudaFuncGetAttributes(&fa, kernel);
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           optin - static_cast<int>(fa.sharedSizeBytes));
      done[dev] = true;
    }
  }
};
// ---- programmatic dependent launch (PDL).  A kernel launched with launch_pdl may start
// while the previous kernel in the stream is still running (once every CTA of that one
// has called pdl_launch_dependents or exited); it must call pdl_wait() before touching
// any memory an earlier kernel writes or reads.  Outside PDL both are no-ops.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;"); }

bool pdl_enabled();  // false when KT_NO_PDL is set (A/B switch)

template <class... KArgs, class... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                       Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

struct PerDeviceInt {
  int v[kMaxDevices] = {};
  int& get() { return v[current_device()]; }
};

// ---- packed fp32x2 FMA (FFMA2).  ptxas folds a scalar broadcast into the
// `Rn.F32` operand form, so `ffma2(s, pair, acc)` costs one issue slot for two FMAs.
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(d)
      : "l"(*reinterpret_cast<unsigned long long*>(&a)),
        "l"(*reinterpret_cast<unsigned long long*>(&b)),
        "l"(*reinterpret_cast<unsigned long long*>(&c)));
  return *reinterpret_cast<float2*>(&d);
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;"
      : "=l"(d)
      : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)));
  return *reinterpret_cast<float2*>(&d);
}
__device__ __forceinline__ float2 fsub2(float2 a, float2 b) {
  unsigned long long d;
  asm("sub.rn.f32x2 %0, %1, %2;"
      : "=l"(d)
      : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)));
  return *reinterpret_cast<float2*>(&d);
}
__device__ __forceinline__ float2 ffma2s(float s, float2 b, float2 c) {
  return ffma2(make_float2(s, s), b, c);
}

// ---- spec-table based encoder pieces (graphs.py:89-126, 305-351) -------------

// Mixed-radix decode, knob 0 most significant (kernels.py:278-286).
__device__ __forceinline__ void decode_choices(const kt_spec_table& T, uint64_t idx, int* ch) {
  if (T.space_size <= 0xffffffffull) {
    uint32_t v = static_cast<uint32_t>(idx);
    for (int j = T.n_knobs - 1; j >= 0; --j) {
      uint32_t c = T.card[j];
      uint32_t q = v / c;
      ch[j] = static_cast<int>(v - q * c);
      v = q;
    }
  } else {
    for (int j = T.n_knobs - 1; j >= 0; --j) {
      uint64_t c = T.card[j];
      uint64_t q = idx / c;
      ch[j] = static_cast<int>(idx - q * c);
      idx = q;
    }
  }
}

// Per-loop extents (outer loops then inner loops), tile choice per axis, unroll flag.
struct LoopInfo {
  int e[KT_MAX_LOOPS];
  int axis_choice[KT_MAX_AXES];
  int unrolled[KT_MAX_AXES];
};

__device__ __forceinline__ void loop_info(const kt_spec_table& T, const int* ch, LoopInfo& L) {
  const int na = T.n_axes;
  const int autov = T.auto_knob >= 0 ? T.auto_vals[ch[T.auto_knob]] : 0;
  const int expl = T.expl_knob >= 0 ? T.expl_vals[ch[T.expl_knob]] : 0;
#pragma unroll
  for (int a = 0; a < KT_MAX_AXES; ++a) {
    if (a < na) {
      const int c = T.axis_knob[a] >= 0 ? ch[T.axis_knob[a]] : 0;
      L.axis_choice[a] = c;
      const int t = T.inner[a][c];
      L.e[a] = T.outer[a][c];
      L.e[na + a] = t;
      L.unrolled[a] = (expl != 0) && (autov > 0) && (t <= autov);
    }
  }
}

}  // namespace kt
