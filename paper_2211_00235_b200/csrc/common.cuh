// Shared helpers for the B200 Evoformer kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdio.h>
#include <atomic>
#include <string>

#include "../../include/evo_b200.h"

namespace evo {

// ---------------------------------------------------------------- errors
void set_error(const char *fmt, ...);
extern std::atomic<int64_t> g_launches;

#define EVO_REQUIRE(cond, code, ...)          \
  do {                                        \
    if (!(cond)) {                            \
      ::evo::set_error(__VA_ARGS__);          \
      return (code);                          \
    }                                         \
  } while (0)

// After a launch: count it and convert launch errors into EVO_ECUDA.
inline int after_launch(const char *what) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return EVO_ECUDA;
  }
  return EVO_OK;
}

#define EVO_LAUNCHED(what)                    \
  do {                                        \
    int _st = ::evo::after_launch(what);      \
    if (_st != EVO_OK) return _st;            \
  } while (0)

// ------------------------------------------------- programmatic launch
// Every kernel of the library starts with evo_pdl_enter(), which waits until
// the previous kernel of the stream has completed and its writes are
// visible (griddepcontrol.wait).  launch_k() launches with programmatic
// stream serialization, so the dependent kernel is staged while its
// predecessor runs and starts the moment it completes -- part of the ~1 us
// per dependent launch a CUDA graph otherwise pays: C2 step 3.11 -> 3.06
// ms.  No kernel triggers its dependents early (griddepcontrol.
// launch_dependents at kernel start measured 3.18 ms: the early CTAs sit
// on the SMs the running kernel still needs).  EVO_PDL=0 in the environment
// launches without the attribute (the waits are then no-ops).
__device__ __forceinline__ void evo_pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
bool pdl_enabled();

template <typename... KArgs, typename... Args>
inline void launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                     Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kern, static_cast<Args &&>(args)...);
}

// ---------------------------------------------------------------- types
typedef __nv_bfloat16 bf16;

template <typename T> struct DType;
template <> struct DType<float> { static constexpr int id = EVO_F32; };
template <> struct DType<bf16> { static constexpr int id = EVO_BF16; };

__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ float to_f(bf16 x) { return __bfloat162float(x); }
template <typename T> __device__ __forceinline__ T from_f(float x);
template <> __device__ __forceinline__ float from_f<float>(float x) { return x; }
template <> __device__ __forceinline__ bf16 from_f<bf16>(float x) {
  return __float2bfloat16_rn(x);
}

// Stable two-branch sigmoid (src/tensor.py:259-269).
__device__ __forceinline__ float sigmoidf_stable(float x) {
  if (x >= 0.f) return 1.f / (1.f + expf(-x));
  float e = expf(x);
  return e / (1.f + e);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Two-level index map of evo_mat (row/col terms).
struct IdxMap {
  int64_t rs, cs, rdiv, rs0, cdiv, cs0;
  __host__ __device__ __forceinline__ int64_t row(int64_t i) const {
    return rdiv > 0 ? (i / rdiv) * rs + (i % rdiv) * rs0 : i * rs;
  }
  __host__ __device__ __forceinline__ int64_t col(int64_t j) const {
    return cdiv > 0 ? (j / cdiv) * cs + (j % cdiv) * cs0 : j * cs;
  }
};

inline IdxMap idxmap_of(const evo_mat &m) {
  IdxMap r;
  r.rs = m.rs; r.cs = m.cs; r.rdiv = m.rdiv; r.rs0 = m.rs0;
  r.cdiv = m.cdiv; r.cs0 = m.cs0;
  return r;
}

inline size_t dtype_size(int dt) { return dt == EVO_BF16 ? 2 : 4; }
inline bool valid_dtype(int dt) { return dt == EVO_F32 || dt == EVO_BF16; }
inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// Raise a kernel's dynamic-smem limit to the device maximum once per
// process (kept out of the per-call path so launches stay graph-capturable).
#define EVO_MAX_SMEM_ONCE(kernel)                                                       \
  do {                                                                                  \
    static bool _done = false;                                                          \
    if (!_done) {                                                                       \
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448); \
      _done = true;                                                                     \
    }                                                                                   \
  } while (0)

inline int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

}  // namespace evo
