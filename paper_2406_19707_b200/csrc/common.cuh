// Shared device helpers for the B200 decode-time KV path (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdlib.h>

#include <utility>

#include "../../include/infinigen_b200.h"

#define IG_CUDA_STATUS(expr)                                         \
  do {                                                               \
    cudaError_t _e = (expr);                                         \
    if (_e != cudaSuccess) return IG_ECUDA + (int)_e;                \
  } while (0)

#define IG_LAUNCH_STATUS() IG_CUDA_STATUS(cudaGetLastError())

namespace ig {

constexpr int kWarp = 32;

// Order-preserving float -> u32 map: a < b  <=>  key(a) < key(b).
// -0.0 is folded onto +0.0 first: NumPy's argsort(-v) treats them as equal
// (linalg.py:184), so they must share a key.  Every finite float maps to a
// key > 0; 0 is reserved as the "empty" value for max reductions.
__device__ __forceinline__ uint32_t order_key(float v) {
  uint32_t u = __float_as_uint(v == 0.0f ? 0.0f : v);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float key_to_float(uint32_t k) {
  uint32_t u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
  return __uint_as_float(u);
}

// Let a programmatic-dependent successor (the packed GEMM, launched with
// cudaLaunchAttributeProgrammaticStreamSerialization) start filling its weight
// rings while this grid runs; the successor reads this grid's outputs only
// after griddepcontrol.wait.  No effect on plainly launched successors.
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Kernels launched with launch_pdl() may start before their predecessor in the
// stream has finished: they must call pdl_wait() before touching anything the
// predecessor writes (it returns once that grid has completed and flushed).
// Only the packed GEMM is launched this way: PDL-launching the layernorm, the
// append and the attention as well measured 880 vs 957 tok/s (their early CTAs
// sit on SM slots while they wait and hold off the speculation stream).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

inline bool pdl_enabled() {
  static const bool v = [] {
    const char* e = getenv("IG_PDL");             // A/B switch: IG_PDL=0 launches plainly
    return !(e && atoi(e) == 0);
  }();
  return v;
}

// cudaLaunchKernelEx with programmatic stream serialization (PDL)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ uint32_t warp_max_u32(uint32_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide sum; `red` needs blockDim.x/32 slots.  Result valid in all threads.
template <typename T>
__device__ __forceinline__ T block_sum(T v, T* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  T t = T(0);
  for (int i = 0; i < nw; ++i) t += red[i];  // fixed order: deterministic
  return t;
}

__device__ __forceinline__ float4 ldg_stream(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}

template <typename T> struct Elt;
template <> struct Elt<float> {
  __device__ static float to_f(float v) { return v; }
  __device__ static float from_f(float v) { return v; }
};
template <> struct Elt<__half> {
  __device__ static float to_f(__half v) { return __half2float(v); }
  __device__ static __half from_f(float v) { return __float2half_rn(v); }
};
template <> struct Elt<__nv_bfloat16> {
  __device__ static float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
  __device__ static __nv_bfloat16 from_f(float v) { return __float2bfloat16_rn(v); }
};

inline int elt_bytes(int elt) {
  return elt == IG_ELT_F32 ? 4 : (elt == IG_ELT_F16 || elt == IG_ELT_BF16 ? 2 : 0);
}

}  // namespace ig
