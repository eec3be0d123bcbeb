// Head-parallel (N > 1) output all-reduce over peer memory (NVLink / NVSwitch
// on a multi-GPU box), replacing the NCCL all-reduce of the row-parallel W_O and
// FFN-out partials (engine.py:360-364 sums all heads).
//
// Every rank owns a receive buffer recv[2 parities][G ranks][n] and flags
// [2][G] (ig_peer_alloc, shared by CUDA IPC handles).  One kernel per call:
//   1. push: each CTA copies its slice of the local partial into slot
//      [parity][rank] of EVERY rank's receive buffer (remote stores);
//   2. the grid's last CTA (ticket) fences at system scope and raises flag
//      [parity][rank] = epoch in every rank;
//   3. every CTA waits for the G flags of its own buffer (acquire, system
//      scope), then sums the G slots in rank order and adds the residual --
//      the same bits on every rank (fixed order), so the replicated residual
//      stream stays identical across ranks.
// epoch = step * calls_per_step + call + 1 comes from the device step counter,
// so the kernel replays inside a CUDA graph.  Slots alternate by call parity:
// a rank can only push call c + 2 (same parity) after its sum of call c + 1,
// which needed this rank's push of c + 1, which follows this rank's sum of c --
// so a slot is never overwritten while it is still being read.
#include <cstring>
#include <type_traits>

#include "common.cuh"

namespace ig {

constexpr int kArThreads = 256;

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// V = 4: float4 slices (n % 4 == 0, 16-B aligned); V = 1: scalar (any n, and
// the int32 head-count sums)
template <typename T, int V, bool PUSH>
__global__ void __launch_bounds__(kArThreads)
allreduce_peer_kernel(const T* __restrict__ src, int n, const uint64_t* __restrict__ peer_recv,
                      const uint64_t* __restrict__ peer_flags, int rank, int G,
                      const ig_step_state* __restrict__ st, int call, int calls_per_step,
                      const T* __restrict__ residual, T* __restrict__ out,
                      uint32_t* __restrict__ ticket) {
  using VT = typename std::conditional<V == 4, float4, T>::type;
  __shared__ int last;
  const uint32_t seqno = (uint32_t)st->step * (uint32_t)calls_per_step + (uint32_t)call;
  const int par = (int)(seqno & 1u);
  const uint32_t epoch = seqno + 1u;
  const int nv = n / V;
  const int tid = threadIdx.x;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const VT* sv = reinterpret_cast<const VT*>(src);
  // 1. push my partial into slot [par][rank] of every rank (PUSH = false: the
  //    producer -- the packed GEMM's epilogue, ig_sgemm_packed_peer -- did it)
  if constexpr (PUSH) {
  for (int r = 0; r < G; ++r) {
    VT* dv = reinterpret_cast<VT*>(reinterpret_cast<T*>(peer_recv[r]) + ((size_t)par * G + rank) * n);
    for (size_t i = blockIdx.x * (size_t)blockDim.x + tid; i < (size_t)nv; i += stride) dv[i] = sv[i];
  }
  __threadfence_system();
  __syncthreads();
  // 2. the last CTA raises my flag in every rank
  if (tid == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (last && tid < G) {
    if (tid == 0) *ticket = 0u;
    __threadfence_system();
    st_release_sys(reinterpret_cast<uint32_t*>(peer_flags[tid]) + par * G + rank, epoch);
  }
  }
  // 3. wait for every rank's slot, sum in rank order, add the residual
  const uint32_t* my_flags = reinterpret_cast<const uint32_t*>(peer_flags[rank]) + par * G;
  if (tid < G) {
    // a peer that never arrives (broken mapping, a rank that died) must fail
    // the context loudly, not hang the GPU: trap after ~10 s of spinning
    const long long t0 = clock64();
    while (ld_acquire_sys(my_flags + tid) != epoch)
      if (clock64() - t0 > 20000000000LL) __trap();
  }
  __syncthreads();
  const T* base = reinterpret_cast<const T*>(peer_recv[rank]) + (size_t)par * G * n;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + tid; i < (size_t)nv; i += stride) {
    if constexpr (V == 4) {
      float4 acc = __ldcg(reinterpret_cast<const float4*>(base) + i);
      for (int r = 1; r < G; ++r) {
        const float4 v = __ldcg(reinterpret_cast<const float4*>(base + (size_t)r * n) + i);
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
      if (residual != nullptr) {
        const float4 rv = reinterpret_cast<const float4*>(residual)[i];
        acc.x = __fadd_rn(acc.x, rv.x); acc.y = __fadd_rn(acc.y, rv.y);
        acc.z = __fadd_rn(acc.z, rv.z); acc.w = __fadd_rn(acc.w, rv.w);
      }
      reinterpret_cast<float4*>(out)[i] = acc;
    } else {
      T acc = __ldcg(base + i);
      for (int r = 1; r < G; ++r) acc += __ldcg(base + (size_t)r * n + i);
      if (residual != nullptr) acc += residual[i];
      out[i] = acc;
    }
  }
}

}  // namespace ig

extern "C" int ig_peer_alloc(int n, int world, void** recv, void** flags) {
  if (n < 1 || world < 1 || !recv || !flags) return IG_EINVAL;
  IG_CUDA_STATUS(cudaMalloc(recv, (size_t)2 * world * n * sizeof(float)));
  IG_CUDA_STATUS(cudaMemset(*recv, 0, (size_t)2 * world * n * sizeof(float)));
  IG_CUDA_STATUS(cudaMalloc(flags, (size_t)2 * world * sizeof(uint32_t) + 16));
  IG_CUDA_STATUS(cudaMemset(*flags, 0, (size_t)2 * world * sizeof(uint32_t) + 16));
  return IG_OK;
}

extern "C" int ig_peer_free(void* recv, void* flags) {
  if (recv) IG_CUDA_STATUS(cudaFree(recv));
  if (flags) IG_CUDA_STATUS(cudaFree(flags));
  return IG_OK;
}

extern "C" int ig_ipc_get_handle(void* dev_ptr, void* handle) {
  if (!dev_ptr || !handle) return IG_EINVAL;
  cudaIpcMemHandle_t h;
  IG_CUDA_STATUS(cudaIpcGetMemHandle(&h, dev_ptr));
  memcpy(handle, &h, sizeof(h));
  return IG_OK;
}

extern "C" int ig_ipc_open_handle(const void* handle, void** dev_ptr) {
  if (!handle || !dev_ptr) return IG_EINVAL;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  IG_CUDA_STATUS(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return IG_OK;
}

extern "C" int ig_ipc_close(void* dev_ptr) {
  if (!dev_ptr) return IG_EINVAL;
  IG_CUDA_STATUS(cudaIpcCloseMemHandle(dev_ptr));
  return IG_OK;
}

namespace ig {
template <typename T, bool PUSH = true>
static int allreduce_peer(const T* src, int n, const uint64_t* peer_recv, const uint64_t* peer_flags,
                          int rank, int world, const ig_step_state* st, int call, int calls_per_step,
                          const T* residual, T* out, uint32_t* ticket, void* stream) {
  if ((PUSH && (!src || !ticket)) || !peer_recv || !peer_flags || !st || !out || n < 1 || world < 1 ||
      world > kArThreads || rank < 0 || rank >= world || call < 0 || call >= calls_per_step)
    return IG_EINVAL;
  const bool vec = std::is_same<T, float>::value && (n & 3) == 0 && !((uintptr_t)src & 15) &&
                   !((uintptr_t)out & 15) && !(residual && ((uintptr_t)residual & 15));
  const int nv = vec ? n / 4 : n;
  // small grid: every CTA is resident while it waits on the flags
  int blocks = (nv + kArThreads - 1) / kArThreads;
  if (blocks > 64) blocks = 64;
  cudaStream_t s = (cudaStream_t)stream;
  if (vec)
    allreduce_peer_kernel<T, 4, PUSH><<<blocks, kArThreads, 0, s>>>(
        src, n, peer_recv, peer_flags, rank, world, st, call, calls_per_step, residual, out, ticket);
  else
    allreduce_peer_kernel<T, 1, PUSH><<<blocks, kArThreads, 0, s>>>(
        src, n, peer_recv, peer_flags, rank, world, st, call, calls_per_step, residual, out, ticket);
  IG_LAUNCH_STATUS();
  return IG_OK;
}
}  // namespace ig

extern "C" int ig_allreduce_peer(const float* src, int n, const uint64_t* peer_recv,
                                 const uint64_t* peer_flags, int rank, int world,
                                 const ig_step_state* st, int call, int calls_per_step,
                                 const float* residual, float* out, uint32_t* ticket, void* stream) {
  return ig::allreduce_peer<float>(src, n, peer_recv, peer_flags, rank, world, st, call,
                                   calls_per_step, residual, out, ticket, stream);
}

extern "C" int ig_allreduce_peer_i32(const int32_t* src, int n, const uint64_t* peer_recv,
                                     const uint64_t* peer_flags, int rank, int world,
                                     const ig_step_state* st, int call, int calls_per_step,
                                     int32_t* out, uint32_t* ticket, void* stream) {
  return ig::allreduce_peer<int32_t>(src, n, peer_recv, peer_flags, rank, world, st, call,
                                     calls_per_step, nullptr, out, ticket, stream);
}

extern "C" int ig_allreduce_peer_sum(int n, const uint64_t* peer_recv, const uint64_t* peer_flags,
                                     int rank, int world, const ig_step_state* st, int call,
                                     int calls_per_step, const float* residual, float* out,
                                     void* stream) {
  return ig::allreduce_peer<float, false>(nullptr, n, peer_recv, peer_flags, rank, world, st, call,
                                          calls_per_step, residual, out, nullptr, stream);
}
