// Resident selection: the fetched set of every speculative layer stays in HBM
// from one decode step to the next, and only the rows that enter the
// selection cross the host link.
//
// The reference fetches every selected row from the host pool at every step
// (KvPool.fetch, pool.py:83-99, called per layer at engine.py:352-356; the
// bytes it accounts are LayerRecord.bytes = H*n*2*d*e, speculation.py:166-168).
// Consecutive selections of one (layer, seq, head) overlap by ~98% (the input
// similarity InfiniGen's speculation itself relies on), so
// B200 keeps a slot table per (layer, b, h) -- at most `cap` rows, the size of
// the reference's own per-step fetch buffer -- and the host pool stays the
// authoritative copy of every row (appends still go to it, engine.py:343).
//
//   ig_resident_plan  per (b, h): drop slots whose row left the selection (or
//                     was overwritten by last step's append: pos_prev), match
//                     the rest against the new ascending selection, assign
//                     free slots to the rows that entered it -> fetch list
//   ig_fetch_slots    gather the fetch list from the mapped host pool into
//                     its slots (zero-copy 16-B loads, ascending rows)
//   ig_stage_put      layer 0 (every row is fetched, engine.py:393-396): the
//                     appended row goes to its HBM mirror in the same step
//   ig_attend_slots   (attend.cu) attention over the slot table
#include "common.cuh"
#include "plan.cuh"

namespace ig {

__global__ void __launch_bounds__(kPlanThreads)
resident_plan_kernel(const int32_t* __restrict__ idx, const int32_t* __restrict__ n_in,
                     const int32_t* __restrict__ pos_prev, int32_t* __restrict__ slot_id,
                     int32_t* __restrict__ slot_used, int Hg, int cap, int32_t* __restrict__ frow,
                     int32_t* __restrict__ fslot, int32_t* __restrict__ fcount,
                     unsigned long long* __restrict__ moved_rows) {
  extern __shared__ int32_t plan_smem[];
  int32_t* freelist = plan_smem;                                   // [cap]
  uint8_t* matched = reinterpret_cast<uint8_t*>(plan_smem + cap);  // [cap]
  __shared__ int wsum[kPlanThreads / kWarp];
  const int b = blockIdx.y, h = blockIdx.x;
  const size_t bh = (size_t)b * Hg + h;
  plan_row(idx + bh * cap, n_in[b], pos_prev ? pos_prev[bh] : -1, slot_id + bh * cap, slot_used + bh,
           frow + bh * cap, fslot + bh * cap, fcount + bh, moved_rows, freelist, matched, wsum);
}

constexpr int kSlotFetchThreads = 128;
constexpr int kSlotFetchUnroll = 4;

// One CTA per (b, h); consecutive threads take consecutive 16-B vectors of
// the fetch list, kSlotFetchUnroll loads in flight per thread.
__global__ void __launch_bounds__(kSlotFetchThreads)
fetch_slots_kernel(const uint8_t* __restrict__ pool, const int32_t* __restrict__ frow,
                   const int32_t* __restrict__ fslot, const int32_t* __restrict__ fcount, int Hg,
                   int S_max, int cap, int row_bytes, uint8_t* __restrict__ stage) {
  const size_t bh = (size_t)blockIdx.y * Hg + blockIdx.x;
  const int cnt = fcount[bh];
  const int vpr = row_bytes >> 4;
  const int total = cnt * vpr;
  const uint8_t* src_bh = pool + bh * S_max * (size_t)row_bytes;
  uint8_t* dst_bh = stage + bh * cap * (size_t)row_bytes;
  for (int base = threadIdx.x; base < total; base += blockDim.x * kSlotFetchUnroll) {
    uint4 v[kSlotFetchUnroll];
    int e[kSlotFetchUnroll];
#pragma unroll
    for (int u = 0; u < kSlotFetchUnroll; ++u) {
      e[u] = base + u * blockDim.x;
      if (e[u] < total) {
        const int k = e[u] / vpr, vec = e[u] - k * vpr;
        const uint4* src = reinterpret_cast<const uint4*>(
            src_bh + (size_t)frow[bh * cap + k] * row_bytes) + vec;
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(src));
      }
    }
#pragma unroll
    for (int u = 0; u < kSlotFetchUnroll; ++u) {
      if (e[u] < total) {
        const int k = e[u] / vpr, vec = e[u] - k * vpr;
        reinterpret_cast<uint4*>(dst_bh + (size_t)fslot[bh * cap + k] * row_bytes)[vec] = v[u];
      }
    }
  }
}

template <typename T>
__global__ void stage_put_kernel(const float* __restrict__ k_cur, const float* __restrict__ v_cur,
                                 int ldkv, const int32_t* __restrict__ pos, int Hg, int d,
                                 int stage_rows, T* __restrict__ stage) {
  const int b = blockIdx.y, h = blockIdx.x;
  const size_t bh = (size_t)b * Hg + h;
  T* dst = stage + (bh * stage_rows + pos[bh]) * (size_t)(2 * d);
  const float* kr = k_cur + (size_t)b * ldkv + (size_t)h * d;
  const float* vr = v_cur + (size_t)b * ldkv + (size_t)h * d;
  for (int i = threadIdx.x; i < d; i += blockDim.x) {   // same rounding as append_kernel
    dst[i] = Elt<T>::from_f(kr[i]);
    dst[d + i] = Elt<T>::from_f(vr[i]);
  }
}

}  // namespace ig

extern "C" int ig_resident_plan(const int32_t* idx, const int32_t* n, const int32_t* pos_prev,
                                int32_t* slot_id, int32_t* slot_used, int B, int Hg, int cap,
                                int32_t* frow, int32_t* fslot, int32_t* fcount,
                                uint64_t* moved_rows, void* stream) {
  using namespace ig;
  if (!idx || !n || !slot_id || !slot_used || !frow || !fslot || !fcount || B < 1 || Hg < 1 ||
      cap < 1)
    return IG_EINVAL;
  const size_t smem = (size_t)cap * 4 + (size_t)cap;
  if (smem > 200 * 1024) return IG_EINVAL;
  if (smem > 32 * 1024)
    IG_CUDA_STATUS(cudaFuncSetAttribute(resident_plan_kernel,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  resident_plan_kernel<<<dim3(Hg, B), kPlanThreads, smem, (cudaStream_t)stream>>>(
      idx, n, pos_prev, slot_id, slot_used, Hg, cap, frow, fslot, fcount,
      reinterpret_cast<unsigned long long*>(moved_rows));
  IG_LAUNCH_STATUS();
  return IG_OK;
}

extern "C" int ig_fetch_slots(const void* pool_dev, const int32_t* frow, const int32_t* fslot,
                              const int32_t* fcount, int B, int Hg, int S_max, int cap,
                              int row_bytes, void* stage, void* stream) {
  using namespace ig;
  if (!pool_dev || !frow || !fslot || !fcount || !stage || B < 1 || Hg < 1 || S_max < 1 ||
      cap < 1 || row_bytes < 16 || (row_bytes & 15))
    return IG_EINVAL;
  fetch_slots_kernel<<<dim3(Hg, B), kSlotFetchThreads, 0, (cudaStream_t)stream>>>(
      (const uint8_t*)pool_dev, frow, fslot, fcount, Hg, S_max, cap, row_bytes, (uint8_t*)stage);
  IG_LAUNCH_STATUS();
  return IG_OK;
}

extern "C" int ig_stage_put(const float* k_cur, const float* v_cur, int ldkv, const int32_t* pos,
                            void* stage, int elt, int B, int Hg, int d, int stage_rows,
                            void* stream) {
  using namespace ig;
  if (!k_cur || !v_cur || !pos || !stage || B < 1 || Hg < 1 || d < 1 || stage_rows < 1 ||
      ldkv < Hg * d)
    return IG_EINVAL;
  dim3 grid(Hg, B);
  cudaStream_t s = (cudaStream_t)stream;
  switch (elt) {
    case IG_ELT_F32:
      stage_put_kernel<float><<<grid, 128, 0, s>>>(k_cur, v_cur, ldkv, pos, Hg, d, stage_rows,
                                                   (float*)stage);
      break;
    case IG_ELT_F16:
      stage_put_kernel<__half><<<grid, 128, 0, s>>>(k_cur, v_cur, ldkv, pos, Hg, d, stage_rows,
                                                    (__half*)stage);
      break;
    case IG_ELT_BF16:
      stage_put_kernel<__nv_bfloat16><<<grid, 128, 0, s>>>(k_cur, v_cur, ldkv, pos, Hg, d,
                                                           stage_rows, (__nv_bfloat16*)stage);
      break;
    default:
      return IG_EINVAL;
  }
  IG_LAUNCH_STATUS();
  return IG_OK;
}
