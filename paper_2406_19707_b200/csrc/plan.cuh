// ig_resident_plan's per-(b, h) step, shared by the plan kernel (resident.cu)
// and the fused select + plan kernel (select.cu).
#pragma once

#include "common.cuh"

namespace ig {

constexpr int kPlanThreads = 256;

__device__ __forceinline__ int lower_bound_i32(const int32_t* __restrict__ a, int n, int v) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Exclusive block-wide prefix of `flag` (ballot per warp, warp totals in
// smem); `total` receives the block total.  Every thread must call it.
__device__ __forceinline__ int block_rank(bool flag, int* wsum, int& total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const unsigned bal = __ballot_sync(0xffffffffu, flag);
  __syncthreads();                     // previous call's wsum reads are done
  if (lane == 0) wsum[w] = __popc(bal);
  __syncthreads();
  int before = 0;
  total = 0;
  for (int i = 0; i < nw; ++i) {
    const int c = wsum[i];
    before += i < w ? c : 0;
    total += c;
  }
  return before + __popc(bal & ((1u << lane) - 1u));
}

// One (b, h): drop the slots whose row left the ascending selection sel[0:n)
// (or was overwritten by last step's append, pp), then give the rows that
// entered it the free slots in ascending order (fresh slots from U up) and
// write the fetch list.  Whole block; freelist [cap] ints, matched [cap] bytes
// and wsum [blockDim/32] in shared memory.
__device__ __forceinline__ void plan_row(const int32_t* __restrict__ sel, int n, int pp, int32_t* __restrict__ ids,
                                         int32_t* __restrict__ slot_used_bh, int32_t* __restrict__ frow,
                                         int32_t* __restrict__ fslot, int32_t* __restrict__ fcount_bh,
                                         unsigned long long* __restrict__ moved_rows, int32_t* freelist,
                                         uint8_t* matched, int* wsum) {
  const int tid = threadIdx.x;
  const int U = *slot_used_bh;
  for (int p = tid; p < n; p += blockDim.x) matched[p] = 0;
  __syncthreads();
  // 1. keep the slots whose row is still selected (and was not overwritten)
  for (int j = tid; j < U; j += blockDim.x) {
    const int id = ids[j];
    bool keep = false;
    if (id >= 0 && id != pp) {
      const int p = lower_bound_i32(sel, n, id);
      if (p < n && sel[p] == id) {
        matched[p] = 1;
        keep = true;
      }
    }
    if (!keep && id != -1) ids[j] = -1;
  }
  __syncthreads();
  // 2. free slots below U, ascending
  int nfree = 0;
  for (int base = 0; base < U; base += blockDim.x) {
    const int j = base + tid;
    const bool f = j < U && ids[j] < 0;
    int tot;
    const int r = block_rank(f, wsum, tot);
    if (f) freelist[nfree + r] = j;
    nfree += tot;
  }
  __syncthreads();
  // 3. rows that entered the selection (ascending) take the free slots in
  //    order, then fresh slots from U up
  int nun = 0;
  for (int base = 0; base < n; base += blockDim.x) {
    const int p = base + tid;
    const bool f = p < n && !matched[p];
    int tot;
    const int r = block_rank(f, wsum, tot);
    if (f) {
      const int k = nun + r;
      const int slot = k < nfree ? freelist[k] : U + (k - nfree);
      const int row = sel[p];
      ids[slot] = row;
      frow[k] = row;
      fslot[k] = slot;
    }
    nun += tot;
  }
  if (tid == 0) {
    *fcount_bh = nun;
    *slot_used_bh = nun > nfree ? U + (nun - nfree) : U;
    if (moved_rows && nun) atomicAdd(moved_rows, (unsigned long long)nun);
  }
}

}  // namespace ig
