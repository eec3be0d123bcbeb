// K2b selection: shared n per (sequence, layer) and per-head top-n rows.
//
// Reference: select_tokens (speculation.py:138-163) and topk_indices
// (linalg.py:177-185): the first n of a STABLE argsort of -score, i.e. the n
// largest scores with ties going to the lower row index.  Implemented as an
// exact 4-pass 8-bit radix select on order-preserving u32 keys (finds the
// n-th largest key P and how many rows equal to P are taken), then one
// ascending pass with warp-ballot compaction that emits
//   { t : key > P }  U  { first `need` t in index order with key == P }
// in ascending row order -- the order the host-pool gather wants (ascending
// rows keep the PCIe reads page-local: 52.7 vs 35 GB/s measured).
#include "common.cuh"

namespace ig {

constexpr int kSelThreads = 512;            // rows up to kSelLongRows keys
constexpr int kSelThreadsLong = 1024;       // longer rows (C4: 32K): 95 vs 124 us per layer
constexpr int kSelLongRows = 8192;
constexpr int kSelWarps = kSelThreadsLong / kWarp;
constexpr size_t kSelMaxSmem = 220 * 1024;  // keys of rows up to 56K tokens

struct SelShared {
  uint32_t hist[256];
  int warp_a[kSelWarps];
  int warp_b[kSelWarps];
  uint32_t prefix;
  int need;
};

// Choose the radix digit: bins are scanned from 255 down; the digit is the
// bin where the running count of larger bins first reaches `need`.  One warp,
// 8 bins per lane, warp prefix sum over lane totals (replaces a 256-step
// serial scan).  Writes sh.prefix / sh.need.
__device__ __forceinline__ void pick_digit(SelShared& sh, uint32_t prefix, int need, int shift) {
  const int lane = threadIdx.x & 31;
  // lane L owns bins 255-8L .. 248-8L (descending)
  int c[8], tot = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i] = (int)sh.hist[255 - 8 * lane - i]; tot += c[i]; }
  int incl = tot;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  const int excl = incl - tot;  // count in bins above my range
  const unsigned hitmask = __ballot_sync(0xffffffffu, excl < need && incl >= need);
  const int src = __ffs(hitmask) - 1;
  if (lane == src) {
    int cum = excl, bin = 255 - 8 * lane;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (cum + c[i] >= need) { bin = 255 - 8 * lane - i; break; }
      cum += c[i];
    }
    sh.prefix = prefix | ((uint32_t)bin << shift);
    sh.need = need - cum;
  }
}

// Top-n rows of a score row, ascending, into out[0:n).  Whole block calls.
// `keys` is this block's shared buffer of s order keys (filled here).
// The radix passes stop early once the boundary bin is taken whole (then
// every key whose resolved digits equal the prefix is selected, no tie rule
// needed); the compaction gives each warp one contiguous row range, counts it
// once, and emits with ballots -- two block barriers instead of two per
// 512-row tile.
__device__ void radix_topn(const float* __restrict__ row, int s, int n, int32_t* __restrict__ out,
                           SelShared& sh, uint32_t* __restrict__ keys) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int nw = blockDim.x >> 5;
  if (n >= s) {
    for (int t = tid; t < s; t += blockDim.x) out[t] = t;
    return;
  }
  if (n <= 0) return;
  for (int t = tid; t < s; t += blockDim.x) keys[t] = order_key(row[t]);
  uint32_t prefix = 0, mask = 0;
  int need = n;
  bool whole = false;      // boundary bin taken entirely: no tie cut inside it
  for (int pass = 0; pass < 4 && !whole; ++pass) {
    const int shift = 24 - 8 * pass;
    for (int i = tid; i < 256; i += blockDim.x) sh.hist[i] = 0;
    __syncthreads();
    for (int t0 = 0; t0 < s; t0 += blockDim.x) {
      const int t = t0 + tid;
      bool live = false;
      uint32_t bin = 0;
      if (t < s) {
        const uint32_t key = keys[t];
        live = (key & mask) == prefix;
        bin = (key >> shift) & 255u;
      }
      // warp-aggregated shared atomics: one add per distinct bin per warp
      const unsigned act = __ballot_sync(0xffffffffu, live);
      if (live) {
        const unsigned peers = __match_any_sync(act, bin);
        if ((__ffs(peers) - 1) == lane) atomicAdd(&sh.hist[bin], (uint32_t)__popc(peers));
      }
    }
    __syncthreads();
    if (w == 0) pick_digit(sh, prefix, need, shift);
    __syncthreads();
    prefix = sh.prefix;
    need = sh.need;
    mask |= 255u << shift;
    whole = (int)sh.hist[(prefix >> shift) & 255u] == need;
    __syncthreads();     // hist is rewritten by the next pass
  }
  // take: (key & mask) > prefix, or == prefix and (whole, or among the first
  // `need` such rows in index order).  Warp w owns rows [w*span, (w+1)*span).
  const int span = ((s + nw - 1) / nw + 31) & ~31;
  const int t_lo = min(s, w * span), t_hi = min(s, t_lo + span);
  const unsigned lt_mask = (1u << lane) - 1u;
  int n_gt = 0, n_eq = 0;
  for (int t0 = t_lo; t0 < t_hi; t0 += 32) {
    const int t = t0 + lane;
    const uint32_t km = t < t_hi ? (keys[t] & mask) : 0u;
    n_gt += __popc(__ballot_sync(0xffffffffu, t < t_hi && km > prefix));
    n_eq += __popc(__ballot_sync(0xffffffffu, t < t_hi && km == prefix));
  }
  if (lane == 0) { sh.warp_a[w] = n_gt; sh.warp_b[w] = n_eq; }
  __syncthreads();
  int out_off = 0, eq_before = 0;
  for (int i = 0; i < w; ++i) {
    const int e = whole ? sh.warp_b[i] : min(sh.warp_b[i], max(0, need - eq_before));
    eq_before += sh.warp_b[i];
    out_off += sh.warp_a[i] + e;
  }
  for (int t0 = t_lo; t0 < t_hi; t0 += 32) {
    const int t = t0 + lane;
    const uint32_t km = t < t_hi ? (keys[t] & mask) : 0u;
    const bool gt = t < t_hi && km > prefix;
    const bool eq = t < t_hi && km == prefix;
    const unsigned eqb = __ballot_sync(0xffffffffu, eq);
    const bool take = gt || (eq && (whole || eq_before + __popc(eqb & lt_mask) < need));
    const unsigned tb = __ballot_sync(0xffffffffu, take);
    if (take) out[out_off + __popc(tb & lt_mask)] = t;
    out_off += __popc(tb);
    eq_before += __popc(eqb);
  }
}

template <int THREADS>
__global__ void __launch_bounds__(THREADS)
select_kernel(const float* __restrict__ scores, const int32_t* __restrict__ count_sum,
              const ig_step_state* __restrict__ st, int Hg, int H_total, int S_max, int cap_max,
              double cap_ratio, int min_select, int32_t* __restrict__ idx,
              int32_t* __restrict__ n_out, int32_t* __restrict__ err_flag) {
  __shared__ SelShared sh;
  extern __shared__ uint32_t keys[];
  const int b = blockIdx.y, h = blockIdx.x;
  const int s = st->s_len;
  // n = floor(sum/H + 0.5) == floor((2 sum + H) / 2H) exactly (integers)
  const long long sum = count_sum[b];
  long long n = (2 * sum + H_total) / (2LL * H_total);
  const long long cap = max((long long)floor(cap_ratio * (double)s), (long long)min_select);
  n = min(max(n, (long long)min_select), cap);
  n = min(n, (long long)s);
  int nn = (int)n;
  if (nn > cap_max) {  // caller sized the index buffer too small: flag and clamp
    if (threadIdx.x == 0) atomicExch(err_flag, 1);
    nn = cap_max;
  }
  if (h == 0 && threadIdx.x == 0) n_out[b] = nn;
  const size_t bh = (size_t)b * Hg + h;
  radix_topn(scores + bh * S_max, s, nn, idx + bh * cap_max, sh, keys);
}

// Rewrite idx[0:n) of each (b, h) into stable descending-score order
// (ties -> lower index), the order topk_indices returns.  O(n^2) rank sort in
// shared memory: drop-in shim only, never on the engine path.
__global__ void order_kernel(const float* __restrict__ scores, const int32_t* __restrict__ n_in,
                             int Hg, int S_max, int cap, int32_t* __restrict__ idx) {
  extern __shared__ uint32_t smem[];
  const int b = blockIdx.y, h = blockIdx.x;
  const int n = n_in[b];
  const size_t bh = (size_t)b * Hg + h;
  uint32_t* keys = smem;
  int32_t* rows = reinterpret_cast<int32_t*>(smem + n);
  int32_t* io = idx + bh * cap;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    rows[i] = io[i];
    keys[i] = order_key(scores[bh * S_max + rows[i]]);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const uint32_t ki = keys[i];
    const int ri = rows[i];
    int rank = 0;
    for (int j = 0; j < n; ++j) {
      const uint32_t kj = keys[j];
      rank += (kj > ki) || (kj == ki && rows[j] < ri);
    }
    io[rank] = ri;
  }
}

__global__ void __launch_bounds__(kSelThreads)
topk_rows_kernel(const float* __restrict__ values, int len, int k, int32_t* __restrict__ out) {
  __shared__ SelShared sh;
  extern __shared__ uint32_t keys[];
  radix_topn(values + (size_t)blockIdx.x * len, len, k, out + (size_t)blockIdx.x * k, sh, keys);
}

}  // namespace ig

extern "C" int ig_select(const float* scores, const int32_t* count_sum, const ig_step_state* st,
                         int B, int Hg, int H_total, int S_max, int cap_max, double cap_ratio,
                         int min_select, int32_t* idx, int32_t* n_out, int32_t* err_flag,
                         void* stream) {
  using namespace ig;
  if (B < 1 || Hg < 1 || H_total < Hg || S_max < 1 || cap_max < 1 || !(cap_ratio > 0) ||
      cap_ratio > 1 || min_select < 1 || !scores || !count_sum || !st || !idx || !n_out ||
      !err_flag)
    return IG_EINVAL;
  const size_t smem = (size_t)S_max * 4;  // the row's order keys
  if (smem > kSelMaxSmem) return IG_EINVAL;
  auto kern = S_max > kSelLongRows ? select_kernel<kSelThreadsLong> : select_kernel<kSelThreads>;
  const int threads = S_max > kSelLongRows ? kSelThreadsLong : kSelThreads;
  if (smem > 32 * 1024)  // dynamic + static must fit: opt in early
    IG_CUDA_STATUS(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)smem));
  kern<<<dim3(Hg, B), threads, smem, (cudaStream_t)stream>>>(
      scores, count_sum, st, Hg, H_total, S_max, cap_max, cap_ratio, min_select, idx, n_out,
      err_flag);
  IG_LAUNCH_STATUS();
  return IG_OK;
}

extern "C" int ig_order_by_score(const float* scores, const int32_t* n, int B, int Hg, int S_max,
                                 int cap, int32_t* idx, void* stream) {
  using namespace ig;
  if (B < 1 || Hg < 1 || cap < 1 || !scores || !n || !idx) return IG_EINVAL;
  const size_t smem = (size_t)cap * 8;
  if (smem > 200 * 1024) return IG_EINVAL;
  if (smem > 32 * 1024)  // dynamic + static must fit: opt in early
    IG_CUDA_STATUS(cudaFuncSetAttribute(order_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)smem));
  order_kernel<<<dim3(Hg, B), 256, smem, (cudaStream_t)stream>>>(scores, n, Hg, S_max, cap, idx);
  IG_LAUNCH_STATUS();
  return IG_OK;
}

extern "C" int ig_topk_rows(const float* values, int rows, int len, int k, int32_t* idx_out,
                            void* stream) {
  using namespace ig;
  if (rows < 1 || len < 1 || k < 0 || k > len || !values || !idx_out) return IG_EINVAL;
  if (k == 0) return IG_OK;
  const size_t smem = (size_t)len * 4;
  if (smem > kSelMaxSmem) return IG_EINVAL;
  if (smem > 32 * 1024)  // dynamic + static must fit: opt in early
    IG_CUDA_STATUS(cudaFuncSetAttribute(topk_rows_kernel,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  topk_rows_kernel<<<rows, kSelThreads, smem, (cudaStream_t)stream>>>(values, len, k, idx_out);
  IG_LAUNCH_STATUS();
  return IG_OK;
}
