// K1 rehearsal + K2a count.
//
// Rehearsal (reference speculation.py:117-135): for layer i, run at layer i-1,
//   score[b,h,t] = (sum_j qspec[b, h*d + cols[b,h,j]] * pk[b,h,j,t]) * scale
// where qspec = x_a(i-1) @ W_Q(i) (the partial query of speculation.py:133 is
// its cols-subset) and pk is the partial key cache stored column-major over
// tokens, so a warp's 32 x float4 loads of one column j are one 512-B burst.
// HBM-bound: each launch streams 4*k*s bytes per (b, h) once.
#include "common.cuh"

namespace ig {

constexpr int kRehearseThreads = 256;
constexpr int kRehearseTok = 4;                                   // tokens per thread (float4)
constexpr int kRehearseChunk = kRehearseThreads * kRehearseTok;   // tokens per CTA
constexpr int kMaxK = 256;

__global__ void __launch_bounds__(kRehearseThreads)
rehearse_kernel(const float* __restrict__ qspec, int ldq, const int32_t* __restrict__ cols,
                const float* __restrict__ pk, const ig_step_state* __restrict__ st, int Hg,
                int d, int k, int S_max, float scale, float* __restrict__ scores,
                uint32_t* __restrict__ maxkey) {
  const int b = blockIdx.z, h = blockIdx.y;
  const int s = st->s_len;
  const int t0 = blockIdx.x * kRehearseChunk;
  if (t0 >= s) return;
  __shared__ float qs[kMaxK];
  __shared__ uint32_t wmax[kRehearseThreads / kWarp];
  const size_t bh = (size_t)b * Hg + h;
  for (int j = threadIdx.x; j < k; j += blockDim.x)
    qs[j] = qspec[(size_t)b * ldq + (size_t)h * d + cols[bh * k + j]];
  __syncthreads();

  const int t = t0 + threadIdx.x * kRehearseTok;
  const float* base = pk + bh * (size_t)k * S_max + t;
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
  uint32_t kmax = 0;
  if (t < s) {
    // fixed ascending-j FMA chain per token: deterministic
#pragma unroll 8
    for (int j = 0; j < k; ++j) {
      const float4 v = ldg_stream(reinterpret_cast<const float4*>(base + (size_t)j * S_max));
      const float q = qs[j];
      a0 = fmaf(q, v.x, a0);
      a1 = fmaf(q, v.y, a1);
      a2 = fmaf(q, v.z, a2);
      a3 = fmaf(q, v.w, a3);
    }
    float r[4] = {a0 * scale, a1 * scale, a2 * scale, a3 * scale};
    float* out = scores + bh * S_max + t;
    if (t + 3 < s) {
      *reinterpret_cast<float4*>(out) = make_float4(r[0], r[1], r[2], r[3]);
#pragma unroll
      for (int i = 0; i < 4; ++i) kmax = max(kmax, order_key(r[i]));
    } else {
      for (int i = 0; i < 4 && t + i < s; ++i) {
        out[i] = r[i];
        kmax = max(kmax, order_key(r[i]));
      }
    }
  }
  kmax = warp_max_u32(kmax);
  if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = kmax;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t m = 0;
    for (int i = 0; i < kRehearseThreads / kWarp; ++i) m = max(m, wmax[i]);
    atomicMax(maxkey + bh, m);  // max is order-independent: exact
  }
}

// count of score > float32(double(max) - alpha) per (b, h), plus per-b sums.
// NumPy 2 compares a float32 array against a Python float by casting the
// scalar to float32 (weak-scalar rule), hence the __double2float_rn.
constexpr int kCountThreads = 256;

__global__ void __launch_bounds__(kCountThreads)
count_kernel(const float* __restrict__ scores, const uint32_t* __restrict__ maxkey,
             const ig_step_state* __restrict__ st, int Hg, int S_max, double alpha,
             int32_t* __restrict__ counts, int32_t* __restrict__ count_sum) {
  __shared__ int red[kCountThreads / kWarp];
  const int b = blockIdx.y, h = blockIdx.x;
  const size_t bh = (size_t)b * Hg + h;
  const int s = st->s_len;
  const float mx = key_to_float(maxkey[bh]);
  const float thr = __double2float_rn((double)mx - alpha);
  const float* row = scores + bh * S_max;
  int c = 0;
  for (int t = threadIdx.x * 4; t < s; t += blockDim.x * 4) {
    if (t + 3 < s) {
      const float4 v = *reinterpret_cast<const float4*>(row + t);
      c += (v.x > thr) + (v.y > thr) + (v.z > thr) + (v.w > thr);
    } else {
      for (int i = t; i < s; ++i) c += row[i] > thr;
    }
  }
  c = block_sum(c, red);
  if (threadIdx.x == 0) {
    counts[bh] = c;
    atomicAdd(count_sum + b, c);  // integer: exact, order-free
  }
}

// Row maxima as order keys, for scores produced outside ig_rehearse.
__global__ void __launch_bounds__(kCountThreads)
score_max_kernel(const float* __restrict__ scores, const ig_step_state* __restrict__ st, int Hg,
                 int S_max, uint32_t* __restrict__ maxkey) {
  __shared__ uint32_t red[kCountThreads / kWarp];
  const size_t bh = (size_t)blockIdx.y * Hg + blockIdx.x;
  const int s = st->s_len;
  uint32_t m = 0;
  for (int t = threadIdx.x; t < s; t += blockDim.x) m = max(m, order_key(scores[bh * S_max + t]));
  m = warp_max_u32(m);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < kCountThreads / kWarp; ++i) m = max(m, red[i]);
    maxkey[bh] = max(m, red[0]);
  }
}

// Fused rehearsal + alpha count (speculation.py:133-134 and :154-157).  The
// rehearsal CTAs are the plain 1024-token tiles of rehearse_kernel (no
// clusters: ~2.7 waves at C3, the shape that streams partial K at ~0.9 of
// HBM peak); each max-reduces its tile into maxkey[b,h] and takes a ticket, and
// the LAST tile of a row to finish counts score > float32(double(max) - alpha)
// over the row (L2-resident, just written), adds it to count_sum[b] and resets
// the row's maxkey/ticket for the next launch.  A cluster/DSMEM version of
// the same fusion measured slower (wave quantization of 2-CTA clusters).
__global__ void __launch_bounds__(kRehearseThreads)
rehearse_count_kernel(const float* __restrict__ qspec, int ldq, const int32_t* __restrict__ cols,
                      const float* __restrict__ pk, const ig_step_state* __restrict__ st, int Hg,
                      int d, int k, int S_max, float scale, double alpha,
                      float* __restrict__ scores, uint32_t* __restrict__ maxkey,
                      int32_t* __restrict__ tickets, int32_t* __restrict__ counts,
                      int32_t* __restrict__ count_sum, uint32_t* __restrict__ row_range) {
  const int b = blockIdx.z, h = blockIdx.y;
  const int s = st->s_len;
  const int t0 = blockIdx.x * kRehearseChunk;
  const int tiles = (s + kRehearseChunk - 1) / kRehearseChunk;
  if (t0 >= s) return;
  __shared__ float qs[kMaxK];
  __shared__ uint32_t wmax[kRehearseThreads / kWarp];
  __shared__ int red[kRehearseThreads / kWarp];
  __shared__ uint32_t wmin[kRehearseThreads / kWarp];
  __shared__ int last;
  const size_t bh = (size_t)b * Hg + h;
  for (int j = threadIdx.x; j < k; j += blockDim.x)
    qs[j] = qspec[(size_t)b * ldq + (size_t)h * d + cols[bh * k + j]];
  __syncthreads();

  const int t = t0 + threadIdx.x * kRehearseTok;
  const float* base = pk + bh * (size_t)k * S_max + t;
  float* row = scores + bh * S_max;
  uint32_t kmax = 0;
  if (t < s) {
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll 8
    for (int j = 0; j < k; ++j) {
      const float4 v = ldg_stream(reinterpret_cast<const float4*>(base + (size_t)j * S_max));
      const float q = qs[j];
      a0 = fmaf(q, v.x, a0);
      a1 = fmaf(q, v.y, a1);
      a2 = fmaf(q, v.z, a2);
      a3 = fmaf(q, v.w, a3);
    }
    float4 r = make_float4(a0 * scale, a1 * scale, a2 * scale, a3 * scale);
    if (t + 1 >= s) r.y = -INFINITY;  // tail of the last quad: never counts, never the max
    if (t + 2 >= s) r.z = -INFINITY;
    if (t + 3 >= s) r.w = -INFINITY;
    *reinterpret_cast<float4*>(row + t) = r;   // S_max % 4 == 0: in bounds
    kmax = max(max(order_key(r.x), order_key(r.y)), max(order_key(r.z), order_key(r.w)));
  }
  kmax = warp_max_u32(kmax);
  if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = kmax;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t m = 0;
    for (int i = 0; i < kRehearseThreads / kWarp; ++i) m = max(m, wmax[i]);
    atomicMax(maxkey + bh, m);       // max is order-independent: exact
    __threadfence();                 // my scores and max before my ticket
    last = atomicAdd(tickets + bh, 1) == tiles - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  const uint32_t rmax = __ldcg(maxkey + bh);
  const float thr = __double2float_rn((double)key_to_float(rmax) - alpha);
  int c = 0;
  uint32_t kmin = 0xffffffffu;       // the row minimum for ig_select (row_range)
  for (int i = threadIdx.x * 4; i < s; i += blockDim.x * 4) {
    const float4 v = __ldcg(reinterpret_cast<const float4*>(row + i));
    c += (v.x > thr) + (v.y > thr) + (v.z > thr) + (v.w > thr);
    if (row_range != nullptr) {
      kmin = min(kmin, order_key(v.x));
      if (i + 1 < s) kmin = min(kmin, order_key(v.y));
      if (i + 2 < s) kmin = min(kmin, order_key(v.z));
      if (i + 3 < s) kmin = min(kmin, order_key(v.w));
    }
  }
  c = block_sum(c, red);
  if (row_range != nullptr) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
    if ((threadIdx.x & 31) == 0) wmin[threadIdx.x >> 5] = kmin;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    counts[bh] = c;
    atomicAdd(count_sum + b, c);     // integer: exact, order-free
    if (row_range != nullptr) {      // the row's (max, min) order keys: ig_select skips its P0 pass
      for (int i = 1; i < kRehearseThreads / kWarp; ++i) kmin = min(kmin, wmin[i]);
      row_range[2 * bh] = rmax;
      row_range[2 * bh + 1] = kmin;
    }
    maxkey[bh] = 0;                  // scratch ready for the next launch
    tickets[bh] = 0;
  }
}

}  // namespace ig

extern "C" int ig_rehearse_count(const float* qspec, int ldq, const int32_t* cols, const float* pk,
                                 const ig_step_state* st, int B, int Hg, int d, int k, int S_max,
                                 float scale, double alpha, float* scores, uint32_t* maxkey,
                                 int32_t* tickets, int32_t* counts, int32_t* count_sum,
                                 uint32_t* row_range, void* stream) {
  using namespace ig;
  if (B < 1 || Hg < 1 || d < 1 || k < 1 || k > d || k > kMaxK || S_max < 1 || (S_max & 3) ||
      ldq < Hg * d || !(alpha > 0) || !qspec || !cols || !pk || !st || !scores || !maxkey ||
      !tickets || !counts || !count_sum)
    return IG_EINVAL;
  dim3 grid((S_max + kRehearseChunk - 1) / kRehearseChunk, Hg, B);
  rehearse_count_kernel<<<grid, kRehearseThreads, 0, (cudaStream_t)stream>>>(
      qspec, ldq, cols, pk, st, Hg, d, k, S_max, scale, alpha, scores, maxkey, tickets, counts,
      count_sum, row_range);
  IG_LAUNCH_STATUS();
  return IG_OK;
}

extern "C" int ig_score_max(const float* scores, const ig_step_state* st, int B, int Hg,
                            int S_max, uint32_t* maxkey, void* stream) {
  using namespace ig;
  if (!scores || !st || !maxkey || B < 1 || Hg < 1 || S_max < 1) return IG_EINVAL;
  score_max_kernel<<<dim3(Hg, B), kCountThreads, 0, (cudaStream_t)stream>>>(scores, st, Hg, S_max,
                                                                           maxkey);
  IG_LAUNCH_STATUS();
  return IG_OK;
}

extern "C" int ig_rehearse(const float* qspec, int ldq, const int32_t* cols, const float* pk,
                           const ig_step_state* st, int B, int Hg, int d, int k, int S_max,
                           float scale, float* scores, uint32_t* maxkey, void* stream) {
  using namespace ig;
  if (B < 1 || Hg < 1 || d < 1 || k < 1 || k > d || k > kMaxK || S_max < 1 || (S_max & 3) ||
      ldq < Hg * d || !qspec || !cols || !pk || !st || !scores || !maxkey)
    return IG_EINVAL;
  dim3 grid((S_max + kRehearseChunk - 1) / kRehearseChunk, Hg, B);
  rehearse_kernel<<<grid, kRehearseThreads, 0, (cudaStream_t)stream>>>(
      qspec, ldq, cols, pk, st, Hg, d, k, S_max, scale, scores, maxkey);
  IG_LAUNCH_STATUS();
  return IG_OK;
}

extern "C" int ig_count(const float* scores, const uint32_t* maxkey, const ig_step_state* st,
                        int B, int Hg, int S_max, double alpha, int32_t* counts,
                        int32_t* count_sum, void* stream) {
  using namespace ig;
  if (B < 1 || Hg < 1 || S_max < 1 || (S_max & 3) || !(alpha > 0) || !scores || !maxkey ||
      !st || !counts || !count_sum)
    return IG_EINVAL;
  count_kernel<<<dim3(Hg, B), kCountThreads, 0, (cudaStream_t)stream>>>(
      scores, maxkey, st, Hg, S_max, alpha, counts, count_sum);
  IG_LAUNCH_STATUS();
  return IG_OK;
}
