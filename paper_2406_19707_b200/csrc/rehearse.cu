// K1 rehearsal + K2a count.
//
// Rehearsal (reference speculation.py:117-135): for layer i, run at layer i-1,
//   score[b,h,t] = (sum_j qspec[b, h*d + cols[b,h,j]] * pk[b,h,j,t]) * scale
// where qspec = x_a(i-1) @ W_Q(i) (the partial query of speculation.py:133 is
// its cols-subset) and pk is the partial key cache stored column-major over
// tokens, so a warp's 32 x float4 loads of one column j are one 512-B burst.
// HBM-bound: each launch streams 4*k*s bytes per (b, h) once.
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

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

// Fused rehearsal + alpha count (speculation.py:133-134 and :154-157) for one
// (b, h) score row split across a thread-block cluster of C CTAs: each CTA
// scores its contiguous token range (kept in shared memory and written out for
// ig_select), the CTAs exchange their maxima through distributed shared memory,
// then count score > float32(double(max) - alpha) locally and rank 0 sums the
// C counts.  Replaces ig_rehearse + ig_count (+ the maxkey memset) on the
// engine path; the row is read from HBM exactly once.
constexpr int kFusedThreads = 256;

__global__ void __launch_bounds__(kFusedThreads)
rehearse_count_kernel(const float* __restrict__ qspec, int ldq, const int32_t* __restrict__ cols,
                      const float* __restrict__ pk, const ig_step_state* __restrict__ st, int Hg,
                      int d, int k, int S_max, float scale, double alpha,
                      float* __restrict__ scores, int32_t* __restrict__ counts,
                      int32_t* __restrict__ count_sum) {
  cg::cluster_group cluster = cg::this_cluster();
  const int C = (int)cluster.num_blocks(), rank = (int)cluster.block_rank();
  extern __shared__ float4 sc_local[];
  __shared__ float qs[kMaxK];
  __shared__ uint32_t red_u[kFusedThreads / kWarp];
  __shared__ int red_i[kFusedThreads / kWarp];
  __shared__ uint32_t cta_max;
  __shared__ int cta_count;
  const int b = blockIdx.z, h = blockIdx.y;
  const size_t bh = (size_t)b * Hg + h;
  const int s = st->s_len;
  const int quads = (s + 3) >> 2;
  const int per = (quads + C - 1) / C;
  const int q0 = rank * per, q1 = min(quads, q0 + per);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (int j = tid; j < k; j += blockDim.x)
    qs[j] = qspec[(size_t)b * ldq + (size_t)h * d + cols[bh * k + j]];
  __syncthreads();

  const float* base = pk + bh * (size_t)k * S_max;
  float* out = scores + bh * S_max;
  uint32_t kmax = 0;
  for (int qd = q0 + tid; qd < q1; qd += blockDim.x) {
    const int t = qd * 4;
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll 8
    for (int j = 0; j < k; ++j) {
      const float4 v = ldg_stream(reinterpret_cast<const float4*>(base + (size_t)j * S_max + t));
      const float q = qs[j];
      a0 = fmaf(q, v.x, a0);
      a1 = fmaf(q, v.y, a1);
      a2 = fmaf(q, v.z, a2);
      a3 = fmaf(q, v.w, a3);
    }
    float4 r = make_float4(a0 * scale, a1 * scale, a2 * scale, a3 * scale);
    // tokens >= s (tail of the last quad) never count and never win the max
    if (t + 1 >= s) r.y = -INFINITY;
    if (t + 2 >= s) r.z = -INFINITY;
    if (t + 3 >= s) r.w = -INFINITY;
    sc_local[qd - q0] = r;
    *reinterpret_cast<float4*>(out + t) = r;  // S_max % 4 == 0: in bounds
    kmax = max(kmax, max(max(order_key(r.x), order_key(r.y)), max(order_key(r.z), order_key(r.w))));
  }
  kmax = warp_max_u32(kmax);
  if (lane == 0) red_u[w] = kmax;
  __syncthreads();
  if (tid == 0) {
    uint32_t m = 0;
    for (int i = 0; i < kFusedThreads / kWarp; ++i) m = max(m, red_u[i]);
    cta_max = m;
  }
  cluster.sync();
  uint32_t gkey = 0;
  for (int r = 0; r < C; ++r) gkey = max(gkey, *cluster.map_shared_rank(&cta_max, r));
  const float thr = __double2float_rn((double)key_to_float(gkey) - alpha);
  int c = 0;
  for (int qd = q0 + tid; qd < q1; qd += blockDim.x) {
    const float4 r = sc_local[qd - q0];
    c += (r.x > thr) + (r.y > thr) + (r.z > thr) + (r.w > thr);
  }
  c = warp_sum(c);
  if (lane == 0) red_i[w] = c;
  __syncthreads();
  if (tid == 0) {
    int t = 0;
    for (int i = 0; i < kFusedThreads / kWarp; ++i) t += red_i[i];
    cta_count = t;
  }
  cluster.sync();
  if (rank == 0 && tid == 0) {
    int t = 0;
    for (int r = 0; r < C; ++r) t += *cluster.map_shared_rank(&cta_count, r);
    counts[bh] = t;
    atomicAdd(count_sum + b, t);
  }
  cluster.sync();  // peers' shared memory stays alive until rank 0 has read it
}

}  // namespace ig

extern "C" int ig_rehearse_count(const float* qspec, int ldq, const int32_t* cols, const float* pk,
                                 const ig_step_state* st, int B, int Hg, int d, int k, int S_max,
                                 float scale, double alpha, int cluster, float* scores,
                                 int32_t* counts, int32_t* count_sum, void* stream) {
  using namespace ig;
  if (B < 1 || Hg < 1 || d < 1 || k < 1 || k > d || k > kMaxK || S_max < 1 || (S_max & 3) ||
      ldq < Hg * d || !(alpha > 0) || !qspec || !cols || !pk || !st || !scores || !counts ||
      !count_sum)
    return IG_EINVAL;
  int C = cluster;
  if (C <= 0) {  // enough CTAs for ~8 per SM, at most the portable cluster size
    const int rows = B * Hg;
    C = (148 * 8 + rows - 1) / rows;
    C = C < 1 ? 1 : (C > 8 ? 8 : C);
  }
  if (C > 8) return IG_EINVAL;
  const int quads = S_max / 4;
  const size_t smem = (size_t)((quads + C - 1) / C) * sizeof(float4);
  if (smem > 200 * 1024) return IG_EINVAL;
  if (smem > 32 * 1024)  // dynamic + static must fit: opt in early
    IG_CUDA_STATUS(cudaFuncSetAttribute(rehearse_count_kernel,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C, Hg, B);
  cfg.blockDim = dim3(kFusedThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  IG_CUDA_STATUS(cudaLaunchKernelEx(&cfg, rehearse_count_kernel, qspec, ldq, cols, pk, st, Hg, d,
                                    k, S_max, scale, alpha, scores, counts, count_sum));
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
