// Skinny f32 GEMM for the decode step's dense projections: Y[M][N] = X[M][K] . W[K][N]
// (+ epilogue), M = sequences <= 32, W row-major (the reference's x @ W layout,
// model.py:63-79).  Weight-streaming / HBM-bound: every weight is read once.
//
// CTA = one 128-column tile x one K slice.  A 4-stage cp.async pipeline
// copies 32-row weight chunks (16 KB) and the matching x slice into shared
// memory, so ~48 KB per CTA is in flight independently of registers (the first
// version loaded W and x straight to registers and stalled on L1TEX: 0.64 TB/s
// under ncu).  Each of the 8 warps consumes 4 rows of a chunk: lane = 4
// columns, 4*M FMAs per 16-B weight element read from shared memory.  The
// warps' partial tiles are summed in shared memory in fixed warp order; the
// K-split partials go to a workspace and the last CTA of a column tile
// (ticket) sums them in fixed split order and applies the epilogue -- the
// result is deterministic.  IEEE f32 throughout (no TF32: x_a feeds the
// rehearsal, whose index parity needs f32).
#include "common.cuh"

namespace ig {

constexpr int kGemmTileN = 128;   // columns per CTA: 32 lanes x float4
constexpr int kGemmKT = 32;       // weight rows per pipeline stage
constexpr int kGemmStages = 4;    // stages in flight (cp.async groups)
constexpr int kGemmWarps = 8;     // each warp owns 4 of the KT rows of a stage

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem);
  const int n = valid ? 16 : 0;   // src-size 0 -> zero fill
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(gmem), "r"(n)
               : "memory");
}

// Stage layout: Ws[stage][KT][128] then Xs[stage][MT][KT] (floats).
template <int MT>
__global__ void __launch_bounds__(kGemmWarps * 32, (MT <= 16 ? 2 : 1))
sgemm_rows_kernel(const float* __restrict__ X, int ldx, const float* __restrict__ W, int ldw,
                  float* __restrict__ Y, int ldy, const float* __restrict__ R, int ldr, int M,
                  int N, int K, int ksplit, int epilogue, float* __restrict__ ws,
                  int32_t* __restrict__ tickets) {
  extern __shared__ __align__(16) float smem[];
  constexpr int kWs = kGemmKT * kGemmTileN, kXs = MT * kGemmKT, kStage = kWs + kXs;
  __shared__ int last;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int tile = blockIdx.x, ks = blockIdx.y;
  const int ncol0 = tile * kGemmTileN;
  // K slice of this CTA in whole stages of KT rows
  const int chunks_all = (K + kGemmKT - 1) / kGemmKT;
  const int cper = (chunks_all + ksplit - 1) / ksplit;
  const int c0 = ks * cper, c1 = min(chunks_all, c0 + cper);
  const int nch = max(0, c1 - c0);

  auto load_stage = [&](int c, int st) {
    float* ws_ = smem + st * kStage;
    float* xs_ = ws_ + kWs;
    const int kb = (c0 + c) * kGemmKT;
    // W: KT x 128 floats = KT*32 float4, 8 per thread
#pragma unroll
    for (int i = 0; i < kGemmKT * 32 / (kGemmWarps * 32); ++i) {
      const int f = tid + i * kGemmWarps * 32;
      const int r = f >> 5, c4 = f & 31;
      const int k = kb + r, n = ncol0 + c4 * 4;
      const bool ok = k < K && n < N;
      cp_async16(ws_ + r * kGemmTileN + c4 * 4, ok ? (const void*)(W + (size_t)k * ldw + n) : (const void*)W, ok);
    }
    // X: MT x KT floats = MT*KT/4 float4
    for (int f = tid; f < MT * kGemmKT / 4; f += kGemmWarps * 32) {
      const int m = f / (kGemmKT / 4), k4 = f % (kGemmKT / 4);
      const int k = kb + k4 * 4;
      const bool ok = m < M && k < K;
      cp_async16(xs_ + m * kGemmKT + k4 * 4, ok ? (const void*)(X + (size_t)m * ldx + k) : (const void*)X, ok);
    }
  };

  float acc[MT][4];
#pragma unroll
  for (int m = 0; m < MT; ++m) acc[m][0] = acc[m][1] = acc[m][2] = acc[m][3] = 0.f;

#pragma unroll
  for (int i = 0; i < kGemmStages - 1; ++i) {
    if (i < nch) load_stage(i, i);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int c = 0; c < nch; ++c) {
    asm volatile("cp.async.wait_group %0;" ::"n"(kGemmStages - 2) : "memory");
    __syncthreads();   // stage c landed for every thread; stage c-1 fully consumed
    const int nx = c + kGemmStages - 1;
    if (nx < nch) load_stage(nx, nx % kGemmStages);
    asm volatile("cp.async.commit_group;" ::: "memory");
    const float* ws_ = smem + (c % kGemmStages) * kStage;
    const float* xs_ = ws_ + kWs;
    const int r0 = w * 4;                                   // my 4 rows of this stage
    float4 wv[4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
      wv[r] = *reinterpret_cast<const float4*>(ws_ + (r0 + r) * kGemmTileN + lane * 4);
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      const float4 xv = *reinterpret_cast<const float4*>(xs_ + m * kGemmKT + r0);   // broadcast
      acc[m][0] = fmaf(xv.x, wv[0].x, acc[m][0]);
      acc[m][1] = fmaf(xv.x, wv[0].y, acc[m][1]);
      acc[m][2] = fmaf(xv.x, wv[0].z, acc[m][2]);
      acc[m][3] = fmaf(xv.x, wv[0].w, acc[m][3]);
      acc[m][0] = fmaf(xv.y, wv[1].x, acc[m][0]);
      acc[m][1] = fmaf(xv.y, wv[1].y, acc[m][1]);
      acc[m][2] = fmaf(xv.y, wv[1].z, acc[m][2]);
      acc[m][3] = fmaf(xv.y, wv[1].w, acc[m][3]);
      acc[m][0] = fmaf(xv.z, wv[2].x, acc[m][0]);
      acc[m][1] = fmaf(xv.z, wv[2].y, acc[m][1]);
      acc[m][2] = fmaf(xv.z, wv[2].z, acc[m][2]);
      acc[m][3] = fmaf(xv.z, wv[2].w, acc[m][3]);
      acc[m][0] = fmaf(xv.w, wv[3].x, acc[m][0]);
      acc[m][1] = fmaf(xv.w, wv[3].y, acc[m][1]);
      acc[m][2] = fmaf(xv.w, wv[3].z, acc[m][2]);
      acc[m][3] = fmaf(xv.w, wv[3].w, acc[m][3]);
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();                 // pipeline buffers are reused for the reduction below
  // warps -> shared memory -> one partial tile (fixed warp order)
  float* red = smem;                                         // [WARPS][MT][128]
#pragma unroll
  for (int m = 0; m < MT; ++m)
    *reinterpret_cast<float4*>(red + ((size_t)w * MT + m) * kGemmTileN + lane * 4) =
        make_float4(acc[m][0], acc[m][1], acc[m][2], acc[m][3]);
  __syncthreads();
  const size_t tile_elems = (size_t)M * kGemmTileN;
  float* part = ws + ((size_t)tile * ksplit + ks) * tile_elems;
  for (int e = tid; e < M * kGemmTileN; e += blockDim.x) {
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < kGemmWarps; ++i) s += red[(size_t)i * MT * kGemmTileN + e];
    part[e] = s;
  }
  if (ksplit == 1) {
    __syncthreads();
  } else {
    __threadfence();
    __syncthreads();
    if (tid == 0) last = atomicAdd(tickets + tile, 1) == ksplit - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
  }
  // the last CTA of this column tile: sum the splits in order, epilogue, store
  const float* tp = ws + (size_t)tile * ksplit * tile_elems;
  for (int e = tid; e < M * kGemmTileN; e += blockDim.x) {
    const int m = e / kGemmTileN, n = ncol0 + (e % kGemmTileN);
    if (n >= N) continue;
    float s = 0.f;
    for (int i = 0; i < ksplit; ++i) s += __ldcg(tp + (size_t)i * tile_elems + e);
    if (epilogue == 1) s = fmaxf(s, 0.f);                              // ReLU (model.py:240)
    else if (epilogue == 2) s = __fadd_rn(R[(size_t)m * ldr + n], s);   // residual add
    Y[(size_t)m * ldy + n] = s;
  }
  if (tid == 0 && ksplit > 1) tickets[tile] = 0;
}

template <int MT>
int launch_sgemm(const float* X, int ldx, const float* W, int ldw, float* Y, int ldy,
                 const float* R, int ldr, int M, int N, int K, int ksplit, int epilogue, float* ws,
                 int32_t* tickets, cudaStream_t s) {
  const int tiles = (N + kGemmTileN - 1) / kGemmTileN;
  const size_t pipe = (size_t)kGemmStages * (kGemmKT * kGemmTileN + MT * kGemmKT) * sizeof(float);
  const size_t red = (size_t)kGemmWarps * MT * kGemmTileN * sizeof(float);
  const size_t smem = pipe > red ? pipe : red;
  if (smem > 32 * 1024)
    IG_CUDA_STATUS(cudaFuncSetAttribute(sgemm_rows_kernel<MT>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  sgemm_rows_kernel<MT><<<dim3(tiles, ksplit), kGemmWarps * 32, smem, s>>>(
      X, ldx, W, ldw, Y, ldy, R, ldr, M, N, K, ksplit, epilogue, ws, tickets);
  IG_LAUNCH_STATUS();
  return IG_OK;
}

}  // namespace ig

extern "C" int ig_sgemm_rows_ksplit(int M, int N, int K) {
  // Fill whole waves: with `slots` resident CTAs (2 per SM at M <= 16, 1 at
  // M = 32), pick the smallest split whose grid reaches >= 1 wave with >= 90%
  // of the last wave occupied (ncu: a 2.03-wave grid left SMs idle 37% of the
  // kernel), else the best-filled; each CTA keeps >= 4 pipeline stages.
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms < 1)
      sms = 148;
  }
  const int slots = sms * (M <= 16 ? 2 : 1);
  const int tiles = (N + ig::kGemmTileN - 1) / ig::kGemmTileN;
  int maxks = ((K + ig::kGemmKT - 1) / ig::kGemmKT) / 4;
  if (maxks < 1) maxks = 1;
  int best = 1;
  double best_fill = -1.0;
  for (int ks = 1; ks <= maxks && ks <= 64; ++ks) {
    const long total = (long)tiles * ks;
    const long waves = (total + slots - 1) / slots;
    const double fill = (double)total / (double)(waves * slots);
    if (total >= slots && fill >= 0.9) return ks;
    if (fill > best_fill + 1e-9) { best_fill = fill; best = ks; }
  }
  return best;
}

extern "C" int ig_sgemm_rows(const float* X, int ldx, const float* W, int ldw, float* Y, int ldy,
                             const float* R, int ldr, int M, int N, int K, int ksplit,
                             int epilogue, float* workspace, size_t workspace_floats,
                             int32_t* tickets, void* stream) {
  using namespace ig;
  if (!X || !W || !Y || !workspace || !tickets || M < 1 || M > 32 || N < 4 || (N & 3) || K < 4 ||
      (K & 3) || ldx < K || (ldx & 3) || ldw < N || (ldw & 3) || ldy < N || ksplit < 1 ||
      epilogue < 0 || epilogue > 2 || (epilogue == 2 && (!R || ldr < N)))
    return IG_EINVAL;
  const int tiles = (N + kGemmTileN - 1) / kGemmTileN;
  if ((size_t)tiles * ksplit * M * kGemmTileN > workspace_floats) return IG_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  if (M <= 8) return launch_sgemm<8>(X, ldx, W, ldw, Y, ldy, R, ldr, M, N, K, ksplit, epilogue, workspace, tickets, s);
  if (M <= 16) return launch_sgemm<16>(X, ldx, W, ldw, Y, ldy, R, ldr, M, N, K, ksplit, epilogue, workspace, tickets, s);
  return launch_sgemm<32>(X, ldx, W, ldw, Y, ldy, R, ldr, M, N, K, ksplit, epilogue, workspace, tickets, s);
}
