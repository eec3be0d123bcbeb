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
#include <cstdlib>

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

// Sum of the K-split partials of one output element in split order 0, 1, ...
// (deterministic); the loads are batched 8 at a time so a 32-way split costs 4
// L2 round trips, not 32 dependent ones (ncu: the serial loop was the tail of
// every column tile).
__device__ __forceinline__ float sum_splits(const float* __restrict__ p, size_t stride, int ks) {
  float s = 0.f;
  int i = 0;
  for (; i + 8 <= ks; i += 8) {
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldcg(p + (size_t)(i + u) * stride);
#pragma unroll
    for (int u = 0; u < 8; ++u) s += v[u];
  }
  for (; i < ks; ++i) s += __ldcg(p + (size_t)i * stride);
  return s;
}

// Per-thread stage loader with the addressing hoisted out of the K loop:
// thread tid copies the 16-B vectors (row w + 8i, column quad lane) of every
// 32-row weight chunk, i = 0..3, and (tid < MT*8) vector tid of the x slice.
// A whole chunk needs one pointer increment per vector; only the last chunk
// of K (rows >= K) and a ragged column tile take the zero-filling path.
template <int MT>
struct StageLoader {
  const char* wp;        // this thread's first W vector of chunk 0
  const char* xp;        // this thread's x vector of chunk 0 (nullptr: none)
  size_t wrow8;          // bytes between rows r and r + 8
  size_t wchunk;         // bytes between chunks
  int krow0, xk, K;      // first row of chunk 0, x column of this thread, K
  bool colok, xok;
  uint32_t wdst, xdst;   // shared offsets within a stage (bytes)

  __device__ void init(const float* W, int ldw, const float* X, int ldx, int M, int N, int K_,
                       int c0, int ncol0, int wpitch, int xpitch, int kWsFloats) {
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    K = K_;
    krow0 = c0 * kGemmKT + w;
    colok = ncol0 + lane * 4 < N;
    wp = reinterpret_cast<const char*>(W + (size_t)krow0 * ldw + ncol0 + lane * 4);
    wrow8 = (size_t)8 * ldw * sizeof(float);
    wchunk = (size_t)kGemmKT * ldw * sizeof(float);
    wdst = (uint32_t)((w * wpitch + lane * 4) * sizeof(float));
    const int m = tid / (kGemmKT / 4), k4 = tid % (kGemmKT / 4);
    xok = tid < MT * (kGemmKT / 4) && m < M;
    xk = c0 * kGemmKT + k4 * 4;
    xp = reinterpret_cast<const char*>(X + (size_t)(m < M ? m : 0) * ldx + xk);
    xdst = (uint32_t)((kWsFloats + m * xpitch + k4 * 4) * sizeof(float));
    (void)lane;
  }
  // chunk c (relative to c0) into the stage at shared address `base`
  __device__ __forceinline__ void load(int c, uint32_t base, int wpitch) const {
    const char* src = wp + (size_t)c * wchunk;
    const int k = krow0 + c * kGemmKT;
    if (colok && k + 24 < K) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(base + wdst + i * 8 * wpitch * 4),
                     "l"(src + i * wrow8) : "memory");
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const bool ok = colok && k + 8 * i < K;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(base + wdst + i * 8 * wpitch * 4),
                     "l"(ok ? src + i * wrow8 : wp), "r"(ok ? 16 : 0) : "memory");
      }
    }
    if (tid_has_x()) {
      const bool ok = xok && xk + c * kGemmKT < K;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(base + xdst),
                   "l"(ok ? xp + (size_t)c * kGemmKT * sizeof(float) : xp), "r"(ok ? 16 : 0) : "memory");
    }
  }
  __device__ __forceinline__ bool tid_has_x() const { return threadIdx.x < MT * (kGemmKT / 4); }
};

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

  StageLoader<MT> ld;
  ld.init(W, ldw, X, ldx, M, N, K, c0, ncol0, kGemmTileN, kGemmKT, kWs);
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  auto load_stage = [&](int c, int st) { ld.load(c, sbase + st * kStage * 4, kGemmTileN); };

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
    s = sum_splits(tp + e, tile_elems, ksplit);
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


// ---------------------------------------------------------------------------
// Tensor-core variant: 3xTF32 split precision on mma.sync m16n8k8.  Every f32
// operand is split into a TF32 head and a tail (v = hi + lo exactly; hi is v
// rounded to TF32 by integer add + mask, lo = v - hi, which the tensor core
// reads truncated to TF32); x.w = x_hi.w_hi + (x_hi.w_lo + x_lo.w_hi) with the
// two tail products in their own accumulator -- f32-level accuracy (the
// neglected terms are ~2^-21 relative).
//
// Weights stream through the same 16-B cp.async pipeline as sgemm_rows_kernel
// (StageLoader: per-thread addressing hoisted out of the K loop).  TMA 1-D
// bulk copies of the 512-B rows were measured slower (1.9 TB/s: the TMA unit
// serves ~one request per ~46 cycles per SM, too few bytes per request).
// CTA = 128 columns x one K slice (fixed-order
// split-K merge as sgemm_rows_kernel); each warp owns 16 columns over the
// whole slice, so no cross-warp reduction.  Shared rows are padded (W: 136
// floats, X: 36) so a warp's fragment loads hit 32 distinct banks.
// ---------------------------------------------------------------------------
constexpr int kTcWPitch = kGemmTileN + 8;    // 136
constexpr int kTcXPitch = kGemmKT + 4;       // 36

__device__ __forceinline__ void split_tf32(float x, uint32_t& hi, uint32_t& lo) {
  hi = (__float_as_uint(x) + 0x1000u) & 0xffffe000u;   // round half away, 10-bit mantissa
  lo = __float_as_uint(x - __uint_as_float(hi));        // exact remainder
}
__device__ __forceinline__ void mma_tf32(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// KIN = 2: the 8 warps form 2 groups over the k8 steps of each stage (warp
// w: columns 32 (w & 3) .. +31, k8 steps 2 (w >> 2), +1) and the groups'
// accumulators are summed through shared memory at the end (fixed order);
// KIN = 1: warp w owns columns 16 w .. +15 over all k8 steps.
template <int MTILES, int STAGES, int KIN>   // 16-row M tiles (M <= 16 * MTILES), pipeline depth
__global__ void __launch_bounds__(kGemmWarps * 32, (MTILES == 1 ? (STAGES <= 3 ? 3 : 2) : 1))
sgemm_tc_kernel(const float* __restrict__ X, int ldx, const float* __restrict__ W, int ldw,
                float* __restrict__ Y, int ldy, const float* __restrict__ R, int ldr, int M, int N,
                int K, int ksplit, int epilogue, float* __restrict__ ws,
                int32_t* __restrict__ tickets) {
  extern __shared__ __align__(128) float smem[];
  constexpr int MT = 16 * MTILES;
  constexpr int kWs = kGemmKT * kTcWPitch, kXs = MT * kTcXPitch, kStage = kWs + kXs;
  __shared__ int last;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int tile = blockIdx.x, ks = blockIdx.y;
  const int ncol0 = tile * kGemmTileN;
  const int chunks_all = (K + kGemmKT - 1) / kGemmKT;
  const int cper = (chunks_all + ksplit - 1) / ksplit;
  const int c0 = ks * cper, c1 = min(chunks_all, c0 + cper);
  const int nch = max(0, c1 - c0);

  StageLoader<MT> ld;
  ld.init(W, ldw, X, ldx, M, N, K, c0, ncol0, kTcWPitch, kTcXPitch, kWs);
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  auto load_stage = [&](int c, int st) { ld.load(c, sbase + st * kStage * 4, kTcWPitch); };

  constexpr int NT = 2 * KIN;                  // n8 tiles per warp
  float big[MTILES][NT][4], small[MTILES][NT][4], small2[MTILES][NT][4];
#pragma unroll
  for (int mt = 0; mt < MTILES; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int i = 0; i < 4; ++i) big[mt][nt][i] = small[mt][nt][i] = small2[mt][nt][i] = 0.f;

#pragma unroll
  for (int i = 0; i < STAGES - 1; ++i) {
    if (i < nch) load_stage(i, i);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  const int wn = KIN == 2 ? (w & 3) * 32 : w * 16;   // my columns of the tile
  const int k8lo = KIN == 2 ? (w >> 2) * 16 : 0;      // my k8 steps of each stage
  for (int c = 0; c < nch; ++c) {
    const int st = c % STAGES;
    asm volatile("cp.async.wait_group %0;" ::"n"(STAGES - 2) : "memory");
    __syncthreads();                           // stage c landed; stage c-1 fully consumed
    const int nx = c + STAGES - 1;
    if (nx < nch) load_stage(nx, nx % STAGES);
    asm volatile("cp.async.commit_group;" ::: "memory");
    const float* ws_ = smem + st * kStage;
    const float* xs_ = ws_ + kWs;
#pragma unroll
    for (int kq = 0; kq < kGemmKT / KIN; kq += 8) {
      const int k8 = k8lo + kq;
      uint32_t ahi[MTILES][4], alo[MTILES][4];
#pragma unroll
      for (int mt = 0; mt < MTILES; ++mt) {
        const float* xr = xs_ + (mt * 16 + g) * kTcXPitch + k8 + t;
        split_tf32(xr[0], ahi[mt][0], alo[mt][0]);
        split_tf32(xr[8 * kTcXPitch], ahi[mt][1], alo[mt][1]);
        split_tf32(xr[4], ahi[mt][2], alo[mt][2]);
        split_tf32(xr[8 * kTcXPitch + 4], ahi[mt][3], alo[mt][3]);
      }
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const float* wr = ws_ + (k8 + t) * kTcWPitch + wn + nt * 8 + g;
        uint32_t bhi0, blo0, bhi1, blo1;
        split_tf32(wr[0], bhi0, blo0);
        split_tf32(wr[4 * kTcWPitch], bhi1, blo1);
#pragma unroll
        for (int mt = 0; mt < MTILES; ++mt) {
          mma_tf32(small[mt][nt], alo[mt], bhi0, bhi1);
          mma_tf32(small2[mt][nt], ahi[mt], blo0, blo1);
          mma_tf32(big[mt][nt], ahi[mt], bhi0, bhi1);
        }
      }
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll
  for (int mt = 0; mt < MTILES; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int i = 0; i < 4; ++i) big[mt][nt][i] += small[mt][nt][i] + small2[mt][nt][i];
  if (KIN == 2) {              // k-group 1 hands its sums to k-group 0 through shared memory
    __syncthreads();           // every warp is past its last stage read
    float* red = smem;         // [4 warps][MTILES][NT][4][32 lanes]
    constexpr int per = MTILES * NT * 4;
    if (w >= 4) {
#pragma unroll
      for (int mt = 0; mt < MTILES; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int i = 0; i < 4; ++i)
            red[(((w - 4) * per) + (mt * NT + nt) * 4 + i) * 32 + lane] = big[mt][nt][i];
    }
    __syncthreads();
    if (w < 4) {
#pragma unroll
      for (int mt = 0; mt < MTILES; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int i = 0; i < 4; ++i)
            big[mt][nt][i] += red[((w * per) + (mt * NT + nt) * 4 + i) * 32 + lane];
    }
  }
  const size_t tile_elems = (size_t)M * kGemmTileN;
  float* part = ws + ((size_t)tile * ksplit + ks) * tile_elems;
#pragma unroll
  for (int mt = 0; mt < MTILES; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      if (KIN == 2 && w >= 4) break;
      const int col = wn + nt * 8 + 2 * t;
      const int r0 = mt * 16 + g, r1 = r0 + 8;
      if (r0 < M)
        *reinterpret_cast<float2*>(part + (size_t)r0 * kGemmTileN + col) =
            make_float2(big[mt][nt][0], big[mt][nt][1]);
      if (r1 < M)
        *reinterpret_cast<float2*>(part + (size_t)r1 * kGemmTileN + col) =
            make_float2(big[mt][nt][2], big[mt][nt][3]);
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
  const float* tp = ws + (size_t)tile * ksplit * tile_elems;
  for (int e = tid; e < M * kGemmTileN; e += blockDim.x) {
    const int m = e / kGemmTileN, n = ncol0 + (e % kGemmTileN);
    if (n >= N) continue;
    float s = 0.f;
    s = sum_splits(tp + e, tile_elems, ksplit);
    if (epilogue == 1) s = fmaxf(s, 0.f);
    else if (epilogue == 2) s = __fadd_rn(R[(size_t)m * ldr + n], s);
    Y[(size_t)m * ldy + n] = s;
  }
  if (tid == 0 && ksplit > 1) tickets[tile] = 0;
}

// Swapped-operand variant: D^T = W^T . X^T, i.e. the weight tile is the MMA's
// A operand (M = output columns) and x the B operand (N = 8 sequences per n
// tile).  A warp owns 32 columns (two m16 tiles) and column m of m-tile mt
// lives at physical column 4 (m % 8) + 2 mt + m / 8 of its 32, so one LDS.128
// at (row k, column 4g) returns the A-fragment pair (g, g + 8) of both m-tiles
// -- one shared load per four weights instead of four (the LDS / MIO queue
// was a top stall of sgemm_tc_kernel).  Same pipeline, K split in two warp
// groups (KIN = 2), split precision and merge as sgemm_tc_kernel.
template <int NB, int STAGES, int KG>   // NB = 8-sequence n tiles (M <= 8 * NB); KG k-groups
__global__ void __launch_bounds__(kGemmWarps * 32, (NB <= 2 && STAGES <= 3 && KG <= 2 ? 3 : 2))
sgemm_tcw_kernel(const float* __restrict__ X, int ldx, const float* __restrict__ W, int ldw,
                 float* __restrict__ Y, int ldy, const float* __restrict__ R, int ldr, int M, int N,
                 int K, int ksplit, int epilogue, float* __restrict__ ws,
                 int32_t* __restrict__ tickets) {
  extern __shared__ __align__(128) float smem[];
  constexpr int MT = 8 * NB;
  constexpr int kWs = kGemmKT * kTcWPitch, kXs = MT * kTcXPitch, kStage = kWs + kXs;
  constexpr int WPG = kGemmWarps / KG;         // warps per k-group
  constexpr int HV = 4 / WPG;                  // 32-column halves per warp (1 or 2)
  constexpr int MTW = 2 * HV;                  // m16 tiles per warp
  __shared__ int last;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int tile = blockIdx.x, ks = blockIdx.y;
  const int ncol0 = tile * kGemmTileN;
  const int chunks_all = (K + kGemmKT - 1) / kGemmKT;
  const int cper = (chunks_all + ksplit - 1) / ksplit;
  const int c0 = ks * cper, c1 = min(chunks_all, c0 + cper);
  const int nch = max(0, c1 - c0);

  StageLoader<MT> ld;
  ld.init(W, ldw, X, ldx, M, N, K, c0, ncol0, kTcWPitch, kTcXPitch, kWs);
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  auto load_stage = [&](int c, int st) { ld.load(c, sbase + st * kStage * 4, kTcWPitch); };

  float big[MTW][NB][4], small[MTW][NB][4];
#pragma unroll
  for (int mt = 0; mt < MTW; ++mt)
#pragma unroll
    for (int nb = 0; nb < NB; ++nb)
#pragma unroll
      for (int i = 0; i < 4; ++i) big[mt][nb][i] = small[mt][nb][i] = 0.f;

#pragma unroll
  for (int i = 0; i < STAGES - 1; ++i) {
    if (i < nch) load_stage(i, i);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  const int kg = w / WPG, wi = w % WPG;
  const int wc = wi * 32 * HV;                 // my columns of the tile
  const int k8lo = kg * (kGemmKT / KG);        // my k8 steps of each stage
  for (int c = 0; c < nch; ++c) {
    const int st = c % STAGES;
    asm volatile("cp.async.wait_group %0;" ::"n"(STAGES - 2) : "memory");
    __syncthreads();
    const int nx = c + STAGES - 1;
    if (nx < nch) load_stage(nx, nx % STAGES);
    asm volatile("cp.async.commit_group;" ::: "memory");
    const float* ws_ = smem + st * kStage;
    const float* xs_ = ws_ + kWs;
#pragma unroll
    for (int kq = 0; kq < kGemmKT / KG; kq += 8) {
      const int k8 = k8lo + kq;
      // A (weights): rows k8+t and k8+t+4; per 32-column half, physical columns
      // 4g .. 4g+3 = (m-tile 0: g, g+8; m-tile 1: g, g+8)
      uint32_t ah[MTW][4], al[MTW][4];
#pragma unroll
      for (int hv = 0; hv < HV; ++hv) {
        const float4 wlo = *reinterpret_cast<const float4*>(ws_ + (k8 + t) * kTcWPitch + wc + 32 * hv + 4 * g);
        const float4 whi = *reinterpret_cast<const float4*>(ws_ + (k8 + t + 4) * kTcWPitch + wc + 32 * hv + 4 * g);
        const int m0 = 2 * hv;
        split_tf32(wlo.x, ah[m0][0], al[m0][0]);
        split_tf32(wlo.y, ah[m0][1], al[m0][1]);
        split_tf32(wlo.z, ah[m0 + 1][0], al[m0 + 1][0]);
        split_tf32(wlo.w, ah[m0 + 1][1], al[m0 + 1][1]);
        split_tf32(whi.x, ah[m0][2], al[m0][2]);
        split_tf32(whi.y, ah[m0][3], al[m0][3]);
        split_tf32(whi.z, ah[m0 + 1][2], al[m0 + 1][2]);
        split_tf32(whi.w, ah[m0 + 1][3], al[m0 + 1][3]);
      }
#pragma unroll
      for (int nb = 0; nb < NB; ++nb) {
        const float* xr = xs_ + (nb * 8 + g) * kTcXPitch + k8 + t;
        uint32_t bh0, bl0, bh1, bl1;
        split_tf32(xr[0], bh0, bl0);
        split_tf32(xr[4], bh1, bl1);
#pragma unroll
        for (int mt = 0; mt < MTW; ++mt) {
          mma_tf32(small[mt][nb], al[mt], bh0, bh1);
          mma_tf32(small[mt][nb], ah[mt], bl0, bl1);
          mma_tf32(big[mt][nb], ah[mt], bh0, bh1);
        }
      }
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll
  for (int mt = 0; mt < MTW; ++mt)
#pragma unroll
    for (int nb = 0; nb < NB; ++nb)
#pragma unroll
      for (int i = 0; i < 4; ++i) big[mt][nb][i] += small[mt][nb][i];
  {                            // k-groups 1.. hand their sums to k-group 0 (fixed order)
    __syncthreads();
    float* red = smem;         // [KG-1][WPG warps][MTW][NB][4][32 lanes]
    constexpr int per = MTW * NB * 4;
    if (kg > 0) {
#pragma unroll
      for (int mt = 0; mt < MTW; ++mt)
#pragma unroll
        for (int nb = 0; nb < NB; ++nb)
#pragma unroll
          for (int i = 0; i < 4; ++i)
            red[((((kg - 1) * WPG + wi) * per) + (mt * NB + nb) * 4 + i) * 32 + lane] = big[mt][nb][i];
    }
    __syncthreads();
    if (kg == 0) {
      for (int gg = 1; gg < KG; ++gg)
#pragma unroll
        for (int mt = 0; mt < MTW; ++mt)
#pragma unroll
          for (int nb = 0; nb < NB; ++nb)
#pragma unroll
            for (int i = 0; i < 4; ++i)
              big[mt][nb][i] += red[((((gg - 1) * WPG + wi) * per) + (mt * NB + nb) * 4 + i) * 32 + lane];
    }
  }
  const size_t tile_elems = (size_t)M * kGemmTileN;
  float* part = ws + ((size_t)tile * ksplit + ks) * tile_elems;
  if (kg == 0) {
#pragma unroll
    for (int mt = 0; mt < MTW; ++mt)
#pragma unroll
      for (int nb = 0; nb < NB; ++nb) {
        // C: (m = g, seq 2t / 2t+1) and (m = g + 8, seq 2t / 2t+1)
        const int col0 = wc + 32 * (mt >> 1) + 4 * g + 2 * (mt & 1), col1 = col0 + 1;
        const int s0 = nb * 8 + 2 * t, s1 = s0 + 1;
        if (s0 < M) {
          part[(size_t)s0 * kGemmTileN + col0] = big[mt][nb][0];
          part[(size_t)s0 * kGemmTileN + col1] = big[mt][nb][2];
        }
        if (s1 < M) {
          part[(size_t)s1 * kGemmTileN + col0] = big[mt][nb][1];
          part[(size_t)s1 * kGemmTileN + col1] = big[mt][nb][3];
        }
      }
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
  const float* tp = ws + (size_t)tile * ksplit * tile_elems;
  for (int e = tid; e < M * kGemmTileN; e += blockDim.x) {
    const int m = e / kGemmTileN, n = ncol0 + (e % kGemmTileN);
    if (n >= N) continue;
    float s = 0.f;
    s = sum_splits(tp + e, tile_elems, ksplit);
    if (epilogue == 1) s = fmaxf(s, 0.f);
    else if (epilogue == 2) s = __fadd_rn(R[(size_t)m * ldr + n], s);
    Y[(size_t)m * ldy + n] = s;
  }
  if (tid == 0 && ksplit > 1) tickets[tile] = 0;
}

template <int NB, int STAGES, int KG = 2>
int launch_sgemm_tcw(const float* X, int ldx, const float* W, int ldw, float* Y, int ldy,
                     const float* R, int ldr, int M, int N, int K, int ksplit, int epilogue,
                     float* ws, int32_t* tickets, cudaStream_t s) {
  const int tiles = (N + kGemmTileN - 1) / kGemmTileN;
  const size_t smem =
      (size_t)STAGES * (kGemmKT * kTcWPitch + 8 * NB * kTcXPitch) * sizeof(float);
  IG_CUDA_STATUS(cudaFuncSetAttribute(sgemm_tcw_kernel<NB, STAGES, KG>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  sgemm_tcw_kernel<NB, STAGES, KG><<<dim3(tiles, ksplit), kGemmWarps * 32, smem, s>>>(
      X, ldx, W, ldw, Y, ldy, R, ldr, M, N, K, ksplit, epilogue, ws, tickets);
  IG_LAUNCH_STATUS();
  return IG_OK;
}

template <int MTILES, int STAGES, int KIN>
int launch_sgemm_tc(const float* X, int ldx, const float* W, int ldw, float* Y, int ldy,
                    const float* R, int ldr, int M, int N, int K, int ksplit, int epilogue,
                    float* ws, int32_t* tickets, cudaStream_t s) {
  const int tiles = (N + kGemmTileN - 1) / kGemmTileN;
  const size_t smem =
      (size_t)STAGES * (kGemmKT * kTcWPitch + 16 * MTILES * kTcXPitch) * sizeof(float);
  IG_CUDA_STATUS(cudaFuncSetAttribute(sgemm_tc_kernel<MTILES, STAGES, KIN>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  sgemm_tc_kernel<MTILES, STAGES, KIN><<<dim3(tiles, ksplit), kGemmWarps * 32, smem, s>>>(
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

extern "C" int ig_sgemm_tc_ksplit(int M, int N, int K) {
  // Measured for sgemm_tcw_kernel (tools/gemm_probe.py --ksplit all, C3 shapes,
  // profiles/r01g_gemm_ksplit_tcw.jsonl): ~1200 CTAs, at most 16 splits and >= 10
  // pipeline chunks per CTA come within noise of the best split of every shape.
  (void)M;
  const int tiles = (N + ig::kGemmTileN - 1) / ig::kGemmTileN;
  const int chunks = (K + ig::kGemmKT - 1) / ig::kGemmKT;
  int ks = (1200 + tiles - 1) / tiles;        // ~1200 CTAs: ~3 waves of 3 CTAs/SM
  if (ks > 16) ks = 16;
  if (ks > chunks / 10) ks = chunks / 10;     // >= 10 pipeline chunks per CTA
  return ks < 1 ? 1 : ks;
}

extern "C" int ig_sgemm_tc(const float* X, int ldx, const float* W, int ldw, float* Y, int ldy,
                           const float* R, int ldr, int M, int N, int K, int ksplit, int epilogue,
                           float* workspace, size_t workspace_floats, int32_t* tickets,
                           void* stream) {
  using namespace ig;
  if (!X || !W || !Y || !workspace || !tickets || M < 1 || M > 32 || N < 4 || (N & 3) || K < 4 ||
      (K & 3) || ldx < K || (ldx & 3) || ldw < N || (ldw & 3) || ldy < N || ksplit < 1 ||
      epilogue < 0 || epilogue > 2 || (epilogue == 2 && (!R || ldr < N)))
    return IG_EINVAL;
  if (((uintptr_t)X & 15) || ((uintptr_t)W & 15)) return IG_EINVAL;   // 16-B vectors
  const int tiles = (N + kGemmTileN - 1) / kGemmTileN;
  if ((size_t)tiles * ksplit * M * kGemmTileN > workspace_floats) return IG_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  static const int variant = [] {
    // tuning sweeps only (profiles/r01e_gemm_variants.md): 4 = swapped operands
    // (sgemm_tcw_kernel, default), 1 = (3 stages, KIN 2), 0 = (3 stages, KIN 1),
    // 2 = (4 stages, KIN 1)
    const char* v = getenv("IG_TC_VARIANT");
    return v ? atoi(v) : 4;
  }();
  if (variant == 4 || variant >= 5) {
    if (M <= 8)
      return launch_sgemm_tcw<1, 3>(X, ldx, W, ldw, Y, ldy, R, ldr, M, N, K, ksplit, epilogue, workspace, tickets, s);
    if (M <= 16)
      return launch_sgemm_tcw<2, 3>(X, ldx, W, ldw, Y, ldy, R, ldr, M, N, K, ksplit, epilogue, workspace, tickets, s);
    return launch_sgemm_tcw<4, 3>(X, ldx, W, ldw, Y, ldy, R, ldr, M, N, K, ksplit, epilogue, workspace, tickets, s);
  }
  if (M <= 16) {
    if (variant == 0)
      return launch_sgemm_tc<1, 3, 1>(X, ldx, W, ldw, Y, ldy, R, ldr, M, N, K, ksplit, epilogue, workspace, tickets, s);
    if (variant == 2)
      return launch_sgemm_tc<1, 4, 1>(X, ldx, W, ldw, Y, ldy, R, ldr, M, N, K, ksplit, epilogue, workspace, tickets, s);
    return launch_sgemm_tc<1, 3, 2>(X, ldx, W, ldw, Y, ldy, R, ldr, M, N, K, ksplit, epilogue, workspace, tickets, s);
  }
  return launch_sgemm_tc<2, 4, 1>(X, ldx, W, ldw, Y, ldy, R, ldr, M, N, K, ksplit, epilogue, workspace, tickets, s);
}
