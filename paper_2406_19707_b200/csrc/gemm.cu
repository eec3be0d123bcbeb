// Skinny f32 GEMM for the decode step's dense projections: Y[M][N] = X[M][K] . W[K][N]
// (+ epilogue), M = sequences <= 32, W row-major (the reference's x @ W layout,
// model.py:63-79).  Weight-streaming / HBM-bound: every weight is read once.
//
// CTA = one 128-column tile x one K slice.  Its warps take interleaved groups
// of 4 weight rows: each lane loads one float4 per row (a warp reads 4 x 512 B)
// and the 4 matching x values per sequence (float4, L1/L2 broadcast), so each
// 16-B weight load feeds 4*M FMAs.  The warps' partial tiles are summed in
// shared memory in fixed warp order; the K-split partials go to a workspace and
// the last CTA of a column tile (ticket) sums them in fixed split order and
// applies the epilogue -- the result is deterministic.  IEEE f32 throughout
// (no TF32: x_a feeds the rehearsal, whose index parity needs f32).
#include "common.cuh"

namespace ig {

constexpr int kGemmTileN = 128;

template <int MT, int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
sgemm_rows_kernel(const float* __restrict__ X, int ldx, const float* __restrict__ W, int ldw,
                  float* __restrict__ Y, int ldy, const float* __restrict__ R, int ldr, int M,
                  int N, int K, int ksplit, int epilogue, float* __restrict__ ws,
                  int32_t* __restrict__ tickets) {
  extern __shared__ float red[];              // [WARPS][MT][kGemmTileN]
  __shared__ int last;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int tile = blockIdx.x, ks = blockIdx.y;
  const int n0 = tile * kGemmTileN + lane * 4;
  const bool colok = n0 < N;                  // N % 4 == 0 (checked on the host)
  // K slice of this CTA, in quads of rows
  const int quads = K >> 2;
  const int qper = (quads + ksplit - 1) / ksplit;
  const int q0 = ks * qper, q1 = min(quads, q0 + qper);

  float acc[MT][4];
#pragma unroll
  for (int m = 0; m < MT; ++m) acc[m][0] = acc[m][1] = acc[m][2] = acc[m][3] = 0.f;

  for (int q = q0 + w; q < q1; q += WARPS) {
    const int k = q * 4;
    float4 wv[4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
      wv[r] = colok ? ldg_stream(reinterpret_cast<const float4*>(W + (size_t)(k + r) * ldw + n0))
                    : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      if (m < M) {
        const float4 xv = __ldg(reinterpret_cast<const float4*>(X + (size_t)m * ldx + k));
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
  }
  // warps -> shared memory -> one partial tile (fixed warp order)
#pragma unroll
  for (int m = 0; m < MT; ++m)
    *reinterpret_cast<float4*>(red + ((size_t)w * MT + m) * kGemmTileN + lane * 4) =
        make_float4(acc[m][0], acc[m][1], acc[m][2], acc[m][3]);
  __syncthreads();
  const size_t tile_elems = (size_t)M * kGemmTileN;
  float* part = ws + ((size_t)tile * ksplit + ks) * tile_elems;
  for (int e = threadIdx.x; e < M * kGemmTileN; e += blockDim.x) {
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < WARPS; ++i) s += red[(size_t)i * MT * kGemmTileN + e];
    part[e] = s;
  }
  if (ksplit == 1) {
    __syncthreads();
  } else {
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(tickets + tile, 1) == ksplit - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
  }
  // the last CTA of this column tile: sum the splits in order, epilogue, store
  const float* tp = ws + (size_t)tile * ksplit * tile_elems;
  for (int e = threadIdx.x; e < M * kGemmTileN; e += blockDim.x) {
    const int m = e / kGemmTileN, n = tile * kGemmTileN + (e % kGemmTileN);
    if (n >= N) continue;
    float s = 0.f;
    for (int i = 0; i < ksplit; ++i) s += __ldcg(tp + (size_t)i * tile_elems + e);
    if (epilogue == 1) s = fmaxf(s, 0.f);                          // ReLU (model.py:240)
    else if (epilogue == 2) s = __fadd_rn(R[(size_t)m * ldr + n], s);   // residual add
    Y[(size_t)m * ldy + n] = s;
  }
  if (threadIdx.x == 0 && ksplit > 1) tickets[tile] = 0;
}

template <int MT, int WARPS>
int launch_sgemm(const float* X, int ldx, const float* W, int ldw, float* Y, int ldy,
                 const float* R, int ldr, int M, int N, int K, int ksplit, int epilogue, float* ws,
                 int32_t* tickets, cudaStream_t s) {
  const int tiles = (N + kGemmTileN - 1) / kGemmTileN;
  const size_t smem = (size_t)WARPS * MT * kGemmTileN * sizeof(float);
  if (smem > 32 * 1024)
    IG_CUDA_STATUS(cudaFuncSetAttribute(sgemm_rows_kernel<MT, WARPS>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  sgemm_rows_kernel<MT, WARPS><<<dim3(tiles, ksplit), WARPS * 32, smem, s>>>(
      X, ldx, W, ldw, Y, ldy, R, ldr, M, N, K, ksplit, epilogue, ws, tickets);
  IG_LAUNCH_STATUS();
  return IG_OK;
}

}  // namespace ig

extern "C" int ig_sgemm_rows_ksplit(int M, int N, int K) {
  // ~4 CTAs per SM in flight, >= 32 rows (8 quads) per CTA
  const int tiles = (N + ig::kGemmTileN - 1) / ig::kGemmTileN;
  int ks = (148 * 4 + tiles - 1) / tiles;
  const int maxks = (K / 4 + 7) / 8;
  ks = ks < 1 ? 1 : (ks > maxks ? maxks : ks);
  (void)M;
  return ks;
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
  if (M <= 8) return launch_sgemm<8, 8>(X, ldx, W, ldw, Y, ldy, R, ldr, M, N, K, ksplit, epilogue, workspace, tickets, s);
  if (M <= 16) return launch_sgemm<16, 8>(X, ldx, W, ldw, Y, ldy, R, ldr, M, N, K, ksplit, epilogue, workspace, tickets, s);
  return launch_sgemm<32, 4>(X, ldx, W, ldw, Y, ldy, R, ldr, M, N, K, ksplit, epilogue, workspace, tickets, s);
}
