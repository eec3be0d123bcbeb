// Prompt-length dense projections on the 5th-generation tensor cores
// (tcgen05.mma, TMEM accumulators, tensor-map TMA) at f32-level accuracy:
// the prefill's x_a @ [W_Q|W_K|W_V], attn @ W_O, relu(x_f @ W_in) @ W_out
// (reference forward_block model.py:195-244 as driven by DecodeSession._prefill
// engine.py:245-291) for M = B x prompt rows, compute-bound.
//
// Split precision.  Each f32 operand x is scaled by a power of two per row of
// A (per output column of W) so that max|x| lands in [2^13, 2^14), then split
// x = hi + lo, hi = f16(x), lo = f16(x - hi): 11 + 11 significand bits, as in
// the decode path's packed GEMM.  The tensor core forms hi.hi + hi.lo + lo.hi
// (each product of two f16 is exact) and accumulates in f32 in TMEM; the lo.lo
// term (2^-22 relative) is dropped.  The power-of-two scales are removed
// exactly in the epilogue.  Operands live in global memory as f16 [rows][2 Kp]
// (hi in columns [0, Kp), lo in [Kp, 2 Kp), Kp = K rounded up to 64, zero
// padded), both K-major: A = activations [M][.], B = W transposed [N][.].
//
// Kernel: persistent, one CTA per SM, 6 warps: warp 0 = TMA producer (2-stage
// ring of 96-KB stages: A hi/lo 128 x 64, B hi/lo 256 x 64, 128-B swizzle),
// warp 1 = TMEM allocator + single-thread MMA issuer (M 128 x N 256 x K 16),
// warps 2-5 = epilogue (tcgen05.ld 32 lanes x 32 columns, scale, ReLU /
// residual, f32 stores).  The tensor core adds each MMA's products into the
// f32 accumulator with truncation (measured: the error vs float64 grows as
// 0.5 ulp x the number of accumulating MMAs), so hi.hi goes to its own
// 256-column accumulator and the two cross terms (2^-11 smaller) to a second
// one, summed with round-to-nearest in the epilogue: a third of the
// accumulation steps on the large term.  Both fill TMEM (512 columns), so the
// epilogue of tile i does not overlap the main loop of tile i+1.
// Tiles are visited in groups of 8 M-tiles per N sweep so concurrently running
// CTAs share their operand tiles in L2.
#include <cuda.h>

#include "common.cuh"
#include "tc05.cuh"

namespace ig {

namespace g5 {
constexpr int BM = 128, BN = 256, BK = 64;
constexpr int kStages = 2;
constexpr int kThreads = 192;
constexpr uint32_t kTileA = BM * BK * 2;            // 16 KB (one of hi / lo)
constexpr uint32_t kTileB = BN * BK * 2;            // 32 KB
constexpr uint32_t kStage = 2 * kTileA + 2 * kTileB;
constexpr size_t kSmem = (size_t)kStages * kStage + 1024 /*align*/ + 256 /*barriers*/ + BN * 4 * 2;
constexpr int kGroupM = 8;
constexpr uint32_t kTmemCols = 512;                 // hi.hi and cross accumulators x 256 columns
}  // namespace g5

__device__ __forceinline__ void g5_tile(int t, int tiles_m, int tiles_n, int& mb, int& nb) {
  const int per_group = g5::kGroupM * tiles_n;
  const int g = t / per_group, r = t % per_group;
  const int m0 = g * g5::kGroupM;
  const int gs = min(g5::kGroupM, tiles_m - m0);
  mb = m0 + r % gs;
  nb = r / gs;
}

__global__ void __launch_bounds__(g5::kThreads, 1)
gemm_tc05_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 int M, int N, int Kp, const float* __restrict__ inv_sa, const float* __restrict__ inv_sb,
                 float* __restrict__ C, int ldc, const float* __restrict__ R, int ldr, int epilogue) {
  using namespace g5;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + kStages * kStage);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;     // [2]
  uint64_t* tempty = tfull + 2;          // [2]
  uint32_t* tmem_base_sh = (uint32_t*)(tempty + 2);
  float* sb_sh = (float*)(smem + kStages * kStage + 256);   // [2][BN] column scales

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles_m = (M + BM - 1) / BM, tiles_n = (N + BN - 1) / BN;
  const int tiles = tiles_m * tiles_n;
  const int nk = Kp / BK;

  if (warp == 0 && lane == 0) {
    tc05::tma_prefetch_desc(&tmA);
    tc05::tma_prefetch_desc(&tmB);
    for (int s = 0; s < kStages; ++s) {
      tc05::mbar_init(&full[s], 1);
      tc05::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc05::mbar_init(&tfull[a], 1);
      tc05::mbar_init(&tempty[a], 4);      // one arrive per epilogue warp
    }
    tc05::fence_barrier_init();
  }
  if (warp == 1) tc05::tmem_alloc<kTmemCols>(tmem_base_sh);
  tc05::fence_before_sync();
  __syncthreads();
  tc05::fence_after_sync();
  const uint32_t tmem = *tmem_base_sh;

  if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        int mb, nb;
        g5_tile(t, tiles_m, tiles_n, mb, nb);
        for (int kb = 0; kb < nk; ++kb) {
          tc05::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* st = smem + stage * kStage;
          tc05::mbar_expect_tx(&full[stage], kStage);
          const int k0 = kb * BK;
          tc05::tma_load_2d(st, &tmA, k0, mb * BM, &full[stage]);
          tc05::tma_load_2d(st + kTileA, &tmA, Kp + k0, mb * BM, &full[stage]);
          tc05::tma_load_2d(st + 2 * kTileA, &tmB, k0, nb * BN, &full[stage]);
          tc05::tma_load_2d(st + 2 * kTileA + kTileB, &tmB, Kp + k0, nb * BN, &full[stage]);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    constexpr uint32_t idesc = tc05::idesc_f16_f32(BM, BN, 0, 0);
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
      const int acc = 0;
      const uint32_t acc_phase = it & 1;
      tc05::mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc05::fence_after_sync();
      const uint32_t d_main = tmem, d_cross = tmem + BN;
      for (int kb = 0; kb < nk; ++kb) {
        tc05::mbar_wait(&full[stage], phase);
        tc05::fence_after_sync();
        if (tc05::elect_one()) {
          const uint32_t s0 = tc05::smem_u32(smem + stage * kStage);
          const uint32_t a_hi = s0, a_lo = s0 + kTileA, b_hi = s0 + 2 * kTileA, b_lo = b_hi + kTileB;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint32_t ko = k * 32;
            const uint32_t first = (kb == 0 && k == 0) ? 0u : 1u;
            tc05::mma_f16(d_main, tc05::desc_kmajor_sw128(a_hi + ko), tc05::desc_kmajor_sw128(b_hi + ko), idesc,
                          first);
            tc05::mma_f16(d_cross, tc05::desc_kmajor_sw128(a_hi + ko), tc05::desc_kmajor_sw128(b_lo + ko), idesc,
                          first);
            tc05::mma_f16(d_cross, tc05::desc_kmajor_sw128(a_lo + ko), tc05::desc_kmajor_sw128(b_hi + ko), idesc,
                          1u);
          }
          tc05::mma_commit(&empty[stage]);
          if (kb == nk - 1) tc05::mma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (++stage == kStages) { stage = 0; phase ^= 1; }
      }
    }
  } else {
    // ---------------- epilogue: warps 2..5 -> TMEM lane quarter (warp % 4)
    const int q = warp & 3;
    const int ep_tid = threadIdx.x - 64;            // 0..127
    int it = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
      int mb, nb;
      g5_tile(t, tiles_m, tiles_n, mb, nb);
      const int acc = 0;
      const uint32_t acc_phase = it & 1;
      float* sb = sb_sh + (it & 1) * BN;
      // column scales of this tile (read while the MMAs run)
      for (int c = ep_tid; c < BN; c += 128) {
        const int n = nb * BN + c;
        sb[c] = n < N ? inv_sb[n] : 0.f;
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      tc05::mbar_wait(&tfull[acc], acc_phase);
      tc05::fence_after_sync();
      const int row = mb * BM + q * 32 + lane;
      const float sa = row < M ? inv_sa[row] : 0.f;
      float* crow = C + (size_t)row * ldc;
      const float* rrow = R ? R + (size_t)row * ldr : nullptr;
      const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16);
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t v[32], w[32];
        tc05::tmem_ld32(tbase + c0, v);
        tc05::tmem_ld32(tbase + BN + c0, w);
        tc05::tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(__uint_as_float(v[j]) + __uint_as_float(w[j]));
        const int n0 = nb * BN + c0;
        if (row < M && n0 < N) {
          if (n0 + 32 <= N && (ldc & 3) == 0 && (!rrow || (ldr & 3) == 0)) {
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
              float4 o;
              o.x = __uint_as_float(v[j]) * sa * sb[c0 + j];
              o.y = __uint_as_float(v[j + 1]) * sa * sb[c0 + j + 1];
              o.z = __uint_as_float(v[j + 2]) * sa * sb[c0 + j + 2];
              o.w = __uint_as_float(v[j + 3]) * sa * sb[c0 + j + 3];
              if (epilogue == 1) {
                o.x = fmaxf(o.x, 0.f); o.y = fmaxf(o.y, 0.f); o.z = fmaxf(o.z, 0.f); o.w = fmaxf(o.w, 0.f);
              } else if (epilogue == 2) {
                const float4 r4 = *(const float4*)(rrow + n0 + j);
                o.x += r4.x; o.y += r4.y; o.z += r4.z; o.w += r4.w;
              }
              *(float4*)(crow + n0 + j) = o;
            }
          } else {
            for (int j = 0; j < 32 && n0 + j < N; ++j) {
              float o = __uint_as_float(v[j]) * sa * sb[c0 + j];
              if (epilogue == 1) o = fmaxf(o, 0.f);
              else if (epilogue == 2) o += rrow[n0 + j];
              crow[n0 + j] = o;
            }
          }
        }
      }
      tc05::fence_before_sync();
      __syncwarp();
      if (lane == 0) tc05::mbar_arrive(&tempty[acc]);
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc05::fence_after_sync();
    tc05::tmem_dealloc<kTmemCols>(tmem);
  }
}

// ---------------------------------------------------------------------------
// Split kernels.  Rows of the output are the K-major operand rows.
// ---------------------------------------------------------------------------
__device__ __forceinline__ float pow2_scale(float amax, float* inv) {
  if (!(amax > 0.f) || !isfinite(amax)) { *inv = 1.f; return 1.f; }
  int e;
  frexpf(amax, &e);              // amax = m 2^e, m in [0.5, 1)
  const int sh = 14 - e;         // amax * 2^sh in [2^13, 2^14)
  *inv = ldexpf(1.f, -sh);
  return ldexpf(1.f, sh);
}

__device__ __forceinline__ void split_store(float x, float s, __half* hi, __half* lo) {
  const float y = x * s;
  const __half h = __float2half_rn(y);
  *hi = h;
  *lo = __float2half_rn(y - __half2float(h));
}

// A: X [rows][cols] (ld), one warp per row -> out [rows][2 Kp]
__global__ void __launch_bounds__(256)
split_rows_kernel(const float* __restrict__ X, int ldx, int rows, int cols, int Kp,
                  __half* __restrict__ out, float* __restrict__ inv_scale) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= rows) return;
  const float* x = X + (size_t)warp * ldx;
  float m = 0.f;
  for (int c = lane; c < cols; c += 32) m = fmaxf(m, fabsf(x[c]));
  m = warp_max(m);
  float inv;
  const float s = pow2_scale(m, &inv);
  __half* o = out + (size_t)warp * 2 * Kp;
  for (int c = lane; c < Kp; c += 32) {
    if (c < cols) split_store(x[c], s, o + c, o + Kp + c);
    else { o[c] = __float2half_rn(0.f); o[Kp + c] = __float2half_rn(0.f); }
  }
  if (lane == 0) inv_scale[warp] = inv;
}

// B: W [K][N] (ld) -> out [N][2 Kp] (transposed), 32 columns per CTA
__global__ void __launch_bounds__(256)
split_cols_kernel(const float* __restrict__ W, int ldw, int K, int N, int Kp,
                  __half* __restrict__ out, float* __restrict__ inv_scale) {
  __shared__ float red[8][33];
  __shared__ float sc[32];
  __shared__ float tile[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 x 8
  const int n0 = blockIdx.x * 32;
  const int n = n0 + tx;
  float m = 0.f;
  if (n < N)
    for (int k = ty; k < K; k += 8) m = fmaxf(m, fabsf(W[(size_t)k * ldw + n]));
  red[ty][tx] = m;
  __syncthreads();
  if (ty == 0) {
    for (int i = 1; i < 8; ++i) m = fmaxf(m, red[i][tx]);
    float inv;
    sc[tx] = pow2_scale(m, &inv);
    if (n < N) inv_scale[n] = inv;
  }
  __syncthreads();
  for (int k0 = 0; k0 < Kp; k0 += 32) {
    for (int r = ty; r < 32; r += 8) {
      const int k = k0 + r;
      tile[r][tx] = (k < K && n < N) ? W[(size_t)k * ldw + n] : 0.f;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {          // r: column within the stripe
      const int nn = n0 + r;
      if (nn < N) {
        __half* o = out + (size_t)nn * 2 * Kp;
        split_store(tile[tx][r], sc[r], o + k0 + tx, o + Kp + k0 + tx);
      }
    }
    __syncthreads();
  }
}

int make_tmap_2d(CUtensorMap* map, CUtensorMapDataType dtype, const void* base, uint64_t inner,
                 uint64_t outer, uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer,
                 CUtensorMapSwizzle swizzle) {
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p)
      return IG_ECUDA + (int)cudaErrorNotSupported;
    fn = (EncodeFn)p;
  }
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {row_bytes};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = fn(map, dtype, 2, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? IG_OK : IG_EINVAL;
}

}  // namespace ig

extern "C" int ig_split_f16(const float* X, int ldx, int rows, int cols, int transpose, int Kp, void* out,
                            float* inv_scale, void* stream) {
  // transpose = 0: X [rows][cols] -> out [rows][2 Kp] (K = cols);
  // transpose = 1: X [rows = K][cols = N] -> out [N][2 Kp] (W transposed)
  const int K = transpose ? rows : cols;
  if (!X || !out || !inv_scale || rows <= 0 || cols <= 0 || Kp < K || Kp % 64 || ldx < cols)
    return IG_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  if (!transpose) {
    const int blocks = (rows + 7) / 8;
    ig::split_rows_kernel<<<blocks, 256, 0, s>>>(X, ldx, rows, cols, Kp, (__half*)out, inv_scale);
  } else {
    ig::split_cols_kernel<<<(cols + 31) / 32, 256, 0, s>>>(X, ldx, rows, cols, Kp, (__half*)out, inv_scale);
  }
  IG_LAUNCH_STATUS();
  return IG_OK;
}

extern "C" int ig_gemm_tc05(const void* A_hl, const float* inv_sa, const void* B_hl, const float* inv_sb, int M,
                            int N, int K, int Kp, float* C, int ldc, const float* R, int ldr, int epilogue,
                            int max_ctas, void* stream) {
  using namespace ig::g5;
  if (!A_hl || !B_hl || !inv_sa || !inv_sb || !C || M <= 0 || N <= 0 || K <= 0 || Kp < K || Kp % BK ||
      ldc < N || (epilogue == 2 && (!R || ldr < N)) || epilogue < 0 || epilogue > 2)
    return IG_EINVAL;
  CUtensorMap ta, tb;
  int rc = ig::make_tmap_2d(&ta, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, A_hl, (uint64_t)2 * Kp, (uint64_t)M,
                            (uint64_t)4 * Kp, BK, BM, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  rc = ig::make_tmap_2d(&tb, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, B_hl, (uint64_t)2 * Kp, (uint64_t)N,
                        (uint64_t)4 * Kp, BK, BN, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    IG_CUDA_STATUS(cudaGetDevice(&dev));
    IG_CUDA_STATUS(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    IG_CUDA_STATUS(cudaFuncSetAttribute(ig::gemm_tc05_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)kSmem));
  }
  const int tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  int grid = tiles < sms ? tiles : sms;
  if (max_ctas > 0 && grid > max_ctas) grid = max_ctas;
  ig::gemm_tc05_kernel<<<grid, kThreads, kSmem, (cudaStream_t)stream>>>(ta, tb, M, N, Kp, inv_sa, inv_sb, C, ldc,
                                                                        R, ldr, epilogue);
  IG_LAUNCH_STATUS();
  return IG_OK;
}
