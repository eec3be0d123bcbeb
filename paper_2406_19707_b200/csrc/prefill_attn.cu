// Prefill causal attention on the 5th-generation tensor cores (SURVEY.md
// s8(f) rank 1): softmax(q k^T / float32(sqrt(d))) v with a causal mask over
// the prompt, per (sequence, head) -- the reference forward_block's attention
// (model.py:156-180 with causal=True, model.py:195-244) as driven by
// DecodeSession._prefill (engine.py:245-291).  f32-level accuracy from exact
// f16 hi/lo splits of q, k, v and p (x = hi + lo, 11 + 11 significand bits):
//
//   S = Q K^T:   qh.kh + qh.kl + ql.kh      (one TMEM accumulator, 128 q x 64 keys)
//   O = P V:     ph.vh  (own accumulator)  +  ph.vl + pl.vh  (cross accumulator)
//
// Two passes over the key tiles of a 128-query block, so the accumulation of
// O needs no rescaling: pass 1 computes S tile by tile for the row maxima only;
// pass 2 recomputes S, writes p = exp(s - m) (split) as the A operand of the
// output MMAs and accumulates l = sum p.  Warp roles as in attend_tc05.cu:
// warp 0 TMA producer (2-D tensor maps, 128-B swizzle, 2-stage ring of K|V
// tiles), warp 1 single-thread tcgen05.mma issuer (score MMAs one tile ahead,
// two TMEM score buffers), warps 2-9 softmax / epilogue (TMEM lane = query
// row, two warps per row: one per half of the key tile / output columns).  One CTA per (q block, head, sequence),
// heaviest (latest) q blocks first.
#include <cuda.h>

#include "common.cuh"
#include "tc05.cuh"

namespace ig {
namespace pa {
constexpr int BQ = 128, BK = 64;
constexpr int kThreads = 320;           // producer, MMA, 8 softmax warps (2 per TMEM lane quarter)
constexpr uint32_t kTmemCols = 512;      // S [0, 64) / [64, 128), O main [128, 128 + D), O cross [256, 256 + D)

template <int D> struct Geo {
  static constexpr int kBoxes = D / 64;                         // 64-element (128-B) boxes per part
  static constexpr uint32_t kQPart = BQ * D * 2;                // one of hi / lo
  static constexpr uint32_t kQBytes = 2 * kQPart;
  static constexpr uint32_t kKPart = BK * D * 2;
  static constexpr uint32_t kKBytes = 2 * kKPart;               // K hi | K lo
  static constexpr uint32_t kStage = 2 * kKBytes;               // K | V
  static constexpr uint32_t kPPart = BQ * BK * 2;               // 16 KB
  static constexpr size_t kSmem = 1024 + kQBytes + 2 * kStage + 2 * kPPart + 128 + 2 * BQ * 4;   // <= 227 KB
};
}  // namespace pa

// qkv [rows = nb N][3 Hg d] f32 (q | k | v) -> hl [3][nb][Hg][N][2 d] f16 (hi | lo)
__global__ void __launch_bounds__(256)
split_qkv_kernel(const float* __restrict__ qkv, int ld, int nb, int N, int Hg, int d,
                 __half* __restrict__ hl) {
  const size_t warp = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const size_t rows = (size_t)3 * nb * Hg * N;
  if (warp >= rows) return;
  // warp -> (which, b, h, n): output row order
  const int n = (int)(warp % N);
  const size_t r1 = warp / N;
  const int h = (int)(r1 % Hg);
  const size_t r2 = r1 / Hg;
  const int b = (int)(r2 % nb);
  const int which = (int)(r2 / nb);
  const float* src = qkv + ((size_t)b * N + n) * ld + (size_t)which * Hg * d + (size_t)h * d;
  __half* dst = hl + warp * 2 * d;
  for (int e = lane; e < d; e += 32) {
    const float x = src[e];
    const __half hi = __float2half_rn(x);
    dst[e] = hi;
    dst[d + e] = __float2half_rn(x - __half2float(hi));
  }
}

template <int D>
__global__ void __launch_bounds__(pa::kThreads, 1)
prefill_attn_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, int nb, int N, int Hg, float sqrt_d,
                    float* __restrict__ out, int ldo) {
  using namespace pa;
  using G = Geo<D>;
  extern __shared__ uint8_t pa_smem_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)pa_smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* qs = sm;                              // Q hi boxes | Q lo boxes
  uint8_t* ring = qs + G::kQBytes;               // [2] stages: K hi | K lo | V hi | V lo
  uint8_t* ps = ring + 2 * G::kStage;            // P hi | P lo (128 q x 64 keys each)
  uint64_t* bars = (uint64_t*)(ps + 2 * G::kPPart);
  uint64_t* qfull = bars;
  uint64_t* full = bars + 1;      // [2]
  uint64_t* empty = bars + 3;     // [2]
  uint64_t* sfull = bars + 5;     // [2] score buffers
  uint64_t* sfree = bars + 7;     // [2]
  uint64_t* pfull = bars + 9;
  uint64_t* pfree = bars + 10;
  uint64_t* ofull = bars + 11;
  uint32_t* tmem_sh = (uint32_t*)(bars + 12);
  // [2 halves][128 rows]: the row max after pass 1, then l at the end (the second
  // use cannot overtake a read of the first: every tile between waits for both halves)
  float* xch = (float*)(bars + 16);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqb = (N + BQ - 1) / BQ;
  const int qb = nqb - 1 - (int)blockIdx.x;      // heaviest blocks launch first
  const int h = blockIdx.y, b = blockIdx.z;
  const int q0 = qb * BQ;
  const int ntk = (N + BK - 1) / BK;
  const int T = min(ntk, (q0 + BQ - 1) / BK + 1);   // causal: key tiles up to the block's last query
  const int rowbase = (b * Hg + h) * N;             // first row of this (b, h) in the hl maps

  if (threadIdx.x == 0) {
    tc05::tma_prefetch_desc(&tmQ);
    tc05::tma_prefetch_desc(&tmK);
    tc05::tma_prefetch_desc(&tmV);
    tc05::mbar_init(qfull, 1);
    for (int s = 0; s < 2; ++s) {
      tc05::mbar_init(&full[s], 1);
      tc05::mbar_init(&empty[s], 1);
    }
    for (int s2 = 0; s2 < 2; ++s2) {
      tc05::mbar_init(&sfull[s2], 1);
      tc05::mbar_init(&sfree[s2], 256);
    }
    tc05::mbar_init(pfull, 256);
    tc05::mbar_init(pfree, 1);
    tc05::mbar_init(ofull, 1);
    tc05::fence_barrier_init();
  }
  if (warp == 1) tc05::tmem_alloc<kTmemCols>(tmem_sh);
  tc05::fence_before_sync();
  __syncthreads();
  tc05::fence_after_sync();
  const uint32_t tmem = *tmem_sh;

  if (warp == 0) {
    // ---------------------------------------------------------------- producer
    if (lane == 0) {
      tc05::mbar_expect_tx(qfull, G::kQBytes);
      for (int part = 0; part < 2; ++part)
        for (int bx = 0; bx < G::kBoxes; ++bx)
          tc05::tma_load_2d(qs + part * G::kQPart + bx * (BQ * 128), &tmQ, part * D + bx * 64, rowbase + q0, qfull);
      int seq = 0;
      for (int pass = 0; pass < 2; ++pass)
        for (int t = 0; t < T; ++t, ++seq) {
          const int stage = seq & 1;
          tc05::mbar_wait(&empty[stage], ((seq >> 1) & 1) ^ 1);
          uint8_t* st = ring + stage * G::kStage;
          tc05::mbar_expect_tx(&full[stage], pass == 0 ? G::kKBytes : G::kStage);
          const int row = rowbase + t * BK;
          for (int part = 0; part < 2; ++part)
            for (int bx = 0; bx < G::kBoxes; ++bx) {
              tc05::tma_load_2d(st + part * G::kKPart + bx * (BK * 128), &tmK, part * D + bx * 64, row, &full[stage]);
              if (pass == 1)
                tc05::tma_load_2d(st + G::kKBytes + part * G::kKPart + bx * (BK * 128), &tmV, part * D + bx * 64,
                                  row, &full[stage]);
            }
        }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    // tile sequence g = 0 .. 2T-1 (pass 0: g = t, pass 1: g = T + t); the score
    // MMAs run one tile ahead of the output MMAs (two TMEM score buffers)
    constexpr uint32_t idS = tc05::idesc_f16_f32(BQ, BK, 0, 0);
    constexpr uint32_t idO = tc05::idesc_f16_f32(BQ, D, 0, 1);
    tc05::mbar_wait(qfull, 0);
    tc05::fence_after_sync();
    const uint32_t qa = tc05::smem_u32(qs);
    const uint32_t pa_ = tc05::smem_u32(ps);
    const int total = 2 * T;
    auto scores = [&](int g) {
      const int stage = g & 1, sb = g & 1;
      tc05::mbar_wait(&full[stage], (g >> 1) & 1);
      if (g >= 2) tc05::mbar_wait(&sfree[sb], ((g - 2) >> 1) & 1);   // buffer's previous scores read
      tc05::fence_after_sync();
      const uint32_t kb = tc05::smem_u32(ring + stage * G::kStage);
      if (tc05::elect_one()) {
#pragma unroll
        for (int j = 0; j < D / 16; ++j) {
          const uint32_t ko = (j & 3) * 32;
          const uint32_t qh = qa + (j >> 2) * (BQ * 128) + ko, ql = qh + G::kQPart;
          const uint32_t kh = kb + (j >> 2) * (BK * 128) + ko, kl = kh + G::kKPart;
          const uint32_t d_s = tmem + 64 * sb;
          tc05::mma_f16(d_s, tc05::desc_kmajor_sw128(qh), tc05::desc_kmajor_sw128(kh), idS, j > 0 ? 1u : 0u);
          tc05::mma_f16(d_s, tc05::desc_kmajor_sw128(qh), tc05::desc_kmajor_sw128(kl), idS, 1u);
          tc05::mma_f16(d_s, tc05::desc_kmajor_sw128(ql), tc05::desc_kmajor_sw128(kh), idS, 1u);
        }
        tc05::mma_commit(&sfull[sb]);
        if (g < T) tc05::mma_commit(&empty[stage]);            // pass 0: only K was needed
      }
      __syncwarp();
    };
    auto outputs = [&](int g) {                                 // pass 1 tile t = g - T
      const int t = g - T, stage = g & 1;
      tc05::mbar_wait(pfull, t & 1);
      tc05::fence_after_sync();
      const uint32_t vb = tc05::smem_u32(ring + stage * G::kStage) + G::kKBytes;
      if (tc05::elect_one()) {
#pragma unroll
        for (int j = 0; j < BK / 16; ++j) {
          const uint32_t ph = pa_ + j * 32, pl = ph + G::kPPart;
          const uint32_t vh = vb + j * 2048, vl = vh + G::kKPart;
          const uint32_t acc = (t > 0 || j > 0) ? 1u : 0u;
          tc05::mma_f16(tmem + 128, tc05::desc_kmajor_sw128(ph), tc05::desc_mnmajor_sw128(vh, BK * 128), idO, acc);
          tc05::mma_f16(tmem + 256, tc05::desc_kmajor_sw128(ph), tc05::desc_mnmajor_sw128(vl, BK * 128), idO, acc);
          tc05::mma_f16(tmem + 256, tc05::desc_kmajor_sw128(pl), tc05::desc_mnmajor_sw128(vh, BK * 128), idO, 1u);
        }
        tc05::mma_commit(&empty[stage]);
        tc05::mma_commit(pfree);
        if (t == T - 1) tc05::mma_commit(ofull);
      }
      __syncwarp();
    };
    scores(0);
    for (int g = 0; g < total; ++g) {
      if (g + 1 < total) scores(g + 1);
      if (g >= T) outputs(g);
    }
  } else {
    // ---------------------------------------------------------------- softmax / epilogue
    // warps 2-9: lane quarter q4 = warp % 4, column half (32 of the 64 keys of a
    // tile, D / 2 output columns); the two halves of a row combine m once (after
    // pass 1) and l once (at the end) through shared memory
    const int q4 = warp & 3, half = (warp - 2) >> 2;
    const int r = q4 * 32 + lane;                // query row of the block (TMEM lane)
    const int qi = q0 + r;
    const uint32_t lanebase = tmem + ((uint32_t)(q4 * 32) << 16);
    constexpr int HK = BK / 2;
    float m = -INFINITY, l = 0.f;
    int sc = 0;
    for (int pass = 0; pass < 2; ++pass) {
      if (pass == 1) {                           // the row max over both halves
        xch[half * 128 + r] = m;
        asm volatile("bar.sync 1, 256;" ::: "memory");
        m = fmaxf(m, xch[(half ^ 1) * 128 + r]);
      }
      for (int t = 0; t < T; ++t) {
        const int sb = sc & 1;
        tc05::mbar_wait(&sfull[sb], (sc >> 1) & 1);
        tc05::fence_after_sync();
        float s[HK];
        {
          uint32_t v[32];
          tc05::tmem_ld32(lanebase + 64 * sb + half * HK, v);
          tc05::tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < HK; ++j) {
            const int key = t * BK + half * HK + j;
            s[j] = (key <= qi && key < N) ? __uint_as_float(v[j]) / sqrt_d : -INFINITY;
          }
        }
        tc05::fence_before_sync();
        tc05::mbar_arrive(&sfree[sb]);
        ++sc;
        if (pass == 0) {
#pragma unroll
          for (int j = 0; j < HK; ++j) m = fmaxf(m, s[j]);
          continue;
        }
        if (t > 0) tc05::mbar_wait(pfree, (t - 1) & 1);        // the previous tile's output MMAs read P
        // p = exp(s - m), split, into row r of the K-major P tiles (128-B swizzle)
        uint8_t* prow_h = ps + (r >> 3) * 1024 + (r & 7) * 128;
        uint8_t* prow_l = prow_h + G::kPPart;
#pragma unroll
        for (int cc = 0; cc < HK / 8; ++cc) {
          const int c = half * (HK / 8) + cc;
          uint32_t hw[4], lw[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float s0 = s[cc * 8 + 2 * u], s1 = s[cc * 8 + 2 * u + 1];
            const float p0 = s0 == -INFINITY ? 0.f : expf(s0 - m);
            const float p1 = s1 == -INFINITY ? 0.f : expf(s1 - m);
            l += p0 + p1;
            const __half2 hh = __floats2half2_rn(p0, p1);
            const float2 hf = __half22float2(hh);
            const __half2 ll = __floats2half2_rn(p0 - hf.x, p1 - hf.y);
            hw[u] = *reinterpret_cast<const uint32_t*>(&hh);
            lw[u] = *reinterpret_cast<const uint32_t*>(&ll);
          }
          const int chunk = (c ^ (r & 7)) * 16;
          *reinterpret_cast<uint4*>(prow_h + chunk) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
          *reinterpret_cast<uint4*>(prow_l + chunk) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
        }
        tc05::fence_proxy_async_smem();
        tc05::mbar_arrive(pfull);
      }
    }
    // ---- output: (O main + O cross) / l, l summed over both halves
    xch[half * 128 + r] = l;
    asm volatile("bar.sync 1, 256;" ::: "memory");
    l += xch[(half ^ 1) * 128 + r];
    tc05::mbar_wait(ofull, 0);
    tc05::fence_after_sync();
    const bool live = qi < N;
    float* orow = out + ((size_t)b * N + (live ? qi : 0)) * ldo + (size_t)h * D;
    const float inv = 1.f / l;
#pragma unroll 1
    for (int c0 = half * (D / 2); c0 < (half + 1) * (D / 2); c0 += 32) {
      uint32_t vm[32], vc[32];
      tc05::tmem_ld32(lanebase + 128 + c0, vm);
      tc05::tmem_ld32(lanebase + 256 + c0, vc);
      tc05::tmem_ld_wait();
      if (live) {
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          float4 o;
          o.x = (__uint_as_float(vm[j]) + __uint_as_float(vc[j])) * inv;
          o.y = (__uint_as_float(vm[j + 1]) + __uint_as_float(vc[j + 1])) * inv;
          o.z = (__uint_as_float(vm[j + 2]) + __uint_as_float(vc[j + 2])) * inv;
          o.w = (__uint_as_float(vm[j + 3]) + __uint_as_float(vc[j + 3])) * inv;
          *reinterpret_cast<float4*>(orow + c0 + j) = o;
        }
      }
    }
    tc05::fence_before_sync();
  }
  __syncthreads();
  if (warp == 1) {
    tc05::fence_after_sync();
    tc05::tmem_dealloc<kTmemCols>(tmem);
  }
}

}  // namespace ig

extern "C" int ig_prefill_attention_scratch(int nb, int N, int Hg, int d, size_t* bytes) {
  if (!bytes || nb < 1 || N < 1 || Hg < 1 || (d != 64 && d != 128)) return IG_EINVAL;
  *bytes = (size_t)3 * nb * Hg * N * 2 * d * 2;
  return IG_OK;
}

extern "C" int ig_prefill_attention(const float* qkv, int ldqkv, int nb, int N, int Hg, int d, void* work,
                                    float* out, int ldo, void* stream) {
  using namespace ig;
  if (!qkv || !work || !out || nb < 1 || N < 1 || Hg < 1 || (d != 64 && d != 128) || ldqkv < 3 * Hg * d ||
      ldo < Hg * d || (ldo & 3) || ((uintptr_t)out & 15) || ((uintptr_t)work & 15))
    return IG_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t rows = (size_t)3 * nb * Hg * N;
  split_qkv_kernel<<<(unsigned)((rows * 32 + 255) / 256), 256, 0, s>>>(qkv, ldqkv, nb, N, Hg, d, (__half*)work);
  IG_LAUNCH_STATUS();
  const size_t part_rows = (size_t)nb * Hg * N;
  const __half* qhl = (const __half*)work;
  const __half* khl = qhl + part_rows * 2 * d;
  const __half* vhl = khl + part_rows * 2 * d;
  CUtensorMap mq, mk, mv;
  int rc = make_tmap_2d(&mq, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, qhl, (uint64_t)2 * d, part_rows, (uint64_t)4 * d, 64,
                        pa::BQ, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  rc = make_tmap_2d(&mk, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, khl, (uint64_t)2 * d, part_rows, (uint64_t)4 * d, 64, pa::BK,
                    CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  rc = make_tmap_2d(&mv, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, vhl, (uint64_t)2 * d, part_rows, (uint64_t)4 * d, 64, pa::BK,
                    CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  const float sqrt_d = (float)sqrt((double)d);      // float32(np.sqrt(d)), model.py:174
  const dim3 grid((N + pa::BQ - 1) / pa::BQ, Hg, nb);
  if (d == 128) {
    const size_t smem = pa::Geo<128>::kSmem;
    IG_CUDA_STATUS(cudaFuncSetAttribute(prefill_attn_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)smem));
    prefill_attn_kernel<128><<<grid, pa::kThreads, smem, s>>>(mq, mk, mv, nb, N, Hg, sqrt_d, out, ldo);
  } else {
    const size_t smem = pa::Geo<64>::kSmem;
    IG_CUDA_STATUS(cudaFuncSetAttribute(prefill_attn_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)smem));
    prefill_attn_kernel<64><<<grid, pa::kThreads, smem, s>>>(mq, mk, mv, nb, N, Hg, sqrt_d, out, ldo);
  }
  IG_LAUNCH_STATUS();
  return IG_OK;
}
