// K4 sparse decode attention on the 5th-generation tensor cores: the
// reference attention_head (model.py:156-180) over the fetch set of
// engine.py:382-418 (selected / slot-table rows + the GPU-resident current
// row), as called at engine.py:352-358.
//
// Data: the staged rows of (b, h) are rows [0, rows_bh) of
// stage[(b Hg + h) cap + r][2d] (K row then V row, 2-byte elements, d = 128),
// row id = idx ? idx[bh cap + r] : r; a row counts if id >= 0 and id != pos.
//
// Work split (stream-K over rows): every (b, h) is cut into 128-row tiles
// (>= 1, so an empty set still yields its current-row output); the tiles of all
// (b, h) are laid end to end and CTA c of the persistent grid (one per SM) takes
// tiles [c T / G, (c+1) T / G).  Its items are the runs of its tiles inside one
// (b, h).  An item covering a whole (b, h) writes the output directly;
// otherwise it writes (m, l, o[d]) to a per-(b, h) slot and the item that
// completes the (b, h)'s tile count merges the slots in tile order
// (deterministic).
//
// Per 128-row tile (whole 512-B rows, one 64-KB ring stage, four 128-B-swizzled
// TMA boxes), warp-specialised and mbarrier-synchronised:
//  * warp 0 (one thread): TMA producer (3-stage ring);
//  * warp 1 (one thread): tcgen05.mma issuer, polling both of its queues and
//    issuing whichever is ready: scores S^T = K_tile (128 x 128, K-major) .
//    [q parts] (N = 16, K-major) as soon as a tile lands, outputs
//    O_t^T = V_tile^T (MN-major: d contiguous) . P_t (N = 16) as soon as the
//    tile's p operand is written -- which releases the stage.  Rows past the
//    row count in an item's last tile are zeroed in shared memory first
//    (0 x NaN must not reach O);
//  * warps 2-5 (128 threads, TMEM lane = tile row): the softmax of tile t per
//    WARP -- each warp's 32 rows take their own max m_w and sum l_w (warp
//    shuffles only) and write their p parts into rows [NS w, NS w + NS) of the
//    P operand (zero elsewhere), so ONE MMA yields the four warps' partial
//    outputs in separate accumulator columns; two tiles later (4-deep TMEM /
//    P rings, so a softmax never waits behind a readout) the tile's four
//    (m_w, l_w, o_w) fold, lane = d index, into the item's running (M, L, acc);
//  * warp 6: q rows -> power-of-two scaled exact split operand tiles, a ring
//    of 4 running ahead of the score MMAs.
// Scores are (q . k) / float32(sqrt(d)) -- a division, model.py:174 -- and
// exp is expf.  f16 pools split q and p in two f16 parts (22 significand bits),
// bf16 pools in three bf16 parts (24 bits); K/V elements are exact in the
// operand type, every product is exact, accumulation is f32.
#include <cuda.h>

#include "common.cuh"
#include "tc05.cuh"

namespace ig {

namespace a5 {
constexpr int kRows = 128;                     // rows per tile (UMMA M)
constexpr int kStages = 3;
constexpr uint32_t kBox = 128 * 128;           // 128 rows x 64 elements x 2 B
constexpr uint32_t kStage = 4 * kBox;          // K0 K1 V0 V1: 128 whole rows
constexpr uint32_t kOpTile = 16 * 128 * 2;     // B operand: 16 rows x 128 K x 2 B
constexpr int kQBufs = 2;                      // q operand ring (the q warp runs ahead)
constexpr int kSBufs = 4;                      // score / output TMEM buffers, P operand tiles
constexpr int kMeta = 8;                       // per-tile row-validity masks (the q warp runs ahead)
constexpr int kThreads = 352;                  // producer, MMA, 4 softmax, 4 readout, q/metadata warp
constexpr int kMaxBH = 2048;
constexpr uint32_t kTmemCols = 128;            // S[4] x 16 + O[4] x 16
constexpr size_t kFixedSmem = 1024 + kStages * kStage + kQBufs * kOpTile + kSBufs * kOpTile + 1024;
}  // namespace a5

template <typename T> struct A5T;
template <> struct A5T<__half> {
  static constexpr int NS = 2, BF = 0;
  __device__ static float rnd(float x) { return __half2float(__float2half_rn(x)); }
  __device__ static uint16_t bits(float x) { return __half_as_ushort(__float2half_rn(x)); }
};
template <> struct A5T<__nv_bfloat16> {
  static constexpr int NS = 3, BF = 1;
  __device__ static float rnd(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }
  __device__ static uint16_t bits(float x) { return __bfloat16_as_ushort(__float2bfloat16_rn(x)); }
};

// byte offset of element (n, k) in a K-major 128-B-swizzled [16][128] operand tile
__device__ __forceinline__ uint32_t a5_op_off(int n, int k) {
  const int atom = k >> 6, kin = k & 63;
  return atom * 2048 + (n >> 3) * 1024 + (n & 7) * 128 + ((((kin >> 3) ^ (n & 7)) & 7) << 4) + (kin & 7) * 2;
}

__device__ __forceinline__ int a5_rows(const int32_t* rows_bh, const int32_t* n_in, const ig_step_state* st,
                                       int b, int bh, int cap) {
  const int r = rows_bh ? rows_bh[bh] : (n_in ? n_in[b] : st->s_len);
  return max(0, min(r, cap));
}

// Optional timeline (tools/attend_trace.py): when set, every CTA records
// globaltimer stamps per role and tile: [cta][kTrStride] u64.
__device__ unsigned long long* a5_trace = nullptr;
constexpr int kTrTiles = 64, kTrStride = 8 + 9 * kTrTiles;
__device__ __forceinline__ unsigned long long a5_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void a5_mark(int ev, int seq) {
  unsigned long long* tb = a5_trace;
  if (tb && seq < kTrTiles) tb[(size_t)blockIdx.x * kTrStride + 8 + ev * kTrTiles + seq] = a5_now();
}
__device__ __forceinline__ void a5_mark_cta(int slot) {
  unsigned long long* tb = a5_trace;
  if (tb) tb[(size_t)blockIdx.x * kTrStride + slot] = a5_now();
}

struct A5Tile {
  int bh, t;          // (b, h) and tile index within it
  int item;           // item ordinal within this CTA
  int t0, nt;         // the item's first tile and tile count
  int seq;            // tile ordinal within this CTA (ring / buffer parity)
  bool first, last;   // first / last tile of its item
};

struct A5Sched {
  const int* prefix;
  int BH, G;
  long long TT, g, g1;
  // tile iterator state
  int bh_, t0_, nt_, k_, item_, seq_;
  bool have_;
  __device__ void init(const int* p, int bh_count, int c, int grid) {
    prefix = p;
    BH = bh_count;
    G = grid;
    TT = p[bh_count];
    g = (long long)c * TT / G;
    g1 = (long long)(c + 1) * TT / G;
    have_ = false;
    k_ = 0;
    item_ = -1;
    seq_ = 0;
  }
  __device__ bool next_item(int& bh, int& t0, int& nt) {
    if (g >= g1) return false;
    int lo = 0, hi = BH - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (prefix[mid] <= g) lo = mid;
      else hi = mid - 1;
    }
    bh = lo;
    t0 = (int)(g - prefix[bh]);
    const int tiles = prefix[bh + 1] - prefix[bh];
    nt = (int)min((long long)(tiles - t0), g1 - g);
    g += nt;
    return true;
  }
  __device__ bool next(A5Tile& x) {
    if (!have_ || k_ >= nt_) {
      if (!next_item(bh_, t0_, nt_)) return false;
      have_ = true;
      k_ = 0;
      ++item_;
    }
    x.bh = bh_;
    x.t = t0_ + k_;
    x.item = item_;
    x.t0 = t0_;
    x.nt = nt_;
    x.seq = seq_++;
    x.first = k_ == 0;
    x.last = k_ == nt_ - 1;
    ++k_;
    return true;
  }
  __device__ bool range_start(long long gg) const {     // some CTA's range starts at gg
    const long long c = (gg * G + TT - 1) / TT;
    return c < G && c * TT / G == gg;
  }
  __device__ bool item_start(int bh, int t) const {
    return t == 0 || range_start((long long)prefix[bh] + t);
  }
};

// 128-thread (readout warps, named barrier 2) block sum, fixed order
__device__ __forceinline__ float a5_bsum(float v, float* red) {
  v = warp_sum(v);
  const int w = (threadIdx.x >> 5) & 3;
  asm volatile("bar.sync 2, 128;" ::: "memory");
  if ((threadIdx.x & 31) == 0) red[4 + w] = v;
  asm volatile("bar.sync 2, 128;" ::: "memory");
  return ((red[4] + red[5]) + red[6]) + red[7];
}

template <typename T>
__global__ void __launch_bounds__(a5::kThreads, 1)
attend_tc05_kernel(const __grid_constant__ CUtensorMap tm, const float* __restrict__ q, int ldq,
                   const float* __restrict__ k_cur, const float* __restrict__ v_cur, int ldkv,
                   const int32_t* __restrict__ idx, const int32_t* __restrict__ n_in,
                   const int32_t* __restrict__ rows_bh, const int32_t* __restrict__ pos_in,
                   const ig_step_state* __restrict__ st, int B, int Hg, int cap, float sqrt_d, int max_chunks,
                   float* __restrict__ partial, int32_t* __restrict__ tickets, float* __restrict__ out, int ldo) {
  using namespace a5;
  constexpr int d = 128, NS = A5T<T>::NS;
  extern __shared__ uint8_t a5_smem_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)a5_smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* ring = sm;
  uint8_t* qt = ring + kStages * kStage;          // [kQBufs] q operand tiles
  uint8_t* pt = qt + kQBufs * kOpTile;            // [kSBufs] p operand tiles
  uint64_t* full = (uint64_t*)(pt + kSBufs * kOpTile);
  uint64_t* empty = full + kStages;
  uint64_t* qfull = empty + kStages;     // [kQBufs]
  uint64_t* qempty = qfull + kQBufs;     // [kQBufs]
  uint64_t* sfull = qempty + kQBufs;     // [kSBufs]
  uint64_t* ofull = sfull + kSBufs;      // [kSBufs]
  uint64_t* pfull = ofull + kSBufs;      // [kSBufs]
  uint64_t* oempty = pfull + kSBufs;     // [kSBufs]
  uint64_t* mfull = oempty + kSBufs;     // [kMeta]
  uint64_t* mempty = mfull + kMeta;      // [kMeta]
  uint32_t* tmem_sh = (uint32_t*)(mempty + kMeta);
  int* flag_sh = (int*)(tmem_sh + 1);
  float* red = (float*)(tmem_sh + 4);    // [8]
  float* qinv_sh = red + 8;              // [8] per item (mod 8) q scale
  // [16] per item (mod 16) current-row score: the q warp runs <= 8 tiles ahead
  // of the softmax, which runs <= 4 tiles ahead of the readout
  float* scur_sh = red + 16;
  // [4][2][4] per tile (seq mod 4: a warp may run one tile's softmax ahead of
  // another warp's readout two tiles back): m_w, l_w
  float* ml_sh = red + 32;
  uint32_t* meta = (uint32_t*)(ml_sh + 32);   // [kMeta][8]: valid-row mask [4], rows in the tile
  int* nrows_sh = (int*)(meta + kMeta * 8);   // [kSBufs] rows in the tile, for the output MMA
  int* prefix = nrows_sh + kSBufs;            // [BH + 1]
  const int BH = B * Hg;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  pdl_trigger();
  if (threadIdx.x == 0) a5_mark_cta(0);

  // tiles per (b, h), then an exclusive scan (warp 0); P tiles zeroed (rows a
  // warp does not own stay zero for the whole kernel)
  for (int i = threadIdx.x; i < BH; i += blockDim.x)
    prefix[i] = max(1, (a5_rows(rows_bh, n_in, st, i / Hg, i, cap) + kRows - 1) / kRows);
  for (int i = threadIdx.x; i < (int)(kSBufs * kOpTile / 16); i += blockDim.x)
    ((uint4*)pt)[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  if (warp == 0) {
    int run = 0;
    for (int base = 0; base < BH; base += 32) {
      const int i = base + lane;
      const int v = i < BH ? prefix[i] : 0;
      int x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (i < BH) prefix[i] = run + x - v;
      run += __shfl_sync(0xffffffffu, x, 31);
    }
    if (lane == 0) {
      prefix[BH] = run;
      tc05::tma_prefetch_desc(&tm);
      for (int s2 = 0; s2 < kStages; ++s2) {
        tc05::mbar_init(&full[s2], 1);
        tc05::mbar_init(&empty[s2], 1);
      }
      for (int b2 = 0; b2 < kQBufs; ++b2) {
        tc05::mbar_init(&qfull[b2], 32);
        tc05::mbar_init(&qempty[b2], 1);
      }
      for (int b2 = 0; b2 < kSBufs; ++b2) {
        tc05::mbar_init(&sfull[b2], 1);
        tc05::mbar_init(&ofull[b2], 1);
        tc05::mbar_init(&pfull[b2], 128);
        tc05::mbar_init(&oempty[b2], 128);
      }
      for (int b2 = 0; b2 < kMeta; ++b2) {
        tc05::mbar_init(&mfull[b2], 32);
        tc05::mbar_init(&mempty[b2], 4);
      }
      tc05::fence_barrier_init();
    }
  }
  if (warp == 1) tc05::tmem_alloc<kTmemCols>(tmem_sh);
  tc05::fence_proxy_async_smem();     // the zeroed P tiles, for the MMAs
  tc05::fence_before_sync();
  __syncthreads();
  tc05::fence_after_sync();
  const uint32_t tmem = *tmem_sh;      // S[j] at 16 j, O[j] at 64 + 16 j (j = seq mod 4)

  A5Sched sc;
  sc.init(prefix, BH, blockIdx.x, gridDim.x);
  if (threadIdx.x == 0) a5_mark_cta(1);

  if (warp == 0) {
    // ---------------------------------------------------------------- producer
    if (lane == 0) {
      A5Tile x;
      while (sc.next(x)) {
        const int stage = x.seq % kStages;
        tc05::mbar_wait(&empty[stage], ((x.seq / kStages) & 1) ^ 1);
        a5_mark(0, x.seq);
        tc05::mbar_expect_tx(&full[stage], kStage);
        const int row = x.bh * cap + x.t * kRows;
        uint8_t* dst = ring + stage * kStage;
#pragma unroll
        for (int bx = 0; bx < 4; ++bx) tc05::tma_load_2d(dst + bx * kBox, &tm, bx * 64, row, &full[stage]);
      }
      a5_mark_cta(3);
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    constexpr uint32_t idS = tc05::idesc_f16_f32(128, 16, 0, 0, A5T<T>::BF);
    constexpr uint32_t idP = tc05::idesc_f16_f32(128, 16, 1, 0, A5T<T>::BF);
    // two cursors over the same tile stream: scores (as tiles land), outputs
    // (as p operands are written); S(t) always precedes O(t)
    A5Sched scp = sc;
    A5Tile xs, xo;
    bool hs = sc.next(xs), ho = scp.next(xo);
    while (ho) {
      bool did = false;
      if (hs) {
        const int qb_i = xs.item % kQBufs, stage = xs.seq % kStages, sb = xs.seq % kSBufs;
        if ((!xs.first || tc05::mbar_test(&qfull[qb_i], (xs.item / kQBufs) & 1)) &&
            tc05::mbar_test(&full[stage], (xs.seq / kStages) & 1)) {
          tc05::fence_after_sync();
          if (lane == 0) a5_mark(1, xs.seq);
          if (tc05::elect_one()) {
            const uint32_t base = tc05::smem_u32(ring + stage * kStage);
            const uint32_t qb = tc05::smem_u32(qt + qb_i * kOpTile);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const uint64_t a = tc05::desc_kmajor_sw128(base + (j >> 2) * kBox + (j & 3) * 32);
              const uint64_t bq = tc05::desc_kmajor_sw128(qb + (j >> 2) * 2048 + (j & 3) * 32);
              tc05::mma_f16(tmem + 16 * sb, a, bq, idS, j > 0 ? 1u : 0u);
            }
            tc05::mma_commit(&sfull[sb]);
            if (xs.last) tc05::mma_commit(&qempty[qb_i]);
          }
          __syncwarp();
          hs = sc.next(xs);
          did = true;
        }
      }
      if (xo.seq < (hs ? xs.seq : 0x7fffffff)) {
        const int stage = xo.seq % kStages, sb = xo.seq % kSBufs;
        if (tc05::mbar_test(&pfull[sb], (xo.seq / kSBufs) & 1)) {
          if (lane == 0) a5_mark(2, xo.seq);
          {
            const int valid = nrows_sh[sb];              // rows of this tile below the count
            if (valid < kRows) {
              // zero the V rows past the row count (masked, but 0 x NaN = NaN)
              uint8_t* vbase = ring + stage * kStage + 2 * kBox;
              const int r0 = max(0, valid);
              const int chunks = (kRows - r0) * 8;         // 16-B chunks per box
              for (int c = lane; c < 2 * chunks; c += 32) {
                const int box = c / chunks, cc = c - box * chunks;
                *(uint4*)(vbase + box * kBox + (size_t)(r0 + cc / 8) * 128 + (cc & 7) * 16) = make_uint4(0, 0, 0, 0);
              }
              tc05::fence_proxy_async_smem();
              __syncwarp();
            }
          }
          tc05::fence_after_sync();
          if (tc05::elect_one()) {
            const uint32_t base = tc05::smem_u32(ring + stage * kStage) + 2 * kBox;
            const uint32_t pb = tc05::smem_u32(pt + sb * kOpTile);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const uint64_t a = tc05::desc_mnmajor_sw128(base + j * 2048, kBox);
              const uint64_t bp = tc05::desc_kmajor_sw128(pb + (j >> 2) * 2048 + (j & 3) * 32);
              tc05::mma_f16(tmem + 64 + 16 * sb, a, bp, idP, j > 0 ? 1u : 0u);
            }
            tc05::mma_commit(&empty[stage]);
            tc05::mma_commit(&ofull[sb]);
          }
          __syncwarp();
          ho = scp.next(xo);
          did = true;
        }
      }
      if (!did) __nanosleep(20);
    }
    if (lane == 0) a5_mark_cta(4);
  } else if (warp == 10) {
    // ---------------------------------------------------------------- q warp
    // per item: its q row -> power-of-two scaled exact split operand tile;
    // per tile: the 128-bit valid-row mask (row < count, id >= 0, id != pos)
    // and the row count -- all global reads of the path's metadata happen
    // here, up to kMeta tiles ahead of the softmax warps
    A5Tile x;
    int rows = 0, pos = 0;
    while (sc.next(x)) {
      const int b = x.bh / Hg, h = x.bh - b * Hg;
      if (x.first) {
        const int i = x.item;
        const int qb_i = i % kQBufs;
        rows = a5_rows(rows_bh, n_in, st, b, x.bh, cap);
        pos = pos_in ? pos_in[x.bh] : st->s_len;
        tc05::mbar_wait(&qempty[qb_i], ((i / kQBufs) & 1) ^ 1);
        const float4 qv = *(const float4*)(q + (size_t)b * ldq + (size_t)h * d + lane * 4);
        float amax = fmaxf(fmaxf(fabsf(qv.x), fabsf(qv.y)), fmaxf(fabsf(qv.z), fabsf(qv.w)));
        amax = warp_max(amax);
        float s2 = 1.f, inv = 1.f;
        if (amax > 0.f && isfinite(amax)) {
          int e;
          frexpf(amax, &e);
          s2 = ldexpf(1.f, 14 - e);
          inv = ldexpf(1.f, e - 14);
        }
        uint8_t* tile = qt + qb_i * kOpTile;
        const float xs[4] = {qv.x * s2, qv.y * s2, qv.z * s2, qv.w * s2};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          float rem = xs[u];
#pragma unroll
          for (int n = 0; n < NS; ++n) {
            const float part = A5T<T>::rnd(rem);
            *(uint16_t*)(tile + a5_op_off(n, lane * 4 + u)) = A5T<T>::bits(part);
            rem -= part;
          }
        }
        // the current token's score: f32 dot with the GPU-resident k row (its
        // row is not in the staged set), consumed by the readout at the item end
        const float4 kv = *(const float4*)(k_cur + (size_t)b * ldkv + (size_t)h * d + lane * 4);
        const float dotc = warp_sum(((qv.x * kv.x + qv.y * kv.y) + qv.z * kv.z) + qv.w * kv.w);
        if (lane == 0) {
          qinv_sh[i & 7] = inv;
          scur_sh[i & 15] = dotc / sqrt_d;
        }
        tc05::fence_proxy_async_smem();
        tc05::mbar_arrive(&qfull[qb_i]);
      }
      const int slot = x.seq % kMeta;
      int ids[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int rr = x.t * kRows + k * 32 + lane;
        ids[k] = rr < rows ? (idx ? idx[(size_t)x.bh * cap + rr] : rr) : -1;
      }
      tc05::mbar_wait(&mempty[slot], ((x.seq / kMeta) & 1) ^ 1);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t m = __ballot_sync(0xffffffffu, ids[k] >= 0 && ids[k] != pos);
        if (lane == 0) meta[slot * 8 + k] = m;
      }
      if (lane == 0) meta[slot * 8 + 4] = (uint32_t)max(0, min(kRows, rows - x.t * kRows));
      __syncwarp();
      tc05::mbar_arrive(&mfull[slot]);
    }
    if (lane == 0) a5_mark_cta(5);
  } else {
    // ---------------------------------------------------------------- softmax (warps 2-5) / readout (6-9)
    const int q4 = warp & 3;
    const int r = q4 * 32 + lane;                 // TMEM lane: tile row / d index
    const uint32_t lanebase = tmem + ((uint32_t)(q4 * 32) << 16);
    // softmax of tile x: per-warp max / sum, p parts -> rows [NS q4, NS q4 + NS)
    auto softmax = [&](const A5Tile& x) {
      const int par = x.seq % kSBufs;
      const int slot = x.seq % kMeta;
      tc05::mbar_wait(&mfull[slot], (x.seq / kMeta) & 1);
      const bool valid = (meta[slot * 8 + q4] >> lane) & 1u;
      const int nrows = (int)meta[slot * 8 + 4];
      __syncwarp();
      if (lane == 0) tc05::mbar_arrive(&mempty[slot]);
      tc05::mbar_wait(&sfull[par], (x.seq / kSBufs) & 1);
      tc05::fence_after_sync();
      if (r == 0) a5_mark(3, x.seq);
      // the readout of tile seq - kSBufs has released this P tile / ml slot / O buffer
      if (x.seq >= kSBufs) tc05::mbar_wait(&oempty[par], ((x.seq / kSBufs) - 1) & 1);
      uint32_t v[4];
      tc05::tmem_ld4(lanebase + 16 * par, v);
      tc05::tmem_ld_wait();
      float dot = __uint_as_float(v[0]) + __uint_as_float(v[1]);
      if (NS > 2) dot += __uint_as_float(v[2]);
      const float sc_ = valid ? (dot * qinv_sh[x.item & 7]) / sqrt_d : -INFINITY;
      const float mw = warp_max(sc_);
      const float p = sc_ == -INFINITY ? 0.f : expf(sc_ - mw);
      const float lw = warp_sum(p);
      uint8_t* tile = pt + par * kOpTile;
      float rem = p;
#pragma unroll
      for (int n = 0; n < NS; ++n) {
        const float part = A5T<T>::rnd(rem);
        *(uint16_t*)(tile + a5_op_off(NS * q4 + n, r)) = A5T<T>::bits(part);
        rem -= part;
      }
      if (lane == 0) {
        ml_sh[(x.seq & 3) * 8 + q4] = mw;
        ml_sh[(x.seq & 3) * 8 + 4 + q4] = lw;
      }
      if (r == 0) nrows_sh[par] = nrows;
      tc05::fence_before_sync();
      tc05::fence_proxy_async_smem();
      tc05::mbar_arrive(&pfull[par]);
      if (r == 0) a5_mark(4, x.seq);
    };
    float M = -INFINITY, L = 0.f, acc = 0.f;     // running state of the readout item
    float vc_i = 0.f;                            // current v row of the readout item (d = r)
    auto readout = [&](const A5Tile& x) {
      const int par = x.seq % kSBufs;
      if (r == 0) a5_mark(6, x.seq);
      const int b = x.bh / Hg, h = x.bh - b * Hg;
      if (x.first) {
        M = -INFINITY;
        L = 0.f;
        acc = 0.f;
        vc_i = v_cur[(size_t)b * ldkv + (size_t)h * d + r];
      }
      tc05::mbar_wait(&ofull[par], (x.seq / kSBufs) & 1);
      tc05::fence_after_sync();
      if (r == 0) a5_mark(7, x.seq);
      uint32_t v[16];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
          : "r"(lanebase + 64 + 16 * par));
      tc05::tmem_ld_wait();
      tc05::fence_before_sync();
      if (r == 0) a5_mark(8, x.seq);
      // the four softmax warps' m_w / l_w of this tile (written before pfull, which
      // the output MMA, and hence ofull, follows)
      const float* ml = ml_sh + (x.seq & 3) * 8;
      float mlv[8];
#pragma unroll
      for (int w = 0; w < 8; ++w) mlv[w] = ml[w];
      tc05::mbar_arrive(&oempty[par]);
      float mt = -INFINITY;
#pragma unroll
      for (int w = 0; w < 4; ++w) mt = fmaxf(mt, mlv[w]);
      if (mt != -INFINITY) {
        const float Mn = fmaxf(M, mt);
        const float so = M == -INFINITY ? 0.f : expf(M - Mn);
        float a2 = acc * so, l2 = L * so;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const float mw = mlv[w];
          const float sw = mw == -INFINITY ? 0.f : expf(mw - Mn);
          float ow = __uint_as_float(v[NS * w]) + __uint_as_float(v[NS * w + 1]);
          if (NS > 2) ow += __uint_as_float(v[NS * w + 2]);
          a2 += ow * sw;
          l2 += mlv[4 + w] * sw;
        }
        acc = a2;
        L = l2;
        M = Mn;
      }
      if (r == 0) a5_mark(5, x.seq);
      if (!x.last) return;
      // ---- end of the item
      const int tiles_bh = prefix[x.bh + 1] - prefix[x.bh];
      bool finalize = x.nt == tiles_bh;
      float* pbase = partial + (size_t)x.bh * max_chunks * (d + 2);
      if (!finalize) {
        float* part = pbase + (size_t)x.t0 * (d + 2);
        part[2 + r] = acc;
        if (r == 0) { part[0] = M; part[1] = L; }
        __threadfence();
        asm volatile("bar.sync 2, 128;" ::: "memory");
        if (r == 0) *flag_sh = atomicAdd(tickets + x.bh, x.nt) + x.nt == tiles_bh;
        asm volatile("bar.sync 2, 128;" ::: "memory");
        finalize = *flag_sh != 0;
        if (finalize) __threadfence();
      }
      if (!finalize) return;
      const float vc = vc_i;
      const float scur = scur_sh[x.item & 15];  // written by the q warp before qfull(item)
      float Mf = scur, Lf = 0.f, Of = 0.f;
      if (x.nt == tiles_bh) {
        Mf = fmaxf(Mf, M);
        const float w = M == -INFINITY ? 0.f : expf(M - Mf);
        Lf = L * w;
        Of = acc * w;
      } else {
        // the (b, h)'s items start at tile 0 and at every CTA range start inside
        // it: walk the ranges (a handful of 64-bit divisions, not one per tile --
        // that walk cost ~30 us at C4's 52-tile row sets)
        const long long g0 = prefix[x.bh], g1 = prefix[x.bh + 1];
        const long long c0 = (g0 * sc.G + sc.TT - 1) / sc.TT;     // first range start >= g0
        for (int pass = 0; pass < 2; ++pass) {
          long long prev = -1;
          for (long long c = c0 - 1; c < sc.G; ++c) {
            const long long gs = c < c0 ? g0 : c * sc.TT / sc.G;  // item start (global tile)
            if (gs == prev) continue;        // tile 0 again, or empty ranges (grid > tiles)
            if (gs >= g1) break;
            prev = gs;
            const float* ps = pbase + (size_t)(gs - g0) * (d + 2);
            if (pass == 0) {
              Mf = fmaxf(Mf, __ldcg(ps));
            } else {
              const float mi = __ldcg(ps);
              const float w = mi == -INFINITY ? 0.f : expf(mi - Mf);
              Lf += __ldcg(ps + 1) * w;
              Of += __ldcg(ps + 2 + r) * w;
            }
          }
        }
        if (r == 0) tickets[x.bh] = 0;
      }
      const float wc = expf(scur - Mf);
      out[(size_t)b * ldo + (size_t)h * d + r] = (Of + wc * vc) / (Lf + wc);
    };
    A5Tile x;
    if (warp < 6) {                    // softmax warps
      while (sc.next(x)) softmax(x);
      if (r == 0) a5_mark_cta(6);
    } else {                           // readout warps
      while (sc.next(x)) readout(x);
      if (r == 0) a5_mark_cta(7);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) a5_mark_cta(2);
  if (warp == 1) {
    tc05::fence_after_sync();
    tc05::tmem_dealloc<kTmemCols>(tmem);
  }
}

int attend_tc05_set_trace(void* buf) {
  unsigned long long* p = (unsigned long long*)buf;
  IG_CUDA_STATUS(cudaMemcpyToSymbol(a5_trace, &p, sizeof(p)));
  return IG_OK;
}

// ----------------------------------------------------------------------------
// host launch (called by attend_dispatch for d = 128, 2-byte pools)
// ----------------------------------------------------------------------------
int attend_tc05_launch(int elt, cudaStream_t s, const float* q, int ldq, const float* k_cur, const float* v_cur,
                       int ldkv, const void* stage, const int32_t* idx, const int32_t* n, const int32_t* rows_bh,
                       const int32_t* pos, const ig_step_state* st, int B, int Hg, int cap, float sqrt_d,
                       int max_chunks, float* partial, int32_t* tickets, float* out, int ldo) {
  using namespace a5;
  const int BH = B * Hg;
  // not applicable (the caller takes the mma.sync kernel): too many (b, h), or a
  // q row the q warp's 16-B loads cannot read
  if (BH > kMaxBH || (((uintptr_t)q) & 15) || (ldq & 3) || (((uintptr_t)stage) & 15)) return -1;
  struct Cached {
    const void* ptr;
    long long rows;
    int elt;
    CUtensorMap map;
  };
  static Cached cache[8];
  static int cache_next = 0;
  const long long total_rows = (long long)BH * cap;
  CUtensorMap* map = nullptr;
  for (auto& c : cache)
    if (c.ptr == stage && c.rows == total_rows && c.elt == elt) map = &c.map;
  if (!map) {
    Cached& c = cache[cache_next++ % 8];
    const int rc = make_tmap_2d(&c.map, elt == IG_ELT_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                                stage, 256, (uint64_t)total_rows, 512, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) { c.ptr = nullptr; return rc; }
    c.ptr = stage;
    c.rows = total_rows;
    c.elt = elt;
    map = &c.map;
  }
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    IG_CUDA_STATUS(cudaGetDevice(&dev));
    IG_CUDA_STATUS(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  }
  const size_t smem = kFixedSmem + (size_t)(BH + 1) * 4;   // <= 227 KB for BH <= kMaxBH
  // an upper bound of the tile count: every (b, h) at cap rows
  const long long max_tiles = (long long)BH * ((cap + kRows - 1) / kRows);
  const int grid = (int)(max_tiles < sms ? max_tiles : sms);
  if (elt == IG_ELT_BF16) {
    IG_CUDA_STATUS(cudaFuncSetAttribute(attend_tc05_kernel<__nv_bfloat16>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attend_tc05_kernel<__nv_bfloat16><<<grid, kThreads, smem, s>>>(*map, q, ldq, k_cur, v_cur, ldkv, idx, n, rows_bh,
                                                                   pos, st, B, Hg, cap, sqrt_d, max_chunks, partial,
                                                                   tickets, out, ldo);
  } else {
    IG_CUDA_STATUS(cudaFuncSetAttribute(attend_tc05_kernel<__half>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)smem));
    attend_tc05_kernel<__half><<<grid, kThreads, smem, s>>>(*map, q, ldq, k_cur, v_cur, ldkv, idx, n, rows_bh, pos,
                                                            st, B, Hg, cap, sqrt_d, max_chunks, partial, tickets,
                                                            out, ldo);
  }
  IG_LAUNCH_STATUS();
  return IG_OK;
}

}  // namespace ig

extern "C" int ig_debug_attend_trace(void* buf) { return ig::attend_tc05_set_trace(buf); }
