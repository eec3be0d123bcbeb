// K4 sparse decode attention over the fetched rows plus the GPU-resident
// current row (reference attention_head model.py:156-180 as called at
// engine.py:352-358 on the fetch set of engine.py:382-418).
//
// Split-KV: CTA (chunk, h, b) streams kAttChunk staged rows; each warp keeps an
// online softmax over its rows; the CTA writes (m, l, acc[d]) and the last CTA
// of a (b, h) to arrive (ticket) merges the chunks in fixed chunk order, so the
// result is deterministic.  Scores are (q . k) / float32(sqrt(d)) -- a division,
// as in model.py:174 -- and exp is the full-precision expf.
#include <cstdlib>
#include <type_traits>

#include "common.cuh"

namespace ig {

constexpr int kAttThreads = 128;
constexpr int kAttWarps = kAttThreads / kWarp;
constexpr int kAttChunk = 128;     // staged rows per CTA
constexpr int kAttMaxPer = 8;      // head_dim <= 256
constexpr int kAttRowsInFlight = 4;

// The current token's pool row: pos_in[b, h] (what ig_append chose), or, with
// pos_in == NULL, the append position below the pool limit (st->s_len) --
// which lets the append run concurrently with the attention when no pool
// limit can make it evict.
__device__ __forceinline__ int att_pos(const int32_t* pos_in, const ig_step_state* st, size_t bh) {
  return pos_in ? pos_in[bh] : st->s_len;
}

// Rows of one (b, h): a per-head count (resident slot tables), the step's
// shared n (selection), or every pool row (identity, layer 0).
__device__ __forceinline__ int att_rows(const int32_t* rows_bh, const int32_t* n_in,
                                        const ig_step_state* st, int b, size_t bh) {
  return rows_bh ? rows_bh[bh] : (n_in ? n_in[b] : st->s_len);
}

// Lane l owns elements l*E .. l*E+E-1 when E > 0 (d == 32*E, vector loads);
// for other head dims (E == 0) lane l owns l, l+32, ... (scalar loads).
template <typename T, int E>
struct RowIO {
  static constexpr int kPer = E > 0 ? E : kAttMaxPer;
  __device__ static int elem(int lane, int j) { return E > 0 ? lane * E + j : lane + 32 * j; }
  __device__ static void load(const T* row, int lane, int d, float* out) {
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const int e = elem(lane, j);
      out[j] = e < d ? Elt<T>::to_f(row[e]) : 0.f;
    }
  }
};

template <typename T, int E>
__global__ void __launch_bounds__(kAttThreads)
attend_kernel(const float* __restrict__ q, int ldq, const float* __restrict__ k_cur,
              const float* __restrict__ v_cur, int ldkv, const T* __restrict__ stage,
              const int32_t* __restrict__ idx, const int32_t* __restrict__ n_in,
              const int32_t* __restrict__ rows_bh, const int32_t* __restrict__ pos_in, const ig_step_state* __restrict__ st, int Hg,
              int d, int cap, float inv_dummy, float sqrt_d, int max_chunks,
              float* __restrict__ partial, int32_t* __restrict__ tickets, float* __restrict__ out,
              int ldo) {
  using IO = RowIO<T, E>;
  constexpr int P = IO::kPer;
  const int b = blockIdx.z, h = blockIdx.y, c = blockIdx.x;
  const size_t bh = (size_t)b * Hg + h;
  const int rows = att_rows(rows_bh, n_in, st, b, bh);
  const int nchunks = max(1, (rows + kAttChunk - 1) / kAttChunk);
  if (c >= nchunks) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int pos = att_pos(pos_in, st, bh);

  float qv[P];
  {
    const float* qr = q + (size_t)b * ldq + (size_t)h * d;
#pragma unroll
    for (int j = 0; j < P; ++j) {
      const int e = IO::elem(lane, j);
      qv[j] = e < d ? qr[e] : 0.f;
    }
  }
  float m = -INFINITY, l = 0.f, acc[P];
#pragma unroll
  for (int j = 0; j < P; ++j) acc[j] = 0.f;

  auto consume = [&](float sc, const float* vv) {
    const float mn = fmaxf(m, sc);
    const float corr = expf(m - mn);  // m == -inf -> 0
    const float p = expf(sc - mn);
    l = l * corr + p;
#pragma unroll
    for (int j = 0; j < P; ++j) acc[j] = fmaf(p, vv[j], acc[j] * corr);
    m = mn;
  };

  const int r0 = c * kAttChunk, r1 = min(rows, r0 + kAttChunk);
  const T* base = stage + bh * (size_t)cap * 2 * d;
  for (int rb = r0 + w * kAttRowsInFlight; rb < r1; rb += kAttWarps * kAttRowsInFlight) {
    float kk[kAttRowsInFlight][P], vv[kAttRowsInFlight][P];
    bool ok[kAttRowsInFlight];
#pragma unroll
    for (int u = 0; u < kAttRowsInFlight; ++u) {
      const int r = rb + u;
      const int id = r < r1 ? (idx ? idx[bh * cap + r] : r) : -1;
      ok[u] = id >= 0 && id != pos;   // id < 0: empty resident slot
      if (ok[u]) {
        IO::load(base + (size_t)r * 2 * d, lane, d, kk[u]);
        IO::load(base + (size_t)r * 2 * d + d, lane, d, vv[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < kAttRowsInFlight; ++u) {
      if (!ok[u]) continue;  // warp-uniform
      float dot = 0.f;
#pragma unroll
      for (int j = 0; j < P; ++j) dot = fmaf(qv[j], kk[u][j], dot);
      dot = warp_sum(dot);
      consume(dot / sqrt_d, vv[u]);
    }
  }
  if (c == 0 && w == 0) {  // the current token: GPU-resident, never fetched
    const float* kr = k_cur + (size_t)b * ldkv + (size_t)h * d;
    const float* vr = v_cur + (size_t)b * ldkv + (size_t)h * d;
    float kk[P], vv[P];
#pragma unroll
    for (int j = 0; j < P; ++j) {
      const int e = IO::elem(lane, j);
      kk[j] = e < d ? kr[e] : 0.f;
      vv[j] = e < d ? vr[e] : 0.f;
    }
    float dot = 0.f;
#pragma unroll
    for (int j = 0; j < P; ++j) dot = fmaf(qv[j], kk[j], dot);
    dot = warp_sum(dot);
    consume(dot / sqrt_d, vv);
  }

  // merge the warps of this CTA (fixed order)
  __shared__ float wm[kAttWarps], wl[kAttWarps];
  __shared__ float wacc[kAttWarps][kAttMaxPer * 32];
  if (lane == 0) { wm[w] = m; wl[w] = l; }
#pragma unroll
  for (int j = 0; j < P; ++j) {
    const int e = IO::elem(lane, j);
    if (e < d) wacc[w][e] = acc[j];
  }
  __syncthreads();
  float* part = partial + (bh * max_chunks + c) * (size_t)(d + 2);
  if (threadIdx.x == 0) {
    float M = -INFINITY;
    for (int i = 0; i < kAttWarps; ++i) M = fmaxf(M, wm[i]);
    float L = 0.f;
    for (int i = 0; i < kAttWarps; ++i) L += wl[i] * (wm[i] == -INFINITY ? 0.f : expf(wm[i] - M));
    part[0] = M;
    part[1] = L;
  }
  {
    float M = -INFINITY;
    for (int i = 0; i < kAttWarps; ++i) M = fmaxf(M, wm[i]);
    for (int e = threadIdx.x; e < d; e += blockDim.x) {
      float a = 0.f;
      for (int i = 0; i < kAttWarps; ++i)
        a += wacc[i][e] * (wm[i] == -INFINITY ? 0.f : expf(wm[i] - M));
      part[2 + e] = a;
    }
  }
  // last CTA of this (b, h) merges all chunks
  __shared__ int last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(tickets + bh, 1) == nchunks - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  const float* pb = partial + bh * max_chunks * (size_t)(d + 2);
  float M = -INFINITY;
  for (int i = 0; i < nchunks; ++i) M = fmaxf(M, __ldcg(pb + (size_t)i * (d + 2)));
  float L = 0.f;
  for (int i = 0; i < nchunks; ++i) {
    const float mi = __ldcg(pb + (size_t)i * (d + 2));
    L += __ldcg(pb + (size_t)i * (d + 2) + 1) * (mi == -INFINITY ? 0.f : expf(mi - M));
  }
  for (int e = threadIdx.x; e < d; e += blockDim.x) {
    float a = 0.f;
    for (int i = 0; i < nchunks; ++i) {
      const float mi = __ldcg(pb + (size_t)i * (d + 2));
      a += __ldcg(pb + (size_t)i * (d + 2) + 2 + e) * (mi == -INFINITY ? 0.f : expf(mi - M));
    }
    out[(size_t)b * ldo + (size_t)h * d + e] = a / L;
  }
  if (threadIdx.x == 0) tickets[bh] = 0;
}

// ---------------------------------------------------------------------------
// Tensor-core 512-B-row path (default for d = 128 with a 2-byte pool).
// Per-row CUDA-core work (f16 -> f32 unpack, 16 FMAs and 5 shuffles per row
// and lane) bounded a register-fed version at ~0.44 of HBM and a TMA-fed one at
// 0.37 (round 1; removed); here both products run on mma.sync m16n8k16 over
// 16-row tiles:
//   scores  S[16 rows x 8] = K_tile[16 x 128] . Qm[128 x 8], Qm's columns
//           0..NS-1 = the f32 query split into NS parts exactly representable
//           in T (q = q0 + q1 (+ q2)), so S[r][0] + .. + S[r][NS-1] is q.k to
//           ~2^-22 (f16: NS = 2, bf16: NS = 3);
//   output  O^T[128 x 8] += V_tile^T[128 x 16 rows] . Pm[16 rows x 8], Pm's
//           columns 0..NS-1 = the split softmax weights p of the tile's rows
//           (d on the MMA's M side: 8 MMAs and 32 accumulator registers per
//           tile instead of 16 / 64 with p on the M side).
// f32 accumulation throughout; scores are (q.k) / float32(sqrt(d)) as in
// model.py:174 and exp is expf.  Rows stream into a per-warp shared-memory
// ring by cp.async (16-B chunk c of row r stored at chunk c ^ (r & 7), so the
// ldmatrix phases are conflict-free); a warp owns every 4th 16-row tile of
// the CTA's chunk and keeps its own online softmax; warps and chunks merge in
// fixed order (deterministic).
// ---------------------------------------------------------------------------
constexpr int kMmaWarps = 4;
constexpr int kMmaTPW = 8;                                  // tiles per warp (default)
constexpr int kMmaTileBytes = 16 * 512;
constexpr int kMmaSlotBytes = kMmaTileBytes + 64;            // + the tile's 16 row ids

template <typename T> struct MmaT;
template <> struct MmaT<__half> {
  static constexpr int NS = 2;
  __device__ static uint32_t pack(float lo_elem, float hi_elem) {
    __half2 h = __floats2half2_rn(lo_elem, hi_elem);
    return *reinterpret_cast<uint32_t*>(&h);
  }
  __device__ static float round(float x) { return __half2float(__float2half_rn(x)); }
  __device__ static void mma(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  }
};
template <> struct MmaT<__nv_bfloat16> {
  static constexpr int NS = 3;
  __device__ static uint32_t pack(float lo_elem, float hi_elem) {
    __nv_bfloat162 h = __floats2bfloat162_rn(lo_elem, hi_elem);
    return *reinterpret_cast<uint32_t*>(&h);
  }
  __device__ static float round(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }
  __device__ static void mma(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  }
};

// part `g` of the exact split x = x0 + x1 (+ x2), each part representable in T
template <typename T>
__device__ __forceinline__ float split_part(float x, int g) {
  const float x0 = MmaT<T>::round(x);
  const float r1 = x - x0;
  const float x1 = MmaT<T>::round(r1);
  if (g == 0) return x0;
  if (g == 1) return x1;
  if (MmaT<T>::NS > 2 && g == 2) return MmaT<T>::round(r1 - x1);
  return 0.f;
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t* r) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t* r) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}

template <typename T, int RING, int TPW>
__global__ void __launch_bounds__(kMmaWarps * 32, RING <= 2 ? 3 : 2)
attend512_mma_kernel(const float* __restrict__ q, int ldq, const float* __restrict__ k_cur,
                     const float* __restrict__ v_cur, int ldkv, const T* __restrict__ stage,
                     const int32_t* __restrict__ idx, const int32_t* __restrict__ n_in,
                     const int32_t* __restrict__ rows_bh, const int32_t* __restrict__ pos_in,
                     const ig_step_state* __restrict__ st, int Hg, int cap, float sqrt_d,
                     int max_chunks, float* __restrict__ partial, int32_t* __restrict__ tickets,
                     float* __restrict__ out, int ldo) {
  constexpr int d = 128, NS = MmaT<T>::NS;
  extern __shared__ __align__(128) uint8_t att_ring[];       // [warps][RING][16 rows][512 B]
  __shared__ float wm[kMmaWarps], wl[kMmaWarps];
  __shared__ float wacc[kMmaWarps][d];
  pdl_trigger();
  __shared__ int last;
  const int b = blockIdx.z, h = blockIdx.y, c = blockIdx.x;
  const size_t bh = (size_t)b * Hg + h;
  const int rows = att_rows(rows_bh, n_in, st, b, bh);
  const int nchunks = max(1, (rows + (kMmaWarps * TPW * 16) - 1) / (kMmaWarps * TPW * 16));
  if (c >= nchunks) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int pos = att_pos(pos_in, st, bh);
  // balanced chunks: nchunks of at most warps*TPW*16 rows, sizes within one 64-row tile group
  const int crows = (((rows + nchunks - 1) / nchunks) + 63) & ~63;
  const int r0 = c * crows, r1 = min(rows, r0 + crows);
  const uint8_t* src = reinterpret_cast<const uint8_t*>(stage + bh * (size_t)cap * 2 * d);
  const uint32_t ring = (uint32_t)__cvta_generic_to_shared(att_ring) + w * RING * kMmaSlotBytes;
  const int* ring_ids = reinterpret_cast<const int*>(att_ring + (size_t)w * RING * kMmaSlotBytes +
                                                     kMmaTileBytes);

  // query split into NS parts: B fragments of the 8 k16-steps (column g < NS)
  uint32_t bq[8][2];
  {
    const float* qr = q + (size_t)b * ldq + (size_t)h * d;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const int k0 = kk * 16 + 2 * t;
      bq[kk][0] = MmaT<T>::pack(split_part<T>(qr[k0], g), split_part<T>(qr[k0 + 1], g));
      bq[kk][1] = MmaT<T>::pack(split_part<T>(qr[k0 + 8], g), split_part<T>(qr[k0 + 9], g));
      if (g >= NS) bq[kk][0] = bq[kk][1] = 0u;
    }
  }
  float m = -INFINITY, l = 0.f;
  float acc[8][4];                 // [m-tile of d][C fragment]: (d, split col) pairs
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;

  // tile j of this warp: rows [tb, tb + 16), tb = r0 + (j * warps + w) * 16; the
  // tile's row ids ride in the same cp.async group (a separate global load of
  // them was the kernel's top stall)
  auto issue = [&](int j) {
    const int tb = r0 + (j * kMmaWarps + w) * 16;
    const uint32_t slot = ring + (j % RING) * kMmaSlotBytes;
#pragma unroll
    for (int rr = 0; rr < 16; ++rr) {
      const int r = tb + rr;
      const bool ok = r < r1;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;"
                   ::"r"(slot + rr * 512 + ((lane ^ (rr & 7)) << 4)),
                   "l"(src + (size_t)(ok ? r : r0) * 512 + lane * 16), "r"(ok ? 16 : 0)
                   : "memory");
    }
    if (idx != nullptr && lane < 16) {
      const int r = tb + lane;
      const bool ok = r < r1;
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;"
                   ::"r"(slot + kMmaTileBytes + lane * 4), "l"(idx + bh * cap + (ok ? r : r0)),
                   "r"(ok ? 4 : 0) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  int ntiles = 0;
#pragma unroll
  for (int j = 0; j < TPW; ++j) ntiles += (r0 + (j * kMmaWarps + w) * 16 < r1) ? 1 : 0;

#pragma unroll
  for (int j = 0; j < RING - 1; ++j)
    if (j < ntiles) issue(j);
#pragma unroll
  for (int j = 0; j < TPW; ++j) {
    if (j >= ntiles) break;
    if (j + RING - 1 < ntiles) {
      issue(j + RING - 1);
      asm volatile("cp.async.wait_group %0;" ::"n"(RING - 1) : "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncwarp();
    const uint32_t slot = ring + (j % RING) * kMmaSlotBytes;
    const int tb = r0 + (j * kMmaWarps + w) * 16;
    const int* sid = ring_ids + (j % RING) * (kMmaSlotBytes / 4);
    // S = K . Qm (two accumulators: half-length dependency chains)
    float sc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
    const int lr = lane & 15, lh = lane >> 4;
    const uint32_t rowaddr = slot + lr * 512;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      uint32_t a[4];
      ldsm_x4(rowaddr + (((2 * kk + lh) ^ (lr & 7)) << 4), a);
      MmaT<T>::mma(sc[kk & 1], a, bq[kk][0], bq[kk][1]);
    }
    float s0 = (sc[0][0] + sc[1][0]) + (sc[0][1] + sc[1][1]);   // columns of this lane's pair
    float s1 = (sc[0][2] + sc[1][2]) + (sc[0][3] + sc[1][3]);
    s0 += __shfl_xor_sync(0xffffffffu, s0, 1);
    s1 += __shfl_xor_sync(0xffffffffu, s1, 1);
    s0 += __shfl_xor_sync(0xffffffffu, s0, 2);
    s1 += __shfl_xor_sync(0xffffffffu, s1, 2);
    const int id0 = tb + g < r1 ? (idx ? sid[g] : tb + g) : -1;
    const int id1 = tb + g + 8 < r1 ? (idx ? sid[g + 8] : tb + g + 8) : -1;
    const bool ok0 = id0 >= 0 && id0 != pos;
    const bool ok1 = id1 >= 0 && id1 != pos;
    s0 = ok0 ? s0 / sqrt_d : -INFINITY;                      // row g
    s1 = ok1 ? s1 / sqrt_d : -INFINITY;                      // row g + 8
    float tm = fmaxf(s0, s1);
    tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, 4));
    tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, 8));
    tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, 16));
    if (tm != -INFINITY) {                                   // warp-uniform
      if (tm > m) {
        const float corr = expf(m - tm);                     // m == -inf -> 0
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          acc[i][0] *= corr; acc[i][1] *= corr; acc[i][2] *= corr; acc[i][3] *= corr;
        }
        l *= corr;
        m = tm;
      }
      const float p0 = expf(s0 - m), p1 = expf(s1 - m);     // exp(-inf) = 0
      l += p0 + p1;
      // Pm fragment: rows 2t, 2t+1 (quads 2t, 2t+1) and 2t+8, 2t+9
      const float pa = __shfl_sync(0xffffffffu, p0, 8 * t);
      const float pb = __shfl_sync(0xffffffffu, p0, 8 * t + 4);
      const float pc = __shfl_sync(0xffffffffu, p1, 8 * t);
      const float pd = __shfl_sync(0xffffffffu, p1, 8 * t + 4);
      // B = Pm: k = tile rows 2t, 2t+1 (b0) and 2t+8, 2t+9 (b1), column g
      uint32_t pb0 = MmaT<T>::pack(split_part<T>(pa, g), split_part<T>(pb, g));
      uint32_t pb1 = MmaT<T>::pack(split_part<T>(pc, g), split_part<T>(pd, g));
      if (g >= NS) pb0 = pb1 = 0u;
      // A = V^T (m = d, k = row): ldmatrix.trans of the blocks (rows 0-7 | 8-15) x
      // (d 0-7 | 8-15) of m-tile mt; lane -> row (lane & 7) + 8 (lane >> 4),
      // chunk 16 + 2 mt + ((lane >> 3) & 1)
      const int vr = (lane & 7) + ((lane >> 4) << 3), vc = (lane >> 3) & 1;
      const uint32_t vaddr = slot + vr * 512;
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) {
        uint32_t a[4];
        ldsm_x4_t(vaddr + (((16 + 2 * mt + vc) ^ (vr & 7)) << 4), a);
        MmaT<T>::mma(acc[mt], a, pb0, pb1);
      }
    }
    __syncwarp();                                            // slot j % RING free for reuse
  }
  if (c == 0 && w == 0) {  // the current token: GPU-resident f32 row, f32 dot
    const float* qr = q + (size_t)b * ldq + (size_t)h * d;
    const float* kr = k_cur + (size_t)b * ldkv + (size_t)h * d;
    float dot = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) dot = fmaf(qr[lane * 4 + i], kr[lane * 4 + i], dot);
    dot = warp_sum(dot);
    const float scur = dot / sqrt_d;
    if (scur > m) {
      const float corr = expf(m - scur);
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        acc[i][0] *= corr; acc[i][1] *= corr; acc[i][2] *= corr; acc[i][3] *= corr;
      }
      l *= corr;
      m = scur;
    }
    const float p = expf(scur - m);
    if (g == 0) l += p;
    if (t == 0) {                  // split column 0 of rows d = 16 mt + g (+ 8)
      const float* vrow = v_cur + (size_t)b * ldkv + (size_t)h * d;
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) {
        acc[mt][0] = fmaf(p, vrow[mt * 16 + g], acc[mt][0]);
        acc[mt][2] = fmaf(p, vrow[mt * 16 + g + 8], acc[mt][2]);
      }
    }
  }
  // O row = sum of the NS split rows; l over the 8 quads
  l += __shfl_xor_sync(0xffffffffu, l, 4);
  l += __shfl_xor_sync(0xffffffffu, l, 8);
  l += __shfl_xor_sync(0xffffffffu, l, 16);
#pragma unroll
  for (int mt = 0; mt < 8; ++mt) {        // sum the split columns (lanes t = 0..3)
    float y0 = acc[mt][0] + acc[mt][1], y1 = acc[mt][2] + acc[mt][3];
    y0 += __shfl_xor_sync(0xffffffffu, y0, 1);
    y1 += __shfl_xor_sync(0xffffffffu, y1, 1);
    y0 += __shfl_xor_sync(0xffffffffu, y0, 2);
    y1 += __shfl_xor_sync(0xffffffffu, y1, 2);
    if (t == 0) {
      wacc[w][mt * 16 + g] = y0;
      wacc[w][mt * 16 + g + 8] = y1;
    }
  }
  if (lane == 0) { wm[w] = m; wl[w] = l; }
  __syncthreads();
  float M = -INFINITY;
  for (int i = 0; i < kMmaWarps; ++i) M = fmaxf(M, wm[i]);
  float* part = partial + (bh * max_chunks + c) * (size_t)(d + 2);
  if (threadIdx.x == 0) {
    float L = 0.f;
    for (int i = 0; i < kMmaWarps; ++i) L += wl[i] * (wm[i] == -INFINITY ? 0.f : expf(wm[i] - M));
    part[0] = M;
    part[1] = L;
  }
  for (int e = threadIdx.x; e < d; e += blockDim.x) {
    float a = 0.f;
    for (int i = 0; i < kMmaWarps; ++i) a += wacc[i][e] * (wm[i] == -INFINITY ? 0.f : expf(wm[i] - M));
    part[2 + e] = a;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(tickets + bh, 1) == nchunks - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  const float* pb = partial + bh * max_chunks * (size_t)(d + 2);
  float MM = -INFINITY;
  for (int i = 0; i < nchunks; ++i) MM = fmaxf(MM, __ldcg(pb + (size_t)i * (d + 2)));
  float LL = 0.f;
  for (int i = 0; i < nchunks; ++i) {
    const float mi = __ldcg(pb + (size_t)i * (d + 2));
    LL += __ldcg(pb + (size_t)i * (d + 2) + 1) * (mi == -INFINITY ? 0.f : expf(mi - MM));
  }
  for (int e = threadIdx.x; e < d; e += blockDim.x) {
    float a = 0.f;
    for (int i = 0; i < nchunks; ++i) {
      const float mi = __ldcg(pb + (size_t)i * (d + 2));
      a += __ldcg(pb + (size_t)i * (d + 2) + 2 + e) * (mi == -INFINITY ? 0.f : expf(mi - MM));
    }
    out[(size_t)b * ldo + (size_t)h * d + e] = a / LL;
  }
  if (threadIdx.x == 0) tickets[bh] = 0;
}

// ---------------------------------------------------------------------------
// Warp-persistent variant of the tensor-core path (default).  Work items are
// 128-row segments of a (b, h) row set; every warp owns a contiguous range of
// items and streams their 16-row tiles through its own cp.async ring, issuing
// the next item's first tile (with the item's query row) before it closes the
// current item -- so the pipeline never drains between items and no CTA-wide
// barrier exists.  A warp closes an item by writing its (m, l, acc) partial
// and taking a per-(b, h) ticket; the last segment to finish merges all
// segments in fixed order (deterministic).  At 819-row selections the
// CTA-per-chunk kernel spent most of its time filling and draining its
// pipeline once per 400-row chunk.
// ---------------------------------------------------------------------------
constexpr int kWpSegDefault = 128;                           // rows per work item
constexpr int kWpWarps = 4;
constexpr int kWpSlotBytes = kMmaTileBytes + 64 + 512;       // rows + ids + query row

template <typename T, int RING, int kWpSeg>
__global__ void __launch_bounds__(kWpWarps * 32, RING <= 2 ? 3 : 2)
attend512_wp_kernel(const float* __restrict__ q, int ldq, const float* __restrict__ k_cur,
                    const float* __restrict__ v_cur, int ldkv, const T* __restrict__ stage,
                    const int32_t* __restrict__ idx, const int32_t* __restrict__ n_in,
                    const int32_t* __restrict__ rows_bh, const int32_t* __restrict__ pos_in,
                    const ig_step_state* __restrict__ st, int B, int Hg, int cap, float sqrt_d,
                    int max_chunks, float* __restrict__ partial, int32_t* __restrict__ tickets,
                    float* __restrict__ out, int ldo) {
  constexpr int d = 128, NS = MmaT<T>::NS;
  extern __shared__ __align__(128) uint8_t wp_ring[];        // [warps][RING][slot]
  pdl_trigger();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  // Items are laid out over the segments the LARGEST row set of this launch
  // needs (read from the device-side counts: every warp computes the same
  // value), not over cap: layers whose selections are well below cap would
  // otherwise leave empty item slots in some warps' ranges and a tail of
  // warps with full ranges.
  int maxrows = 0;
  for (int i = lane; i < B * Hg; i += 32) maxrows = max(maxrows, att_rows(rows_bh, n_in, st, i / Hg, (size_t)i));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) maxrows = max(maxrows, __shfl_xor_sync(0xffffffffu, maxrows, o));
  const int maxseg = max(1, min((cap + kWpSeg - 1) / kWpSeg, (maxrows + kWpSeg - 1) / kWpSeg));
  // 32-bit item arithmetic (64-bit division is a subroutine call per item)
  const int items = B * Hg * maxseg;
  const int tw = gridDim.x * kWpWarps, gw = blockIdx.x * kWpWarps + w;
  // ceil(items / tw) items per warp (the balanced floor/ceil split and 256-row
  // items both measured slower at 819 rows: 74-77 vs 70 us)
  const int per = (items + tw - 1) / tw;
  const int it_lo = gw * per, it_hi = min(items, it_lo + per);
  uint8_t* wbase = wp_ring + (size_t)w * RING * kWpSlotBytes;
  const uint32_t sring = (uint32_t)__cvta_generic_to_shared(wbase);

  // item geometry; an item exists if seg < nseg(bh) (segment 0 always: the current row)
  auto geom = [&](int it, int& bh, int& seg, int& r0, int& r1, int& ntl) -> bool {
    bh = it / maxseg;
    seg = it - bh * maxseg;
    const int b = bh / Hg;
    const int rows = att_rows(rows_bh, n_in, st, b, (size_t)bh);
    const int nseg = max(1, (rows + kWpSeg - 1) / kWpSeg);
    if (seg >= nseg) return false;
    r0 = seg * kWpSeg;
    r1 = min(rows, r0 + kWpSeg);
    ntl = max(0, (r1 - r0 + 15) / 16);
    return true;
  };
  auto next_item = [&](int it) -> int {                    // first existing item > it
    for (int j = it + 1; j < it_hi; ++j) {
      int bh, seg, r0, r1, ntl;
      if (geom(j, bh, seg, r0, r1, ntl)) return j;
    }
    return -1;
  };
  // issue tile `tl` of item (bh, r0, r1) into ring slot `slot_i`; tile 0 also
  // brings the item's query row
  auto issue = [&](int bh, int r0, int r1, int tl, int slot_i) {
    const uint32_t slot = sring + slot_i * kWpSlotBytes;
    const uint8_t* src = reinterpret_cast<const uint8_t*>(stage + (size_t)bh * cap * 2 * d);
    const int tb = r0 + tl * 16;
#pragma unroll
    for (int rr = 0; rr < 16; ++rr) {
      const int r = tb + rr;
      const bool ok = r < r1;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;"
                   ::"r"(slot + rr * 512 + ((lane ^ (rr & 7)) << 4)),
                   "l"(src + (size_t)(ok ? r : 0) * 512 + lane * 16), "r"(ok ? 16 : 0)
                   : "memory");
    }
    if (idx != nullptr && lane < 16) {
      const int r = tb + lane;
      const bool ok = r < r1;
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;"
                   ::"r"(slot + kMmaTileBytes + lane * 4),
                   "l"(idx + (size_t)bh * cap + (ok ? r : 0)), "r"(ok ? 4 : 0) : "memory");
    }
    if (tl == 0) {
      const int b = bh / Hg, h = bh - b * Hg;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;"
                   ::"r"(slot + kMmaTileBytes + 64 + lane * 16),
                   "l"(q + (size_t)b * ldq + (size_t)h * d + lane * 4) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  int cur = -1;
  {
    int bh, seg, r0, r1, ntl;
    if (it_lo < it_hi && geom(it_lo, bh, seg, r0, r1, ntl)) cur = it_lo;
    else if (it_lo < it_hi) cur = next_item(it_lo);
  }
  // Issue cursor: runs up to RING - 1 tiles ahead of the compute cursor,
  // across item boundaries (an empty item still takes its q-carrying slot).
  int icur = cur;
  int itl = 0, ibh = 0, iseg = 0, ir0 = 0, ir1 = 0, intl = 0;
  if (icur >= 0) geom(icur, ibh, iseg, ir0, ir1, intl);
  int slot_ctr = 0;                     // ring slot of the next tile to issue
  int pending = 0;                      // tiles issued and not yet consumed
  auto issue_next = [&]() {
    issue(ibh, ir0, ir1, itl, slot_ctr % RING);
    ++slot_ctr;
    ++pending;
    if (++itl >= max(1, intl)) {
      icur = next_item(icur);
      itl = 0;
      if (icur >= 0) geom(icur, ibh, iseg, ir0, ir1, intl);
    }
  };
  int cslot = 0;                        // ring slot of the tile being computed
  while (cur >= 0) {
    int bh, seg, r0, r1, ntl;
    geom(cur, bh, seg, r0, r1, ntl);
    const int b = bh / Hg, h = bh - b * Hg;
    const int pos = att_pos(pos_in, st, bh);
    const int nxt = next_item(cur);
    float m = -INFINITY, l = 0.f;
    float acc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
    uint32_t bq[8][2];
    const int ntiles = max(1, ntl);     // an empty item still consumes its q-carrying slot
    for (int tl = 0; tl < ntiles; ++tl) {
      // keep RING tiles in the ring (this one included), then wait for this one
      while (pending < RING && icur >= 0) issue_next();
      if (pending >= 4) asm volatile("cp.async.wait_group 3;" ::: "memory");
      else if (pending == 3) asm volatile("cp.async.wait_group 2;" ::: "memory");
      else if (pending == 2) asm volatile("cp.async.wait_group 1;" ::: "memory");
      else asm volatile("cp.async.wait_group 0;" ::: "memory");
      --pending;
      __syncwarp();
      const uint32_t slot = sring + cslot * kWpSlotBytes;
      const uint8_t* gslot = wbase + (size_t)cslot * kWpSlotBytes;
      if (tl == 0) {                    // the item's query row -> split B fragments
        const float* qs = reinterpret_cast<const float*>(gslot + kMmaTileBytes + 64);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const int k0 = kk * 16 + 2 * t;
          bq[kk][0] = MmaT<T>::pack(split_part<T>(qs[k0], g), split_part<T>(qs[k0 + 1], g));
          bq[kk][1] = MmaT<T>::pack(split_part<T>(qs[k0 + 8], g), split_part<T>(qs[k0 + 9], g));
          if (g >= NS) bq[kk][0] = bq[kk][1] = 0u;
        }
      }
      if (tl < ntl) {
        const int tb = r0 + tl * 16;
        const int* sid = reinterpret_cast<const int*>(gslot + kMmaTileBytes);
        float sc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
        const int lr = lane & 15, lh = lane >> 4;
        const uint32_t rowaddr = slot + lr * 512;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          uint32_t a[4];
          ldsm_x4(rowaddr + (((2 * kk + lh) ^ (lr & 7)) << 4), a);
          MmaT<T>::mma(sc[kk & 1], a, bq[kk][0], bq[kk][1]);
        }
        float s0 = (sc[0][0] + sc[1][0]) + (sc[0][1] + sc[1][1]);
        float s1 = (sc[0][2] + sc[1][2]) + (sc[0][3] + sc[1][3]);
        s0 += __shfl_xor_sync(0xffffffffu, s0, 1);
        s1 += __shfl_xor_sync(0xffffffffu, s1, 1);
        s0 += __shfl_xor_sync(0xffffffffu, s0, 2);
        s1 += __shfl_xor_sync(0xffffffffu, s1, 2);
        const int id0 = tb + g < r1 ? (idx ? sid[g] : tb + g) : -1;
        const int id1 = tb + g + 8 < r1 ? (idx ? sid[g + 8] : tb + g + 8) : -1;
        s0 = (id0 >= 0 && id0 != pos) ? s0 / sqrt_d : -INFINITY;
        s1 = (id1 >= 0 && id1 != pos) ? s1 / sqrt_d : -INFINITY;
        float tm = fmaxf(s0, s1);
        tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, 4));
        tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, 8));
        tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, 16));
        if (tm != -INFINITY) {
          if (tm > m) {
            const float corr = expf(m - tm);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              acc[i][0] *= corr; acc[i][1] *= corr; acc[i][2] *= corr; acc[i][3] *= corr;
            }
            l *= corr;
            m = tm;
          }
          const float p0 = expf(s0 - m), p1 = expf(s1 - m);
          l += p0 + p1;
          const float pa = __shfl_sync(0xffffffffu, p0, 8 * t);
          const float pb = __shfl_sync(0xffffffffu, p0, 8 * t + 4);
          const float pc = __shfl_sync(0xffffffffu, p1, 8 * t);
          const float pd = __shfl_sync(0xffffffffu, p1, 8 * t + 4);
          uint32_t pb0 = MmaT<T>::pack(split_part<T>(pa, g), split_part<T>(pb, g));
          uint32_t pb1 = MmaT<T>::pack(split_part<T>(pc, g), split_part<T>(pd, g));
          if (g >= NS) pb0 = pb1 = 0u;
          const int vr = (lane & 7) + ((lane >> 4) << 3), vc = (lane >> 3) & 1;
          const uint32_t vaddr = slot + vr * 512;
#pragma unroll
          for (int mt = 0; mt < 8; ++mt) {
            uint32_t a[4];
            ldsm_x4_t(vaddr + (((16 + 2 * mt + vc) ^ (vr & 7)) << 4), a);
            MmaT<T>::mma(acc[mt], a, pb0, pb1);
          }
        }
      }
      __syncwarp();
      cslot = (cslot + 1) % RING;
    }
    if (seg == 0) {                     // the current token: GPU-resident f32 row, f32 dot
      const float* qr = q + (size_t)b * ldq + (size_t)h * d;
      const float* kr = k_cur + (size_t)b * ldkv + (size_t)h * d;
      float dot = 0.f;
#pragma unroll
      for (int i = 0; i < 4; ++i) dot = fmaf(qr[lane * 4 + i], kr[lane * 4 + i], dot);
      dot = warp_sum(dot);
      const float scur = dot / sqrt_d;
      if (scur > m) {
        const float corr = expf(m - scur);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          acc[i][0] *= corr; acc[i][1] *= corr; acc[i][2] *= corr; acc[i][3] *= corr;
        }
        l *= corr;
        m = scur;
      }
      const float p = expf(scur - m);
      if (g == 0) l += p;
      if (t == 0) {
        const float* vrow = v_cur + (size_t)b * ldkv + (size_t)h * d;
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
          acc[mt][0] = fmaf(p, vrow[mt * 16 + g], acc[mt][0]);
          acc[mt][2] = fmaf(p, vrow[mt * 16 + g + 8], acc[mt][2]);
        }
      }
    }
    // close the item: partial (m, l, acc) of segment seg
    l += __shfl_xor_sync(0xffffffffu, l, 4);
    l += __shfl_xor_sync(0xffffffffu, l, 8);
    l += __shfl_xor_sync(0xffffffffu, l, 16);
    float* part = partial + ((size_t)bh * max_chunks + seg) * (size_t)(d + 2);
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) {
      float y0 = acc[mt][0] + acc[mt][1], y1 = acc[mt][2] + acc[mt][3];
      y0 += __shfl_xor_sync(0xffffffffu, y0, 1);
      y1 += __shfl_xor_sync(0xffffffffu, y1, 1);
      y0 += __shfl_xor_sync(0xffffffffu, y0, 2);
      y1 += __shfl_xor_sync(0xffffffffu, y1, 2);
      if (t == 0) {
        part[2 + mt * 16 + g] = y0;
        part[2 + mt * 16 + g + 8] = y1;
      }
    }
    if (lane == 0) { part[0] = m; part[1] = l; }
    __threadfence();
    __syncwarp();
    const int rows = att_rows(rows_bh, n_in, st, b, (size_t)bh);
    const int nseg = max(1, (rows + kWpSeg - 1) / kWpSeg);
    int lastw = 0;
    if (lane == 0) lastw = atomicAdd(tickets + bh, 1) == nseg - 1;
    lastw = __shfl_sync(0xffffffffu, lastw, 0);
    if (lastw) {                        // merge every segment of (b, h) in order
      __threadfence();
      const float* pb = partial + (size_t)bh * max_chunks * (d + 2);
      // lane i holds segment i's (m, l) (segments 32.. folded in order), so the
      // max and the scales take one L2 round trip, not one per segment
      float MM = -INFINITY;
      for (int i = lane; i < nseg; i += 32) MM = fmaxf(MM, __ldcg(pb + (size_t)i * (d + 2)));
      MM = warp_max(MM);
      float LL = 0.f, o[4] = {0.f, 0.f, 0.f, 0.f};
      for (int i0 = 0; i0 < nseg; i0 += 32) {
        const int i = i0 + lane;
        float sc = 0.f, li = 0.f;
        if (i < nseg) {
          const float mi = __ldcg(pb + (size_t)i * (d + 2));
          li = __ldcg(pb + (size_t)i * (d + 2) + 1);
          sc = mi == -INFINITY ? 0.f : expf(mi - MM);
        }
        const int cnt = min(32, nseg - i0);
        for (int j0 = 0; j0 < cnt; j0 += 8) {   // accumulator rows 8 segments per batch
          float2 v[8][2];                      // rows are 8-B aligned ((d + 2) floats)
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (j0 + u < cnt) {
              const float2* r = reinterpret_cast<const float2*>(pb + (size_t)(i0 + j0 + u) * (d + 2) + 2);
              v[u][0] = __ldcg(r + 2 * lane);
              v[u][1] = __ldcg(r + 2 * lane + 1);
            }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            if (j0 + u >= cnt) break;
            const float scu = __shfl_sync(0xffffffffu, sc, j0 + u);
            const float lu = __shfl_sync(0xffffffffu, li, j0 + u);
            LL += lu * scu;
            o[0] += v[u][0].x * scu; o[1] += v[u][0].y * scu; o[2] += v[u][1].x * scu; o[3] += v[u][1].y * scu;
          }
        }
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) out[(size_t)b * ldo + (size_t)h * d + lane * 4 + e] = o[e] / LL;
      if (lane == 0) tickets[bh] = 0;
    }
    cur = nxt;
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// IG_ATTEND_IMPL: 'm' (default: mma.sync), 'c' (tcgen05, attend_tc05.cu)
inline char attend_impl() {
  static const char impl = [] {
    const char* v = getenv("IG_ATTEND_IMPL");
    return v && v[0] == 'c' ? 'c' : 'm';
  }();
  return impl;
}

int attend_tc05_launch(int elt, cudaStream_t s, const float* q, int ldq, const float* k_cur, const float* v_cur,
                       int ldkv, const void* stage, const int32_t* idx, const int32_t* n, const int32_t* rows_bh,
                       const int32_t* pos, const ig_step_state* st, int B, int Hg, int cap, float sqrt_d,
                       int max_chunks, float* partial, int32_t* tickets, float* out, int ldo);

template <typename T>
int launch_attend(dim3 grid, cudaStream_t s, const float* q, int ldq, const float* k_cur,
                  const float* v_cur, int ldkv, const void* stage, const int32_t* idx,
                  const int32_t* n, const int32_t* rows_bh, const int32_t* pos,
                  const ig_step_state* st, int Hg, int d, int cap, float sqrt_d, int max_chunks,
                  float* partial, int32_t* tickets, float* out, int ldo) {
  if constexpr (sizeof(T) == 2) {
    // tcgen05 (attend_tc05.cu) only on request (IG_ATTEND_IMPL=c).  Alone it is the
    // faster kernel on long row sets (640 x 4K rows: 6.42 vs 5.98 TB/s; C4's
    // 128 x 6.5K: 82 vs 89 us) and the slower one on C3's 819-row sets (72 vs 62 us);
    // inside the step its one CTA per SM with a 192-KB ring holds the SMs the
    // speculation stream needs, so both C3 (962 vs 987 tok/s) and C4 (324 vs 329)
    // run faster with the mma.sync kernels below (profiles/r02ae*, r02af*).
    // -1 from the launcher: not applicable here.
    if (d == 128 && attend_impl() == 'c') {
      const int rc = attend_tc05_launch(std::is_same<T, __half>::value ? IG_ELT_F16 : IG_ELT_BF16, s, q, ldq, k_cur,
                                        v_cur, ldkv, stage, idx, n, rows_bh, pos, st, (int)grid.z, Hg, cap, sqrt_d,
                                        max_chunks, partial, tickets, out, ldo);
      if (rc >= 0) return rc;
    }
    if (d == 128) {  // 512-B rows, mma.sync
      // IG_ATT_VARIANT (tuning sweeps): 0 = CTA per chunk, ring 2 x 8 tiles/warp (3 CTAs/SM),
      // 1 = ring 2 x 4 tiles, 2 = ring 3 x 8 tiles (2 CTAs/SM), 3 = ring 2 x 16 tiles,
      // 4 = warp-persistent (attend512_wp_kernel)
      static const int forced = [] {
        const char* v = getenv("IG_ATT_VARIANT");
        return v ? atoi(v) : -1;
      }();
      // default: warp-persistent for short row sets (selections of <= 2K rows, where
      // the CTA kernel's per-chunk pipeline fill dominates), CTA-per-chunk otherwise
      // (tools/attend_probe.py: 819 rows 4.07 vs 3.75 TB/s; 4K-32K rows 5.8-6.0 vs 5.2-5.5)
      const int variant = forced >= 0 ? forced : (cap <= 2048 ? 4 : 0);
#define IG_ATT_MMA(RING, TPW)                                                                  \
  do {                                                                                         \
    const int chunk = kMmaWarps * (TPW) * 16;                                                  \
    const dim3 g3((cap + chunk - 1) / chunk, grid.y, grid.z);                                  \
    const size_t smem = (size_t)kMmaWarps * (RING) * kMmaSlotBytes;                            \
    IG_CUDA_STATUS(cudaFuncSetAttribute(attend512_mma_kernel<T, RING, TPW>,                    \
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    attend512_mma_kernel<T, RING, TPW><<<g3, kMmaWarps * 32, smem, s>>>(                       \
        q, ldq, k_cur, v_cur, ldkv, (const T*)stage, idx, n, rows_bh, pos, st, Hg, cap, sqrt_d, \
        max_chunks, partial, tickets, out, ldo);                                               \
  } while (0)
      if (variant == 4) {   // warp-persistent
        static int sms = 0;
        if (sms == 0) {
          int dev = 0;
          if (cudaGetDevice(&dev) != cudaSuccess ||
              cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
            sms = 148;
        }
        // ring depth: 2 tiles per warp at 3 CTAs/SM (default) or 3 at 2 CTAs/SM
        // (IG_WP_RING=3: more bytes in flight per SM, fewer warps -- measured
        // 3.48 vs 3.76 TB/s at 819 rows, so per-warp latency, not bytes in
        // flight, bounds this kernel); IG_WP_SEG=256: 256-row work items
        static const int ring = [] {
          const char* e = getenv("IG_WP_RING");
          return e && atoi(e) == 3 ? 3 : 2;
        }();
        static const int seg = [] {
          const char* e = getenv("IG_WP_SEG");
          // (no 64-row option: the partial scratch holds cap / kAttChunk = cap / 128
          // segments per (b, h), so smaller items would overrun a row's slots)
          return e && atoi(e) == 256 ? 256 : kWpSegDefault;
        }();
        const int per_sm = ring == 2 ? 3 : 2;
        const int maxseg = (cap + seg - 1) / seg;
        const long long items = (long long)grid.z * grid.y * maxseg;
        const int ctas = (int)min((long long)sms * per_sm, (items + kWpWarps - 1) / kWpWarps);
        const size_t smem = (size_t)kWpWarps * ring * kWpSlotBytes;
#define IG_ATT_WP(RING, SEG)                                                                    \
  do {                                                                                         \
    IG_CUDA_STATUS(cudaFuncSetAttribute(attend512_wp_kernel<T, RING, SEG>,                     \
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    attend512_wp_kernel<T, RING, SEG><<<ctas, kWpWarps * 32, smem, s>>>(                        \
        q, ldq, k_cur, v_cur, ldkv, (const T*)stage, idx, n, rows_bh, pos, st, (int)grid.z,     \
        (int)grid.y, cap, sqrt_d, max_chunks, partial, tickets, out, ldo);                      \
  } while (0)
        if (ring == 2 && seg == 256) IG_ATT_WP(2, 256);
        else if (ring == 3 && seg == 256) IG_ATT_WP(3, 256);
        else if (ring == 3) IG_ATT_WP(3, kWpSegDefault);
        else IG_ATT_WP(2, kWpSegDefault);
#undef IG_ATT_WP
        IG_LAUNCH_STATUS();
        return IG_OK;
      }
      switch (variant) {
        case 1: IG_ATT_MMA(2, 4); break;
        case 2: IG_ATT_MMA(3, 8); break;
        case 3: IG_ATT_MMA(2, 16); break;
        default: IG_ATT_MMA(2, 8); break;
      }
#undef IG_ATT_MMA
      IG_LAUNCH_STATUS();
      return IG_OK;
    }
  }
#define IG_ATT(E)                                                                              \
  attend_kernel<T, E><<<grid, kAttThreads, 0, s>>>(q, ldq, k_cur, v_cur, ldkv,                \
      (const T*)stage, idx, n, rows_bh, pos, st, Hg, d, cap, 0.f, sqrt_d, max_chunks, partial, \
      tickets, out, ldo)
  switch (d) {
    case 32: IG_ATT(1); break;
    case 64: IG_ATT(2); break;
    case 128: IG_ATT(4); break;
    case 256: IG_ATT(8); break;
    default: IG_ATT(0); break;
  }
#undef IG_ATT
  IG_LAUNCH_STATUS();
  return IG_OK;
}

}  // namespace ig

extern "C" int ig_attend_scratch(int B, int Hg, int d, int cap, size_t* partial_floats,
                                 size_t* tickets) {
  using namespace ig;
  if (B < 1 || Hg < 1 || d < 1 || cap < 1 || !partial_floats || !tickets) return IG_EINVAL;
  const int max_chunks = (cap + kAttChunk - 1) / kAttChunk;
  *partial_floats = (size_t)B * Hg * max_chunks * (d + 2);
  *tickets = (size_t)B * Hg;
  return IG_OK;
}

namespace ig {
static int attend_dispatch(const float* q, int ldq, const float* k_cur, const float* v_cur,
                           int ldkv, const void* stage, int elt, const int32_t* idx,
                           const int32_t* n, const int32_t* rows_bh, const int32_t* pos,
                           const ig_step_state* st, int B, int Hg, int d, int cap, float* partial,
                           int32_t* tickets, float* out, int ldo, void* stream) {
  if (!q || !k_cur || !v_cur || !stage || !st || !partial || !tickets || !out || B < 1 ||
      Hg < 1 || d < 1 || d > 32 * kAttMaxPer || cap < 1 || ldq < Hg * d || ldkv < Hg * d ||
      ldo < Hg * d)
    return IG_EINVAL;
  const int max_chunks = (cap + kAttChunk - 1) / kAttChunk;
  dim3 grid(max_chunks, Hg, B);
  const float sqrt_d = (float)sqrt((double)d);  // float32(np.sqrt(d)), model.py:174
  cudaStream_t s = (cudaStream_t)stream;
  switch (elt) {
    case IG_ELT_F32:
      return launch_attend<float>(grid, s, q, ldq, k_cur, v_cur, ldkv, stage, idx, n, rows_bh, pos,
                                  st, Hg, d, cap, sqrt_d, max_chunks, partial, tickets, out, ldo);
    case IG_ELT_F16:
      return launch_attend<__half>(grid, s, q, ldq, k_cur, v_cur, ldkv, stage, idx, n, rows_bh,
                                   pos, st, Hg, d, cap, sqrt_d, max_chunks, partial, tickets, out,
                                   ldo);
    case IG_ELT_BF16:
      return launch_attend<__nv_bfloat16>(grid, s, q, ldq, k_cur, v_cur, ldkv, stage, idx, n,
                                          rows_bh, pos, st, Hg, d, cap, sqrt_d, max_chunks,
                                          partial, tickets, out, ldo);
    default:
      return IG_EINVAL;
  }
}
}  // namespace ig

extern "C" int ig_attend(const float* q, int ldq, const float* k_cur, const float* v_cur, int ldkv,
                         const void* stage, int elt, const int32_t* idx, const int32_t* n,
                         const int32_t* pos, const ig_step_state* st, int B, int Hg, int d, int cap,
                         float* partial, int32_t* tickets, float* out, int ldo, void* stream) {
  return ig::attend_dispatch(q, ldq, k_cur, v_cur, ldkv, stage, elt, idx, n, nullptr, pos, st, B,
                             Hg, d, cap, partial, tickets, out, ldo, stream);
}

extern "C" int ig_attend_slots(const float* q, int ldq, const float* k_cur, const float* v_cur,
                               int ldkv, const void* stage, int elt, const int32_t* slot_id,
                               const int32_t* slot_used, const int32_t* pos,
                               const ig_step_state* st, int B, int Hg, int d, int cap,
                               float* partial, int32_t* tickets, float* out, int ldo,
                               void* stream) {
  if (!slot_id || !slot_used) return IG_EINVAL;
  return ig::attend_dispatch(q, ldq, k_cur, v_cur, ldkv, stage, elt, slot_id, nullptr, slot_used,
                             pos, st, B, Hg, d, cap, partial, tickets, out, ldo, stream);
}
