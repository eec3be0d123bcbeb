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
#include "plan.cuh"

namespace ig {

constexpr int kSelThreads = 512;            // rows up to kSelLongRows keys
constexpr int kSelThreadsLong = 1024;       // longer rows (C4: 32K): 95 vs 124 us per layer
constexpr int kSelLongRows = 8192;
constexpr int kSelWarps = kSelThreadsLong / kWarp;
constexpr size_t kSelMaxSmem = 220 * 1024;  // ig_topk_rows: keys of rows up to 56K

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

// ---------------------------------------------------------------------------
// ig_select: value-bin select (one CTA per (b, h) row, the row streamed from
// L2 -- rehearse_count wrote it just before -- so no shared-memory copy of the
// keys and no row-length ceiling beyond the 1-bit-per-row take mask).
//
//   P0  min / max of the row;
//   P1  histogram over kBins value bins: bin(x) = min(kBins-1, (hi - x) * scale),
//       a monotone non-increasing map of the score (IEEE subtraction and
//       multiplication round monotonically), so every row of a lower bin
//       outranks every row of a higher bin; a block scan finds the boundary
//       bin b* holding the n-th largest score and `need`, how many of its rows
//       are taken;
//   P2  the rows of b* are gathered (typically a few dozen: kBins bins over the
//       score range) and ranked exactly by (order key desc, row asc) -- the
//       reference's stable argsort (linalg.py:184), -0.0 == +0.0 -- and the
//       taken ones marked in a row bitmap; a boundary bin too full for the
//       candidate buffer (huge outliers, mass ties) is resolved instead by an
//       8-bit radix select over the order keys of its rows;
//   P3  ascending emission with warp ballots / scans, each warp owning one
//       contiguous row range whose count was taken in P2.
// ---------------------------------------------------------------------------
constexpr int kBins = 2048;
constexpr int kCandMax = 1024;
constexpr int kSelMaxRows = 1 << 20;        // take bitmap: 128 KB of shared memory

struct BinShared {
  uint32_t hist[kBins];
  uint32_t cand_key[kCandMax];
  int32_t cand_t[kCandMax];
  uint32_t kmin[kSelWarps], kmax[kSelWarps];
  int scan[kSelWarps];
  int warp_a[kSelWarps];      // rows of the warp's range surely taken
  int warp_b[kSelWarps];      // radix mode: rows of b* whose key == P
  int bstar, need, m, ncand, nn;
  SelShared rx;               // radix fallback
};

__device__ __forceinline__ int vbin(float x, float hi, float scale) {
  return (int)fminf((hi - x) * scale, (float)(kBins - 1));
}

// inclusive block scan of one int per thread (warp scans + a scan of warp totals)
__device__ __forceinline__ int block_incl_scan(int v, int* warp_tot) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += y;
  }
  if (lane == 31) warp_tot[w] = v;
  __syncthreads();
  if (w == 0) {
    int t = lane < nw ? warp_tot[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < nw) warp_tot[lane] = t;
  }
  __syncthreads();
  const int r = v + (w > 0 ? warp_tot[w - 1] : 0);
  __syncthreads();
  return r;
}

// 4 consecutive scores of a row as a float4 (rows t >= s are masked by callers)
__device__ __forceinline__ float4 row4(const float* row, int t) {
  return __ldcg(reinterpret_cast<const float4*>(row + t));
}

// The select of one (b, h) row; returns the number of rows written to
// idx[bh][0:n) (ascending).
template <int THREADS>
__device__ __forceinline__ int select_row(const float* __restrict__ scores, const int32_t* __restrict__ count_sum,
                                          const ig_step_state* __restrict__ st, int Hg, int H_total, int S_max,
                                          int cap_max, double cap_ratio, int min_select, int32_t* __restrict__ idx,
                                          int32_t* __restrict__ n_out, int32_t* __restrict__ err_flag,
                                          const uint32_t* __restrict__ row_range, BinShared& sh,
                                          uint32_t* __restrict__ bits) {
  constexpr int NW = THREADS / kWarp;
  constexpr int PER = kBins / THREADS;
  const int b = blockIdx.y, h = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int s = st->s_len;
  const size_t bh = (size_t)b * Hg + h;
  const float* row = scores + bh * S_max;
  int32_t* out = idx + bh * cap_max;
  if (tid == 0) {
    // n = floor(sum/H + 0.5) == floor((2 sum + H) / 2H) exactly (integers)
    const long long sum = count_sum[b];
    long long n = (2 * sum + H_total) / (2LL * H_total);
    const long long cap = max((long long)floor(cap_ratio * (double)s), (long long)min_select);
    n = min(max(n, (long long)min_select), cap);
    n = min(n, (long long)s);
    int nn = (int)n;
    if (nn > cap_max) {  // caller sized the index buffer too small: flag and clamp
      // a plain store (the flag may live in mapped host memory, where device
      // atomics are not guaranteed): only ever 0 -> 1
      *reinterpret_cast<volatile int32_t*>(err_flag) = 1;
      nn = cap_max;
    }
    if (h == 0) n_out[b] = nn;
    sh.nn = nn;
  }

  // ---- P0: row min / max (order keys) -- from ig_rehearse_count's last-tile
  // pass when it recorded them (row_range), else one pass over the row
  uint32_t kmin = 0xffffffffu, kmax = 0u;
  if (row_range != nullptr) {
    kmax = __ldcg(row_range + 2 * bh);
    kmin = __ldcg(row_range + 2 * bh + 1);
  } else {
    for (int t = tid * 4; t < s; t += THREADS * 4) {
      const float4 v = row4(row, t);
      const float x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (t + i < s) {
          const uint32_t k = order_key(x[i]);
          kmin = min(kmin, k);
          kmax = max(kmax, k);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
      kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
    }
    if (lane == 0) { sh.kmin[w] = kmin; sh.kmax[w] = kmax; }
  }
  for (int i = tid; i < kBins; i += THREADS) sh.hist[i] = 0;
  __syncthreads();
  const int nn = sh.nn;
  if (nn >= s) {
    for (int t = tid; t < s; t += THREADS) out[t] = t;
    return s;
  }
  if (nn <= 0) return 0;
  if (row_range == nullptr) {
    kmin = sh.kmin[0];
    kmax = sh.kmax[0];
    for (int i = 1; i < NW; ++i) { kmin = min(kmin, sh.kmin[i]); kmax = max(kmax, sh.kmax[i]); }
  }
  const float hi = key_to_float(kmax), lo = key_to_float(kmin);
  float scale = (float)kBins / (hi - lo);
  if (!(scale < 1e30f)) scale = 0.f;            // flat (or denormal-range) row: one bin

  // warp w owns rows [t_lo, t_hi), a multiple of 128 (its float4 lanes)
  const int span = ((s + NW - 1) / NW + 127) & ~127;
  const int t_lo = min(s, w * span), t_hi = min(s, t_lo + span);
  // ---- P1: value-bin histogram, boundary bin
  for (int t = tid * 4; t < s; t += THREADS * 4) {
    const float4 v = row4(row, t);
    const float x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (t + i < s) atomicAdd(&sh.hist[vbin(x[i], hi, scale)], 1u);
  }
  __syncthreads();
  {
    int c[PER], tot = 0;
#pragma unroll
    for (int i = 0; i < PER; ++i) { c[i] = (int)sh.hist[tid * PER + i]; tot += c[i]; }
    const int incl = block_incl_scan(tot, sh.scan);
    const int excl = incl - tot;
    if (excl < nn && incl >= nn) {
      int cum = excl;
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        if (cum + c[i] >= nn) {
          sh.bstar = tid * PER + i;
          sh.need = nn - cum;
          sh.m = c[i];
          break;
        }
        cum += c[i];
      }
    }
    if (tid == 0) sh.ncand = 0;
  }
  for (int i = tid; i < (s + 31) / 32; i += THREADS) bits[i] = 0;
  __syncthreads();
  const int bstar = sh.bstar, need = sh.need, m = sh.m;
  // 0: the whole boundary bin is taken; 1: candidates ranked; 2: radix select in b*
  const int mode = (m == need) ? 0 : (m <= kCandMax ? 1 : 2);


  // ---- P2: per-warp counts (+ candidate gather / radix resolve of b*)
  uint32_t P = 0u;          // radix mode: the key of the need-th largest row in b*
  int need_eq = 0;          // radix mode: rows with key == P to take (index order)
  if (mode == 2) {
    SelShared& rx = sh.rx;
    uint32_t prefix = 0u, mask = 0u;
    int nd = need;
    for (int pass = 0; pass < 4; ++pass) {
      const int shift = 24 - 8 * pass;
      for (int i = tid; i < 256; i += THREADS) rx.hist[i] = 0;
      __syncthreads();
      for (int t0 = 0; t0 < s; t0 += THREADS) {
        const int t = t0 + tid;
        bool live = false;
        uint32_t bin = 0;
        if (t < s) {
          const float x = __ldcg(row + t);
          const uint32_t key = order_key(x);
          live = vbin(x, hi, scale) == bstar && (key & mask) == prefix;
          bin = (key >> shift) & 255u;
        }
        const unsigned act = __ballot_sync(0xffffffffu, live);
        if (live) {
          const unsigned peers = __match_any_sync(act, bin);
          if ((__ffs(peers) - 1) == lane) atomicAdd(&rx.hist[bin], (uint32_t)__popc(peers));
        }
      }
      __syncthreads();
      if (w == 0) pick_digit(rx, prefix, nd, shift);
      __syncthreads();
      prefix = rx.prefix;
      nd = rx.need;
      mask |= 255u << shift;
      __syncthreads();
    }
    P = prefix;
    need_eq = nd;
  }
  int a = 0, e = 0;
  // short rows, no tie cut: the warp compacts the rows of bins <= b* of its
  // range into shared memory as it counts them (b* rows flagged in bit 31),
  // so P3 is a copy of those entries instead of a second pass over the row
  constexpr bool kCompact = THREADS <= 512;
  int32_t* wbuf = reinterpret_cast<int32_t*>(bits + (S_max + 31) / 32) + t_lo;
  int wcount = 0;
  const unsigned lt_mask = (1u << lane) - 1u;
  if (kCompact && mode != 2) {
    for (int t0 = t_lo; t0 < t_hi; t0 += 128) {
      const int t = t0 + lane * 4;
      int bn[4] = {kBins, kBins, kBins, kBins};
      float x[4] = {0.f, 0.f, 0.f, 0.f};
      if (t < t_hi) {
        const float4 v = row4(row, t);
        x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (t + i < t_hi) bn[i] = vbin(x[i], hi, scale);
      }
      int before = 0, total = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const unsigned mb = __ballot_sync(0xffffffffu, bn[i] <= bstar);
        before += __popc(mb & lt_mask);
        total += __popc(mb);
      }
      int pos = wcount + before;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (bn[i] < bstar || (bn[i] == bstar && mode == 0)) {
          ++a;
          wbuf[pos++] = t + i;
        } else if (bn[i] == bstar) {
          wbuf[pos++] = (t + i) | (int)0x80000000;
          const int slot = atomicAdd(&sh.ncand, 1);
          sh.cand_key[slot] = order_key(x[i]);
          sh.cand_t[slot] = t + i;
        }
      }
      wcount += total;
    }
  } else
  for (int t = t_lo + lane * 4; t < t_hi; t += 128) {
    const float4 v = row4(row, t);
    const float x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (t + i >= t_hi) break;
      const int bn = vbin(x[i], hi, scale);
      if (bn < bstar) {
        ++a;
      } else if (bn == bstar) {
        if (mode == 0) {
          ++a;
        } else if (mode == 1) {
          const int slot = atomicAdd(&sh.ncand, 1);
          sh.cand_key[slot] = order_key(x[i]);
          sh.cand_t[slot] = t + i;
        } else {
          const uint32_t k = order_key(x[i]);
          a += k > P;
          e += k == P;
        }
      }
    }
  }
  a = warp_sum(a);
  e = warp_sum(e);
  __syncthreads();
  if (mode == 1) {
    // rank the m candidates: (key desc, row asc) -- the reference's stable order
    for (int i = tid; i < m; i += THREADS) {
      const uint32_t ki = sh.cand_key[i];
      const int ti = sh.cand_t[i];
      int rank = 0;
      for (int j = 0; j < m; ++j) {
        const uint32_t kj = sh.cand_key[j];
        rank += (kj > ki) || (kj == ki && sh.cand_t[j] < ti);
      }
      if (rank < need) atomicOr(&bits[ti >> 5], 1u << (ti & 31));
    }
    __syncthreads();
    int tk = 0;     // taken candidates in my range (a is already the warp total)
    for (int wd = (t_lo >> 5) + lane; wd < (t_hi + 31) >> 5; wd += 32) tk += __popc(bits[wd]);
    a += warp_sum(tk);
  }
  if (lane == 0) { sh.warp_a[w] = a; sh.warp_b[w] = e; }
  __syncthreads();

  // ---- P3: ascending emission
  int out_off = 0, eq_before = 0;
  if (kCompact && mode != 2) {
    out_off = warp_sum(lane < w ? sh.warp_a[lane] : 0);      // rows of the warps before mine
    for (int j0 = 0; j0 < wcount; j0 += 32) {
      const int j = j0 + lane;
      const int ent = j < wcount ? wbuf[j] : 0;
      const int t = ent & 0x7fffffff;
      const bool take = j < wcount && (ent >= 0 || ((bits[t >> 5] >> (t & 31)) & 1u));
      const unsigned mb = __ballot_sync(0xffffffffu, take);
      if (take) out[out_off + __popc(mb & lt_mask)] = t;
      out_off += __popc(mb);
    }
    return nn;
  }
  if (mode != 2) {
    out_off = warp_sum(lane < w ? sh.warp_a[lane] : 0);      // rows of the warps before mine
    // no tie cut inside b*: a row is taken iff its bin is < b*, or == b* and
    // (whole bin, or its candidate bit is set).  Ranks from four ballots (one
    // per float4 position): the rows before (lane, i) are every taken row of
    // lanes < lane plus this lane's taken rows at positions < i.
    for (int t0 = t_lo; t0 < t_hi; t0 += 128) {
      const int t = t0 + lane * 4;
      int bn[4] = {kBins, kBins, kBins, kBins};
      if (t < t_hi) {
        const float4 v = row4(row, t);
        const float x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (t + i < t_hi) bn[i] = vbin(x[i], hi, scale);
      }
      bool take[4];
      int before = 0, total = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        take[i] = bn[i] < bstar ||
                  (bn[i] == bstar && (mode == 0 || ((bits[(t + i) >> 5] >> ((t + i) & 31)) & 1u)));
        const unsigned mb = __ballot_sync(0xffffffffu, take[i]);
        before += __popc(mb & lt_mask);
        total += __popc(mb);
      }
      int pos = out_off + before;
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (take[i]) out[pos++] = t + i;
      out_off += total;
    }
    return nn;
  }
  for (int i = 0; i < w; ++i) {
    const int ee = min(sh.warp_b[i], max(0, need_eq - eq_before));
    eq_before += sh.warp_b[i];
    out_off += sh.warp_a[i] + ee;
  }
  for (int t0 = t_lo; t0 < t_hi; t0 += 128) {
    const int t = t0 + lane * 4;
    float x[4] = {0.f, 0.f, 0.f, 0.f};
    if (t < t_hi) {
      const float4 v = row4(row, t);
      x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
    }
    bool sure[4], eq[4];
    int ns = 0, ne = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      sure[i] = eq[i] = false;
      if (t + i < t_hi) {
        const int bn = vbin(x[i], hi, scale);
        if (bn < bstar) {
          sure[i] = true;
        } else if (bn == bstar) {
          if (mode == 0) sure[i] = true;
          else if (mode == 1) sure[i] = (bits[(t + i) >> 5] >> ((t + i) & 31)) & 1u;
          else {
            const uint32_t k = order_key(x[i]);
            sure[i] = k > P;
            eq[i] = k == P;
          }
        }
      }
      ne += eq[i];
    }
    // eq rows before this lane (index order), then within the lane
    int e_incl = ne;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, e_incl, o);
      if (lane >= o) e_incl += y;
    }
    int e_run = eq_before + e_incl - ne;
    bool take[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      take[i] = sure[i] || (eq[i] && e_run < need_eq);
      e_run += eq[i];
      ns += take[i];
    }
    int incl = ns;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    int pos = out_off + incl - ns;
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (take[i]) out[pos++] = t + i;
    out_off += __shfl_sync(0xffffffffu, incl, 31);
    eq_before += __shfl_sync(0xffffffffu, e_incl, 31);
  }
  return nn;
}


// ig_select (plan == false) / ig_select_plan (plan == true: the resident plan
// of the same (b, h) runs in the same CTA on the selection just written --
// one launch and one dependent hop fewer on the speculation chain)
template <int THREADS, bool PLAN>
__global__ void __launch_bounds__(THREADS) __maxnreg__(THREADS == 1024 ? 64 : THREADS == 256 ? 40 : 32)   // no spills; 256: 6 CTAs/SM
select_kernel(const float* __restrict__ scores, const int32_t* __restrict__ count_sum,
              const ig_step_state* __restrict__ st, int Hg, int H_total, int S_max, int cap_max,
              double cap_ratio, int min_select, int32_t* __restrict__ idx,
              int32_t* __restrict__ n_out, int32_t* __restrict__ err_flag, const int32_t* __restrict__ pos_prev,
              int32_t* __restrict__ slot_id, int32_t* __restrict__ slot_used, int32_t* __restrict__ frow,
              int32_t* __restrict__ fslot, int32_t* __restrict__ fcount,
              unsigned long long* __restrict__ moved_rows, const uint32_t* __restrict__ row_range) {
  __shared__ BinShared sh;
  extern __shared__ uint32_t bits[];            // take bitmap, ceil(S_max / 32) words (+ plan scratch)
  const int n = select_row<THREADS>(scores, count_sum, st, Hg, H_total, S_max, cap_max, cap_ratio, min_select,
                                    idx, n_out, err_flag, row_range, sh, bits);
  if constexpr (PLAN) {
    const size_t bh = (size_t)blockIdx.y * Hg + blockIdx.x;
    // after the take bitmap and the compaction buffer (short-row kernels)
    int32_t* freelist = reinterpret_cast<int32_t*>(bits + (S_max + 31) / 32) + (THREADS <= 512 ? S_max : 0);
    uint8_t* matched = reinterpret_cast<uint8_t*>(freelist + cap_max);
    __syncthreads();                  // the selection (global) and the bitmap reads are done
    plan_row(idx + bh * cap_max, n, pos_prev ? pos_prev[bh] : -1, slot_id + bh * cap_max, slot_used + bh,
             frow + bh * cap_max, fslot + bh * cap_max, fcount + bh, moved_rows, freelist, matched, sh.scan);
  }
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

namespace ig {
static int select_launch(const float* scores, const int32_t* count_sum, const ig_step_state* st, int B, int Hg,
                         int H_total, int S_max, int cap_max, double cap_ratio, int min_select, int32_t* idx,
                         int32_t* n_out, int32_t* err_flag, const int32_t* pos_prev, int32_t* slot_id,
                         int32_t* slot_used, int32_t* frow, int32_t* fslot, int32_t* fcount, int64_t* moved_rows,
                         const uint32_t* row_range, void* stream) {
  if (B < 1 || Hg < 1 || H_total < Hg || S_max < 1 || cap_max < 1 || !(cap_ratio > 0) ||
      cap_ratio > 1 || min_select < 1 || !scores || !count_sum || !st || !idx || !n_out ||
      !err_flag)
    return IG_EINVAL;
  if (S_max > kSelMaxRows) return IG_EINVAL;
  const bool plan = slot_id != nullptr;
  if (plan && (!slot_used || !frow || !fslot || !fcount)) return IG_EINVAL;
  // the take bitmap (+ the plan's free list and match flags)
  const bool short_rows = S_max <= kSelLongRows;
  const size_t smem = (size_t)(S_max + 31) / 32 * 4 + (short_rows ? (size_t)S_max * 4 : 0) +
                      (plan ? (size_t)cap_max * 5 : 0);
  if (smem > 200 * 1024) return IG_EINVAL;
  // rows up to kSelLongRows: 256 threads (5 CTAs/SM: C3's 640 rows in one wave);
  // IG_SELECT_THREADS=512 for the A/B
  static const int short_threads = [] {
    const char* e = getenv("IG_SELECT_THREADS");
    return e && atoi(e) == 512 ? kSelThreads : 256;
  }();
  const int threads = S_max > kSelLongRows ? kSelThreadsLong : short_threads;
  auto pick = [&](auto k512, auto k256, auto k1024) {
    return S_max > kSelLongRows ? k1024 : (short_threads == 256 ? k256 : k512);
  };
  auto kern = plan ? pick(select_kernel<kSelThreads, true>, select_kernel<256, true>,
                          select_kernel<kSelThreadsLong, true>)
                   : pick(select_kernel<kSelThreads, false>, select_kernel<256, false>,
                          select_kernel<kSelThreadsLong, false>);
  if (smem > 16 * 1024)  // dynamic + static (~25 KB) must fit: opt in early
    IG_CUDA_STATUS(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<dim3(Hg, B), threads, smem, (cudaStream_t)stream>>>(
      scores, count_sum, st, Hg, H_total, S_max, cap_max, cap_ratio, min_select, idx, n_out, err_flag, pos_prev,
      slot_id, slot_used, frow, fslot, fcount, reinterpret_cast<unsigned long long*>(moved_rows), row_range);
  IG_LAUNCH_STATUS();
  return IG_OK;
}
}  // namespace ig

extern "C" int ig_select(const float* scores, const int32_t* count_sum, const ig_step_state* st,
                         int B, int Hg, int H_total, int S_max, int cap_max, double cap_ratio,
                         int min_select, int32_t* idx, int32_t* n_out, int32_t* err_flag,
                         const uint32_t* row_range, void* stream) {
  return ig::select_launch(scores, count_sum, st, B, Hg, H_total, S_max, cap_max, cap_ratio, min_select, idx, n_out,
                           err_flag, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, row_range,
                           stream);
}

extern "C" int ig_select_plan(const float* scores, const int32_t* count_sum, const ig_step_state* st, int B,
                              int Hg, int H_total, int S_max, int cap_max, double cap_ratio, int min_select,
                              int32_t* idx, int32_t* n_out, int32_t* err_flag, const int32_t* pos_prev,
                              int32_t* slot_id, int32_t* slot_used, int32_t* frow, int32_t* fslot,
                              int32_t* fcount, int64_t* moved_rows, const uint32_t* row_range, void* stream) {
  if (!slot_id) return IG_EINVAL;
  return ig::select_launch(scores, count_sum, st, B, Hg, H_total, S_max, cap_max, cap_ratio, min_select, idx, n_out,
                           err_flag, pos_prev, slot_id, slot_used, frow, fslot, fcount, moved_rows, row_range,
                           stream);
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
