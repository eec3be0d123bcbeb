// Weight-streaming skinny GEMM over PACKED weights: Y[M][N] = X[M][K] . W[K][N]
// (+ epilogue), M <= 32 sequences, 3xTF32 split precision on the tensor cores
// (same arithmetic as sgemm_tcw_kernel in gemm.cu: f32-level accuracy).
//
// Why a packed layout.  The decode step streams ~54 GB of f32 weights per
// step (C3) through these projections; the row-major kernels issue one 16-B
// cp.async per thread per vector (issue-bound) or 512-B TMA rows
// (request-rate-bound), and their fixed (tile, K-slice) grid leaves pipeline
// fill/drain bubbles per CTA.  The weights are the engine's own HBM objects,
// so they are re-laid ONCE at load time (ig_sgemm_pack) into 16-KB blocks:
//
//   P[tile][kc] = block of 32 weight rows (kc) x 128 output columns (tile),
//   inside a block: [k8 (4)][warp column slab wi (4)][j (2)][lane (32)][4]
//   with lane = 4 g + t holding W[k][c0 + g], W[k][c0 + g + 8],
//   W[k][c0 + g + 16], W[k][c0 + g + 24] at
//   k = 32 kc + 16 (k8 / 2) + 4 t + 2 (k8 % 2) + j, c0 = 128 tile + 32 wi --
//   exactly the A fragments (rows g / g+8 of the two m16 tiles, k columns
//   t / t+4) of mma.m16n8k8 with the weights as the A operand, so every
//   shared load is one conflict-free 512-B LDS.128 per warp.  The MMA's k
//   order is permuted (the sum over k does not care) so that a lane's x
//   fragments for a block are 4 consecutive floats: one 16-B load.  Blocks are contiguous in (tile, kc) order: the whole GEMM is ONE
//   sequential stream.
//
// Kernel: persistent, stream-K.  CTA c of G owns global chunks
// [c T / G, (c+1) T / G) of the T = tiles x chunks_per_tile blocks.  A
// producer warp moves each block into a STAGES-deep shared ring with one
// 16-KB cp.async.bulk (mbarrier complete_tx); 8 consumer warps (2 k-groups x
// 4 column slabs) release stages through an `empty` mbarrier, so the ring
// stays full across tile boundaries and no CTA ever drains its pipeline
// before the kernel's end.  x fragments come straight from global memory
// (L2-resident, 2 KB per block; one float4 per lane and 8-row group) two
// blocks ahead in registers.  At the end of
// a tile segment the k-groups are summed in shared memory (fixed order); a
// segment covering its whole tile writes Y directly, otherwise it goes to a
// per-CTA workspace slot and the last CTA of the tile (ticket) sums the
// segments in CTA order and applies the epilogue -- deterministic for a given
// grid.
#include <cstdlib>

#include "common.cuh"

namespace ig {
namespace packed {

constexpr int kTileN = 128;            // output columns per tile
constexpr int kChunkK = 64;            // weight rows per block
constexpr int kBlockFloats = kTileN * kChunkK;   // 8192 floats = 32 KB
// A CTA = KG k-groups x 4 column slabs of 32 columns: KG = 2 (8 warps, 2 CTAs
// per SM) or KG = 4 (16 warps, 1 CTA per SM with a deeper ring); each k-group
// takes 4 / KG of a block's k16 steps.
// (CTAs per SM, ring stages): M <= 16 runs 2 x 3 (96-KB rings); M <= 32 (64
// accumulator registers per lane) 1 x 6.  Registers: an SM
// sub-partition holds 16K, i.e. 2 CTAs x 8 warps -> 128 per thread, 3 -> 80.
template <int WARPS_PER_SM> struct RegCap {   // 64K registers per SM, 16K per sub-partition
  static constexpr int v = WARPS_PER_SM <= 8 ? 255 : (WARPS_PER_SM <= 16 ? 128 : 80);
};

__device__ __forceinline__ void bar_init(uint32_t bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void bar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void bar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W_%=;\n}" ::"r"(bar), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
template <int THREADS>
__device__ __forceinline__ void consumers_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(THREADS) : "memory");
}

constexpr float kLoScale = 2048.f;           // lo parts carry the next 11 bits
constexpr float kLoScaleInv = 1.f / 2048.f;

// (x0, x1) -> hi = f16x2(x), lo = f16x2((x - hi) * 2^11): x = hi + lo 2^-11 to
// ~22 bits (the same 11 + 11 significand bits as a 3xTF32 split)
__device__ __forceinline__ void split_h2(float x0, float x1, uint32_t& hi, uint32_t& lo) {
  const __half2 h = __floats2half2_rn(x0, x1);
  const float2 f = __half22float2(h);
  const __half2 l = __floats2half2_rn((x0 - f.x) * kLoScale, (x1 - f.y) * kLoScale);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
}
__device__ __forceinline__ void mma_h(float* c, const uint4& a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b0), "r"(b1));
}

// Optional all-reduce push (head-parallel W_O / FFN-out, csrc/collective.cu):
// final values go to slot [parity][rank] of every rank's IPC-mapped receive
// buffer instead of Y, and the grid's last CTA raises this rank's flag in
// every rank -- the collective's push folded into the GEMM epilogue.
struct PeerOut {
  const uint64_t* recv = nullptr;    // [world] receive-buffer bases (u64)
  const uint64_t* flags = nullptr;   // [world] flag-array bases
  const ig_step_state* st = nullptr;
  uint32_t* done = nullptr;          // grid-completion counter (local, left zeroed)
  int rank = 0, world = 1, call = 0, calls = 1;
  int l2pf = 0;                      // prefetch this CTA's blocks beyond the ring into L2 (IG_PACKED_L2PF)
};

// chunk index -> CTA that owns it, for the split [c T / G, (c+1) T / G)
__device__ __forceinline__ int owner(int x, int T, int G) { return (int)(((long)(x + 1) * G - 1) / T); }
__device__ __forceinline__ int first_chunk(int c, int T, int G) { return (int)((long)c * T / G); }

template <int NB, int CPS, int kStages, int KG>   // NB 8-sequence MMA n tiles: M <= 8 NB
__global__ void __launch_bounds__(KG * 4 * 32) __maxnreg__(RegCap<CPS * KG * 4>::v)
sgemm_packed_kernel(const float* __restrict__ X, int ldx, const float* __restrict__ P,
                    float* __restrict__ Y, int ldy, const float* __restrict__ R, int ldr, int M,
                    int N, int K, int C, int epilogue, float* __restrict__ ws,
                    int32_t* __restrict__ tickets, const PeerOut po) {
  extern __shared__ __align__(128) float smem[];
  constexpr int MTW = 2;                        // m16 tiles per warp (32 columns)
  constexpr int PER = MTW * NB * 4;             // accumulator floats per lane
  constexpr int kWarps = KG * 4, kSteps = 4 / KG;
  float* ring = smem;                                        // [kStages][4096]
  float* red = smem + kStages * kBlockFloats;                // [KG-1][4 warps][PER][32]
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
  __shared__ int last;

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int G = gridDim.x, c = blockIdx.x;
  const int tiles = (N + kTileN - 1) / kTileN;
  const int T = tiles * C;
  const int g0 = first_chunk(c, T, G), g1 = first_chunk(c + 1, T, G);
  const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring);
  const uint32_t full_s = (uint32_t)__cvta_generic_to_shared(full);
  const uint32_t empty_s = (uint32_t)__cvta_generic_to_shared(empty);

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      bar_init(full_s + 8 * s, 1);
      bar_init(empty_s + 8 * s, kWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // Thread 0 keeps the ring full: chunks g0 .. g0 + S - 1 now, then at
  // iteration j the stage released at iteration j - 1 gets chunk j - 1 + S
  // (one iteration of slack, so the wait on `empty` rarely blocks).
  auto issue = [&](int jj, int st) {
    bar_expect_tx(full_s + 8 * st, kBlockFloats * 4);
    bulk_g2s(ring_s + st * kBlockFloats * 4, P + (size_t)(g0 + jj) * kBlockFloats,
             kBlockFloats * 4, full_s + 8 * st);
  };
  if (tid == 0) {
    for (int jj = 0; jj < kStages && g0 + jj < g1; ++jj) issue(jj, jj);
    // small GEMMs (few blocks per CTA): the rest of this CTA's blocks into L2
    // while the previous kernel drains
    if (g1 - g0 <= po.l2pf)
      for (int jj = kStages; g0 + jj < g1; ++jj)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(P + (size_t)(g0 + jj) * kBlockFloats),
                     "r"(kBlockFloats * 4)
                     : "memory");
  }
  // Programmatic dependent launch: the weight stream above does not depend on
  // the previous kernel, so this grid may start (and fill its rings) while
  // that kernel drains; x, R, Y, the workspace and the tickets are touched
  // only after the wait (full completion + visibility of the previous grid).
  // The next GEMM may likewise launch as soon as SMs free up.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  uint32_t po_epoch = 0;
  size_t po_off = 0;                      // my slot within every rank's receive buffer
  if (po.recv != nullptr) {
    const uint32_t seqno = (uint32_t)po.st->step * (uint32_t)po.calls + (uint32_t)po.call;
    po_epoch = seqno + 1u;
    po_off = ((size_t)(seqno & 1u) * po.world + po.rank) * (size_t)M * N;
  }
  auto store = [&](int m, int n, float v) {
    if (po.recv == nullptr) {
      Y[(size_t)m * ldy + n] = v;
    } else {
      for (int r = 0; r < po.world; ++r)
        reinterpret_cast<float*>(po.recv[r])[po_off + (size_t)m * N + n] = v;
    }
  };

  // ---- kg = k-group (k16 steps 2 kg, 2 kg + 1 of a block), wi = 32-column
  // slab of the tile
  const int g = lane >> 2, t = lane & 3;
  const int kg = w >> 2, wi = w & 3;
  float big[MTW][NB][4], small[MTW][NB][4];
#pragma unroll
  for (int mt = 0; mt < MTW; ++mt)
#pragma unroll
    for (int nb = 0; nb < NB; ++nb)
#pragma unroll
      for (int e = 0; e < 4; ++e) big[mt][nb][e] = small[mt][nb][e] = 0.f;

  // x fragments of a block at row kc: rows m = 8 nb + g,
  // k = 64 kc + 32 kg + 16 s + 4 t + (0..3) for k16 step s
  const float* xrow[NB];
  bool mok[NB];
#pragma unroll
  for (int nb = 0; nb < NB; ++nb) {
    mok[nb] = 8 * nb + g < M;
    xrow[nb] = X + (size_t)(mok[nb] ? 8 * nb + g : 0) * ldx + kSteps * 16 * kg + 4 * t;
  }
  auto load_x = [&](int kc, bool ok, float4 (&xv)[NB][kSteps]) {
#pragma unroll
    for (int nb = 0; nb < NB; ++nb)
#pragma unroll
      for (int s2 = 0; s2 < kSteps; ++s2) {
        const int k = kc * kChunkK + kSteps * 16 * kg + 16 * s2 + 4 * t;
        xv[nb][s2] = (ok && mok[nb] && k < K)
                         ? __ldg(reinterpret_cast<const float4*>(xrow[nb] + kc * kChunkK + 16 * s2))
                         : make_float4(0.f, 0.f, 0.f, 0.f);
      }
  };
  float4 xa[NB][kSteps], xb[NB][kSteps];
  int kc = g0 % C, tile = g0 / C;          // chunk g0 + j = (tile, kc)
  int kcn = kc + 1 == C ? 0 : kc + 1;      // row block of the next chunk
  load_x(kc, true, xb);
  int st = 0, ph = 0;                      // ring stage and its phase parity

  for (int j = 0, i = g0; i < g1; ++i, ++j) {
    // xb (loaded one iteration ago) becomes current before the next block's
    // load reuses it: the copy waits only if that load has not landed yet
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) { xa[nb][0] = xb[nb][0]; xa[nb][1] = xb[nb][1]; }
    load_x(kcn, i + 1 < g1, xb);
    if (tid == 0 && j >= 1 && i - 1 + kStages < g1) {
      const int sp = st == 0 ? kStages - 1 : st - 1;        // stage of iteration j - 1
      bar_wait(empty_s + 8 * sp, (sp == kStages - 1 ? ph ^ 1 : ph));
      issue(j - 1 + kStages, sp);
    }
    bar_wait(full_s + 8 * st, ph);
    const uint4* blk = reinterpret_cast<const uint4*>(ring + st * kBlockFloats);
#pragma unroll
    for (int s2 = 0; s2 < kSteps; ++s2) {
      const int k16 = kSteps * kg + s2;
      uint4 a[MTW][2];
#pragma unroll
      for (int mt = 0; mt < MTW; ++mt)
#pragma unroll
        for (int pt = 0; pt < 2; ++pt) a[mt][pt] = blk[(((k16 * 4 + wi) * 2 + mt) * 2 + pt) * 32 + lane];
#pragma unroll
      for (int nb = 0; nb < NB; ++nb) {
        uint32_t bh0, bl0, bh1, bl1;
        split_h2(xa[nb][s2].x, xa[nb][s2].y, bh0, bl0);
        split_h2(xa[nb][s2].z, xa[nb][s2].w, bh1, bl1);
#pragma unroll
        for (int mt = 0; mt < MTW; ++mt) {
          mma_h(small[mt][nb], a[mt][1], bh0, bh1);
          mma_h(small[mt][nb], a[mt][0], bl0, bl1);
          mma_h(big[mt][nb], a[mt][0], bh0, bh1);
        }
      }
    }
    __syncwarp();
    if (lane == 0) bar_arrive(empty_s + 8 * st);
    if (++st == kStages) { st = 0; ph ^= 1; }
    const bool seg_end = kc == C - 1 || i == g1 - 1;
    const int seg_tile = tile;
    kc = kcn;
    if (kc == 0) ++tile;
    kcn = kc + 1 == C ? 0 : kc + 1;
    if (!seg_end) continue;

    // ---- end of a tile segment: k-group 1 hands its sums to k-group 0
#pragma unroll
    for (int mt = 0; mt < MTW; ++mt)
#pragma unroll
      for (int nb = 0; nb < NB; ++nb)
#pragma unroll
        for (int e = 0; e < 4; ++e) big[mt][nb][e] = fmaf(small[mt][nb][e], kLoScaleInv, big[mt][nb][e]);
    if (kg > 0) {
#pragma unroll
      for (int mt = 0; mt < MTW; ++mt)
#pragma unroll
        for (int nb = 0; nb < NB; ++nb)
#pragma unroll
          for (int e = 0; e < 4; ++e)
            red[(((kg - 1) * 4 + wi) * PER + (mt * NB + nb) * 4 + e) * 32 + lane] = big[mt][nb][e];
    }
    consumers_sync<kWarps * 32>();
    const int t0 = seg_tile * C;
    const int cf = owner(t0, T, G), cl = owner(t0 + C - 1, T, G);
    const bool whole = cf == cl;
    const size_t seg_elems = (size_t)M * kTileN;
    const float inv_scale = __ldg(P + (size_t)T * kBlockFloats + seg_tile);
    // my workspace slot: 0 if this tile holds my first chunk, else 1
    float* part = ws + ((size_t)c * 2 + (g0 / C == seg_tile ? 0 : 1)) * seg_elems;
    if (kg == 0) {
#pragma unroll
      for (int mt = 0; mt < MTW; ++mt)
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            float v = big[mt][nb][e];
#pragma unroll
            for (int gg = 1; gg < KG; ++gg)             // k-groups in fixed order
              v += red[(((gg - 1) * 4 + wi) * PER + (mt * NB + nb) * 4 + e) * 32 + lane];
            v *= inv_scale;
            // C fragment: e = 0/1 -> (column g, seq 2t / 2t+1), e = 2/3 -> (column g + 8, ...)
            const int col = 32 * wi + 16 * mt + g + 8 * (e >> 1);
            const int m = 8 * nb + 2 * t + (e & 1);
            if (m < M) {
              if (whole) {
                const int n = seg_tile * kTileN + col;
                if (n < N) {
                  if (epilogue == 1) v = fmaxf(v, 0.f);
                  else if (epilogue == 2) v = __fadd_rn(R[(size_t)m * ldr + n], v);
                  store(m, n, v);
                }
              } else {
                part[(size_t)m * kTileN + col] = v;
              }
            }
          }
        }
    }
#pragma unroll
    for (int mt = 0; mt < MTW; ++mt)
#pragma unroll
      for (int nb = 0; nb < NB; ++nb)
#pragma unroll
        for (int e = 0; e < 4; ++e) big[mt][nb][e] = small[mt][nb][e] = 0.f;
    if (whole) {
      consumers_sync<kWarps * 32>();          // red is rewritten at the next segment end
      continue;
    }
    __threadfence();
    consumers_sync<kWarps * 32>();
    if (tid == 0) last = atomicAdd(tickets + seg_tile, 1) == cl - cf;
    consumers_sync<kWarps * 32>();
    if (!last) continue;
    __threadfence();
    // segment s of the tile = CTA cf + s; only CTA cf can have started in an
    // earlier tile (then its segment is in slot 1).  Each thread sums float4s
    // of all segments with the loads batched 8 deep (one L2 round trip per 8
    // segments, not one per segment), in segment order.
    const int nseg = cl - cf + 1;
    const float* seg0 = ws + ((size_t)cf * 2 + (first_chunk(cf, T, G) < t0 ? 1 : 0)) * seg_elems;
    for (int e4 = tid; e4 < M * (kTileN / 4); e4 += kWarps * 32) {
      float4 acc = __ldcg(reinterpret_cast<const float4*>(seg0) + e4);
      for (int sg = 1; sg < nseg; sg += 8) {
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (sg + u < nseg)
            v[u] = __ldcg(reinterpret_cast<const float4*>(ws + (size_t)(cf + sg + u) * 2 * seg_elems) + e4);
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (sg + u < nseg) {
            acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w;
          }
      }
      const int m = (4 * e4) / kTileN, n0 = seg_tile * kTileN + (4 * e4) % kTileN;
      const float a4[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int n = n0 + q;
        if (n >= N) continue;
        float v = a4[q];
        if (epilogue == 1) v = fmaxf(v, 0.f);
        else if (epilogue == 2) v = __fadd_rn(R[(size_t)m * ldr + n], v);
        store(m, n, v);
      }
    }
    if (tid == 0) tickets[seg_tile] = 0;
    consumers_sync<kWarps * 32>();
  }
  if (po.recv != nullptr) {               // every final value of this grid is pushed
    consumers_sync<kWarps * 32>();
    if (tid == 0) {
      __threadfence_system();
      if (atomicAdd(po.done, 1u) == gridDim.x - 1) {
        *po.done = 0u;
        __threadfence_system();
        const int par = (int)((po_epoch - 1u) & 1u);
        for (int r = 0; r < po.world; ++r)
          asm volatile("st.release.sys.global.u32 [%0], %1;"
                       ::"l"(reinterpret_cast<uint32_t*>(po.flags[r]) + par * po.world + po.rank),
                       "r"(po_epoch) : "memory");
      }
    }
  }
}

// Per column tile: scale = 2^(14 - e), max |W| < 2^e, so every scaled weight
// and its lo part are f16 normals down to 2^-28 of the tile's max; the
// kernel's epilogue multiplies by the stored 1 / scale (exact).
__global__ void tile_scale_kernel(const float* __restrict__ W, int ldw, int N, int K,
                                  float* __restrict__ inv_scale, float* __restrict__ scale) {
  __shared__ float red[32];
  const int tile = blockIdx.x;
  float mx = 0.f;
  for (int e = threadIdx.x; e < K * kTileN; e += blockDim.x) {
    const int k = e / kTileN, n = tile * kTileN + e % kTileN;
    if (n < N) mx = fmaxf(mx, fabsf(W[(size_t)k * ldw + n]));
  }
  mx = warp_max(mx);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) mx = fmaxf(mx, red[i]);
    mx = fmaxf(mx, red[0]);
    int e = 0;
    if (mx > 0.f) frexpf(mx, &e);            // mx = f 2^e, 0.5 <= f < 1
    scale[tile] = ldexpf(1.f, 14 - e);
    inv_scale[tile] = ldexpf(1.f, e - 14);
  }
}

// one 16-B unit per thread: unit u of block (tile, kc) =
// (((k16 * 4 + wi) * 2 + mt) * 2 + part) * 32 + lane, holding A registers
// a0..a3 of mma.m16n8k16 (f16 pairs): register r, half q is
// W[k][n] with k = 32 kc + 16 k16 + 4 t + 2 (r >> 1) + q,
// n = 128 tile + 32 wi + 16 mt + g + 8 (r & 1); part 0 = hi, 1 = lo.
__global__ void pack_kernel(const float* __restrict__ W, int ldw, int N, int K, int C,
                            const float* __restrict__ scale, uint4* __restrict__ P, size_t units) {
  for (size_t u = blockIdx.x * (size_t)blockDim.x + threadIdx.x; u < units;
       u += (size_t)gridDim.x * blockDim.x) {
    const int lane = (int)(u & 31), part = (int)((u >> 5) & 1), mt = (int)((u >> 6) & 1);
    const int wi = (int)((u >> 7) & 3), k16 = (int)((u >> 9) & 3);
    const size_t blk = u >> 11;
    const int kc = (int)(blk % C), tile = (int)(blk / C);
    const int g = lane >> 2, t = lane & 3;
    const float sc = scale[tile];
    uint32_t r32[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      float h2[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int k = kc * kChunkK + 16 * k16 + 4 * t + 2 * (r >> 1) + q;
        const int n = tile * kTileN + 32 * wi + 16 * mt + g + 8 * (r & 1);
        const float w = (k < K && n < N) ? W[(size_t)k * ldw + n] * sc : 0.f;
        const float hi = __half2float(__float2half_rn(w));
        h2[q] = part == 0 ? hi : (w - hi) * kLoScale;
      }
      const __half2 hv = __floats2half2_rn(h2[0], h2[1]);
      r32[r] = *reinterpret_cast<const uint32_t*>(&hv);
    }
    P[u] = make_uint4(r32[0], r32[1], r32[2], r32[3]);
  }
}

inline int num_sms() {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms < 1)
      sms = 148;
  }
  return sms;
}

inline int grid_for(int N, int K, int cps) {
  const long T = (long)((N + kTileN - 1) / kTileN) * ((K + kChunkK - 1) / kChunkK);
  long G = (long)num_sms() * cps;
  if (G > T) G = T;
  return (int)G;
}

// IG_PACKED_CTA: 0 (default) 2 x 8-warp CTAs per SM; 16: one 16-warp CTA, 6-deep
// ring; 8: one 8-warp CTA, 3-deep ring (half the SM's registers and shared
// memory left to the kernels of the other streams)
inline int packed_cta_mode() {
  static const int m = [] {
    const char* e = getenv("IG_PACKED_CTA");
    return e ? atoi(e) : 0;
  }();
  return m == 16 || m == 8 ? m : 0;
}

// IG_PACKED_L2PF=N: a CTA with <= N blocks prefetches the ones beyond its ring
// into L2 before griddepcontrol.wait (A/B; 0 = off)
inline int packed_l2pf() {
  static const int n = [] {
    const char* e = getenv("IG_PACKED_L2PF");
    return e ? atoi(e) : 0;
  }();
  return n;
}

inline int ctas_per_sm(int M) {
  // IG_PACKED_CTA=16: one 16-warp CTA per SM with a 6-deep ring (more bytes in
  // flight, fewer CTA fix-ups) -- measured equal or slower (ffn_out 4.7 vs 5.6
  // TB/s), so 2 x 8-warp CTAs stay the default
  return M <= 16 && packed_cta_mode() == 0 ? 2 : 1;
}

template <int NB, int CPS, int STAGES, int KG>
int launch(const float* X, int ldx, const float* P, float* Y, int ldy, const float* R, int ldr,
           int M, int N, int K, int epilogue, float* ws, int32_t* tickets, cudaStream_t s,
           const PeerOut& po) {
  const int C = (K + kChunkK - 1) / kChunkK;
  const int G = grid_for(N, K, CPS);
  const size_t smem = (size_t)(STAGES * kBlockFloats + (KG - 1) * 4 * 2 * NB * 4 * 32) * sizeof(float);
  auto kern = sgemm_packed_kernel<NB, CPS, STAGES, KG>;
  IG_CUDA_STATUS(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(KG * 4 * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  PeerOut pl = po;
  pl.l2pf = packed_l2pf();
  IG_CUDA_STATUS(cudaLaunchKernelEx(&cfg, kern, X, ldx, P, Y, ldy, R, ldr, M, N, K, C, epilogue, ws,
                                    tickets, pl));
  IG_LAUNCH_STATUS();
  return IG_OK;
}

}  // namespace packed
}  // namespace ig

extern "C" int ig_sgemm_packed_sizes(int M, int N, int K, size_t* packed_floats,
                                     size_t* workspace_floats, size_t* tickets) {
  using namespace ig::packed;
  if (M < 1 || M > 32 || N < 1 || K < 1) return IG_EINVAL;
  const size_t tiles = (N + kTileN - 1) / kTileN, C = (K + kChunkK - 1) / kChunkK;
  if (packed_floats) *packed_floats = tiles * C * kBlockFloats + 2 * tiles;   // + 1/scale, scale
  if (workspace_floats) *workspace_floats = (size_t)grid_for(N, K, ctas_per_sm(M)) * 2 * M * kTileN;
  if (tickets) *tickets = tiles;
  return IG_OK;
}

extern "C" int ig_sgemm_pack(const float* W, int ldw, int N, int K, float* P, void* stream) {
  using namespace ig::packed;
  if (!W || !P || N < 1 || K < 1 || ldw < N) return IG_EINVAL;
  const int C = (K + kChunkK - 1) / kChunkK, tiles = (N + kTileN - 1) / kTileN;
  const size_t units = (size_t)tiles * C * (kBlockFloats / 4);
  float* inv_scale = P + (size_t)tiles * C * kBlockFloats;
  cudaStream_t s = (cudaStream_t)stream;
  tile_scale_kernel<<<tiles, 1024, 0, s>>>(W, ldw, N, K, inv_scale, inv_scale + tiles);
  IG_LAUNCH_STATUS();
  const int blocks = (int)((units + 255) / 256 < 65536 ? (units + 255) / 256 : 65536);
  pack_kernel<<<blocks, 256, 0, s>>>(W, ldw, N, K, C, inv_scale + tiles,
                                     reinterpret_cast<uint4*>(P), units);
  IG_LAUNCH_STATUS();
  return IG_OK;
}

namespace ig {
namespace packed {
static int sgemm_packed_any(const float* X, int ldx, const float* P, int N, int K, float* Y, int ldy,
                            const float* R, int ldr, int M, int epilogue, float* workspace,
                            size_t workspace_floats, int32_t* tickets, size_t ntickets,
                            cudaStream_t s, const PeerOut& po) {
  if (!X || !P || (!Y && !po.recv) || !workspace || !tickets || M < 1 || M > 32 || N < 1 || K < 1 ||
      ldx < K || (Y && ldy < N) || epilogue < 0 || epilogue > 2 || (epilogue == 2 && (!R || ldr < N)))
    return IG_EINVAL;
  if (((uintptr_t)P & 15) || ((uintptr_t)X & 15) || ((uintptr_t)workspace & 15) || (ldx & 3) || (K & 3))
    return IG_EINVAL;                                  // 16-B bulk copies and x vectors
  size_t ws_need = 0, tk_need = 0;
  ig_sgemm_packed_sizes(M, N, K, nullptr, &ws_need, &tk_need);
  if (ws_need > workspace_floats || tk_need > ntickets) return IG_EINVAL;
  if (M > 16) return launch<4, 1, 6, 2>(X, ldx, P, Y, ldy, R, ldr, M, N, K, epilogue, workspace, tickets, s, po);
  if (ctas_per_sm(M) == 1 && packed_cta_mode() == 8) {      // 8 warps, 3-deep ring, 1 CTA/SM
    if (M <= 8) return launch<1, 1, 3, 2>(X, ldx, P, Y, ldy, R, ldr, M, N, K, epilogue, workspace, tickets, s, po);
    return launch<2, 1, 3, 2>(X, ldx, P, Y, ldy, R, ldr, M, N, K, epilogue, workspace, tickets, s, po);
  }
  if (ctas_per_sm(M) == 1) {      // 16 warps, 6-deep ring
    if (M <= 8) return launch<1, 1, 6, 4>(X, ldx, P, Y, ldy, R, ldr, M, N, K, epilogue, workspace, tickets, s, po);
    return launch<2, 1, 6, 4>(X, ldx, P, Y, ldy, R, ldr, M, N, K, epilogue, workspace, tickets, s, po);
  }
  if (M <= 8) return launch<1, 2, 3, 2>(X, ldx, P, Y, ldy, R, ldr, M, N, K, epilogue, workspace, tickets, s, po);
  return launch<2, 2, 3, 2>(X, ldx, P, Y, ldy, R, ldr, M, N, K, epilogue, workspace, tickets, s, po);
}
}  // namespace packed
}  // namespace ig

extern "C" int ig_sgemm_packed(const float* X, int ldx, const float* P, int N, int K, float* Y,
                               int ldy, const float* R, int ldr, int M, int epilogue,
                               float* workspace, size_t workspace_floats, int32_t* tickets,
                               size_t ntickets, void* stream) {
  if (!Y) return IG_EINVAL;
  return ig::packed::sgemm_packed_any(X, ldx, P, N, K, Y, ldy, R, ldr, M, epilogue, workspace,
                                      workspace_floats, tickets, ntickets, (cudaStream_t)stream,
                                      ig::packed::PeerOut{});
}

extern "C" int ig_sgemm_packed_peer(const float* X, int ldx, const float* P, int N, int K, int M,
                                    const uint64_t* peer_recv, const uint64_t* peer_flags, int rank,
                                    int world, const ig_step_state* st, int call, int calls_per_step,
                                    uint32_t* done, float* workspace, size_t workspace_floats,
                                    int32_t* tickets, size_t ntickets, void* stream) {
  if (!peer_recv || !peer_flags || !st || !done || world < 1 || rank < 0 || rank >= world ||
      call < 0 || call >= calls_per_step)
    return IG_EINVAL;
  ig::packed::PeerOut po;
  po.recv = peer_recv;
  po.flags = peer_flags;
  po.st = st;
  po.done = done;
  po.rank = rank;
  po.world = world;
  po.call = call;
  po.calls = calls_per_step;
  return ig::packed::sgemm_packed_any(X, ldx, P, N, K, nullptr, N, nullptr, 0, M, 0, workspace,
                                      workspace_floats, tickets, ntickets, (cudaStream_t)stream, po);
}
