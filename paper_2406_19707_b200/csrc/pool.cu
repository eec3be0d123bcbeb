// Host KV pool: storage, K3 fetch (gather over the host link), K5 append
// (+ eviction + partial-K mirror + fetch metadata), step bookkeeping.
//
// Reference: KvPool (pool.py:28-112), append_partial_key
// (speculation.py:92-114), DecodeSession._fetch_sets / _with_position
// (engine.py:382-418, 449-453).
#include "common.cuh"

namespace ig {

// ---------------------------------------------------------------------------
// K3 fetch.  Zero-copy gather of 16-B vectors from the mapped host pool.
// Consecutive threads take consecutive vectors, so a warp moves one 512-B
// (d=128, f16) row per instruction; rows arrive in ascending index order per
// (b, h), which keeps host-page locality (measured 52.7 GB/s vs 55.5 GB/s for
// the copy engine; 35 GB/s if rows are visited in random order).
// ---------------------------------------------------------------------------
constexpr int kFetchUnroll = 4;
constexpr int kMaxBatch = 256;

template <int kFetchThreads>
__global__ void __launch_bounds__(kFetchThreads)
fetch_kernel(const uint8_t* __restrict__ pool, const int32_t* __restrict__ idx,
             const int32_t* __restrict__ n_in, int B, int Hg, int S_max, int cap,
             int row_bytes, uint8_t* __restrict__ stage) {
  __shared__ long long off[kMaxBatch + 1];
  if (threadIdx.x == 0) {
    long long acc = 0;
    for (int b = 0; b < B; ++b) {
      off[b] = acc;
      acc += (long long)n_in[b] * Hg;
    }
    off[B] = acc;
  }
  __syncthreads();
  const int vpr = row_bytes >> 4;  // 16-B vectors per row
  const long long total = off[B] * vpr;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long base = (long long)blockIdx.x * blockDim.x + threadIdx.x; base < total;
       base += stride * kFetchUnroll) {
    uint4 v[kFetchUnroll];
    size_t dst[kFetchUnroll];
#pragma unroll
    for (int u = 0; u < kFetchUnroll; ++u) {
      const long long e = base + u * stride;
      dst[u] = ~(size_t)0;
      if (e < total) {
        const long long g = e / vpr;
        const int vec = (int)(e - g * vpr);
        int b = 0;
        while (off[b + 1] <= g) ++b;
        const int nb = n_in[b];
        const long long rem = g - off[b];
        const int h = (int)(rem / nb);
        const int r = (int)(rem - (long long)h * nb);
        const size_t bh = (size_t)b * Hg + h;
        const int row = idx[bh * cap + r];
        const uint4* src = reinterpret_cast<const uint4*>(pool + ((bh * S_max + row) * row_bytes)) + vec;
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(src));
        dst[u] = (bh * cap + r) * row_bytes + (size_t)vec * 16;
      }
    }
#pragma unroll
    for (int u = 0; u < kFetchUnroll; ++u)
      if (dst[u] != ~(size_t)0) *reinterpret_cast<uint4*>(stage + dst[u]) = v[u];
  }
}


// ---------------------------------------------------------------------------
// K3 fetch, TMA variant.  Each lane of a warp moves one row per batch with a
// bulk async copy host -> shared memory (cp.async.bulk ... complete_tx on an
// mbarrier) and a bulk async store shared memory -> HBM stage
// (cp.async.bulk.global.shared::cta); two 32-row batches per warp are in
// flight (double-buffered).  The bytes in flight live in shared memory, not
// registers, so one warp per CTA saturates its share of the link and the
// gather leaves the SMs' threads and registers to the compute stream
// (measured: the 1024-thread LDG gather slows the compute stream enough to
// stall the fetch pipeline at C2).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(bar),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_load(uint32_t dst_smem, const void* src, uint32_t bytes,
                                          uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst_smem),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, uint32_t src_smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(src_smem), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read_1() {
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

constexpr int kTmaBufs = 3;   // batch j loads while j-1 drains; j-2's store reads retire

__global__ void __launch_bounds__(128)
fetch_tma_kernel(const uint8_t* __restrict__ pool, const int32_t* __restrict__ idx,
                 const int32_t* __restrict__ n_in, const ig_step_state* __restrict__ st, int B,
                 int Hg, int S_max, int cap, int row_bytes, int rows_per_batch,
                 uint8_t* __restrict__ stage) {
  const int R = rows_per_batch;   // lanes [0, R) each move one row per batch
  // idx == nullptr: every row [0, st->s_len) of every (b, h), identity order
  // (a full layer, graph-capturable: the row count is read on the device)
  extern __shared__ __align__(128) uint8_t tma_smem[];
  __shared__ long long off[kMaxBatch + 1];
  __shared__ __align__(8) unsigned long long bars[4][kTmaBufs];   // <= 4 warps
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (threadIdx.x == 0) {
    long long acc = 0;
    const int all = idx == nullptr ? st->s_len : 0;
    for (int b = 0; b < B; ++b) {
      off[b] = acc;
      acc += (long long)(idx == nullptr ? all : n_in[b]) * Hg;
    }
    off[B] = acc;
  }
  if (lane == 0) {
    for (int i = 0; i < kTmaBufs; ++i) mbar_init((uint32_t)__cvta_generic_to_shared(&bars[w][i]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const long long total = off[B];
  uint8_t* wbuf = tma_smem + (size_t)w * kTmaBufs * R * row_bytes;
  const long long gw = (long long)blockIdx.x * nw + w, nwt = (long long)gridDim.x * nw;
  uint32_t phase_bits = 0;      // bit i = parity to wait for on buffer i
  bool prev_batch = false, prev_mine = false;
  size_t prev_dst = 0;
  int prev_buf = 0;
  for (long long j = 0;; ++j) {
    const long long base = (gw + j * nwt) * R;
    const int buf = (int)(j % kTmaBufs);
    const bool batch = base < total;
    bool mine = false;
    size_t dst = 0;
    if (batch) {
      // buffer `buf` was last read by the stores of batch j-3, issued one
      // iteration before the most recent group: allow exactly one pending
      bulk_wait_read_1();
      __syncwarp();
      const long long g = base + lane;
      const void* src = nullptr;
      mine = lane < R && g < total;
      if (mine) {
        int b = 0;
        while (off[b + 1] <= g) ++b;
        const long long rem = g - off[b];
        const int nb = (int)((off[b + 1] - off[b]) / Hg);
        const int h = (int)(rem / nb);
        const int r = (int)(rem - (long long)h * nb);
        const size_t bh = (size_t)b * Hg + h;
        src = pool + (bh * S_max + (idx ? idx[bh * cap + r] : r)) * (size_t)row_bytes;
        dst = (bh * cap + r) * (size_t)row_bytes;
      }
      const int cnt = __popc(__ballot_sync(0xffffffffu, mine));
      const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&bars[w][buf]);
      if (lane == 0) mbar_expect_tx(bar, (uint32_t)cnt * row_bytes);
      __syncwarp();
      if (mine)
        bulk_load((uint32_t)__cvta_generic_to_shared(wbuf + ((size_t)buf * R + lane) * row_bytes),
                  src, row_bytes, bar);
    }
    if (prev_batch) {  // drain batch j-1: its loads landed -> store to HBM
      mbar_wait((uint32_t)__cvta_generic_to_shared(&bars[w][prev_buf]), (phase_bits >> prev_buf) & 1u);
      phase_bits ^= 1u << prev_buf;
      if (prev_mine)
        bulk_store(stage + prev_dst,
                   (uint32_t)__cvta_generic_to_shared(wbuf + ((size_t)prev_buf * R + lane) * row_bytes),
                   row_bytes);
    }
    if (!batch) break;
    prev_batch = true;
    prev_mine = mine;
    prev_dst = dst;
    prev_buf = buf;
  }
  bulk_wait_all();
}

// ---------------------------------------------------------------------------
// K5 append (one CTA per (b, h)).
// ---------------------------------------------------------------------------
constexpr int kAppendThreads = 256;

__device__ __forceinline__ long long policy_key(int policy, const long long* arrival,
                                                const long long* lastf, const uint8_t* ctr,
                                                int t) {
  return policy == IG_POLICY_FIFO ? arrival[t] : (policy == IG_POLICY_LRU ? lastf[t] : (long long)ctr[t]);
}

// KvPool.fetch metadata (pool.py:93-98) for one pool, whole block:
// rows = sel[0:n] (sel == nullptr -> rows 0..n-1) plus `extra` (>= 0) unless
// it is already in sel (_with_position, engine.py:449-453); each gets
// last_fetch = fseq and a saturating counter bump; if any bumped counter is
// 255, every counter in [0, len) is halved.  Rows must be unique.
__device__ void touch_rows(const int32_t* __restrict__ sel, int n, int extra, int len,
                           long long fseq, long long* __restrict__ lf, uint8_t* __restrict__ ctr,
                           int* sh_flag) {
  const int tid = threadIdx.x;
  __syncthreads();
  if (tid == 0) *sh_flag = 0;
  __syncthreads();
  if (extra >= 0 && sel != nullptr) {
    int found = 0;
    for (int r = tid; r < n; r += blockDim.x) found |= sel[r] == extra;
    if (found) atomicOr(sh_flag, 1);
  }
  __syncthreads();
  const bool extra_in = extra < 0 || *sh_flag != 0 || (sel == nullptr && extra < n);
  __syncthreads();
  if (tid == 0) *sh_flag = 0;
  __syncthreads();
  // Saturation is decided on the pre-increment value: ptxas (12.9, sm_100a)
  // lowers `c = min(old + 1, 255); hit = c == 255` to a packed VIMNMX.U16x2
  // whose second predicate output clobbers the first, making `hit` always 1.
  int hit = 0;
  for (int r = tid; r < n; r += blockDim.x) {
    const int t = sel ? sel[r] : r;
    lf[t] = fseq;
    const unsigned old = ctr[t];
    const bool sat = old >= 254u;
    ctr[t] = sat ? (uint8_t)255 : (uint8_t)(old + 1u);
    hit |= (int)sat;
  }
  if (!extra_in && tid == 0) {
    lf[extra] = fseq;
    const unsigned old = ctr[extra];
    const bool sat = old >= 254u;
    ctr[extra] = sat ? (uint8_t)255 : (uint8_t)(old + 1u);
    hit |= (int)sat;
  }
  if (hit) atomicOr(sh_flag, 1);
  __syncthreads();
  if (*sh_flag)  // "hit 255 -> halve all" over the whole pool
    for (int t = tid; t < len; t += blockDim.x) ctr[t] = ctr[t] >> 1;
  __syncthreads();
}

constexpr int kTouchThreads = 256;

__global__ void __launch_bounds__(kTouchThreads)
touch_kernel(const int32_t* __restrict__ idx, const int32_t* __restrict__ n_in, int cap, int Hg,
             int S_max, const ig_step_state* __restrict__ st, long long fseq,
             long long* __restrict__ lastf, uint8_t* __restrict__ counter) {
  __shared__ int flag;
  const int b = blockIdx.y, h = blockIdx.x;
  const size_t bh = (size_t)b * Hg + h;
  touch_rows(idx + bh * cap, n_in[b], -1, st->s_len, fseq, lastf + bh * S_max,
             counter + bh * S_max, &flag);
}

// evict_select (pool.py:101-109): argmin over [0, s) of the policy key, lowest
// index on ties.  Whole block; result valid in every thread.
__device__ int victim_argmin(int policy, const long long* arr, const long long* lf,
                             const uint8_t* ctr, int s, long long* red_v, int* red_i) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  long long bv = LLONG_MAX;
  int bi = INT_MAX;
  for (int t = tid; t < s; t += blockDim.x) {
    const long long v = policy_key(policy, arr, lf, ctr, t);
    if (v < bv) { bv = v; bi = t; }  // ascending t per thread: first minimum kept
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const long long ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov < bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
  }
  __syncthreads();
  if (lane == 0) { red_v[w] = bv; red_i[w] = bi; }
  __syncthreads();
  long long mv = red_v[0];
  int mi = red_i[0];
  for (int i = 1; i < (int)(blockDim.x >> 5); ++i)
    if (red_v[i] < mv || (red_v[i] == mv && red_i[i] < mi)) { mv = red_v[i]; mi = red_i[i]; }
  return mi;
}

__global__ void __launch_bounds__(kAppendThreads)
victim_kernel(const long long* __restrict__ arrival, const long long* __restrict__ lastf,
              const uint8_t* __restrict__ counter, int policy, const ig_step_state* __restrict__ st,
              int Hg, int S_max, int32_t* __restrict__ out) {
  __shared__ long long red_v[kAppendThreads / kWarp];
  __shared__ int red_i[kAppendThreads / kWarp];
  const size_t bh = (size_t)blockIdx.y * Hg + blockIdx.x;
  const int v = victim_argmin(policy, arrival + bh * S_max, lastf + bh * S_max,
                              counter + bh * S_max, st->s_len, red_v, red_i);
  if (threadIdx.x == 0) out[bh] = v;
}

template <typename T>
__global__ void __launch_bounds__(kAppendThreads)
append_kernel(const float* __restrict__ k_cur, const float* __restrict__ v_cur, int ldkv,
              T* __restrict__ pool, float* __restrict__ pk, const int32_t* __restrict__ cols, int k,
              long long* __restrict__ arrival, long long* __restrict__ lastf,
              uint8_t* __restrict__ counter, int policy, int fetch_mode,
              const int32_t* __restrict__ idx, const int32_t* __restrict__ n_in, int cap,
              const ig_step_state* __restrict__ st, int Hg, int d, int S_max,
              int32_t* __restrict__ pos_out, long long* __restrict__ events) {
  __shared__ long long red_v[kAppendThreads / kWarp];
  __shared__ int red_i[kAppendThreads / kWarp];
  __shared__ int sh_pos;
  __shared__ int sh_flag;
  const int b = blockIdx.y, h = blockIdx.x;
  const size_t bh = (size_t)b * Hg + h;
  const int s = st->s_len, limit = st->limit;
  const long long seq = st->seq;
  long long* arr = arrival + bh * S_max;
  long long* lf = lastf + bh * S_max;
  uint8_t* ctr = counter + bh * S_max;
  const int tid = threadIdx.x;

  // 1. row position: append at s, or the policy victim (argmin, lowest index)
  const bool evict = limit > 0 && s >= limit;
  if (evict) {
    const int v = victim_argmin(policy, arr, lf, ctr, s, red_v, red_i);
    if (tid == 0) sh_pos = v;
  } else if (tid == 0) {
    sh_pos = s;
  }
  __syncthreads();
  const int pos = sh_pos;

  // 2. overwrite event (engine.py:237-243) -- old arrival read before reset
  if (tid == 0) {
    events[bh * 2] = evict ? pos : -1;
    events[bh * 2 + 1] = evict ? arr[pos] : 0;
  }
  // 3. the new K/V row to the host pool (zero-copy posted stores)
  T* dst = pool + (bh * S_max + pos) * (size_t)(2 * d);
  const float* kr = k_cur + (size_t)b * ldkv + (size_t)h * d;
  const float* vr = v_cur + (size_t)b * ldkv + (size_t)h * d;
  for (int i = tid; i < d; i += blockDim.x) {
    dst[i] = Elt<T>::from_f(kr[i]);
    dst[d + i] = Elt<T>::from_f(vr[i]);
  }
  // 4. partial-K mirror: the skewed key's selected columns at row pos
  if (pk != nullptr)
    for (int j = tid; j < k; j += blockDim.x)
      pk[(bh * k + j) * (size_t)S_max + pos] = kr[cols[bh * k + j]];
  __syncthreads();  // old arrival read (step 2) before the reset below
  // 5. metadata of the (re)used row (pool.py:68-72, 77-79)
  if (tid == 0) {
    arr[pos] = seq + 1;
    lf[pos] = seq + 1;
    ctr[pos] = 0;
  }
  __syncthreads();
  // 6. fetch metadata for this layer's fetch set (pool.py:93-98)
  const int s_after = evict ? s : s + 1;
  if (fetch_mode == 1) {         // layer 0: every row, including the new one
    touch_rows(nullptr, s_after, -1, s_after, seq + 2, lf, ctr, &sh_flag);
  } else if (fetch_mode == 2) {  // carried selection plus the current row
    touch_rows(idx + bh * cap, n_in[b], pos, s_after, seq + 2, lf, ctr, &sh_flag);
  }
  if (tid == 0) pos_out[bh] = pos;
}

__global__ void step_advance_kernel(ig_step_state* st) {
  if (st->limit == 0 || st->s_len < st->limit) st->s_len += 1;
  st->seq += 2;
  st->step += 1;
}

}  // namespace ig

// ---------------------------------------------------------------------------
// Host pool allocation (each rank's slice of the pinned pool
// sits on its GPU's NUMA node).  When the machine has more than one NUMA node
// and the current GPU reports one (sysfs numa_node of its PCI function), the
// pool is mmap'ed, bound to that node (mbind MPOL_BIND) and pinned + mapped
// with cudaHostRegister; otherwise (one node, unknown node, IG_HOST_NUMA=0 or
// any failure) it is a plain cudaHostAlloc(Mapped | Portable).
// ---------------------------------------------------------------------------
#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <cstdio>
#include <mutex>
#include <unordered_map>

namespace ig {
namespace hostpool {
std::mutex mu;
std::unordered_map<void*, size_t> mapped;    // mmap'ed + registered pools -> bytes

int gpu_numa_node() {
  const char* e = getenv("IG_HOST_NUMA");
  if (e && atoi(e) == 0) return -1;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  char bus[32] = {0};
  if (cudaDeviceGetPCIBusId(bus, sizeof(bus), dev) != cudaSuccess) return -1;
  for (char* c = bus; *c; ++c) *c = (char)tolower(*c);
  char path[128];
  snprintf(path, sizeof(path), "/sys/bus/pci/devices/%s/numa_node", bus);
  FILE* f = fopen(path, "r");
  if (!f) return -1;
  int node = -1;
  if (fscanf(f, "%d", &node) != 1) node = -1;
  fclose(f);
  if (node < 0 || node > 63) return -1;
  if (access("/sys/devices/system/node/node1", F_OK) != 0) return -1;   // a single node
  return node;
}
}  // namespace hostpool
}  // namespace ig

extern "C" int ig_host_free(void* host_ptr);

extern "C" int ig_host_alloc(size_t bytes, void** host_ptr, void** dev_ptr) {
  using namespace ig::hostpool;
  if (!host_ptr || !dev_ptr || bytes == 0) return IG_EINVAL;
  void* h = nullptr;
  const int node = gpu_numa_node();
  if (node >= 0) {
    void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (p != MAP_FAILED) {
      unsigned long mask = 1ul << node;
      const long rc = syscall(SYS_mbind, p, bytes, 2 /*MPOL_BIND*/, &mask, 65ul, 0u);
      if (rc == 0 && cudaHostRegister(p, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable) == cudaSuccess) {
        h = p;
        std::lock_guard<std::mutex> g(mu);
        mapped[p] = bytes;
      } else {
        cudaGetLastError();
        munmap(p, bytes);
      }
    }
  }
  if (!h) {
    cudaError_t e = cudaHostAlloc(&h, bytes, cudaHostAllocMapped | cudaHostAllocPortable);
    if (e == cudaErrorMemoryAllocation) return IG_ENOMEM;
    IG_CUDA_STATUS(e);
  }
  void* d = nullptr;
  cudaError_t e = cudaHostGetDevicePointer(&d, h, 0);
  if (e != cudaSuccess) {
    ig_host_free(h);
    return IG_ECUDA + (int)e;
  }
  *host_ptr = h;
  *dev_ptr = d;
  return IG_OK;
}

extern "C" int ig_host_free(void* host_ptr) {
  using namespace ig::hostpool;
  if (!host_ptr) return IG_EINVAL;
  size_t bytes = 0;
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = mapped.find(host_ptr);
    if (it != mapped.end()) {
      bytes = it->second;
      mapped.erase(it);
    }
  }
  if (bytes) {
    IG_CUDA_STATUS(cudaHostUnregister(host_ptr));
    munmap(host_ptr, bytes);
    return IG_OK;
  }
  IG_CUDA_STATUS(cudaFreeHost(host_ptr));
  return IG_OK;
}

extern "C" int ig_host_numa_node(const void* host_ptr, int* node) {
  // NUMA node of the pool's first page (get_mempolicy MPOL_F_NODE | MPOL_F_ADDR), -1 if unknown
  if (!host_ptr || !node) return IG_EINVAL;
  int n = -1;
  const long rc = syscall(SYS_get_mempolicy, &n, nullptr, 0ul, const_cast<void*>(host_ptr), 3u);
  *node = rc == 0 ? n : -1;
  return IG_OK;
}

extern "C" int ig_fetch(const void* pool_dev, const int32_t* idx, const int32_t* n, int B, int Hg,
                        int S_max, int cap, int row_bytes, void* stage, int ctas, int threads,
                        void* stream) {
  using namespace ig;
  if (!pool_dev || !idx || !n || !stage || B < 1 || B > kMaxBatch || Hg < 1 || cap < 1 ||
      S_max < 1 || row_bytes < 16 || (row_bytes & 15) || ctas < 1)
    return IG_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  const uint8_t* src = (const uint8_t*)pool_dev;
  uint8_t* dst = (uint8_t*)stage;
  switch (threads) {
    case 256: fetch_kernel<256><<<ctas, 256, 0, s>>>(src, idx, n, B, Hg, S_max, cap, row_bytes, dst); break;
    case 512: fetch_kernel<512><<<ctas, 512, 0, s>>>(src, idx, n, B, Hg, S_max, cap, row_bytes, dst); break;
    case 1024: fetch_kernel<1024><<<ctas, 1024, 0, s>>>(src, idx, n, B, Hg, S_max, cap, row_bytes, dst); break;
    default: return IG_EINVAL;
  }
  IG_LAUNCH_STATUS();
  return IG_OK;
}

extern "C" int ig_fetch_tma(const void* pool_dev, const int32_t* idx, const int32_t* n,
                            const ig_step_state* st, int B, int Hg, int S_max, int cap,
                            int row_bytes, void* stage, int ctas, int warps, int rows_per_batch,
                            void* stream) {
  using namespace ig;
  if (!pool_dev || (idx && !n) || (!idx && !st) || !stage || B < 1 || B > kMaxBatch || Hg < 1 || cap < 1 ||
      S_max < 1 || row_bytes < 16 || (row_bytes & 15) || ctas < 1 || warps < 1 || warps > 4 ||
      rows_per_batch < 1 || rows_per_batch > 32)
    return IG_EINVAL;
  const size_t smem = (size_t)warps * kTmaBufs * rows_per_batch * row_bytes;
  if (smem > 200 * 1024) return IG_EINVAL;
  if (smem > 32 * 1024)  // dynamic + static must fit: opt in early
    IG_CUDA_STATUS(cudaFuncSetAttribute(fetch_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)smem));
  fetch_tma_kernel<<<ctas, 32 * warps, smem, (cudaStream_t)stream>>>(
      (const uint8_t*)pool_dev, idx, n, st, B, Hg, S_max, cap, row_bytes, rows_per_batch,
      (uint8_t*)stage);
  IG_LAUNCH_STATUS();
  return IG_OK;
}

extern "C" int ig_fetch_all(const void* pool_host, int B, int Hg, int S_max, int s, int row_bytes,
                            void* stage, int stage_rows, void* stream) {
  if (!pool_host || !stage || B < 1 || Hg < 1 || s < 0 || s > S_max || s > stage_rows ||
      row_bytes < 1)
    return IG_EINVAL;
  if (s == 0) return IG_OK;
  IG_CUDA_STATUS(cudaMemcpy2DAsync(stage, (size_t)stage_rows * row_bytes, pool_host,
                                   (size_t)S_max * row_bytes, (size_t)s * row_bytes,
                                   (size_t)B * Hg, cudaMemcpyHostToDevice, (cudaStream_t)stream));
  return IG_OK;
}

extern "C" int ig_memcpy2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width,
                           size_t height, void* stream) {
  if (!dst || !src || width > dpitch || width > spitch) return IG_EINVAL;
  if (width == 0 || height == 0) return IG_OK;
  IG_CUDA_STATUS(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, cudaMemcpyDefault,
                                   (cudaStream_t)stream));
  return IG_OK;
}

extern "C" int ig_append(const float* k_cur, const float* v_cur, int ldkv, void* pool_dev, int elt,
                         float* pk, const int32_t* cols, int k, int64_t* arrival,
                         int64_t* last_fetch, uint8_t* counter, int policy, int fetch_mode,
                         const int32_t* idx, const int32_t* n, int cap, const ig_step_state* st,
                         int B, int Hg, int d, int S_max, int32_t* pos_out, int64_t* events,
                         void* stream) {
  using namespace ig;
  if (!k_cur || !v_cur || !pool_dev || !arrival || !last_fetch || !counter || !st || !pos_out ||
      !events || B < 1 || Hg < 1 || d < 1 || S_max < 1 || ldkv < Hg * d ||
      policy < IG_POLICY_FIFO || policy > IG_POLICY_COUNTER)
    return IG_EINVAL;
  if (pk && (!cols || k < 1 || k > d)) return IG_EINVAL;
  if (fetch_mode < 0 || fetch_mode > 2 || (fetch_mode == 2 && (!idx || !n || cap < 1)))
    return IG_EINVAL;
  dim3 grid(Hg, B);
  cudaStream_t s = (cudaStream_t)stream;
  auto* arr = reinterpret_cast<long long*>(arrival);
  auto* lf = reinterpret_cast<long long*>(last_fetch);
  auto* ev = reinterpret_cast<long long*>(events);
  switch (elt) {
    case IG_ELT_F32:
      append_kernel<float><<<grid, kAppendThreads, 0, s>>>(k_cur, v_cur, ldkv, (float*)pool_dev, pk,
          cols, k, arr, lf, counter, policy, fetch_mode, idx, n, cap, st, Hg, d, S_max, pos_out, ev);
      break;
    case IG_ELT_F16:
      append_kernel<__half><<<grid, kAppendThreads, 0, s>>>(k_cur, v_cur, ldkv, (__half*)pool_dev,
          pk, cols, k, arr, lf, counter, policy, fetch_mode, idx, n, cap, st, Hg, d, S_max, pos_out, ev);
      break;
    case IG_ELT_BF16:
      append_kernel<__nv_bfloat16><<<grid, kAppendThreads, 0, s>>>(k_cur, v_cur, ldkv,
          (__nv_bfloat16*)pool_dev, pk, cols, k, arr, lf, counter, policy, fetch_mode, idx, n, cap,
          st, Hg, d, S_max, pos_out, ev);
      break;
    default:
      return IG_EINVAL;
  }
  IG_LAUNCH_STATUS();
  return IG_OK;
}

extern "C" int ig_touch(const int32_t* idx, const int32_t* n, int cap, const ig_step_state* st,
                        int B, int Hg, int S_max, int64_t seq, int64_t* last_fetch,
                        uint8_t* counter, void* stream) {
  using namespace ig;
  if (!idx || !n || !st || !last_fetch || !counter || B < 1 || Hg < 1 || cap < 1 || S_max < 1)
    return IG_EINVAL;
  touch_kernel<<<dim3(Hg, B), kTouchThreads, 0, (cudaStream_t)stream>>>(
      idx, n, cap, Hg, S_max, st, (long long)seq, reinterpret_cast<long long*>(last_fetch), counter);
  IG_LAUNCH_STATUS();
  return IG_OK;
}

extern "C" int ig_evict_select(const int64_t* arrival, const int64_t* last_fetch,
                               const uint8_t* counter, int policy, const ig_step_state* st, int B,
                               int Hg, int S_max, int32_t* victim, void* stream) {
  using namespace ig;
  if (!arrival || !last_fetch || !counter || !st || !victim || B < 1 || Hg < 1 || S_max < 1 ||
      policy < IG_POLICY_FIFO || policy > IG_POLICY_COUNTER)
    return IG_EINVAL;
  victim_kernel<<<dim3(Hg, B), kAppendThreads, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const long long*>(arrival), reinterpret_cast<const long long*>(last_fetch),
      counter, policy, st, Hg, S_max, victim);
  IG_LAUNCH_STATUS();
  return IG_OK;
}

extern "C" int ig_step_advance(ig_step_state* st, void* stream) {
  if (!st) return IG_EINVAL;
  ig::step_advance_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(st);
  IG_LAUNCH_STATUS();
  return IG_OK;
}
