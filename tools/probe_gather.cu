// Gather-variant probe: 512-B rows, ascending random subset (20%) of a host
// region laid out like the pool ([bh][S][512 B]), into HBM.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <random>
#include <algorithm>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

template <int U, int HINT>
__global__ void g_ld(const int4* __restrict__ src, const int* __restrict__ rows, int4* __restrict__ dst, long long nvec) {
  long long stride = (long long)gridDim.x * blockDim.x;
  for (long long base = (long long)blockIdx.x * blockDim.x + threadIdx.x; base < nvec; base += stride * U) {
    int4 v[U]; long long e[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      e[u] = base + u * stride;
      if (e[u] < nvec) {
        const int4* p = src + (long long)rows[e[u] >> 5] * 32 + (e[u] & 31);
        if (HINT == 0) asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(p));
        else if (HINT == 1) asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(p));
        else if (HINT == 2) asm volatile("ld.global.nc.L1::no_allocate.L2::128B.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(p));
        else asm volatile("ld.global.cv.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(p));
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) if (e[u] < nvec) dst[e[u]] = v[u];
  }
}

// TMA bulk: each warp's lane 0 issues row copies host->smem (512 B each) on an
// mbarrier, then the warp writes smem->HBM. ROWS rows per batch per warp.
template <int ROWS>
__global__ void g_tma(const char* __restrict__ src, const int* __restrict__ rows, char* __restrict__ dst, int nrows) {
  extern __shared__ __align__(128) char sm[];
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  char* buf = sm + warp * ROWS * 512;
  __shared__ __align__(8) unsigned long long bar[32];
  unsigned b = (unsigned)__cvta_generic_to_shared(&bar[warp]);
  if (lane == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(b));
  __syncwarp();
  asm volatile("fence.proxy.async.shared::cta;");
  unsigned phase = 0;
  int gw = blockIdx.x * nw + warp, gnw = gridDim.x * nw;
  for (int r0 = gw * ROWS; r0 < nrows; r0 += gnw * ROWS) {
    int cnt = min(ROWS, nrows - r0);
    if (lane == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(b), "r"(cnt * 512));
      for (int i = 0; i < cnt; ++i) {
        unsigned d = (unsigned)__cvta_generic_to_shared(buf + i * 512);
        const char* s = src + (long long)rows[r0 + i] * 512;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 512, [%2];" :: "r"(d), "l"(s), "r"(b) : "memory");
      }
    }
    // wait
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" :: "r"(b), "r"(phase) : "memory");
    phase ^= 1;
    const int4* s4 = (const int4*)buf;
    int4* d4 = (int4*)(dst + (long long)r0 * 512);
    for (int i = lane; i < cnt * 32; i += 32) d4[i] = s4[i];
    __syncwarp();
  }
}

int main() {
  const int BH = 640, S = 4096;
  size_t host_bytes = (size_t)BH * S * 512;  // 1.34 GB
  char* h; CK(cudaHostAlloc((void**)&h, host_bytes, cudaHostAllocMapped | cudaHostAllocPortable));
  for (size_t i = 0; i < host_bytes; i += 4096) h[i] = 1;
  char* dh; CK(cudaHostGetDevicePointer((void**)&dh, h, 0));
  std::vector<int> rows; std::mt19937 rng(3);
  for (int bh = 0; bh < BH; ++bh) {
    std::vector<int> r(S); for (int i = 0; i < S; ++i) r[i] = i;
    std::shuffle(r.begin(), r.end(), rng); r.resize(820); std::sort(r.begin(), r.end());
    for (int x : r) rows.push_back(bh * S + x);
  }
  int nrows = rows.size(); long long nvec = (long long)nrows * 32;
  int* drows; CK(cudaMalloc(&drows, nrows * 4)); CK(cudaMemcpy(drows, rows.data(), nrows * 4, cudaMemcpyHostToDevice));
  char* d; CK(cudaMalloc(&d, (size_t)nrows * 512));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  auto timeit = [&](const char* name, int ctas, int thr, auto fn) {
    fn(); CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
    cudaEventRecord(a); for (int i = 0; i < 3; ++i) fn(); cudaEventRecord(b); CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&ms, a, b);
    printf("{\"variant\":\"%s\",\"ctas\":%d,\"threads\":%d,\"gbs\":%.2f}\n", name, ctas, thr, 3.0 * nrows * 512 / ms / 1e6);
  };
  for (int ctas : {16, 32, 64, 148}) {
    timeit("ld_u4", ctas, 1024, [&] { g_ld<4, 0><<<ctas, 1024>>>((const int4*)dh, drows, (int4*)d, nvec); });
    timeit("ld_u8", ctas, 1024, [&] { g_ld<8, 0><<<ctas, 1024>>>((const int4*)dh, drows, (int4*)d, nvec); });
    timeit("ld_u8_L2_256B", ctas, 1024, [&] { g_ld<8, 1><<<ctas, 1024>>>((const int4*)dh, drows, (int4*)d, nvec); });
    timeit("ld_u8_L2_128B", ctas, 1024, [&] { g_ld<8, 2><<<ctas, 1024>>>((const int4*)dh, drows, (int4*)d, nvec); });
    timeit("ld_u8_cv", ctas, 1024, [&] { g_ld<8, 3><<<ctas, 1024>>>((const int4*)dh, drows, (int4*)d, nvec); });
    timeit("ld_u16_L2_256B", ctas, 512, [&] { g_ld<16, 1><<<ctas, 512>>>((const int4*)dh, drows, (int4*)d, nvec); });
  }
  for (int ctas : {16, 32, 64, 148}) {
    for (int thr : {256, 512}) {
      size_t smem = (thr / 32) * 8 * 512;
      CK(cudaFuncSetAttribute(g_tma<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      timeit("tma_bulk_8rows", ctas, thr, [&] { g_tma<8><<<ctas, thr, smem>>>(dh, drows, d, nrows); });
      size_t smem16 = (thr / 32) * 16 * 512;
      if (smem16 <= 200 * 1024) {
        CK(cudaFuncSetAttribute(g_tma<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem16));
        timeit("tma_bulk_16rows", ctas, thr, [&] { g_tma<16><<<ctas, thr, smem16>>>(dh, drows, d, nrows); });
      }
    }
  }
  return 0;
}
