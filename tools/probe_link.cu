// Host-link probe: copy-engine H2D/D2H and SM zero-copy gathers of 512-B rows
// from pinned, mapped host memory. Standalone; prints one JSON object per line.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <random>
#include <algorithm>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

template <int UNROLL>
__global__ void gather_rows(const int4* __restrict__ src, const int* __restrict__ idx,
                            int4* __restrict__ dst, int nrows, int row_vec) {
  // one warp handles UNROLL rows per iteration; row_vec int4 per row (32 for 512 B)
  int lane = threadIdx.x & 31;
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int base = warp * UNROLL; base < nrows; base += nwarps * UNROLL) {
    int4 v[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      int r = base + u;
      if (r < nrows && lane < row_vec) v[u] = src[(size_t)idx[r] * row_vec + lane];
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      int r = base + u;
      if (r < nrows && lane < row_vec) dst[(size_t)r * row_vec + lane] = v[u];
    }
  }
}

__global__ void store_rows(int4* __restrict__ dst_host, const int* __restrict__ idx,
                           const int4* __restrict__ src, int nrows, int row_vec) {
  int lane = threadIdx.x & 31;
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int r = warp; r < nrows; r += nwarps)
    if (lane < row_vec) dst_host[(size_t)idx[r] * row_vec + lane] = src[(size_t)r * row_vec + lane];
}

int main(int argc, char** argv) {
  size_t host_bytes = (argc > 1 ? atoll(argv[1]) : 8) << 30;
  int dev = 0; CK(cudaSetDevice(dev));
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  printf("{\"probe\":\"device\",\"name\":\"%s\",\"sms\":%d,\"pci_bus\":%d,\"can_map\":%d,\"uva\":%d,\"pageable_access\":%d}\n",
         p.name, p.multiProcessorCount, p.pciBusID, p.canMapHostMemory, p.unifiedAddressing,
         p.pageableMemoryAccess);
  char* h; CK(cudaHostAlloc((void**)&h, host_bytes, cudaHostAllocMapped | cudaHostAllocPortable));
  for (size_t i = 0; i < host_bytes; i += 4096) h[i] = (char)i;
  char* dh; CK(cudaHostGetDevicePointer((void**)&dh, h, 0));
  size_t dev_bytes = 2ull << 30;
  char* d; CK(cudaMalloc(&d, dev_bytes));
  cudaStream_t s; CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  float ms;
  // copy-engine H2D / D2H
  for (size_t mb : {64ull, 512ull, 2048ull}) {
    size_t n = mb << 20;
    for (int rep = 0; rep < 2; ++rep) CK(cudaMemcpyAsync(d, h, n, cudaMemcpyHostToDevice, s));
    CK(cudaEventRecord(a, s));
    for (int rep = 0; rep < 5; ++rep) CK(cudaMemcpyAsync(d, h, n, cudaMemcpyHostToDevice, s));
    CK(cudaEventRecord(b, s)); CK(cudaEventSynchronize(b)); CK(cudaEventElapsedTime(&ms, a, b));
    printf("{\"probe\":\"ce_h2d\",\"mb\":%zu,\"gbs\":%.2f}\n", mb, 5.0 * n / ms / 1e6);
    CK(cudaEventRecord(a, s));
    for (int rep = 0; rep < 5; ++rep) CK(cudaMemcpyAsync(h, d, n, cudaMemcpyDeviceToHost, s));
    CK(cudaEventRecord(b, s)); CK(cudaEventSynchronize(b)); CK(cudaEventElapsedTime(&ms, a, b));
    printf("{\"probe\":\"ce_d2h\",\"mb\":%zu,\"gbs\":%.2f}\n", mb, 5.0 * n / ms / 1e6);
  }
  // 2-D copy: 640 chunks of 2 MB at pitch 2.1 MB (layer-0 style bulk fetch)
  {
    size_t w = 2ull << 20, pitch = w + (64 << 10); int hgt = 640;
    if (pitch * hgt <= host_bytes && w * hgt <= dev_bytes) {
      CK(cudaMemcpy2DAsync(d, w, h, pitch, w, hgt, cudaMemcpyHostToDevice, s));
      CK(cudaEventRecord(a, s));
      for (int rep = 0; rep < 3; ++rep) CK(cudaMemcpy2DAsync(d, w, h, pitch, w, hgt, cudaMemcpyHostToDevice, s));
      CK(cudaEventRecord(b, s)); CK(cudaEventSynchronize(b)); CK(cudaEventElapsedTime(&ms, a, b));
      printf("{\"probe\":\"ce_h2d_2d\",\"chunk_mb\":2,\"chunks\":%d,\"gbs\":%.2f}\n", hgt, 3.0 * w * hgt / ms / 1e6);
    }
  }
  // zero-copy gathers of random rows
  for (int row_bytes : {256, 512, 1024}) {
    int row_vec = row_bytes / 16;
    size_t host_rows = host_bytes / row_bytes;
    int nrows = (int)std::min<size_t>((size_t)(1u << 20), dev_bytes / row_bytes);
    std::vector<int> hi(nrows);
    std::mt19937_64 rng(1);
    for (int i = 0; i < nrows; ++i) hi[i] = (int)(rng() % host_rows);
    std::vector<int> sorted_idx = hi; std::sort(sorted_idx.begin(), sorted_idx.end());
    int* didx; CK(cudaMalloc(&didx, nrows * sizeof(int)));
    for (int sorted = 0; sorted < 2; ++sorted) {
      CK(cudaMemcpy(didx, sorted ? sorted_idx.data() : hi.data(), nrows * sizeof(int), cudaMemcpyHostToDevice));
      for (int ctas : {16, 32, 64, 148, 296, 592}) {
        for (int threads : {256, 1024}) {
          if (row_vec > 32) continue;  // one warp per row in this probe
          auto launch = [&]() { gather_rows<8><<<ctas, threads, 0, s>>>((const int4*)dh, didx, (int4*)d, nrows, row_vec); };
          launch(); CK(cudaGetLastError());
          CK(cudaEventRecord(a, s));
          for (int rep = 0; rep < 3; ++rep) launch();
          CK(cudaEventRecord(b, s)); CK(cudaEventSynchronize(b)); CK(cudaEventElapsedTime(&ms, a, b));
          printf("{\"probe\":\"zc_gather\",\"row_bytes\":%d,\"sorted\":%d,\"ctas\":%d,\"threads\":%d,\"gbs\":%.2f}\n",
                 row_bytes, sorted, ctas, threads, 3.0 * nrows * row_bytes / ms / 1e6);
        }
      }
    }
    // zero-copy scattered stores (append path)
    if (row_vec <= 32) {
      for (int ctas : {16, 148}) {
        store_rows<<<ctas, 256, 0, s>>>((int4*)dh, didx, (const int4*)d, nrows, row_vec);
        CK(cudaEventRecord(a, s));
        for (int rep = 0; rep < 3; ++rep) store_rows<<<ctas, 256, 0, s>>>((int4*)dh, didx, (const int4*)d, nrows, row_vec);
        CK(cudaEventRecord(b, s)); CK(cudaEventSynchronize(b)); CK(cudaEventElapsedTime(&ms, a, b));
        printf("{\"probe\":\"zc_store\",\"row_bytes\":%d,\"ctas\":%d,\"gbs\":%.2f}\n", row_bytes, ctas, 3.0 * nrows * row_bytes / ms / 1e6);
      }
    }
    CK(cudaFree(didx));
  }
  // concurrency: CE H2D and zero-copy gather at once
  {
    int row_vec = 32, nrows = 1 << 20; size_t host_rows = host_bytes / 512;
    std::vector<int> hi(nrows); std::mt19937_64 rng(2);
    for (int i = 0; i < nrows; ++i) hi[i] = (int)(rng() % host_rows);
    int* didx; CK(cudaMalloc(&didx, nrows * sizeof(int)));
    CK(cudaMemcpy(didx, hi.data(), nrows * sizeof(int), cudaMemcpyHostToDevice));
    cudaStream_t s2; CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
    cudaEvent_t c; CK(cudaEventCreate(&c));
    size_t n = 512ull << 20;
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(a, s));
    CK(cudaStreamWaitEvent(s2, a, 0));
    CK(cudaMemcpyAsync(d + (1ull << 30), h, n, cudaMemcpyHostToDevice, s2));
    gather_rows<8><<<148, 1024, 0, s>>>((const int4*)dh, didx, (int4*)d, nrows, row_vec);
    CK(cudaEventRecord(c, s2)); CK(cudaStreamWaitEvent(s, c, 0));
    CK(cudaEventRecord(b, s)); CK(cudaEventSynchronize(b)); CK(cudaEventElapsedTime(&ms, a, b));
    printf("{\"probe\":\"ce_plus_zc\",\"bytes\":%zu,\"gbs\":%.2f}\n", n + (size_t)nrows * 512, (n + (double)nrows * 512) / ms / 1e6);
  }
  return 0;
}
