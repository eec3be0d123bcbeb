// ABI metadata and the reference layernorm (produces the rehearsal input x_a).
#include "common.cuh"

namespace ig {

constexpr int kLnThreads = 1024;
constexpr int kLnCache = 8;      // row elements per thread kept in registers (D <= 8192)

// linalg.py:50-69: mean, centered, var = mean(c*c), c / sqrt(var + eps) * g + b.
// Sums are accumulated in f64 and rounded once (the reference sums pairwise in
// f32; both are within a few ulps of the exact value).  The elementwise tail is
// f32 with explicit _rn intrinsics so nvcc cannot contract (x*g)+b into an FMA:
// NumPy rounds the product and the sum separately.  One CTA of 1024 threads
// per row; the row is read once into registers (D <= 8192) and the three
// passes run from there (the 256-thread version re-read it and took ~20 us).
__global__ void __launch_bounds__(kLnThreads)
layernorm_kernel(const float* __restrict__ x, const float* __restrict__ g,
                 const float* __restrict__ bias, float eps, int D, float* __restrict__ out) {
  __shared__ double red[kLnThreads / kWarp];
  pdl_trigger();
  pdl_wait();        // launched with PDL (ln_pdl()): the producer of x has completed
  const float* xr = x + (size_t)blockIdx.x * D;
  float* yr = out + (size_t)blockIdx.x * D;
  const bool cached = D <= kLnCache * kLnThreads;
  float xv[kLnCache];
  double s = 0.0;
  if (cached) {
#pragma unroll
    for (int j = 0; j < kLnCache; ++j) {
      const int i = threadIdx.x + j * kLnThreads;
      xv[j] = i < D ? xr[i] : 0.f;
      s += (double)xv[j];
    }
  } else {
    for (int i = threadIdx.x; i < D; i += blockDim.x) s += (double)xr[i];
  }
  s = block_sum(s, red);
  const float mean = (float)(s / (double)D);
  double v = 0.0;
  if (cached) {
#pragma unroll
    for (int j = 0; j < kLnCache; ++j) {
      const int i = threadIdx.x + j * kLnThreads;
      const float c = __fsub_rn(xv[j], mean);
      if (i < D) v += (double)__fmul_rn(c, c);
    }
  } else {
    for (int i = threadIdx.x; i < D; i += blockDim.x) {
      const float c = __fsub_rn(xr[i], mean);
      v += (double)__fmul_rn(c, c);
    }
  }
  v = block_sum(v, red);
  const float var = (float)(v / (double)D);
  const float den = sqrtf(__fadd_rn(var, eps));
  if (cached) {
#pragma unroll
    for (int j = 0; j < kLnCache; ++j) {
      const int i = threadIdx.x + j * kLnThreads;
      if (i < D) yr[i] = __fadd_rn(__fmul_rn(__fdiv_rn(__fsub_rn(xv[j], mean), den), g[i]), bias[i]);
    }
  } else {
    for (int i = threadIdx.x; i < D; i += blockDim.x) {
      const float c = __fsub_rn(xr[i], mean);
      yr[i] = __fadd_rn(__fmul_rn(__fdiv_rn(c, den), g[i]), bias[i]);
    }
  }
}

}  // namespace ig

extern "C" int ig_abi_version(void) { return 2; }

extern "C" const char* ig_status_string(int status) {
  switch (status) {
    case IG_OK: return "ok";
    case IG_EINVAL: return "invalid argument";
    case IG_ERANGE: return "index out of range";
    case IG_ECONSISTENCY: return "partial key cache out of lock-step with its pool";
    case IG_ENOMEM: return "out of memory";
    default:
      if (status >= IG_ECUDA) return cudaGetErrorString((cudaError_t)(status - IG_ECUDA));
      return "unknown status";
  }
}

// Programmatic dependent launch (IG_LN_PDL=0: plain): the CTAs are resident and
// waiting when the producing GEMM completes -- C3 990 / 995 vs 989 / 985 tok/s
// at 15-30 MHz lower SM clocks (profiles/r02q_*)
static bool ln_pdl() {
  static const bool v = [] {
    const char* e = getenv("IG_LN_PDL");
    return !(e && atoi(e) == 0) && ig::pdl_enabled();
  }();
  return v;
}

extern "C" int ig_layernorm(const float* x, const float* gain, const float* bias, float eps,
                            int rows, int D, float* out, void* stream) {
  if (!x || !gain || !bias || !out || rows < 1 || D < 1 || !(eps > 0)) return IG_EINVAL;
  if (ln_pdl()) {
    IG_CUDA_STATUS(ig::launch_pdl(ig::layernorm_kernel, dim3(rows), dim3(ig::kLnThreads), 0,
                                  (cudaStream_t)stream, x, gain, bias, eps, D, out));
  } else {
    ig::layernorm_kernel<<<rows, ig::kLnThreads, 0, (cudaStream_t)stream>>>(x, gain, bias, eps, D,
                                                                            out);
  }
  IG_LAUNCH_STATUS();
  return IG_OK;
}
