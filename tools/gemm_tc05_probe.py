#!/usr/bin/env python3
"""Throughput of the tcgen05 prefill GEMM (ig_gemm_tc05) at the C3 prefill
shapes vs torch fp32 (IEEE, cuBLAS) and TF32.  One JSON line per shape."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2406_19707_b200 import tcgemm
    torch.backends.cuda.matmul.allow_tf32 = False
    shapes = [(65536, 15360, 5120), (65536, 5120, 5120), (65536, 20480, 5120), (65536, 5120, 20480),
              (8192, 5120, 5120)]
    if len(sys.argv) > 1:
        shapes = [tuple(int(v) for v in s.split("x")) for s in sys.argv[1:]]
    for M, N, K in shapes:
        X = torch.randn(M, K, device="cuda")
        W = torch.randn(K, N, device="cuda") / K ** 0.5
        A, B = tcgemm.split_rows(X), tcgemm.split_weight(W)
        out = torch.empty(M, N, device="cuda")

        def t(fn, reps=3):
            fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                fn()
            e1.record()
            e1.synchronize()
            return e0.elapsed_time(e1) / reps

        fl = 2.0 * M * N * K
        ms_tc = t(lambda: tcgemm.gemm(A, B, out))
        ms_split = t(lambda: tcgemm.split_rows(X, A))
        ms_f32 = t(lambda: torch.matmul(X, W, out=out))
        torch.backends.cuda.matmul.allow_tf32 = True
        ms_tf32 = t(lambda: torch.matmul(X, W, out=out))
        torch.backends.cuda.matmul.allow_tf32 = False
        print(json.dumps({"M": M, "N": N, "K": K, "tc05_ms": ms_tc, "tc05_tflops": fl / ms_tc / 1e9,
                          "split_a_ms": ms_split, "cublas_f32_tflops": fl / ms_f32 / 1e9,
                          "cublas_tf32_tflops": fl / ms_tf32 / 1e9}), flush=True)
        del X, W, A, B, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
