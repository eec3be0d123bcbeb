"""Time the skinny dense-projection kernels (ig_sgemm_rows, ig_sgemm_tc) at
the decode step's shapes with CUDA events (best of N), for each ksplit.

    python tools/gemm_probe.py [--shape opt-13b] [--batch 16] [--ksplit auto|all]
Prints one JSON line per (kernel, shape, ksplit)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2406_19707_b200 import _lib
    from paper_2406_19707_b200.model import SHAPES
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="opt-13b")
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--ksplit", default="auto")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--chain", type=int, default=10,
                    help="launches back to back between one event pair (amortises host launch cost)")
    ap.add_argument("--fns", default="ig_sgemm_rows,ig_sgemm_tc")
    ap.add_argument("--only", default=None, help="N,K of a single shape")
    a = ap.parse_args()
    lib = _lib.load()
    sh = SHAPES[a.shape]
    D, F, M = sh["model_dim"], sh["ffn_dim"], a.batch
    shapes = {"fused_qkv_qspec": (4 * D, D), "qkv": (3 * D, D), "wo": (D, D), "ffn_in": (F, D),
              "ffn_out": (D, F)}
    if a.only:
        n_, k_ = (int(v) for v in a.only.split(","))
        shapes = {"only": (n_, k_)}
    for name, (N, K) in shapes.items():
        X = torch.randn(M, K, device="cuda")
        W = torch.randn(K, N, device="cuda")
        Y = torch.empty(M, N, device="cuda")
        for fn in a.fns.split(","):
            if fn == "ig_sgemm_packed":
                import ctypes
                pf, wf, tf = ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_size_t()
                _lib.call("ig_sgemm_packed_sizes", M, N, K, ctypes.byref(pf), ctypes.byref(wf),
                          ctypes.byref(tf), kernels=0)
                P = torch.empty(pf.value, device="cuda")
                _lib.call("ig_sgemm_pack", W.data_ptr(), N, N, K, P.data_ptr(), _lib.stream_handle())
                ws = torch.empty(wf.value, device="cuda")
                tk = torch.zeros(tf.value, dtype=torch.int32, device="cuda")
                ref = X @ W
                best = 1e9
                for _ in range(a.reps):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for _ in range(a.chain):
                        _lib.call(fn, X.data_ptr(), K, P.data_ptr(), N, K, Y.data_ptr(), N, None, 0, M, 0,
                                  ws.data_ptr(), ws.numel(), tk.data_ptr(), tk.numel(), _lib.stream_handle())
                    e1.record()
                    e1.synchronize()
                    best = min(best, e0.elapsed_time(e1) / a.chain)
                err = float((Y - ref).abs().max() / ref.abs().max())
                nbytes = 4 * (K * N + M * K + M * N)
                print(json.dumps({"fn": fn, "shape": name, "M": M, "N": N, "K": K, "us": best * 1e3,
                                  "gbs": nbytes / (best * 1e6), "relerr_vs_tf32_torch": err}), flush=True)
                del P
                continue
            auto = getattr(lib, fn + "_ksplit")(M, N, K)
            kss = [auto] if a.ksplit == "auto" else sorted({1, 2, 3, 4, 5, 6, 8, 10, 12, 16, 24, 32, auto})
            for ks in kss:
                ws = torch.empty(((N + 127) // 128) * ks * M * 128, device="cuda")
                tk = torch.zeros((N + 127) // 128, dtype=torch.int32, device="cuda")
                best = 1e9
                for _ in range(a.reps):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for _ in range(a.chain):
                        _lib.call(fn, X.data_ptr(), K, W.data_ptr(), N, Y.data_ptr(), N, None, 0, M, N, K, ks,
                                  0, ws.data_ptr(), ws.numel(), tk.data_ptr(), _lib.stream_handle())
                    e1.record()
                    e1.synchronize()
                    best = min(best, e0.elapsed_time(e1) / a.chain)
                nbytes = 4 * (K * N + M * K + M * N)
                print(json.dumps({"fn": fn, "shape": name, "M": M, "N": N, "K": K, "ksplit": ks,
                                  "auto": ks == auto, "us": best * 1e3, "gbs": nbytes / (best * 1e6)}),
                      flush=True)


if __name__ == "__main__":
    main()
