"""Time the packed dense-projection GEMM (ig_sgemm_pack + ig_sgemm_packed) at
the decode step's shapes with CUDA events: best of --reps, each a chain of
--chain launches between one event pair (amortises the host launch cost).

    python tools/gemm_probe.py [--shape opt-13b] [--batch 16] [--only N,K]
Prints one JSON line per shape."""
import argparse
import ctypes
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
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--chain", type=int, default=10)
    ap.add_argument("--only", default=None, help="N,K of a single shape")
    a = ap.parse_args()
    _lib.load()
    sh = SHAPES[a.shape]
    D, F, M = sh["model_dim"], sh["ffn_dim"], a.batch
    shapes = {"fused_qkv_qspec": (4 * D, D), "qkv": (3 * D, D), "wo": (D, D), "ffn_in": (F, D),
              "ffn_out": (D, F)}
    if a.only:
        n_, k_ = (int(v) for v in a.only.split(","))
        shapes = {"only": (n_, k_)}
    h = _lib.stream_handle()
    for name, (N, K) in shapes.items():
        X = torch.randn(M, K, device="cuda")
        W = torch.randn(K, N, device="cuda")
        Y = torch.empty(M, N, device="cuda")
        pf, wf, tf = ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_size_t()
        _lib.call("ig_sgemm_packed_sizes", M, N, K, ctypes.byref(pf), ctypes.byref(wf), ctypes.byref(tf),
                  kernels=0)
        P = torch.empty(pf.value, device="cuda")
        _lib.call("ig_sgemm_pack", W.data_ptr(), N, N, K, P.data_ptr(), h)
        ws = torch.empty(wf.value, device="cuda")
        tk = torch.zeros(tf.value, dtype=torch.int32, device="cuda")
        ref = X.double() @ W.double()
        best = 1e9
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.chain):
                _lib.call("ig_sgemm_packed", X.data_ptr(), K, P.data_ptr(), N, K, Y.data_ptr(), N, None, 0, M,
                          0, ws.data_ptr(), ws.numel(), tk.data_ptr(), tk.numel(), h)
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1) / a.chain)
        err = float((Y.double() - ref).abs().max() / ref.abs().max())
        nbytes = 4 * (K * N + M * K + M * N)
        print(json.dumps({"fn": "ig_sgemm_packed", "shape": name, "M": M, "N": N, "K": K, "us": best * 1e3,
                          "gbs": nbytes / (best * 1e6), "relerr_vs_f64": err}), flush=True)
        del P, W


if __name__ == "__main__":
    main()
