"""Drive every path kernel once at a small size, for compute-sanitizer:

    compute-sanitizer --tool memcheck  python tools/sanitize_path.py
    compute-sanitizer --tool racecheck python tools/sanitize_path.py
    compute-sanitizer --tool synccheck python tools/sanitize_path.py

Engine decode on a 3-layer D=256 / d=128 model (the 512-B-row tensor-core
attention, the three GEMMs, rehearse/select/plan/fetch/append) in resident and
refetch modes with f16 and f32 pools, plus a pool-limit run (eviction)."""
import copy
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    from oracle import speckv_port as O
    import paper_2406_19707_b200 as G
    spec = O.ModelSpec(layers=3, model_dim=256, heads=2, ffn_dim=1024, outlier_channels=8,
                       outlier_scale=2.0, seed=3)
    sk = O.skew_model(O.generate_synthetic(spec), calib_seed=0)
    for limit in (None, 44):
        ocfg = O.RunConfig(scheme="speculative", prompt_len=40, gen_len=4, batch=2, pool_limit=limit)
        sessions = [O.Session(sk, ocfg, O.random_prompt(40, 256, b)) for b in range(2)]
        for pool in ("f16", "f32"):
            for resident in (True, False):
                for dense in ("packed", "cublas"):
                    cfg = G.RunConfig(scheme="speculative", prompt_len=40, gen_len=4, batch=2,
                                      pool_limit=limit)
                    eng = G.DecodeEngine.from_sessions(sk, cfg, copy.deepcopy(sessions), pool_dtype=pool,
                                                       resident=resident, dense=dense)
                    try:
                        for _ in range(4):
                            out = eng.decode_step()
                        assert np.all(np.isfinite(out.cpu().numpy()))
                    finally:
                        eng.close()
    # the packed GEMM alone at M = 16 with tile segments split over CTAs (stream-K
    # fix-ups through the workspace), chained as FFN-in -> FFN-out (PDL overlap)
    import ctypes
    import torch
    from paper_2406_19707_b200 import _lib
    M, D, F = 16, 512, 4096
    x = torch.randn(M, D, device="cuda")
    w1, w2 = torch.randn(D, F, device="cuda") * 0.05, torch.randn(F, D, device="cuda") * 0.05
    packs = []
    for W in (w1, w2):
        K, N = W.shape
        pf, wf, tf = ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_size_t()
        _lib.call("ig_sgemm_packed_sizes", M, N, K, ctypes.byref(pf), ctypes.byref(wf), ctypes.byref(tf),
                  kernels=0)
        P = torch.empty(pf.value, device="cuda")
        _lib.call("ig_sgemm_pack", W.data_ptr(), N, N, K, P.data_ptr(), _lib.stream_handle())
        packs.append((P, wf.value, tf.value))
    ws = torch.empty(max(p[1] for p in packs), device="cuda")
    tk = torch.zeros(max(p[2] for p in packs), dtype=torch.int32, device="cuda")
    h, y = torch.empty(M, F, device="cuda"), torch.empty(M, D, device="cuda")
    for _ in range(2):
        _lib.call("ig_sgemm_packed", x.data_ptr(), D, packs[0][0].data_ptr(), F, D, h.data_ptr(), F, None, 0,
                  M, 1, ws.data_ptr(), ws.numel(), tk.data_ptr(), tk.numel(), _lib.stream_handle())
        _lib.call("ig_sgemm_packed", h.data_ptr(), F, packs[1][0].data_ptr(), D, F, y.data_ptr(), D,
                  x.data_ptr(), D, M, 2, ws.data_ptr(), ws.numel(), tk.data_ptr(), tk.numel(),
                  _lib.stream_handle())
    ref = torch.relu(x.double() @ w1.double()) @ w2.double() + x.double()
    assert torch.allclose(y.double(), ref, rtol=1e-5, atol=1e-4)
    print("sanitize_path: all configurations ran")


if __name__ == "__main__":
    main()
