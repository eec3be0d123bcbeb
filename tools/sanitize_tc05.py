"""Drive the tcgen05 kernels once at small sizes, for compute-sanitizer:

    compute-sanitizer --tool memcheck  python tools/sanitize_tc05.py
    compute-sanitizer --tool racecheck python tools/sanitize_tc05.py
    compute-sanitizer --tool synccheck python tools/sanitize_tc05.py

ig_split_f16 + ig_gemm_tc05 (ragged M / N / K, all epilogues, several tiles per
CTA) and the tcgen05 attention (IG_ATTEND_IMPL=c, set here before the library
reads it: slot tables with holes, an empty set, rows split over CTAs with
ticket merges, f16 and bf16), plus the prefill path on a 2-layer model."""
import ctypes
import os
import sys

os.environ["IG_ATTEND_IMPL"] = "c"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2406_19707_b200 import _lib, tcgemm
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    for M, N, K in ((130, 300, 100), (257, 512, 640)):
        X = torch.randn(M, K, device="cuda", generator=g)
        W = torch.randn(K, N, device="cuda", generator=g)
        R = torch.randn(M, N, device="cuda", generator=g)
        for ep in (0, 1, 2):
            tcgemm.matmul(X, W, epilogue=ep, R=R if ep == 2 else None)
        A, B = tcgemm.split_rows(X), tcgemm.split_weight(W)
        tcgemm.gemm(A, B, max_ctas=2)
    torch.cuda.synchronize()
    for T, elt in ((torch.float16, 1), (torch.bfloat16, 2)):
        B_, Hg, d, cap = 2, 3, 128, 600
        q = torch.randn(B_, 3 * Hg * d, device="cuda", generator=g)
        stage = torch.randn(B_, Hg, cap, 2 * d, device="cuda", generator=g).to(T)
        used = torch.tensor([[600, 257, 0], [130, 1, 599]], dtype=torch.int32, device="cuda")
        slot = torch.arange(cap, device="cuda", dtype=torch.int32).repeat(B_, Hg, 1).contiguous()
        slot[:, :, 2::9] = -1
        pos = torch.full((B_, Hg), 4, dtype=torch.int32, device="cuda")
        st = torch.zeros(8, dtype=torch.int32, device="cuda")
        pf, tk = ctypes.c_size_t(), ctypes.c_size_t()
        _lib.call("ig_attend_scratch", B_, Hg, d, cap, ctypes.byref(pf), ctypes.byref(tk), kernels=0)
        part = torch.empty(pf.value, device="cuda")
        tick = torch.zeros(tk.value, dtype=torch.int32, device="cuda")
        out = torch.empty(B_, Hg * d, device="cuda")
        _lib.call("ig_attend_slots", q.data_ptr(), 3 * Hg * d, q.data_ptr() + 4 * Hg * d, q.data_ptr() + 8 * Hg * d,
                  3 * Hg * d, stage.data_ptr(), elt, slot.data_ptr(), used.data_ptr(), pos.data_ptr(), st.data_ptr(),
                  B_, Hg, d, cap, part.data_ptr(), tick.data_ptr(), out.data_ptr(), Hg * d, _lib.stream_handle())
    torch.cuda.synchronize()
    # the prefill on tcgen05 GEMMs
    import numpy as np
    from oracle import speckv_port as O
    import paper_2406_19707_b200 as G
    spec = O.ModelSpec(layers=2, model_dim=256, heads=2, ffn_dim=1024, outlier_channels=8, outlier_scale=2.0, seed=3)
    sk = O.skew_model(O.generate_synthetic(spec), calib_seed=0)
    cfg = G.RunConfig(scheme="speculative", prompt_len=48, gen_len=2, batch=2)
    eng = G.DecodeEngine(sk, cfg, pool_dtype="f16")
    eng.prefill(np.stack([O.random_prompt(48, 256, b) for b in range(2)]))
    eng.decode_step()
    torch.cuda.synchronize()
    eng.close()
    print("sanitize_tc05 done")


if __name__ == "__main__":
    main()
