"""Time ig_attend / ig_attend_slots alone at the C3 per-layer shapes (CUDA
events, best of N), one JSON line per case.  The kernel variant comes from
IG_ATTEND_IMPL / IG_ATT_VARIANT (read once per process).

    IG_ATT_VARIANT=1 python tools/attend_probe.py [--batch 16 --heads 40 --ctx 4096]
"""
import argparse
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2406_19707_b200 import _lib
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--heads", type=int, default=40)
    ap.add_argument("--ctx", type=int, default=4096)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--sweep", type=str, default="",
                    help="comma-separated row counts at the 20%% cap (fixed-cost fit), e.g. 16,256,819")
    ap.add_argument("--chain", type=int, default=10,
                    help="launches back to back between one event pair (amortises host launch cost)")
    a = ap.parse_args()
    _lib.load()
    B, Hg, d = a.batch, a.heads, 128
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    cases = [("layer>=1 (n = 20% cap)", a.ctx // 5, a.ctx // 5 + 1),
             ("layer 0 (all rows)", a.ctx, a.ctx + 4)]
    if a.sweep:
        cases = [(f"sweep rows {r}", int(r), a.ctx // 5 + 1) for r in a.sweep.split(",")]
    for name, rows, cap in cases:
        q = torch.randn(B, 3 * Hg * d, device="cuda", generator=g)
        stage = torch.randn(B, Hg, cap, 2 * d, device="cuda", generator=g).half()
        n = torch.full((B,), rows, dtype=torch.int32, device="cuda")
        idx = torch.arange(cap, dtype=torch.int32, device="cuda").repeat(B, Hg, 1).contiguous()
        pos = torch.full((B, Hg), -1, dtype=torch.int32, device="cuda")
        st = torch.zeros(8, dtype=torch.int32, device="cuda")
        pf, tk = ctypes.c_size_t(), ctypes.c_size_t()
        _lib.call("ig_attend_scratch", B, Hg, d, cap, ctypes.byref(pf), ctypes.byref(tk), kernels=0)
        part = torch.empty(pf.value, device="cuda")
        tick = torch.zeros(tk.value, dtype=torch.int32, device="cuda")
        out = torch.empty(B, Hg * d, device="cuda")
        def launch():
            _lib.call("ig_attend", q.data_ptr(), 3 * Hg * d, q.data_ptr() + 4 * Hg * d,
                      q.data_ptr() + 8 * Hg * d, 3 * Hg * d, stage.data_ptr(), _lib.ELT["f16"],
                      idx.data_ptr(), n.data_ptr(), pos.data_ptr(), st.data_ptr(), B, Hg, d, cap,
                      part.data_ptr(), tick.data_ptr(), out.data_ptr(), Hg * d, _lib.stream_handle())
        launch()
        best = 1e9
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.chain):
                launch()
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1) / a.chain)
        nbytes = B * Hg * rows * 2 * d * 2
        print(json.dumps({"case": name, "impl": os.environ.get("IG_ATTEND_IMPL", "mma"),
                          "variant": os.environ.get("IG_ATT_VARIANT", "0"), "rows": rows,
                          "us": best * 1e3, "gbs": nbytes / (best * 1e6)}), flush=True)


if __name__ == "__main__":
    main()
