"""ig_select at the bench's C3 workload: which path each (b, h) row takes and
how long the kernel runs alone.

Builds the bench's synthetic OPT-13B-shaped model (--layers of it), prefills
the batch, decodes two steps, then for each layer li >= 1 takes the
rehearsal scores of the speculation hook (DecodeEngine.speculate) and
  * replays csrc/select.cu's value binning in numpy (f32, same formulas) to
    report the boundary-bin size m per row and the mode split
    (0: boundary bin taken whole, 1: <= 1024 candidates ranked, 2: radix
    select inside the boundary bin);
  * times ig_select on those scores (chained launches between one event pair).
Prints one JSON line per layer."""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

KBINS, KCAND = 2048, 1024


def order_key(x: np.ndarray) -> np.ndarray:
    u = np.where(x == 0, np.float32(0), x).astype(np.float32).view(np.uint32)   # -0.0 keyed as +0.0
    return np.where(u & 0x80000000, ~u, u | 0x80000000).astype(np.uint32)


def modes(scores: np.ndarray, nn: int) -> np.ndarray:
    """[rows] boundary-bin size m, [rows] mode, as select_row computes them."""
    out_m, out_mode = [], []
    for row in scores.reshape(-1, scores.shape[-1]):
        k = order_key(row)
        hi = np.float32(row[np.argmax(k)])
        lo = np.float32(row[np.argmin(k)])
        with np.errstate(divide="ignore", over="ignore"):
            scale = np.float32(KBINS) / np.float32(hi - lo)
        if not scale < np.float32(1e30):
            scale = np.float32(0)
        b = np.minimum((np.float32(hi) - row.astype(np.float32)) * scale, np.float32(KBINS - 1)).astype(np.int32)
        h = np.bincount(b, minlength=KBINS)
        c = np.cumsum(h)
        bstar = int(np.searchsorted(c, nn))
        need = nn - (int(c[bstar - 1]) if bstar else 0)
        m = int(h[bstar])
        out_m.append(m)
        out_mode.append(0 if m == need else (1 if m <= KCAND else 2))
    return np.array(out_m), np.array(out_mode)


def main():
    import ctypes
    import torch
    from paper_2406_19707_b200 import _lib
    from paper_2406_19707_b200.engine import DecodeEngine, RunConfig
    from paper_2406_19707_b200.model import SHAPES, ModelSpec, generate_synthetic_gpu, skew_model_gpu
    from paper_2406_19707_b200.speculation import SpeculationConfig
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="opt-13b")
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--prompt", type=int, default=4096)
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--chain", type=int, default=20)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    sh = dict(SHAPES[a.shape])
    sh["layers"] = a.layers
    spec = ModelSpec(**sh, outlier_channels=8, outlier_scale=2.0, seed=0)
    model = generate_synthetic_gpu(spec, device=dev)
    skew_model_gpu(model)
    cfg = RunConfig(scheme="speculative", prompt_len=a.prompt, gen_len=8, batch=a.batch,
                    speculation=SpeculationConfig(0.3, 4.0, 0.2, 1))
    eng = DecodeEngine(model, cfg, pool_dtype="f16", device=dev, cuda_graph=False)
    g = torch.Generator(device=dev)
    g.manual_seed(1234)
    prompts = torch.empty(a.batch, a.prompt, spec.model_dim, device=dev).normal_(generator=g)
    eng.prefill(prompts)
    del prompts
    for _ in range(2):
        eng.decode_step()
    torch.cuda.synchronize()
    B, Hg, S = eng.B, eng.Hg, eng.S_max
    h = _lib.stream_handle()
    for li in range(1, a.layers):
        out = eng.speculate(li)
        sc = out["scores"]                    # [B, Hg, s]
        s = sc.shape[-1]
        nn = int(out["n"][0])
        m, mode = modes(sc[0], nn)
        dsc = torch.zeros((B, Hg, S), dtype=torch.float32, device=dev)
        dsc[:, :, :s] = torch.from_numpy(sc).to(dev)
        csum = torch.from_numpy(out["count_sum"].astype(np.int32)).to(dev)
        idx = torch.zeros((B, Hg, eng.cap), dtype=torch.int32, device=dev)
        n = torch.zeros(B, dtype=torch.int32, device=dev)
        err = torch.zeros(1, dtype=torch.int32, device=dev)

        keys = order_key(sc.reshape(-1, s)).reshape(B, Hg, s)
        rr = torch.from_numpy(np.stack([keys.max(-1), keys.min(-1)], -1).view(np.int32)).to(dev)
        times = {}
        for name, rrp in (("select_us", None), ("select_ranged_us", rr.data_ptr())):
            def launch():
                _lib.call("ig_select", dsc.data_ptr(), csum.data_ptr(), eng.st.data_ptr(), B, Hg, eng.H, S,
                          eng.cap, 0.2, 1, idx.data_ptr(), n.data_ptr(), err.data_ptr(), rrp, h)
            launch()
            torch.cuda.synchronize()
            best = 1e9
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(a.chain):
                    launch()
                e1.record()
                e1.synchronize()
                best = min(best, e0.elapsed_time(e1) / a.chain)
            times[name] = best * 1e3
            same = bool((idx.cpu().numpy() == out["idx"]).all())
            if not same:
                break
        print(json.dumps({"layer": li, "s": s, "n_b0": nn, **times,
                          "mode_counts_b0": np.bincount(mode, minlength=3).tolist(),
                          "m_median_b0": float(np.median(m)), "m_max_b0": int(m.max()),
                          "same_idx_as_hook": same}), flush=True)
    del ctypes


if __name__ == "__main__":
    main()
