#!/usr/bin/env python3
"""Timeline of the tcgen05 attention (csrc/attend_tc05.cu) on a C3-shaped slot
table: B 16 x Hg 40 (b, h), `--rows` resident rows each, f16.  Prints the
kernel time (CUDA events, 10 launches chained) and, from one traced launch,
per-CTA averages of the pipeline gaps (globaltimer, ns)."""
import argparse
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=819)
    ap.add_argument("--B", type=int, default=16)
    ap.add_argument("--Hg", type=int, default=40)
    ap.add_argument("--cap", type=int, default=820)
    a = ap.parse_args()
    import numpy as np
    import torch
    from paper_2406_19707_b200 import _lib
    B, Hg, d, cap = a.B, a.Hg, 128, a.cap
    g = torch.Generator(device="cuda")
    g.manual_seed(1)
    q = torch.randn(B, 4 * Hg * d, device="cuda", generator=g)
    stage = torch.randn(B, Hg, cap, 2 * d, device="cuda", generator=g).half()
    slot = torch.arange(cap, device="cuda", dtype=torch.int32).repeat(B, Hg, 1).contiguous()
    used = torch.full((B, Hg), a.rows, dtype=torch.int32, device="cuda")
    pos = torch.full((B, Hg), 5, dtype=torch.int32, device="cuda")
    st = torch.zeros(8, dtype=torch.int32, device="cuda")
    pf, tk = ctypes.c_size_t(), ctypes.c_size_t()
    _lib.call("ig_attend_scratch", B, Hg, d, cap, ctypes.byref(pf), ctypes.byref(tk), kernels=0)
    part = torch.empty(pf.value, device="cuda")
    tick = torch.zeros(tk.value, dtype=torch.int32, device="cuda")
    out = torch.empty(B, Hg * d, device="cuda")
    Hgd = Hg * d
    ld = q.stride(0)

    def launch():
        _lib.call("ig_attend_slots", q.data_ptr(), ld, q.data_ptr() + 4 * Hgd, q.data_ptr() + 8 * Hgd, ld,
                  stage.data_ptr(), 1, slot.data_ptr(), used.data_ptr(), pos.data_ptr(), st.data_ptr(), B, Hg, d,
                  cap, part.data_ptr(), tick.data_ptr(), out.data_ptr(), Hgd, _lib.stream_handle())

    launch()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        launch()
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 10
    nbytes = B * Hg * a.rows * 512
    res = {"rows": a.rows, "us": ms * 1e3, "gbs": nbytes / ms / 1e6}
    if os.environ.get("IG_ATTEND_IMPL", "c")[0] != "c":
        print(json.dumps(res))
        return
    G, stride, T = 148, 8 + 9 * 64, 64
    buf = torch.zeros(G * stride, dtype=torch.int64, device="cuda")
    _lib.call("ig_debug_attend_trace", buf.data_ptr(), kernels=0)
    launch()
    torch.cuda.synchronize()
    _lib.call("ig_debug_attend_trace", None, kernels=0)
    tr = buf.cpu().numpy().reshape(G, stride).astype(np.int64)
    t0 = tr[:, 0].min()
    ev = tr[:, 8:].reshape(G, 9, T)
    stats = {}
    n_t = (ev[:, 0] > 0).sum(axis=1)
    res["tiles_per_cta"] = [int(n_t.min()), int(n_t.max())]
    res["cta_start_spread_us"] = float((tr[:, 0].max() - t0) / 1e3)
    res["setup_us"] = float(np.median(tr[:, 1] - tr[:, 0]) / 1e3)
    res["cta_end_us"] = [float((tr[:, 2].min() - t0) / 1e3), float((tr[:, 2].max() - t0) / 1e3)]
    ends = (tr[:, 2] - t0) / 1e3
    res["cta_end_by_block"] = [round(float(v), 1) for v in ends]
    roles = ["producer", "mma", "qwarp", "softmax", "readout"]
    res["role_end_by_block"] = {nm: [round(float((tr[c, 3 + i] - t0) / 1e3), 1) for c in range(G)]
                                for i, nm in enumerate(roles)}
    names = ["load_issue", "s_issue", "pv_issue", "softmax_start", "softmax_end", "readout_end"]
    # per tile latencies, median over CTAs and tiles 1..n-2
    for i in range(1, 6):
        lat = []
        for c in range(G):
            for t in range(1, int(n_t[c]) - 1):
                if ev[c, i, t] > 0 and ev[c, i - 1, t] > 0:
                    lat.append(ev[c, i, t] - ev[c, i - 1, t])
        stats[f"{names[i - 1]}->{names[i]}_ns"] = float(np.median(lat)) if lat else None
    per = []
    for c in range(G):
        k = int(n_t[c])
        if k > 2:
            per.append((ev[c, 0, k - 1] - ev[c, 0, 1]) / (k - 2))
    stats["load_issue_interval_ns"] = float(np.median(per))
    def span(i, j):
        lat = [ev[c, j, t] - ev[c, i, t] for c in range(G) for t in range(1, int(n_t[c]) - 1)
               if ev[c, i, t] > 0 and ev[c, j, t] > 0]
        return float(np.median(lat)) if lat else None
    stats["readout_start->ofull_ns"] = span(6, 7)
    stats["ofull->tmem_ld_ns"] = span(7, 8)
    stats["tmem_ld->readout_end_ns"] = span(8, 5)
    stats["pv_issue->ofull_ns"] = span(2, 7)
    stats["pv_issue(t-3)->load_issue(t)_ns"] = float(np.median(
        [ev[c, 0, t] - ev[c, 2, t - 3] for c in range(G) for t in range(4, int(n_t[c]) - 1)]))
    res["median"] = stats
    # raw per-tile stamps (us from the CTA's start) of one CTA
    c = G // 2
    res["cta"] = {names_i: [round((ev[c, i, t] - tr[c, 0]) / 1e3, 2) for t in range(int(n_t[c]))]
                  for i, names_i in enumerate(names + ["readout_start", "ofull_seen", "o_loaded"])}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
