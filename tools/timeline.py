#!/usr/bin/env python3
"""Kernel timeline of the bench's decode step (CUPTI via torch.profiler).

    python tools/timeline.py [--shape opt-13b --batch 16 --prompt 4096] [--steps 3]
                             [--layers N] [--out gpurun_out/timeline.json]

Builds the bench engine (same defaults as bench.py), warms up, then records
`--steps` decode steps (CUDA-graph replays by default) and writes, per kernel
launch: name, stream, start / end (us, relative to the first kernel), plus a
summary: step time, per-stream busy time, per-kernel-kind totals and the
compute stream's idle gaps (what the critical path waits on).  No ncu, no
serialisation: this is the concurrent schedule as it runs.
"""

from __future__ import annotations

import argparse
import collections
import json
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="opt-13b")
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--prompt", type=int, default=4096)
    ap.add_argument("--layers", type=int, default=None)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--no-cuda-graph", dest="cuda_graph", action="store_false")
    ap.add_argument("--out", default="gpurun_out/timeline.json")
    a = ap.parse_args()
    import torch
    from paper_2406_19707_b200.engine import DecodeEngine, RunConfig
    from paper_2406_19707_b200.model import SHAPES, ModelSpec, generate_synthetic_gpu, skew_model_gpu
    from paper_2406_19707_b200.speculation import SpeculationConfig

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    sh = dict(SHAPES[a.shape])
    if a.layers:
        sh["layers"] = a.layers
    spec = ModelSpec(**sh, outlier_channels=8, outlier_scale=2.0, seed=0)
    model = generate_synthetic_gpu(spec, device=dev)
    skew_model_gpu(model)
    cfg = RunConfig(scheme="speculative", prompt_len=a.prompt, gen_len=a.steps + 16, batch=a.batch,
                    speculation=SpeculationConfig(0.3, 4.0, 0.2, 1))
    eng = DecodeEngine(model, cfg, pool_dtype="f16", device=dev, cuda_graph=a.cuda_graph)
    del model
    torch.cuda.empty_cache()
    g = torch.Generator(device=dev)
    g.manual_seed(1234)
    prompts = torch.empty(a.batch, a.prompt, spec.model_dim, device=dev).normal_(generator=g)
    eng.prefill(prompts)
    del prompts
    eng.release_model()
    torch.cuda.empty_cache()
    for _ in range(4):
        eng.decode_step()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(a.steps):
            eng.decode_step()
        torch.cuda.synchronize()
    with tempfile.NamedTemporaryFile(suffix=".json", delete=False) as f:
        path = f.name
    prof.export_chrome_trace(path)
    with open(path) as f:
        tr = json.load(f)
    os.unlink(path)
    ks = [e for e in tr["traceEvents"] if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy",
                                                                                     "gpu_memset")]
    ks.sort(key=lambda e: e["ts"])
    t0 = ks[0]["ts"]
    launches = [{"name": e["name"][:90], "stream": e.get("args", {}).get("stream", e.get("tid")),
                 "t": round(e["ts"] - t0, 3), "dur": round(e["dur"], 3), "cat": e["cat"]} for e in ks]
    span = max(x["t"] + x["dur"] for x in launches)
    # per stream busy (union of intervals) and the busiest stream's gaps
    by_stream = collections.defaultdict(list)
    for x in launches:
        by_stream[x["stream"]].append(x)
    streams = {}
    for sid, xs in by_stream.items():
        busy, end, gaps = 0.0, None, []
        for x in xs:
            s0, s1 = x["t"], x["t"] + x["dur"]
            if end is None or s0 >= end:
                if end is not None:
                    gaps.append((round(s0 - end, 2), x["name"][:50]))
                busy += s1 - s0
                end = s1
            elif s1 > end:
                busy += s1 - end
                end = s1
        gaps.sort(reverse=True)
        streams[str(sid)] = {"launches": len(xs), "busy_us": round(busy, 1),
                             "gap_us_total": round(sum(g_[0] for g_ in gaps), 1),
                             "gaps_over_2us": sum(1 for g_ in gaps if g_[0] > 2),
                             "largest_gaps": gaps[:12]}
    kinds = collections.defaultdict(lambda: [0, 0.0])
    for x in launches:
        k = x["name"].split("(")[0].split("<")[0].replace("void ", "")
        kinds[k][0] += 1
        kinds[k][1] += x["dur"]
    summary = {"steps": a.steps, "span_us": round(span, 1), "us_per_step": round(span / a.steps, 1),
               "config": {"shape": a.shape, "batch": a.batch, "prompt": a.prompt, "layers": eng.L,
                          "cuda_graph": a.cuda_graph},
               "streams": streams,
               "kinds": {k: {"launches": v[0], "us_total": round(v[1], 1),
                             "us_per_step": round(v[1] / a.steps, 1),
                             "us_per_launch": round(v[1] / max(v[0], 1), 2)}
                         for k, v in sorted(kinds.items(), key=lambda kv: -kv[1][1])}}
    os.makedirs(os.path.dirname(os.path.abspath(a.out)), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump({"summary": summary, "launches": launches}, f)
    print(json.dumps(summary, indent=1))
    eng.close()


if __name__ == "__main__":
    main()
