#!/usr/bin/env python3
"""Kernel-time breakdown of the GPU prefill (torch.profiler / CUPTI) at a
bench shape with a few layers: python tools/prefill_profile.py [--layers 4]"""
import argparse
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="opt-13b")
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--prompt", type=int, default=4096)
    ap.add_argument("--layers", type=int, default=4)
    a = ap.parse_args()
    import time
    import torch
    from torch.profiler import ProfilerActivity, profile
    from paper_2406_19707_b200.engine import DecodeEngine, RunConfig
    from paper_2406_19707_b200.model import SHAPES, ModelSpec, generate_synthetic_gpu, skew_model_gpu
    from paper_2406_19707_b200.speculation import SpeculationConfig
    dev = torch.device("cuda", 0)
    sh = dict(SHAPES[a.shape], layers=a.layers)
    spec = ModelSpec(**sh, outlier_channels=8, outlier_scale=2.0, seed=0)
    model = generate_synthetic_gpu(spec, device=dev)
    skew_model_gpu(model)
    cfg = RunConfig(scheme="speculative", prompt_len=a.prompt, gen_len=4, batch=a.batch,
                    speculation=SpeculationConfig(0.3, 4.0, 0.2, 1))
    eng = DecodeEngine(model, cfg, pool_dtype="f16", device=dev)
    g = torch.Generator(device=dev)
    g.manual_seed(1)
    prompts = torch.empty(a.batch, a.prompt, spec.model_dim, device=dev).normal_(generator=g)
    torch.cuda.synchronize()
    t0 = time.time()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        eng.prefill(prompts)
        torch.cuda.synchronize()
    wall = time.time() - t0
    kinds = collections.defaultdict(float)
    for e in prof.events():
        if e.device_type.name == "CUDA":
            k = e.name.split("(")[0].split("<")[0].replace("void ", "")[:60]
            kinds[k] += e.device_time_total / 1e3 if hasattr(e, "device_time_total") else e.cuda_time_total / 1e3
    top = sorted(kinds.items(), key=lambda kv: -kv[1])[:15]
    print(json.dumps({"layers": a.layers, "wall_s": wall, "per_layer_s": wall / a.layers,
                      "kernels_ms": {k: round(v, 2) for k, v in top}}, indent=1))


if __name__ == "__main__":
    main()
