"""Where the end-to-end step's extra time goes: the same engine timed as
back-to-back graph replays (bench `value`) and through step_host (bench `e2e`),
with host perf_counter splits of the step_host path.  A truncated C3 (few
layers) keeps the setup short; the host turnaround does not depend on depth.

    python tools/e2e_probe.py [--layers 4] [--steps 50]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch
    from paper_2406_19707_b200.engine import DecodeEngine, RunConfig
    from paper_2406_19707_b200.model import SHAPES, ModelSpec, generate_synthetic_gpu, skew_model_gpu
    from paper_2406_19707_b200.speculation import SpeculationConfig
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--prompt", type=int, default=4096)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    sh = dict(SHAPES["opt-13b"])
    sh["layers"] = a.layers
    spec = ModelSpec(**sh, outlier_channels=8, outlier_scale=2.0, seed=0)
    model = generate_synthetic_gpu(spec, device=dev)
    skew_model_gpu(model)
    cfg = RunConfig(scheme="speculative", prompt_len=a.prompt, gen_len=4 * a.steps + 16, batch=a.batch,
                    speculation=SpeculationConfig(0.3, 4.0, 0.2, 1))
    eng = DecodeEngine(model, cfg, pool_dtype="f16", device=dev, cuda_graph=True, resident=True)
    del model
    g = torch.Generator(device=dev)
    g.manual_seed(1234)
    eng.prefill(torch.empty(a.batch, a.prompt, spec.model_dim, device=dev).normal_(generator=g))
    eng.release_model()
    for _ in range(3):
        eng.decode_step()
    torch.cuda.synchronize()
    cur = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(cur)
    for _ in range(a.steps):
        eng.decode_step()
    e1.record(cur)
    torch.cuda.synchronize()
    dev_ms = e0.elapsed_time(e1) / a.steps
    # host wall of back-to-back replays, synchronised each step (GPU idle = launch path)
    t0 = time.perf_counter()
    for _ in range(a.steps):
        eng.decode_step()
        cur.synchronize()
    sync_ms = (time.perf_counter() - t0) * 1e3 / a.steps
    # step_host with the bench's feedback loop, split by phase
    x_host = torch.empty((a.batch, spec.model_dim), dtype=torch.float32).pin_memory()
    x_host.copy_(eng.x.cpu())
    ph = {"h2d_issue": 0.0, "replay_issue": 0.0, "d2h_issue": 0.0, "wait": 0.0, "out_copy": 0.0,
          "feedback": 0.0}
    t_all = time.perf_counter()
    for _ in range(a.steps):
        t = time.perf_counter()
        eng.x.copy_(torch.from_numpy(x_host.numpy()).reshape(a.batch, spec.model_dim), non_blocking=True)
        t1 = time.perf_counter(); ph["h2d_issue"] += t1 - t
        y = eng.decode_step()
        t2 = time.perf_counter(); ph["replay_issue"] += t2 - t1
        if eng._out_host is None:
            eng._out_host = torch.empty(y.shape, dtype=y.dtype).pin_memory()
        eng._out_host.copy_(y, non_blocking=True)
        t3 = time.perf_counter(); ph["d2h_issue"] += t3 - t2
        cur.synchronize()
        t4 = time.perf_counter(); ph["wait"] += t4 - t3
        eng.check_errors()
        out = eng._out_host.numpy().copy()
        t5 = time.perf_counter(); ph["out_copy"] += t5 - t4
        x_host.copy_(torch.from_numpy(out))
        ph["feedback"] += time.perf_counter() - t5
    split_ms = (time.perf_counter() - t_all) * 1e3 / a.steps
    t0 = time.perf_counter()
    for _ in range(a.steps):
        out = eng.step_host(x_host.numpy())
        x_host.copy_(torch.from_numpy(out))
    e2e_ms = (time.perf_counter() - t0) * 1e3 / a.steps
    print(json.dumps({"layers": a.layers, "device_ms_per_step": dev_ms, "replay_sync_ms": sync_ms,
                      "step_host_ms": e2e_ms, "split_loop_ms": split_ms,
                      "split_us": {k: v * 1e6 / a.steps for k, v in ph.items()}}), flush=True)
    eng.close()


if __name__ == "__main__":
    main()
