#!/usr/bin/env python3
"""Decode-throughput benchmark of the B200 InfiniGen KV path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Workload (BASELINE.json metric "decode tok/s (OPT-13B, KV on host)"):
OPT-13B-shaped decode (40 layers, D 5120, 40 heads, d 128, FFN 20480),
batch 16, 4096-token prompt (context 4096 + steps), KV pool in pinned host
memory (fp16, e = 2 B, the reference accounting), speculation ratio 0.3,
alpha 4, cap 20%.  Weights: random init with the reference's synthetic
recipe (outlier scale 2.0) drawn by torch's RNG on the GPU; skew by GPU SVD;
prompts N(0, 1); GPU prefill (TF32) builds the pool -- all outside the timed
region.  A "step" = one decode iteration of all 16 sequences.

N > 1 (torchrun): heads are sharded over the ranks (each owns H/N heads,
their pool shard and partial keys); NCCL all-reduces the per-layer head
counts and W_O output.  Total work is fixed -> "scaling": "strong".

--impl reference times the reference algorithm (the NumPy oracle port; the
reference is Python, so there is nothing to compile) on the host cores: a
3-layer truncation of the same shape at the same context with injected
state, extrapolated to 40 layers and to the serial batch (engine.py:468-476).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOAD = dict(name="OPT-13B-shaped decode, batch 16, 4K context (BASELINE.json configs[2])",
                shape="opt-13b", batch=16, prompt=4096, alpha=4.0, ratio=0.3, cap=0.2,
                outlier_scale=2.0)
METRIC = "decode tok/s (OPT-13B, KV on host)"
UNIT = "tok/s"


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--batch", type=int, default=WORKLOAD["batch"])
    ap.add_argument("--prompt", type=int, default=WORKLOAD["prompt"])
    ap.add_argument("--shape", default=WORKLOAD["shape"])
    ap.add_argument("--layers", type=int, default=None, help="override (debug only)")
    ap.add_argument("--fetch-ctas", type=int, default=32)
    ap.add_argument("--fetch-threads", type=int, default=32)
    ap.add_argument("--fetch-priority", type=int, default=0, help="CUDA stream priority (-1 = high)")
    ap.add_argument("--fetch-impl", default="tma", choices=["ldg", "tma"])
    ap.add_argument("--fetch-rows", type=int, default=16, help="TMA rows per warp batch")
    ap.add_argument("--dense", default="packed", choices=["cublas", "packed"])
    ap.add_argument("--no-cuda-graph", dest="cuda_graph", action="store_false",
                    help="launch every kernel eagerly instead of replaying a captured decode step")
    ap.add_argument("--no-resident", dest="resident", action="store_false",
                    help="refetch every selected row each step (the reference's data movement) "
                         "instead of keeping each layer's fetched set resident in HBM")
    ap.add_argument("--no-spec-stream", dest="spec_stream", action="store_false",
                    help="run the speculation chain on the compute stream (A/B of the overlap)")
    ap.add_argument("--append-stream", action="store_true",
                    help="run ig_append beside the attention on its own stream (measured neutral)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo lets N ranks share one GPU (tests of the N > 1 path)")
    ap.add_argument("--no-variant", "--no-hbm-variant", dest="no_variant", action="store_true",
                    help="skip the secondary run (resident: refetch every step; else layer 0 in HBM)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-steps", type=int, default=None,
                    help="timed 3-layer steps of the CPU baseline (default: --steps, as the reference arm)")
    return ap.parse_args()


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self._p = index, [], None

    def __enter__(self):
        try:
            self._p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                        "-i", str(self.index), "-lms", "100"],
                                       stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except OSError:
            self._p = None
        return self

    def _read(self):
        for line in self._p.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self._p is not None:
            self._p.terminate()
            try:
                self._p.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self._p.kill()

    def summary(self) -> dict:
        sm = [float(r[1]) for r in self.rows if len(r) > 2 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 2 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 9
                          for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# --------------------------------------------------------- reference (CPU)
def cpu_reference(shape: str, batch: int, prompt: int, steps: int, warmup: int = 1, ctx: dict | None = None) -> dict:
    """Time the reference algorithm (oracle port, NumPy/OpenBLAS, all host
    cores) on a 3-layer truncation of the workload with injected state;
    extrapolate T_step = T0 + (L-2) * T1 + T_last per sequence, x batch.
    ctx (a dict): filled with the truncation's model, state and the oracle's
    outputs and selections, for the GPU parity check of the same run."""
    import numpy as np
    from oracle import speckv_port as O
    from paper_2406_19707_b200.model import SHAPES
    sh = SHAPES[shape]
    L_full, D, H, F = sh["layers"], sh["model_dim"], sh["heads"], sh["ffn_dim"]
    d = D // H
    Lt = 3
    rng = np.random.default_rng(0)
    spec = O.ModelSpec(layers=Lt, model_dim=D, heads=H, ffn_dim=F, outlier_channels=8,
                       outlier_scale=2.0, seed=0)

    def mat(r, c):
        return rng.standard_normal((r, c), dtype=np.float32) * np.float32(1.0 / np.sqrt(r))

    layers = []
    for _ in range(Lt):
        g = (1 + 0.02 * rng.standard_normal(D)).astype(np.float32)
        layers.append(O.Layer(mat(D, D), mat(D, D), mat(D, D), mat(D, D), mat(D, F), mat(F, D),
                              g, np.zeros(D, np.float32), g.copy(), np.zeros(D, np.float32)))
    model = O.Model(spec, layers, np.zeros(0, np.int64), skewed=True)
    kc = int(np.ceil(0.3 * d))
    # K / V f16-representable: the bench's f16 host pool then holds the oracle's values
    kv = [[tuple(rng.standard_normal((prompt, d), dtype=np.float32).astype(np.float16).astype(np.float32)
                 for _ in range(2)) for _ in range(H)] for _ in range(Lt)]
    cols = [[np.sort(rng.choice(d, kc, replace=False)) for _ in range(H)] for _ in range(Lt)]
    cfg = O.RunConfig(scheme="speculative", prompt_len=prompt, gen_len=steps + warmup, batch=1,
                      speculation=O.SpeculationConfig(WORKLOAD["ratio"], WORKLOAD["alpha"], WORKLOAD["cap"], 1),
                      record_selection=ctx is not None)
    x0 = rng.standard_normal(D, dtype=np.float32)
    sess = O.Session.from_state(model, cfg, x0, kv, cols)
    marks = []
    orig = O.layernorm

    def timed_ln(x, g, b, eps):  # LN1 of each layer opens a layer: a free layer clock
        if g is sess.model.layers[len(marks) % Lt].ln1_gain:
            marks.append(time.perf_counter())
        return orig(x, g, b, eps)

    O.layernorm = timed_ln
    per_layer = []
    outs = []
    try:
        for i in range(steps + warmup):
            marks.clear()
            t0 = time.perf_counter()
            outs.append(sess.decode_step())
            t1 = time.perf_counter()
            if i >= warmup and len(marks) == Lt:
                per_layer.append([marks[1] - marks[0], marks[2] - marks[1], t1 - marks[2]])
    finally:
        O.layernorm = orig
    if ctx is not None:
        ctx.update(model=model, x0=x0, kv=kv, cols=cols, prompt=prompt, outs=outs, records=sess.records,
                   steps=steps + warmup)
    t0_, t1_, tl_ = (statistics.median(x) for x in zip(*per_layer))
    t_seq = t0_ + (L_full - 2) * t1_ + tl_
    import threadpoolctl
    threads = sum(p.get("num_threads", 0) for p in threadpoolctl.threadpool_info()
                  if p.get("user_api") == "blas") or os.cpu_count()
    return {"value": 1.0 / t_seq, "unit": UNIT, "cores": int(threads), "kind": "port",
            "sample": (f"oracle port (reference algorithm, NumPy/OpenBLAS) decode_step of a {Lt}-layer "
                       f"{shape} truncation, s={prompt}, 1 sequence, {len(per_layer)} timed steps; "
                       f"T_step = T0 + {L_full - 2}*T1 + T_last = {t_seq:.3f} s/seq, batch {batch} "
                       f"runs serially -> {batch} tok per {batch * t_seq:.2f} s (extrapolated)"),
            "t_layer0_s": t0_, "t_layer_mid_s": t1_, "t_layer_last_s": tl_, "t_seq_s": t_seq,
            "measured": {"what": f"median {Lt}-layer truncation decode_step, 1 sequence (wall clock)",
                         "step_s": t0_ + t1_ + tl_, "timed_steps": len(per_layer)},
            "extrapolated": {"what": f"{L_full} layers x batch {batch} (run() serialises the batch, "
                                     "engine.py:468-476)",
                             "step_s": batch * t_seq}}


def run_reference_arm(a) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cb = cpu_reference(a.shape, a.batch, a.prompt, steps=a.steps, warmup=min(a.warmup, 1))
    line = {"metric": METRIC, "value": cb["value"], "unit": UNIT, "impl": "reference",
            "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": 1000.0 * a.batch / cb["value"], "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": _config(a), "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _config(a) -> dict:
    from paper_2406_19707_b200.model import SHAPES
    sh = SHAPES[a.shape]
    default = (a.shape, a.batch, a.prompt) == (WORKLOAD["shape"], WORKLOAD["batch"], WORKLOAD["prompt"])
    name = WORKLOAD["name"] if default else (f"{a.shape.upper()}-shaped decode, batch {a.batch}, "
                                             f"{a.prompt}-token context (non-default config)")
    return {"workload": name, "model": a.shape, "layers": a.layers or sh["layers"],
            "model_dim": sh["model_dim"], "heads": sh["heads"], "ffn_dim": sh["ffn_dim"],
            "global_batch": a.batch, "context": a.prompt, "partial_ratio": WORKLOAD["ratio"],
            "alpha": WORKLOAD["alpha"], "cap_ratio": WORKLOAD["cap"],
            "outlier_scale": WORKLOAD["outlier_scale"], "kv_pool": "pinned host, f16",
            "fetch": (f"{a.fetch_impl} x {a.fetch_ctas} CTAs x {a.fetch_threads} threads"
                      + (f" x {a.fetch_rows} rows/batch" if a.fetch_impl == "tma" else "")),
            "parallelism": f"tp{a.gpus} (attention heads + FFN columns)" if a.gpus > 1 else "single GPU",
            "dense": {"packed": "ig_sgemm_packed (packed f16 hi/lo weights, 2xf16-split tensor cores, stream-K)",
                      "cublas": "cuBLAS f32 (TF32 off)"}[a.dense],
            "cuda_graph": bool(a.cuda_graph), "resident": bool(a.resident),
            "l2": "inputs larger than L2 (partial K >= 1.6 GB streamed per layer set; host pool 54 GB)"}


def _graph_kernel_us(eng, steps: int) -> dict:
    """Per kernel kind: launches per step and mean device time per launch over
    `steps` CUDA-graph replays (CUPTI kernel records; no events in the graph)."""
    import tempfile

    import torch
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(steps):
            eng.decode_step()
        torch.cuda.synchronize()
    fd, path = tempfile.mkstemp(suffix=".json")
    os.close(fd)
    try:
        prof.export_chrome_trace(path)
        with open(path) as f:
            tr = json.load(f)
    finally:
        os.unlink(path)
    acc = {}
    pats = (("rehearse", "rehearse_count_kernel"), ("attend", "attend512"), ("select", "select_kernel"))
    for e in tr.get("traceEvents", []):
        if e.get("ph") != "X" or e.get("cat") != "kernel":
            continue
        for key, pat in pats:
            if pat in e.get("name", ""):
                c = acc.setdefault(key, [0, 0.0])
                c[0] += 1
                c[1] += float(e.get("dur", 0.0))
    return {k: {"launches_per_step": v[0] / steps, "us_per_launch": v[1] / v[0]}
            for k, v in acc.items() if v[0]}


# --------------------------------------------------------------- B200 arm
def run_b200(a) -> None:
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2406_19707_b200 import _lib
    from paper_2406_19707_b200.engine import DecodeEngine, RunConfig
    from paper_2406_19707_b200.model import SHAPES, ModelSpec, generate_synthetic_gpu, skew_model_gpu
    from paper_2406_19707_b200.speculation import SpeculationConfig

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local = local % torch.cuda.device_count()          # N ranks may share a GPU (gloo tests)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    group = None
    if world > 1:
        if a.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
        group = dist.group.WORLD
    if (world > 1 and a.cuda_graph and a.dist_backend != "nccl"
            and os.environ.get("IG_PEER_AR", "1") == "0"):
        a.cuda_graph = False            # gloo collectives cannot be captured
    sh = dict(SHAPES[a.shape])
    if a.layers:
        sh["layers"] = a.layers
    spec = ModelSpec(**sh, outlier_channels=8, outlier_scale=WORKLOAD["outlier_scale"], seed=0)
    t_setup = time.time()
    model = generate_synthetic_gpu(spec, device=dev)
    skew_model_gpu(model)
    # warmup + timed + e2e + (HBM variant: 2 + timed) decode steps, plus slack
    steps_total = a.warmup + 4 * a.steps + 12
    cfg = RunConfig(scheme="speculative", prompt_len=a.prompt, gen_len=steps_total, batch=a.batch,
                    speculation=SpeculationConfig(WORKLOAD["ratio"], WORKLOAD["alpha"], WORKLOAD["cap"], 1))
    eng = DecodeEngine(model, cfg, pool_dtype="f16", device=dev, group=group, fetch_ctas=a.fetch_ctas,
                       fetch_threads=a.fetch_threads, fetch_priority=a.fetch_priority,
                       fetch_impl=a.fetch_impl, fetch_rows=a.fetch_rows, dense=a.dense,
                       cuda_graph=a.cuda_graph, resident=a.resident, append_stream=a.append_stream,
                       spec_stream=a.spec_stream)
    del model               # the engine holds the only reference until the prefill is done
    torch.cuda.empty_cache()
    g = torch.Generator(device=dev)
    g.manual_seed(1234)
    prompts = torch.empty(a.batch, a.prompt, spec.model_dim, device=dev).normal_(generator=g)
    t_pf = time.time()
    eng.prefill(prompts)
    prefill_s = time.time() - t_pf
    del prompts
    if a.dense == "packed":
        eng.release_model()  # decode reads only the packed weights: one copy in HBM
    torch.cuda.empty_cache()
    footprint = eng.hbm_footprint()
    setup_s = time.time() - t_setup

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    for i in range(a.warmup):
        if i == 0 and a.cuda_graph and world > 1:
            # the first step captures the graph, NCCL all-reduces included (verified
            # on a one-rank NCCL group: tests/test_tp_gpu.py); if the capture fails
            # on this box, time eager steps instead of failing the run
            try:
                eng.decode_step()
            except Exception as e:  # noqa: BLE001
                sys.stderr.write(f"bench: CUDA-graph capture with NCCL failed ({e!r}); "
                                 "timing eager steps\n")
                torch.cuda.synchronize(dev)
                eng._graph, eng.cuda_graph, a.cuda_graph = None, False, False
        else:
            eng.decode_step()
    barrier()
    # -------- device-timed region: K steps, inputs resident in HBM / host pool
    # (no per-kernel events here: they are recorded in a separate pass below)
    launches0 = _lib.launches
    cur = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    prof = os.environ.get("IG_PROFILE_WINDOW") == "1"   # ncu --profile-from-start off
    with ClockSampler(local) as clk:
        barrier()
        if prof:
            torch.cuda.profiler.start()
        e0.record(cur)
        for _ in range(a.steps):
            eng.decode_step()
        e1.record(cur)
        barrier()
        if prof:
            torch.cuda.profiler.stop()
    ms = e0.elapsed_time(e1)
    launches = _lib.launches - launches0
    if a.cuda_graph:   # one eager step's launches are replayed per step
        launches = eng.graph_launches * a.steps
    # -------- per-kernel CUDA events over another K eager steps (not the headline)
    eng.cuda_graph = False
    try:
        eng.instrument(a.steps)
        i0, i1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        i0.record(cur)
        for _ in range(a.steps):
            eng.decode_step()
        i1.record(cur)
        barrier()
        stats = eng.kernel_stats()
        stats["instrumented_ms_per_step"] = i0.elapsed_time(i1) / a.steps
        eng._inst = None
    finally:
        eng.cuda_graph = a.cuda_graph
    iso = eng.isolated_kernel_times(li=eng.L // 2) if eng.L > 2 else {}
    # -------- end-to-end: public API with host input/output rows each step
    x_host = torch.empty((a.batch, spec.model_dim), dtype=torch.float32).pin_memory()
    x_host.copy_(eng.x.cpu())
    barrier()
    t0 = time.perf_counter()
    xh = x_host.numpy()
    for _ in range(a.steps):
        eng.step_host(xh, out=xh)       # rows in from pinned memory, the step's rows back into it
    barrier()
    e2e_ms = (time.perf_counter() - t0) * 1000.0
    # -------- in-graph durations of the non-PDL path kernels (CUPTI via torch.profiler
    # over graph replays: these launch plainly, so start..end is their own time)
    graph_k = None
    if a.cuda_graph and os.environ.get("IG_BENCH_GRAPH_KERNELS", "1") == "1":
        try:
            graph_k = _graph_kernel_us(eng, 3)
        except Exception as e:  # noqa: BLE001
            sys.stderr.write(f"bench: in-graph kernel timing failed ({e!r})\n")
    # -------- secondary variant: resident -> refetch every selected row each
    # step (the reference's data movement, host-link bound); else layer 0 in HBM
    var_ms = 0.0
    var_stats = None
    var_kind = None
    if not a.no_variant and a.resident:
        var_kind = "refetch"
        eng.cuda_graph = False          # the variant is timed eagerly, with its kernel events
        eng.set_resident(False)
        for _ in range(2):
            eng.decode_step()
        eng.instrument(a.steps)
        barrier()
        v0, v1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        v0.record(cur)
        for _ in range(a.steps):
            eng.decode_step()
        v1.record(cur)
        barrier()
        var_ms = v0.elapsed_time(v1)
        var_stats = eng.kernel_stats()
        eng._inst = None
    elif not a.no_variant and not a.resident:
        var_kind = "layer0_in_hbm"
        eng.set_hbm_layers(1)
        for _ in range(2):
            eng.decode_step()
        eng.instrument(a.steps)
        barrier()
        v0, v1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        v0.record(cur)
        for _ in range(a.steps):
            eng.decode_step()
        v1.record(cur)
        barrier()
        var_ms = v0.elapsed_time(v1)
        var_stats = eng.kernel_stats()
        eng._inst = None
        eng.set_hbm_layers(0)
    ms_t = torch.tensor([ms, e2e_ms, var_ms], dtype=torch.float64, device=dev)
    # per rank (N > 1: the scaling curve's evidence): its own step time, the
    # kernels on its GPU, what its fetch stream moved over its host link, and
    # where its host pool lives
    mine = {"rank": rank, "ms_per_step": ms / a.steps, "heads": eng.Hg,
            "host_pool_numa_node": eng.pool.numa_node,
            "kernels_ms_per_step": {k: v["ms"] / a.steps for k, v in stats.items()
                                    if isinstance(v, dict) and v.get("ms")},
            "hbm_footprint_gb": footprint["torch_allocated"] / 1e9}
    fk = [v for k, v in stats.items() if isinstance(v, dict) and k.startswith("fetch") and v.get("ms")]
    if fk:
        fb, fm = sum(v["bytes"] for v in fk), sum(v["ms"] for v in fk)
        mine["fetch_link_gbs"] = fb / (fm * 1e6) if fm else None
        mine["fetch_bytes_per_step"] = fb / a.steps
    per_rank = [mine]
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
        per_rank = [None] * world
        dist.all_gather_object(per_rank, mine)
    ms, e2e_ms, var_ms = float(ms_t[0]), float(ms_t[1]), float(ms_t[2])

    if rank == 0:
        tok = a.batch * a.steps
        value = tok / (ms / 1000.0)
        hbm_peak = _peak("hbm_gbs", 6452.8)
        link_peak = _link_peak(dev)
        tr = _traffic_ratios()
        ms_inst = stats.get("instrumented_ms_per_step", ms / a.steps) * a.steps   # stats' own steps
        link_roof = _link_roofline(stats, link_peak, tr, ms_inst, a)
        f_bytes = link_roof.pop("_bytes")
        # the step's dominant kernel kind (device time inside the timed steps)
        kinds = {k: v["ms"] for k, v in stats.items() if isinstance(v, dict) and v.get("ms")}
        fetch_ms = sum(v for k, v in kinds.items() if k.startswith("fetch"))
        other = {k: v for k, v in kinds.items() if not k.startswith("fetch")}
        top = max(other, key=other.get) if other else None
        if top is not None and other[top] > fetch_ms:
            st = stats[top]
            roof = {"kernel": {"dense": f"dense projections ({_config(a)['dense']})",
                               "rehearse": "ig_rehearse_count", "attend": "ig_attend",
                               "select": "ig_select"}.get(top, top),
                    "bound": "hbm", "achieved": st["gbs"], "peak": hbm_peak,
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy bandwidth)", "unit": "GB/s",
                    "frac": st["gbs"] / hbm_peak if st["gbs"] else None,
                    "traffic": (st["bytes"] / st["launches"] * tr[top]["dram_per_algorithmic"]
                                if tr and top in tr else None),
                    "traffic_source": ("dram bytes per algorithmic byte from the committed ncu capture "
                                       "profiles/r01_traffic.json") if tr and top in tr else None,
                    "bytes_per_launch": st["bytes"] / st["launches"],
                    "ms_per_launch": st["ms"] / st["launches"], "launches": st["launches"],
                    "step_share": st["ms"] / ms_inst if ms_inst else None,
                    "how": "CUDA events around every launch on the compute stream, timed steps"}
        else:
            roof = link_roof
        hbm = {}
        for k in ("rehearse_count", "attend", "select", "dense_ffn_in"):   # alone: own roofline
            if k in iso:
                gbs = iso[k]["gbs"]
                hbm[k] = {"achieved": gbs, "peak": hbm_peak, "unit": "GB/s",
                          "frac": gbs / hbm_peak, "bytes_per_launch": iso[k]["bytes"],
                          "ms_per_launch": iso[k]["ms"],
                          "how": f"alone on the GPU (fetch stream idle), layer {eng.L // 2}, 10 launches back to back per event pair, best of 5"}
                if k == "rehearse_count" and tr and "rehearse_count" in tr:
                    hbm[k]["traffic"] = iso[k]["bytes"] * tr["rehearse_count"]["dram_per_algorithmic"]
        for k in ("rehearse", "attend", "select"):          # in situ, sharing the GPU with the gather
            if k in stats:
                gbs = stats[k]["gbs"]
                hbm[k + "_in_situ"] = {"achieved": gbs, "peak": hbm_peak, "unit": "GB/s",
                                       "frac": gbs / hbm_peak if gbs else None,
                                       "bytes_per_launch": stats[k]["bytes"] / stats[k]["launches"],
                                       "ms_per_launch": stats[k]["ms"] / stats[k]["launches"],
                                       "how": "CUDA events around each launch in eager instrumented steps"}
                if graph_k and k in graph_k and graph_k[k]["us_per_launch"] > 0:
                    bpl = stats[k]["bytes"] / stats[k]["launches"]
                    gg = bpl / graph_k[k]["us_per_launch"] / 1e3
                    hbm[k + "_in_graph"] = {
                        "achieved": gg, "peak": hbm_peak, "unit": "GB/s", "frac": gg / hbm_peak,
                        "bytes_per_launch": bpl, "us_per_launch": graph_k[k]["us_per_launch"],
                        "launches_per_step": graph_k[k]["launches_per_step"],
                        "how": "CUPTI kernel records (torch.profiler) over 3 CUDA-graph replays of the "
                               "step; plain launches, so start..end is the kernel's own time beside "
                               "the other streams"}
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
                "warmup": a.warmup, "ms_per_step": ms / a.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None,
                "dtype": "f32 compute (rehearsal, attention, dense), f16 host KV pool",
                "data": ("synthetic: random-init OPT-13B-shaped weights (reference recipe, torch RNG), "
                         "GPU-SVD skew, N(0,1) prompts, GPU prefill"),
                "config": _config(a), "roofline": roof, "roofline_link": link_roof,
                "roofline_hbm": hbm,
                "kernel_stats": stats, "clocks": clk.summary(),
                "e2e": {"value": tok / (e2e_ms / 1000.0), "unit": UNIT,
                        "h2d_bytes_per_step": a.batch * spec.model_dim * 4,
                        "d2h_bytes_per_step": a.batch * spec.model_dim * 4},
                "gpu_launches": launches, "setup_s": setup_s, "prefill_s": prefill_s,
                "per_rank": per_rank,
                "hbm_footprint_gb": {k: (v / 1e9 if isinstance(v, int) else v)
                                     for k, v in footprint.items()},
                "link_bytes_per_step": {"reference_accounted": _ref_bytes(stats, eng, a.steps),
                                        "moved": f_bytes / a.steps}}
        if var_stats is not None and var_kind == "refetch":
            vroof = _link_roofline(var_stats, link_peak, tr, var_ms, a)
            line["variant_refetch"] = {
                "value": tok / (var_ms / 1000.0), "unit": UNIT, "ms_per_step": var_ms / a.steps,
                "note": "same engine and state with resident selection off: every selected row "
                        "(and all of layer 0) fetched from the host pool every step -- the "
                        "reference's data movement, host-link bound",
                "link_bytes_per_step_moved": vroof.pop("_bytes") / a.steps,
                "roofline": vroof, "kernel_stats": var_stats}
        elif var_stats is not None:
            vk = [k for k in ("fetch_gather", "fetch_all_ce") if k in var_stats]
            line["variant_layer0_in_hbm"] = {
                "value": tok / (var_ms / 1000.0), "unit": UNIT, "ms_per_step": var_ms / a.steps,
                "note": "same workload; layer 0's KV (1.3 GB, read in full every step) resident in HBM, "
                        "layers 1-39 on the host pool",
                "link_bytes_per_step_moved": sum(var_stats[k]["bytes"] for k in vk) / a.steps,
                "kernel_stats": var_stats}
        if not a.no_cpu_baseline and world == 1:
            ctx: dict = {}
            try:
                line["cpu_baseline"] = cpu_reference(a.shape, a.batch, a.prompt,
                                                     a.cpu_sample_steps or a.steps, ctx=ctx)
            except Exception as e:  # reported, never fatal to the GPU number
                line["cpu_baseline"] = {"error": repr(e)}
            if ctx:
                try:
                    line["cpu_baseline"]["parity"] = _bench_parity(ctx, a, dev)
                except Exception as e:  # noqa: BLE001
                    line["cpu_baseline"]["parity"] = {"error": repr(e)}
        print(json.dumps(line), flush=True)
    eng.close()
    if world > 1:
        dist.destroy_process_group()


def _bench_parity(ctx: dict, a, dev) -> dict:
    """The B200 engine, with this run's settings (f16 host pool, resident
    selection, CUDA graph, packed GEMMs, spec stream), decoding the very
    truncation the CPU baseline just timed (same weights, injected state,
    steps): per (step, layer >= 1, head) index sets and n vs the oracle's,
    and the outputs' scaled error."""
    import numpy as np
    import torch
    from paper_2406_19707_b200.engine import DecodeEngine, RunConfig
    from paper_2406_19707_b200.speculation import SpeculationConfig
    model, steps, kv, cols = ctx["model"], ctx["steps"], ctx["kv"], ctx["cols"]
    cfg = RunConfig(scheme="speculative", prompt_len=ctx["prompt"], gen_len=steps, batch=1,
                    speculation=SpeculationConfig(WORKLOAD["ratio"], WORKLOAD["alpha"], WORKLOAD["cap"], 1))
    eng = DecodeEngine(model, cfg, pool_dtype="f16", device=dev, dense=a.dense, cuda_graph=a.cuda_graph,
                       resident=a.resident, append_stream=a.append_stream, spec_stream=a.spec_stream)
    try:
        eng.load_state(ctx["x0"][None], lambda li, b, h: kv[li][h], lambda li, b, h: cols[li][h])
        L, H = model.spec.layers, model.spec.heads
        rows = flipped = sets = set_flips = n_exact = n_cmp = 0
        first = None
        err = 0.0
        for it in range(steps):
            out = eng.decode_step().cpu().numpy()[0]
            torch.cuda.synchronize(dev)
            ref = np.asarray(ctx["outs"][it], np.float64)
            err = max(err, float(np.abs(out - ref).max() / max(1.0, np.abs(ref).max())))
            n_dev, idx = eng.n.cpu().numpy(), eng.idx.cpu().numpy()
            for li in range(1, L):
                rr = ctx["records"][it][li]
                gn = int(n_dev[li, 0])
                n_cmp += 1
                n_exact += int(gn == int(rr["n_selected"]))
                for h in range(H):
                    g = set(int(i) for i in idx[li, 0, h, :gn])
                    r = set(int(i) for i in rr["selected"][h])
                    sets += 1
                    rows += len(r)
                    if g != r:
                        set_flips += 1
                        flipped += max(len(g - r), len(r - g))
            if it == 0:
                first = {"set_flips": set_flips, "rows_flipped": flipped, "out_scaled_err": err}
    finally:
        eng.close()
    return {"what": "B200 engine (this run's settings) vs the oracle on the timed truncation: "
                    f"{steps} steps x {L - 1} selecting layers x {H} heads, 1 sequence",
            "selections": sets, "set_flips": set_flips, "rows": rows, "rows_flipped": flipped,
            "set_agreement": 1.0 - flipped / max(rows, 1), "n_exact": n_exact, "n_compared": n_cmp,
            "out_scaled_err": err, "first_step": first,
            "note": "free-running: from the first step on, the trajectories carry the f32-level "
                    "differences, so later steps compare slightly different inputs; n sits at the "
                    "20% cap here, inside the dense middle of the score distribution "
                    "(tests/test_parity_shapes_gpu.py holds the per-flip explanation)"}


def _link_roofline(stats, link_peak, tr, ms, a) -> dict:
    """Host-link roofline of the fetch stream (gather + copy-engine rows)."""
    keys = [k for k in ("fetch_gather", "fetch_slots", "fetch_all_ce") if k in stats]
    f_bytes = sum(stats[k]["bytes"] for k in keys)
    f_ms = sum(stats[k]["ms"] for k in keys)
    f_launch = sum(stats[k]["launches"] for k in keys)
    gbs = f_bytes / (f_ms * 1e6) if f_ms else None
    per_launch = f_bytes / max(f_launch, 1)
    fr = tr.get("fetch") if tr else None
    return {"kernel": ("fetch (" + " + ".join(keys) + ")") if keys else "fetch",
            "bound": "host_link", "achieved": gbs, "peak": link_peak["gbs"],
            "peak_source": link_peak["source"], "unit": "GB/s",
            "frac": (gbs / link_peak["gbs"]) if gbs else None,
            "traffic": per_launch * fr["sysmem_per_payload"] if fr else None,
            "traffic_pcie": per_launch * fr["pcie_per_payload"] if fr else None,
            "traffic_source": ("host-memory bytes read (and raw PCIe bytes) per algorithmic byte from "
                               "the committed ncu capture profiles/r01_traffic.json, scaled to this "
                               "run's average launch") if fr else None,
            "bytes_per_launch": per_launch, "launches": f_launch,
            "step_share": f_ms / ms if ms else None, "_bytes": f_bytes}


def _traffic_ratios():
    """Per-algorithmic-byte traffic measured by ncu (committed with the repo)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r01_traffic.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return None


def _graph_stats(eng, steps) -> dict:
    """Graph replays carry no per-kernel events: report the step's moved bytes."""
    s = eng.s_host
    return {"n_mean_per_layer": [float(x) for x in eng.n.float().mean(dim=1).cpu()],
            "note": "cuda_graph: per-kernel timings unavailable (replayed graph)",
            "fetch_gather": {"launches": steps * (eng.L - 1), "ms": 0.0,
                             "bytes": int(eng.n[1:].sum()) * eng.Hg * eng.row_bytes * steps, "gbs": None},
            "fetch_all_ce": {"launches": steps, "ms": 0.0,
                             "bytes": eng.B * eng.Hg * s * eng.row_bytes * steps, "gbs": None}}


def _ref_bytes(stats, eng, steps) -> float:
    """The reference's LayerRecord.bytes summed over a step (engine.py:429):
    layer 0 = all s rows, layers >= 1 = n rows, per head, 2*d*e bytes."""
    n = stats["n_mean_per_layer"]
    s = eng.s_host
    per_row = eng.Hg * eng.row_bytes   # this rank's heads, pool element bytes
    return float(eng.B * per_row * (s + sum(n[1:])))


def _peak(key, fallback):
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)[key])
    except (OSError, KeyError, ValueError):
        return fallback


def _link_peak(dev) -> dict:
    """Host link peak measured live: copy-engine H2D of 1 GiB pinned (best of 5)."""
    import torch
    n = 1 << 30
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    best = 0.0
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        d.copy_(h, non_blocking=True)
        e1.record()
        e1.synchronize()
        best = max(best, n / (e0.elapsed_time(e1) * 1e6))
    return {"gbs": best, "source": "measured live: copy-engine H2D, 1 GiB pinned, best of 5"}


def main():
    a = _args()
    if a.impl == "reference":
        run_reference_arm(a)
    else:
        run_b200(a)


if __name__ == "__main__":
    main()
