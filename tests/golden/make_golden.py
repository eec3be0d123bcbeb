"""Generate golden fixtures from the REAL reference (run in the build container).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/*.npz / *.json.  These pin oracle/speckv_port.py to the
reference (tests/test_oracle_golden.py) and give the GPU tests known answers
that do not need /root/reference at run time.  The CPU model, NumPy and
OpenBLAS versions are recorded in meta.json.
"""

import json
import os
import platform
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from speckv import engine, linalg, model, pool, skewing, speculation  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
F32 = np.float32


def small_models():
    """(name, ModelSpec) pairs used by the fixtures."""
    return [
        ("m64", model.ModelSpec(layers=3, model_dim=64, heads=4, ffn_dim=256,
                                outlier_channels=8, outlier_scale=2.0, seed=0)),
        ("m256", model.ModelSpec(layers=3, model_dim=256, heads=2, ffn_dim=1024,
                                 outlier_channels=8, outlier_scale=2.0, seed=3)),
    ]


def run_cfgs():
    S = speculation.SpeculationConfig
    P = pool.EvictionPolicy
    return [
        ("spec", dict(scheme=engine.Scheme.SPECULATIVE, prompt_len=48, gen_len=6, batch=2)),
        ("spec_counter", dict(scheme=engine.Scheme.SPECULATIVE, prompt_len=40, gen_len=12,
                              batch=1, pool_limit=int(0.8 * 52), pool_policy=P.COUNTER)),
        ("spec_lru", dict(scheme=engine.Scheme.SPECULATIVE, prompt_len=40, gen_len=12,
                          batch=1, pool_limit=36, pool_policy=P.LRU)),
        ("spec_fifo", dict(scheme=engine.Scheme.SPECULATIVE, prompt_len=40, gen_len=12,
                           batch=1, pool_limit=36, pool_policy=P.FIFO)),
        ("spec_alpha2_cap05", dict(scheme=engine.Scheme.SPECULATIVE, prompt_len=64, gen_len=5,
                                   batch=1, speculation=S(0.3, 2.0, 0.5, 1))),
        ("spec_identity", dict(scheme=engine.Scheme.SPECULATIVE, prompt_len=32, gen_len=4,
                               batch=1, speculation=S(0.3, 1e9, 1.0, 1))),
        ("full", dict(scheme=engine.Scheme.FULL, prompt_len=32, gen_len=4, batch=1)),
    ]


def main():
    arrays = {}
    digests = {}
    traces = {}
    for mname, spec in small_models():
        plain = model.generate_synthetic(spec)
        sk, skews = skewing.skew_model(plain, calib_seed=0)
        for li, lw in enumerate(plain.layers):
            for f in ("w_q", "w_k", "w_v", "w_o", "ffn_in", "ffn_out",
                      "ln1_gain", "ln1_bias", "ln2_gain", "ln2_bias"):
                digests[f"{mname}.plain.{li}.{f}"] = _sha(getattr(lw, f))
            digests[f"{mname}.skewed.{li}.w_q"] = _sha(sk.layers[li].w_q)
            digests[f"{mname}.skewed.{li}.w_k"] = _sha(sk.layers[li].w_k)
            # skew blocks are small: keep the values for a tolerance fallback
            arrays[f"{mname}.skew.{li}"] = np.stack(skews.matrices[li])
        arrays[f"{mname}.outliers"] = plain.outlier_indices
        for rname, kw in run_cfgs():
            cfg = engine.RunConfig(record_selection=True, record_scores=(mname == "m64"), **kw)
            use = sk if cfg.scheme is engine.Scheme.SPECULATIVE else plain
            # per-step outputs as well as finals
            steps = []
            for b in range(cfg.batch):
                prompt = model.random_prompt(cfg.prompt_len, spec.model_dim, cfg.prompt_seed + b)
                sess = engine.DecodeSession(use, cfg, prompt)
                rows = [sess.x[0].copy()]
                for _ in range(cfg.gen_len):
                    rows.append(sess.decode_step())
                steps.append(np.stack(rows))
            arrays[f"{mname}.{rname}.outputs"] = np.stack(steps)
            trace, finals = engine.run(use, cfg)
            traces[f"{mname}.{rname}"] = trace.to_json()
            assert np.array_equal(np.stack(finals), np.stack(steps)[:, -1])

    # operator-level known answers
    rng = np.random.default_rng(123)
    sel_cases = []
    S = speculation.SpeculationConfig
    for case in range(40):
        H = int(rng.integers(1, 6))
        s = int(rng.integers(1, 300))
        alpha = float(rng.choice([0.5, 1.0, 4.0, 5.0, 1e9]))
        cap = float(rng.choice([0.05, 0.2, 0.5, 1.0]))
        mins = int(rng.choice([1, 2, 7]))
        quant = rng.choice([0.0, 0.25, 1.0])  # 0.0 -> continuous, else ties
        sc = rng.standard_normal((H, s)).astype(F32) * F32(3.0)
        if quant:
            sc = (np.round(sc / quant) * quant).astype(F32)
        cfg = S(0.3, alpha, cap, mins)
        picks, n = speculation.select_tokens([sc[h] for h in range(H)], cfg)
        arrays[f"sel.{case}.scores"] = sc
        arrays[f"sel.{case}.picks"] = np.stack(picks) if n else np.zeros((H, 0), np.int64)
        sel_cases.append({"case": case, "alpha": alpha, "cap_ratio": cap,
                          "min_select": mins, "n": int(n)})

    for case in range(12):
        m = int(rng.integers(1, 70))
        d = int(rng.choice([8, 64, 128]))
        q = rng.standard_normal((1, d)).astype(F32)
        k = rng.standard_normal((m, d)).astype(F32) * F32(2.0)
        v = rng.standard_normal((m, d)).astype(F32)
        o, w = model.attention_head(q, k, v)
        arrays.update({f"attn.{case}.q": q, f"attn.{case}.k": k, f"attn.{case}.v": v,
                       f"attn.{case}.out": o, f"attn.{case}.w": w})

    for case in range(12):
        n = int(rng.integers(2, 60))
        d = int(rng.choice([10, 64, 128]))
        qt = rng.standard_normal((n, d)).astype(F32)
        kt = rng.standard_normal((n, d)).astype(F32)
        ratio = float(rng.choice([0.1, 0.3, 0.5, 1.0]))
        arrays.update({f"bp.{case}.qt": qt, f"bp.{case}.kt": kt,
                       f"bp.{case}.cols": speculation.build_partial(qt, kt, ratio)})
        sel_cases.append({"bp_case": case, "ratio": ratio})

    # KvPool random op sequences (append / fetch / evict, all policies)
    pool_log = []
    for case, pol in enumerate(["fifo", "lru", "counter", "counter"]):
        d = 4
        limit = 9
        pl = pool.KvPool(d, limit=limit, policy=pool.EvictionPolicy(pol))
        ops = []
        for step in range(600 if case == 3 else 200):
            if len(pl) == 0 or rng.random() < 0.3:
                k = rng.standard_normal(d).astype(F32)
                pos = pl.append(k, -k)
                ops.append(["a", [float(x) for x in k], int(pos)])
            else:
                cnt = int(rng.integers(1, len(pl) + 1))
                idx = rng.choice(len(pl), size=cnt, replace=False)
                if case == 3:  # hammer a few rows so counters saturate and halve
                    idx = np.unique(np.concatenate([idx, [0, 1]])[: len(pl)])
                    idx = idx[idx < len(pl)]
                K, V = pl.fetch(idx)
                ops.append(["f", [int(i) for i in idx], float(K.sum())])
        pool_log.append({"policy": pol, "limit": limit, "ops": ops,
                         "final": {"keys": pl.keys.tolist(),
                                   "arrival_seq": pl.arrival_seq.tolist(),
                                   "last_fetch_seq": pl.last_fetch_seq.tolist(),
                                   "fetch_counter": pl.fetch_counter.tolist()}})

    np.savez_compressed(os.path.join(OUT, "golden_small.npz"), **arrays)
    with open(os.path.join(OUT, "golden_traces.json"), "w") as f:
        json.dump(traces, f)
    with open(os.path.join(OUT, "golden_ops.json"), "w") as f:
        json.dump({"select": sel_cases, "pool": pool_log, "digests": digests}, f)
    import threadpoolctl
    meta = {"numpy": np.__version__, "python": platform.python_version(),
            "machine": platform.machine(), "processor": platform.processor(),
            "cpu_model": _cpu_model(), "blas": threadpoolctl.threadpool_info(),
            "reference": REF}
    with open(os.path.join(OUT, "meta.json"), "w") as f:
        json.dump(meta, f, indent=1, default=str)
    print("wrote", sorted(os.listdir(OUT)))


def _sha(a):
    import hashlib
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.dtype.str.encode() + str(a.shape).encode() + a.tobytes()).hexdigest()


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


if __name__ == "__main__":
    main()
