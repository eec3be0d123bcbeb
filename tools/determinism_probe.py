"""Run-to-run determinism of the engine at a shape-parity case: the same engine
(same weights, state, settings) built and decoded several times in one process;
per step, the max |difference| of the outputs against the first run.  Bisects
the engine features (CUDA graph, resident selection, speculation stream, pool
dtype) that make two identical runs differ.

    python tools/determinism_probe.py [--case c2] [--steps 4] [--runs 3]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    from tests.shape_parity import Case
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="c2")
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--runs", type=int, default=3)
    ap.add_argument("--configs", default="all")
    ap.add_argument("--save", default=None, help="save the first run's outputs (.npy) for cross-process checks")
    a = ap.parse_args()
    case = Case(a.case)
    configs = [
        dict(pool_dtype="f16", cuda_graph=True),
        dict(pool_dtype="f16", cuda_graph=False),
        dict(pool_dtype="f16", cuda_graph=True, resident=False),
        dict(pool_dtype="f16", cuda_graph=True, spec_stream=False),
        dict(pool_dtype="f32", cuda_graph=True),
        dict(pool_dtype="f32", cuda_graph=False),
    ]
    if a.configs != "all":
        configs = [configs[int(i)] for i in a.configs.split(",")]
    for kw in configs:
        outs = []
        for _ in range(a.runs):
            eng = case.engine(a.steps, **kw)
            try:
                o = []
                for _ in range(a.steps):
                    o.append(eng.decode_step().cpu().numpy().copy())
                    torch.cuda.synchronize()
                outs.append((np.stack(o), eng.n.cpu().numpy().copy(), eng.idx.cpu().numpy().copy()))
            finally:
                eng.close()
                del eng
                torch.cuda.empty_cache()
        ref = outs[0]
        if a.save:
            np.save(a.save, ref[0])
        per_run = []
        for o in outs[1:]:
            per_run.append({"step_max_abs_diff": [float(np.abs(o[0][i] - ref[0][i]).max())
                                                  for i in range(a.steps)],
                            "n_equal": bool(np.array_equal(o[1], ref[1])),
                            "idx_equal_last": bool(np.array_equal(o[2], ref[2]))})
        print(json.dumps({"config": kw, "runs": per_run}), flush=True)


if __name__ == "__main__":
    main()
