"""Find engine buffers read before they are written: build the C2 shape-parity
engine (tests/shape_parity.py, bench defaults: f16 pool, resident, CUDA graph),
fill ONE device buffer with NaN after load_state, decode a few steps and compare
with an unpoisoned run.  A buffer whose poison reaches the outputs is read
before the step writes it.

    python tools/poison_probe.py [--case c2] [--steps 4]
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
    a = ap.parse_args()
    case = Case(a.case)

    def run(poison=None):
        eng = case.engine(a.steps, pool_dtype="f16", cuda_graph=True)
        try:
            if poison is not None:
                obj = getattr(eng, poison)
                ts = obj if isinstance(obj, (list, tuple)) else [obj]
                for t in ts:
                    if t is None:
                        continue
                    if t.dtype.is_floating_point:
                        t.fill_(float("nan"))
                    else:
                        t.fill_(-7 if t.dtype != torch.uint8 else 0xAB)
            torch.cuda.synchronize()
            outs = [eng.decode_step().cpu().numpy().copy() for _ in range(a.steps)]
            return np.stack(outs)
        finally:
            eng.close()
            del eng
            torch.cuda.empty_cache()

    base = run()
    again = run()
    print(json.dumps({"buffer": "(none, repeat)", "max_abs_diff": float(np.abs(base - again).max())}),
          flush=True)
    names = ["x_a", "x_f", "qkvq_buf", "attn", "o", "hidden", "scores", "stage_full", "att_partial",
             "att_tickets", "gemm_ws", "gemm_tickets", "stage_res", "slot_id", "slot_used", "frow",
             "fslot", "fcount", "maxkey", "rtickets", "counts", "count_sum", "row_range", "idx", "n",
             "pos", "xbuf"]
    for nm in names:
        eng_has = True
        try:
            got = run(nm)
        except AttributeError:
            eng_has = False
        except Exception as e:  # noqa: BLE001
            print(json.dumps({"buffer": nm, "error": repr(e)[:200]}), flush=True)
            continue
        if not eng_has:
            print(json.dumps({"buffer": nm, "missing": True}), flush=True)
            continue
        d = np.abs(got - base)
        print(json.dumps({"buffer": nm, "nan": bool(np.isnan(got).any()),
                          "max_abs_diff": float(np.nanmax(d)) if np.isfinite(d).any() else None}),
              flush=True)


if __name__ == "__main__":
    main()
