"""speckv-compatible command line for the B200 path.

Mirrors the reference's `run` and `bench` verbs (cli.py:168-208, argument
surface cli.py:83-105, error convention cli.py:28-33: ValueError / OSError /
KeyError -> exit 2 and one JSON line on stderr), so a user's scripts keep
working:

    python -m paper_2406_19707_b200 run   --model m.json --scheme speculative -o trace.json
    python -m paper_2406_19707_b200 bench --model m.json --schemes full,speculative -o cmp.json

`run` writes the schema-v1 trace (engine.py:83-196) of the B200 engine and
prints {"written", "scheme", "total_bytes"} like the reference.  `bench`
writes, per scheme, total_bytes, mean_selected_fraction, native_style and
final_output_norm like the reference, plus the MEASURED decode time on the
GPU ("measured_decode_s") in place of the reference's cost-model simulation
("simulated_total_s", costmodel.py -- out of scope here).
Only the schemes on the B200 path exist (speculative, full); the others
(h2o, int4, oracle) raise ValueError -> exit 2, as an unknown scheme does in
the reference.  gen-model / skew / report stay with the reference (offline
tooling; model files it writes load here, model.load_model).
"""

from __future__ import annotations

import argparse
import json
import sys
import time

import numpy as np

POLICIES = ("fifo", "lru", "counter")
SCHEMES = ("full", "speculative")


def main(argv: list[str] | None = None) -> int:
    parser = _build_parser()
    args = parser.parse_args(argv)
    try:
        return args.func(args)
    except (ValueError, OSError, KeyError) as e:
        print(json.dumps({"error": type(e).__name__, "message": str(e)}), file=sys.stderr)
        return 2


def _build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="speckv-b200")
    sub = parser.add_subparsers(required=True)
    p = sub.add_parser("run", help="run one scheme on the B200 path and write a trace")
    _add_run_args(p)
    p.add_argument("-o", "--output", required=True, help="trace JSON path")
    p.set_defaults(func=_cmd_run)
    p = sub.add_parser("bench", help="run several schemes and compare (measured on the GPU)")
    _add_run_args(p, scheme_list=True)
    p.add_argument("-o", "--output", required=True, help="comparison JSON path")
    p.set_defaults(func=_cmd_bench)
    return parser


def _add_run_args(p: argparse.ArgumentParser, scheme_list: bool = False) -> None:
    p.add_argument("--model", required=True)
    if scheme_list:
        p.add_argument("--schemes", default="full,speculative", help="comma-separated scheme list")
    else:
        p.add_argument("--scheme", default="full")
    p.add_argument("--prompt-len", type=int, default=64)
    p.add_argument("--gen-len", type=int, default=16)
    p.add_argument("--batch", type=int, default=1)
    p.add_argument("--alpha", type=float, default=4.0)
    p.add_argument("--partial-ratio", type=float, default=0.3)
    p.add_argument("--cap-ratio", type=float, default=0.2)
    p.add_argument("--min-select", type=int, default=1)
    p.add_argument("--pool-limit", default=None, help="max pool rows, or a fraction of prompt+gen length")
    p.add_argument("--policy", default="counter", choices=POLICIES)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--record-scores", action="store_true")
    p.add_argument("--record-selection", action="store_true")
    p.add_argument("--pool-dtype", default="f16", choices=("f16", "bf16", "f32"),
                   help="host KV pool element (B200 path; the reference accounts 2 bytes)")


def _parse_pool_limit(raw, total_rows: int) -> int | None:
    """cli.py:108-116: a row count, or a fraction of prompt + gen length."""
    if raw is None:
        return None
    value = float(raw)
    if 0 < value < 1:
        return max(1, int(value * total_rows))
    if value != int(value) or value < 1:
        raise ValueError(f"pool limit must be a row count or fraction, got {raw}")
    return int(value)


def _scheme(name: str) -> str:
    if name not in SCHEMES:
        raise ValueError(f"scheme {name!r} is not on the B200 path (speculative, full)")
    return name


def _run_config(args, scheme: str):
    from .engine import RunConfig
    from .speculation import SpeculationConfig
    total = args.prompt_len + args.gen_len
    return RunConfig(scheme=scheme, prompt_len=args.prompt_len, gen_len=args.gen_len,
                     batch=args.batch,
                     speculation=SpeculationConfig(partial_ratio=args.partial_ratio, alpha=args.alpha,
                                                   cap_ratio=args.cap_ratio, min_select=args.min_select),
                     pool_limit=_parse_pool_limit(args.pool_limit, total), pool_policy=args.policy,
                     prompt_seed=args.seed, record_scores=args.record_scores,
                     record_selection=args.record_selection)


def total_bytes(trace: dict) -> int:
    """Trace.total_bytes (engine.py:174-175)."""
    return sum(r["bytes"] for s in trace["sequences"] for it in s["iterations"] for r in it)


def mean_selected_fraction(trace: dict) -> float:
    """cli.py:219-223: mean over records of bytes / full_bytes (full_bytes > 0)."""
    fr = [r["bytes"] / r["full_bytes"] for s in trace["sequences"] for it in s["iterations"] for r in it
          if r["full_bytes"] > 0]
    return float(np.mean(fr)) if fr else 0.0


def _cmd_run(args) -> int:
    from .engine import run
    from .model import load_model
    model = load_model(args.model)
    config = _run_config(args, _scheme(args.scheme))
    trace, _ = run(model, config, pool_dtype=args.pool_dtype)
    with open(args.output, "w", encoding="utf-8") as f:
        json.dump(trace, f)
    print(json.dumps({"written": args.output, "scheme": args.scheme, "total_bytes": total_bytes(trace)}))
    return 0


def _cmd_bench(args) -> int:
    import torch
    from .engine import run
    from .model import load_model
    model = load_model(args.model)
    schemes = [_scheme(s.strip()) for s in args.schemes.split(",") if s.strip()]
    comparison = {}
    for scheme in schemes:
        config = _run_config(args, scheme)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        trace, finals = run(model, config, pool_dtype=args.pool_dtype)
        torch.cuda.synchronize()
        comparison[scheme] = {
            "total_bytes": total_bytes(trace),
            "mean_selected_fraction": mean_selected_fraction(trace),
            "native_style": "selective_prefetch" if scheme == "speculative" else "prefetch_all",
            "measured_decode_s": time.perf_counter() - t0,
            "final_output_norm": [float(np.linalg.norm(f)) for f in finals],
        }
    with open(args.output, "w", encoding="utf-8") as f:
        json.dump(comparison, f, indent=1)
    print(json.dumps({"written": args.output, "schemes": schemes}))
    return 0


if __name__ == "__main__":
    sys.exit(main())
