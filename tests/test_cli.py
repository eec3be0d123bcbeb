"""The speckv-compatible CLI (paper_2406_19707_b200/cli.py) vs the reference's
verbs (cli.py:168-208) and error convention (cli.py:28-33)."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TINY = os.path.join(ROOT, "tests", "golden", "tiny_skewed.json")


def _cli(*args):
    return subprocess.run([sys.executable, "-m", "paper_2406_19707_b200", *args], cwd=ROOT,
                          capture_output=True, text=True, timeout=600)


@pytest.mark.parametrize("args,err", [
    (["run", "--model", TINY, "--scheme", "h2o", "-o", "/tmp/x.json"], "ValueError"),
    (["run", "--model", TINY, "--pool-limit", "2.5", "-o", "/tmp/x.json"], "ValueError"),
    (["run", "--model", "/nonexistent/m.json", "-o", "/tmp/x.json"], None),
    (["bench", "--model", TINY, "--schemes", "full,int4", "-o", "/tmp/x.json"], "ValueError"),
])
def test_cli_errors_exit_2_with_json(args, err):
    r = _cli(*args)
    assert r.returncode == 2, r.stderr
    line = json.loads(r.stderr.strip().splitlines()[-1])
    assert set(line) == {"error", "message"}
    if err:
        assert line["error"] == err
    else:
        assert line["error"] in ("FileNotFoundError", "OSError")


def test_cli_pool_limit_parsing_matches_reference():
    from paper_2406_19707_b200.cli import _parse_pool_limit
    assert _parse_pool_limit(None, 100) is None
    assert _parse_pool_limit("0.8", 100) == 80
    assert _parse_pool_limit("0.001", 100) == 1
    assert _parse_pool_limit("42", 100) == 42
    with pytest.raises(ValueError):
        _parse_pool_limit("0", 100)


@pytest.mark.gpu
def test_cli_run_trace_equals_oracle(tmp_path):
    """`run` on a model file the real reference wrote: the trace equals the
    oracle run()'s (selected lists as sets), total_bytes as the reference prints."""
    from oracle import speckv_port as O
    from paper_2406_19707_b200.model import load_model
    out = tmp_path / "trace.json"
    r = _cli("run", "--model", TINY, "--scheme", "speculative", "--prompt-len", "40", "--gen-len", "5",
             "--batch", "2", "--pool-limit", "42", "--record-selection", "--pool-dtype", "f32",
             "-o", str(out))
    assert r.returncode == 0, r.stderr
    msg = json.loads(r.stdout.strip().splitlines()[-1])
    trace = json.load(open(out))
    m = load_model(TINY)
    oracle_model = O.Model(O.ModelSpec(2, 32, 2, 64), [O.Layer(*[np.asarray(getattr(lw, f)) for f in
                           ("w_q", "w_k", "w_v", "w_o", "ffn_in", "ffn_out", "ln1_gain", "ln1_bias",
                            "ln2_gain", "ln2_bias")]) for lw in m.layers], np.zeros(0, np.int64), True)
    ocfg = O.RunConfig(scheme="speculative", prompt_len=40, gen_len=5, batch=2, record_selection=True,
                       pool_limit=42, pool_policy=O.Policy.COUNTER)
    ref_trace, _ = O.run(oracle_model, ocfg)
    ref_total = sum(rr["bytes"] for s in ref_trace["sequences"] for it in s["iterations"] for rr in it)
    assert msg == {"written": str(out), "scheme": "speculative", "total_bytes": ref_total}
    for sm, sr in zip(trace["sequences"], ref_trace["sequences"]):
        assert sm["prefill"] == sr["prefill"]
        for im, ir in zip(sm["iterations"], sr["iterations"]):
            for rm, rr in zip(im, ir):
                assert rm["n_selected"] == rr["n_selected"] and rm["bytes"] == rr["bytes"]
                assert [sorted(x) for x in rm["selected"]] == [sorted(x) for x in rr["selected"]]
    b = tmp_path / "cmp.json"
    r = _cli("bench", "--model", TINY, "--prompt-len", "40", "--gen-len", "3", "-o", str(b))
    assert r.returncode == 0, r.stderr
    cmp = json.load(open(b))
    assert set(cmp) == {"full", "speculative"}
    assert cmp["speculative"]["total_bytes"] <= cmp["full"]["total_bytes"]
    assert cmp["full"]["mean_selected_fraction"] == pytest.approx(1.0)
