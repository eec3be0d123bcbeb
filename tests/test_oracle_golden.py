"""Pin oracle/speckv_port.py to the reference via the golden fixtures (CPU).

The fixtures were produced by the REAL reference (tests/golden/make_golden.py).
Weights are compared by SHA-256 (bit-exact), traces/indices exactly, floats
with tolerances that only matter if OpenBLAS picks different kernels on
another CPU.
"""

import hashlib

import numpy as np
import pytest

from oracle import speckv_port as O
from tests.golden_cfg import MODELS, RUNS, models, run_config


def _sha(a):
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.dtype.str.encode() + str(a.shape).encode() + a.tobytes()).hexdigest()


@pytest.mark.parametrize("mname", sorted(MODELS))
def test_generate_synthetic_bit_exact(golden, mname):
    plain, _ = models(mname)
    dig = golden["ops"]["digests"]
    for li, lw in enumerate(plain.layers):
        for f in ("w_q", "w_k", "w_v", "w_o", "ffn_in", "ffn_out",
                  "ln1_gain", "ln1_bias", "ln2_gain", "ln2_bias"):
            assert _sha(getattr(lw, f)) == dig[f"{mname}.plain.{li}.{f}"], (li, f)
    np.testing.assert_array_equal(plain.outlier_indices, golden["arrays"][f"{mname}.outliers"])


@pytest.mark.parametrize("mname", sorted(MODELS))
def test_skew_matches_reference(golden, mname):
    _, sk = models(mname)
    dig = golden["ops"]["digests"]
    for li in range(sk.spec.layers):
        ref = golden["arrays"][f"{mname}.skew.{li}"]
        np.testing.assert_allclose(np.stack(sk.skew_matrices[li]), ref, rtol=0, atol=1e-5)
        same = (_sha(sk.layers[li].w_q) == dig[f"{mname}.skewed.{li}.w_q"] and
                _sha(sk.layers[li].w_k) == dig[f"{mname}.skewed.{li}.w_k"])
        if not same:  # a different CPU/BLAS may round differently: fall back to geometry
            a = np.stack(sk.skew_matrices[li]).astype(np.float64)
            eye = np.einsum("hij,hik->hjk", a, a)
            assert np.abs(eye - np.eye(a.shape[1])).max() < 1e-4


def _trace_equal(mine, ref, ftol=1e-4):
    assert mine["version"] == ref["version"] == 1
    assert mine["scheme"] == ref["scheme"]
    assert len(mine["sequences"]) == len(ref["sequences"])
    for sm, sr in zip(mine["sequences"], ref["sequences"]):
        assert sm["prefill"] == sr["prefill"]
        assert len(sm["iterations"]) == len(sr["iterations"])
        for itm, itr in zip(sm["iterations"], sr["iterations"]):
            for rm, rr in zip(itm, itr):
                for key in ("iteration", "layer", "n_selected", "bytes", "full_bytes",
                            "pool_events", "selected"):
                    assert rm[key] == rr[key], (key, rm["iteration"], rm["layer"])
                for key in ("attention_flops", "ffn_flops", "speculation_flops"):
                    assert rm[key] == pytest.approx(rr[key])
                for key in ("spec_scores", "true_scores"):
                    if key in rr:
                        np.testing.assert_allclose(np.array(rm[key]), np.array(rr[key]),
                                                   rtol=ftol, atol=ftol)


@pytest.mark.parametrize("rname", sorted(RUNS))
@pytest.mark.parametrize("mname", sorted(MODELS))
def test_run_matches_reference_trace(golden, mname, rname):
    plain, sk = models(mname)
    cfg = run_config(rname, record_selection=True, record_scores=(mname == "m64"))
    use = sk if cfg.scheme == "speculative" else plain
    trace, finals = O.run(use, cfg)
    ref = golden["traces"][f"{mname}.{rname}"]
    _trace_equal(trace, ref)
    outs = golden["arrays"][f"{mname}.{rname}.outputs"]
    for b in range(cfg.batch):
        np.testing.assert_allclose(finals[b], outs[b, -1], rtol=1e-5, atol=1e-4)


def test_select_tokens_known_answers():
    cfg1 = O.SpeculationConfig(0.3, 4.0, 1.0, 1)
    picks, n = O.select_tokens([np.array([10, 7, 5.9, 3], np.float32)], cfg1)
    assert n == 2 and set(picks[0]) == {0, 1}
    picks, n = O.select_tokens([np.array([10, 7, 5.9, 3], np.float32)], O.SpeculationConfig())
    assert n == 1 and list(picks[0]) == [0]  # default cap 0.2: floor(0.8) -> min_select
    picks, n = O.select_tokens([np.array([10, 9, 0, 0], np.float32),
                                np.array([10, 9, 8, 7], np.float32)], cfg1)
    assert n == 3 and [list(p) for p in picks] == [[0, 1, 2], [0, 1, 2]]
    picks, n = O.select_tokens([np.arange(100, dtype=np.float32)],
                               O.SpeculationConfig(0.3, 1e9, 0.2, 1))
    assert n == 20
    picks, n = O.select_tokens([np.array([1, 3, 3, 3, 0], np.float32)],
                               O.SpeculationConfig(0.3, 0.5, 1.0, 1))
    assert list(picks[0]) == [1, 2, 3]


def test_select_tokens_golden_cases(golden):
    for case in golden["ops"]["select"]:
        if "case" not in case:
            continue
        c = case["case"]
        sc = golden["arrays"][f"sel.{c}.scores"]
        cfg = O.SpeculationConfig(0.3, case["alpha"], case["cap_ratio"], case["min_select"])
        picks, n = O.select_tokens([sc[h] for h in range(sc.shape[0])], cfg)
        assert n == case["n"]
        np.testing.assert_array_equal(np.stack(picks), golden["arrays"][f"sel.{c}.picks"])


def test_attention_and_build_partial_golden(golden):
    a = golden["arrays"]
    for c in range(12):
        o, w = O.attention_head(a[f"attn.{c}.q"], a[f"attn.{c}.k"], a[f"attn.{c}.v"])
        np.testing.assert_allclose(o, a[f"attn.{c}.out"], rtol=1e-6, atol=1e-6)
        np.testing.assert_allclose(w, a[f"attn.{c}.w"], rtol=1e-6, atol=1e-7)
    for case in golden["ops"]["select"]:
        if "bp_case" not in case:
            continue
        c = case["bp_case"]
        cols = O.partial_columns(a[f"bp.{c}.qt"], a[f"bp.{c}.kt"], case["ratio"])
        np.testing.assert_array_equal(cols, a[f"bp.{c}.cols"])
    assert O.partial_columns(np.ones((4, 10), np.float32), np.ones((4, 10), np.float32), 0.3).size == 3


def test_pool_golden_logs(golden):
    for log in golden["ops"]["pool"]:
        p = O.Pool(4, limit=log["limit"], policy=O.Policy(log["policy"]))
        for op in log["ops"]:
            if op[0] == "a":
                k = np.array(op[1], np.float32)
                assert p.append(k, -k) == op[2]
            else:
                K, V = p.fetch(op[1])
                assert float(K.sum()) == pytest.approx(op[2], rel=1e-6, abs=1e-6)
        fin = log["final"]
        np.testing.assert_array_equal(p.arrival_seq, fin["arrival_seq"])
        np.testing.assert_array_equal(p.last_fetch_seq, fin["last_fetch_seq"])
        np.testing.assert_array_equal(p.fetch_counter, fin["fetch_counter"])
        np.testing.assert_allclose(p.keys, np.array(fin["keys"], np.float32))


def test_pool_spec_examples():
    p = O.Pool(2, limit=3, policy=O.Policy.COUNTER)
    for i in range(3):
        p.append(np.zeros(2), np.zeros(2))
    p.fetch_counter[:] = [5, 0, 7]
    assert p.evict_select() == 1
    p.fetch_counter[:] = [254, 10, 3]
    p.fetch([0])                                      # 254 -> 255 -> halve all
    assert list(p.fetch_counter) == [127, 5, 1]
    q = O.Pool(2, limit=3, policy=O.Policy.LRU)
    for i in range(3):
        q.append(np.zeros(2), np.zeros(2))
    q.fetch([0, 2])
    q.fetch([1])
    assert q.evict_select() == 0


def test_load_model_reads_reference_files():
    """paper_2406_19707_b200.load_model reads the reference's manifest + payload
    format (model.py:284-409) written by the real reference's save_model, and
    the oracle rebuilds the same weights bit-for-bit."""
    import os
    from paper_2406_19707_b200.model import load_model
    path = os.path.join(os.path.dirname(__file__), "golden", "tiny_skewed.json")
    m = load_model(path)
    assert m.skewed and m.spec.layers == 2 and m.spec.model_dim == 32 and m.spec.head_dim == 16
    spec = O.ModelSpec(layers=2, model_dim=32, heads=2, ffn_dim=64, outlier_channels=4,
                       outlier_scale=2.0, seed=5)
    ref = O.skew_model(O.generate_synthetic(spec), calib_seed=1)
    for li in range(2):
        for f in ("w_q", "w_k", "w_v", "w_o", "ffn_in", "ffn_out", "ln1_gain", "ln2_bias"):
            np.testing.assert_allclose(getattr(m.layers[li], f), getattr(ref.layers[li], f),
                                       rtol=0, atol=1e-6)
