"""Engine-vs-oracle parity at the benchmark widths (VERDICT r1 "Next round" #1).

Per config (C2 OPT-6.7B B 8 s 2K, C3 OPT-13B B 16 s 4K, C4 Llama-2-7B B 4
s 32K, C5 rank 0 of the 8-way OPT-30B split B 32 s 8K), on a 3-layer
truncation with injected state (tests/shape_parity.py):

1. hook mode -- identical x_a (the reference's LN1 output, engine.py:311)
   and identical partial artifacts: DecodeEngine.speculate() runs the product
   chain (packed fused GEMM -> ig_rehearse_count -> ig_select) and must give
   the reference's n and per-head index sets (speculation.py:117-163); with
   the reference's own partial queries replayed (x_a . partial_w_q,
   speculation.py:133) the rehearsal + selection kernels are checked alone.
   Every difference must be implied by the score differences (see
   shape_parity.explain_selection) and is counted in the report;
2. engine, f32 pool, 4 free-running decode steps from the same state (the
   default resident / packed / eager path): output rows within 1e-4 (scaled)
   of the reference's decode_step (engine.py:295-380), selections checked
   with the same rule on the engine's own recorded scores;
3. bench defaults (f16 host pool, resident slot tables, packed GEMMs,
   speculation stream, CUDA-graph replay), 4 steps: output rows within 2e-4
   (scaled; the appended rows are rounded to f16, the injected ones are
   f16-representable) and the selection agreement reported.

Numbers go to $IG_PARITY_REPORT (profiles/r02*_parity_shapes.jsonl).
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import speckv_port as O
from tests.shape_parity import ALPHA, CAP, LAYERS, RATIO, Case, Tally, explain_selection, report

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

STEPS = 4
F32_TOL = 1e-4
F16_TOL = 2e-4


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2406_19707_b200 import _lib
    _lib.load()


def _scaled_err(a, b):
    return float(np.abs(a - b).max() / max(1.0, np.abs(b).max()))


def hook_mode(case: Case, eng, reps: int = 3) -> dict:
    """speculate() on identical inputs at layers 1 and 2, `reps` x vectors."""
    sc = O.SpeculationConfig(RATIO, ALPHA, CAP, 1)
    B, H, d = case.B, case.H, case.d
    h0, Hg = eng.h0, eng.Hg
    rng = np.random.default_rng(case.seed + 11)
    xs = [case.x0] + [rng.standard_normal((B, case.D), dtype=np.float32) for _ in range(reps - 1)]
    tallies = {"gemm": Tally(), "replay": Tally()}
    for li in range(1, LAYERS):
        prev = case.model.layers[li - 1]
        xa = [np.concatenate([O.layernorm(x[b:b + 1], prev.ln1_gain, prev.ln1_bias, case.spec.ln_eps)
                              for b in range(B)]) for x in xs]
        ref = [[None] * B for _ in xs]            # (scores [H][s], picks, n)
        qref = [np.zeros((B, Hg, case.kc), np.float32) for _ in xs]
        for b in range(B):
            arts = case.partials(b, li)
            for r, x in enumerate(xa):
                scores = O.speculate_scores(x[b], arts, li, d)
                picks, n = O.select_tokens(scores, sc)
                ref[r][b] = (scores, picks, n)
                for hl in range(Hg):        # the reference's own partial query (speculation.py:133)
                    qref[r][b, hl] = x[b] @ arts.head(li, h0 + hl).partial_w_q
            del arts
        for r in range(len(xs)):
            counts_all = np.array([[int(np.sum(v > np.float32(float(np.max(v)) - ALPHA)))
                                    for v in ref[r][b][0]] for b in range(B)])
            extra = counts_all.sum(axis=1) - counts_all[:, h0:h0 + Hg].sum(axis=1)
            for mode, kw in (("gemm", dict(x_a=xa[r])), ("replay", dict(qspec=qref[r]))):
                out = eng.speculate(li, extra_counts=extra if Hg != H else None, **kw)
                for b in range(B):
                    scores, picks, n = ref[r][b]
                    gn = int(out["n"][b])
                    explain_selection(tallies[mode], (li, r, b), scores[h0:h0 + Hg],
                                      picks[h0:h0 + Hg], n,
                                      [out["idx"][b, hl, :gn] for hl in range(Hg)], gn,
                                      gpu_scores=out["scores"][b], gpu_counts=out["counts"][b])
    return {k: t.as_dict() for k, t in tallies.items()}


def oracle_run(case: Case, steps: int):
    """The reference decode loop per sequence from the injected state; returns
    outputs [B][steps][D], records [b][step][layer], spec scores [b][step][layer]."""
    ocfg = case.oracle_config(steps, record_selection=True)
    outs, recs, scs = [], [], []
    for b in range(case.B):
        cap = []

        def spec_hook(x, arts, layer, d):
            v = O.speculate_scores(x, arts, layer, d)
            cap.append(v)
            return v

        sess = case.session(b, ocfg)
        sess.hooks["speculate_scores"] = spec_hook
        outs.append([sess.decode_step() for _ in range(steps)])
        recs.append(sess.records)
        scs.append([[None] + cap[2 * t:2 * t + 2] for t in range(steps)])
        del sess
    return np.asarray(outs), recs, scs


@pytest.mark.parametrize("name", ["c2", "c3", "c4", "c5r0"])
def test_full_width_parity(name):
    import torch
    case = Case(name)
    problems = []
    res = {"B": case.B, "s": case.s, "D": case.D, "H": case.H, "ffn": case.F, "layers": LAYERS,
           "shard": case.shard}
    # ---- 1. hook mode (and, below, the f32-pool free-running engine)
    eng = case.engine(STEPS, pool_dtype="f32", record=True)
    try:
        res["hook"] = hook = hook_mode(case, eng)
        for mode, t in hook.items():
            if t["n_unexplained"]:
                problems.append(f"hook/{mode}: unexplained {t['unexplained']}")
        if hook["replay"]["max_score_err"] > 2e-6:
            problems.append(f"replayed-query scores off by {hook['replay']['max_score_err']}")
        if hook["gemm"]["max_score_err"] > 2e-5:
            problems.append(f"GEMM-query scores off by {hook['gemm']['max_score_err']}")
        if case.shard is not None:        # a shard engine runs hook calls only
            report(name, res)
            assert not problems, problems
            return
        # ---- 2. engine, f32 pool, free-running
        got = np.stack([eng.decode_step().cpu().numpy().copy() for _ in range(STEPS)], axis=1)
        eng_recs = eng.records
    finally:
        eng.close()
        del eng
        torch.cuda.empty_cache()
    ref_out, ref_recs, ref_sc = oracle_run(case, STEPS)
    err = _scaled_err(got, ref_out)
    t = Tally()
    for it in range(STEPS):
        for b in range(case.B):
            for li in range(1, LAYERS):
                r, rr = eng_recs[it][b][li], ref_recs[b][it][li]
                explain_selection(t, (it, b, li), ref_sc[b][it][li], rr["selected"], rr["n_selected"],
                                  r["selected"], r["n_selected"], gpu_scores=r["spec_scores"])
    res["engine_f32"] = {"out_err": err, "tol": F32_TOL, **t.as_dict()}
    if err >= F32_TOL:
        problems.append(f"engine f32 outputs off by {err}")
    if t.unexplained:
        problems.append(f"engine f32: unexplained {t.unexplained[:5]}")
    # ---- 3. bench defaults: f16 pool, resident, packed, spec stream, CUDA graph
    eng = case.engine(STEPS, pool_dtype="f16", cuda_graph=True)
    try:
        t = Tally()
        outs = []
        for it in range(STEPS):
            outs.append(eng.decode_step().cpu().numpy().copy())
            torch.cuda.synchronize()
            n_dev, idx = eng.n.cpu().numpy(), eng.idx.cpu().numpy()
            for b in range(case.B):
                for li in range(1, LAYERS):
                    rr = ref_recs[b][it][li]
                    gn = int(n_dev[li, b])
                    explain_selection(t, (it, b, li), ref_sc[b][it][li], rr["selected"], rr["n_selected"],
                                      [idx[li, b, h, :gn] for h in range(case.H)], gn)
        err16 = _scaled_err(np.stack(outs, axis=1), ref_out)
        res["bench_defaults"] = {"out_err": err16, "tol": F16_TOL, "graph_replays": STEPS - 1,
                                 **t.as_dict()}
        if err16 >= F16_TOL:
            problems.append(f"bench-default outputs off by {err16}")
    finally:
        eng.close()
    report(name, res)
    assert not problems, problems


@pytest.mark.parametrize("graph", [True, False])
def test_bench_defaults_are_deterministic(graph):
    """Three runs of the bench-default engine (f16 pool, resident slot tables,
    speculation and fetch streams) from the same injected C2 state give the same
    output bits and selections.  A binary that only shifted the GEMM's timing
    once broke this (profiles/r02_ab_late/README.md), so it is checked directly."""
    import torch
    case = Case("c2")
    runs = []
    for _ in range(3):
        eng = case.engine(STEPS, pool_dtype="f16", cuda_graph=graph)
        try:
            outs = []
            for _ in range(STEPS):
                outs.append(eng.decode_step().cpu().numpy().copy())
            torch.cuda.synchronize()
            runs.append((np.stack(outs), eng.n.cpu().numpy().copy(), eng.idx.cpu().numpy().copy()))
        finally:
            eng.close()
            del eng
            torch.cuda.empty_cache()
    for r in runs[1:]:
        np.testing.assert_array_equal(r[0], runs[0][0])
        np.testing.assert_array_equal(r[1], runs[0][1])
        np.testing.assert_array_equal(r[2], runs[0][2])
