"""Resident selection (csrc/resident.cu, DecodeEngine(resident=True)).

The fetched set of every speculative layer stays in HBM across decode steps
and only rows that enter the selection cross the host link.  The attended
rows must be exactly the reference's fetch set (engine.py:382-418), so:

* ig_resident_plan vs a NumPy statement of its contract (random slot tables,
  selections, overwritten rows);
* engine, f32 pool: every selection / n / byte count / pool event identical to
  the oracle for every speculative fixture config (incl. COUNTER/LRU/FIFO
  eviction, where an overwritten row may sit in a slot), outputs within 1e-4;
* a 300-step eviction run (victims churn through the slot tables);
* f16 pool within the 2-byte tolerance; CUDA-graph replay identical to eager;
* fewer rows fetched than the reference accounts.
"""

import copy

import numpy as np
import pytest

from oracle import speckv_port as O
from tests.golden_cfg import RUNS, models, run_config
from tests.test_engine_gpu import _cmp_records, _scaled_err, engine_cfg, oracle_decode, oracle_sessions

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2406_19707_b200 import _lib
    _lib.load()


def _plan_reference(ids, used, sel, pos_prev):
    """The contract of ig_resident_plan for one (b, h) (include/infinigen_b200.h)."""
    ids = ids.copy()
    sel_set = set(int(x) for x in sel)
    for j in range(used):
        if ids[j] >= 0 and (ids[j] == pos_prev or ids[j] not in sel_set):
            ids[j] = -1
    resident = set(int(x) for x in ids[:used] if x >= 0)
    free = [j for j in range(used) if ids[j] < 0]
    enter = [int(x) for x in sel if int(x) not in resident]
    slots = []
    for k, row in enumerate(enter):
        slot = free[k] if k < len(free) else used + (k - len(free))
        ids[slot] = row
        slots.append(slot)
    return ids, max(used, used + len(enter) - len(free)), enter, slots


@pytest.mark.parametrize("seed", range(6))
def test_resident_plan_matches_contract(seed):
    import torch
    from paper_2406_19707_b200 import _lib
    rng = np.random.default_rng(seed)
    B, Hg, cap, S = 3, 5, [7, 64, 700, 300, 1, 33][seed], 2000
    ids = np.full((B, Hg, cap), -1, np.int32)
    used = np.zeros((B, Hg), np.int32)
    idx = np.zeros((B, Hg, cap), np.int32)
    n = rng.integers(0, cap + 1, size=B).astype(np.int32)
    pos_prev = np.full((B, Hg), -1, np.int32)
    for b in range(B):
        for h in range(Hg):
            u = int(rng.integers(0, cap + 1))
            held = rng.choice(S, size=u, replace=False).astype(np.int32)
            held[rng.random(u) < 0.2] = -1                         # freed slots
            ids[b, h, :u], used[b, h] = held, u
            live = held[held >= 0]
            keep = live[rng.random(len(live)) < 0.7][: n[b]]
            rest = np.setdiff1d(np.arange(S), live)
            new = rng.choice(rest, size=n[b] - len(keep), replace=False)
            idx[b, h, :n[b]] = np.sort(np.concatenate([keep, new]).astype(np.int32))
            if len(live) and rng.random() < 0.5:
                pos_prev[b, h] = live[rng.integers(len(live))]     # an overwritten row
    t = {k: torch.from_numpy(v).cuda() for k, v in
         dict(ids=ids, used=used, idx=idx, n=n, pos=pos_prev).items()}
    frow = torch.full((B, Hg, cap), -7, dtype=torch.int32, device="cuda")
    fslot = torch.full((B, Hg, cap), -7, dtype=torch.int32, device="cuda")
    fcount = torch.zeros((B, Hg), dtype=torch.int32, device="cuda")
    moved = torch.zeros(1, dtype=torch.int64, device="cuda")
    _lib.call("ig_resident_plan", t["idx"].data_ptr(), t["n"].data_ptr(), t["pos"].data_ptr(),
              t["ids"].data_ptr(), t["used"].data_ptr(), B, Hg, cap, frow.data_ptr(),
              fslot.data_ptr(), fcount.data_ptr(), moved.data_ptr(), _lib.stream_handle())
    got_ids, got_used = t["ids"].cpu().numpy(), t["used"].cpu().numpy()
    fr, fs, fc = frow.cpu().numpy(), fslot.cpu().numpy(), fcount.cpu().numpy()
    total = 0
    for b in range(B):
        for h in range(Hg):
            e_ids, e_used, e_rows, e_slots = _plan_reference(ids[b, h], int(used[b, h]),
                                                             idx[b, h, :n[b]], int(pos_prev[b, h]))
            assert got_used[b, h] == e_used
            np.testing.assert_array_equal(got_ids[b, h, :e_used], e_ids[:e_used])
            assert fc[b, h] == len(e_rows)
            np.testing.assert_array_equal(fr[b, h, :fc[b, h]], e_rows)
            np.testing.assert_array_equal(fs[b, h, :fc[b, h]], e_slots)
            live = got_ids[b, h, :e_used]
            assert sorted(live[live >= 0].tolist()) == sorted(idx[b, h, :n[b]].tolist())
            total += len(e_rows)
    assert int(moved.item()) == total


def test_fetch_slots_and_stage_put():
    import torch
    from paper_2406_19707_b200 import _lib
    rng = np.random.default_rng(0)
    B, Hg, S, cap, d = 2, 3, 50, 9, 128
    pool = torch.from_numpy(rng.standard_normal((B, Hg, S, 2 * d)).astype(np.float16)).pin_memory()
    pool_dev = pool.data_ptr()          # UVA: pinned host memory is device-addressable
    stage = torch.zeros((B, Hg, cap, 2 * d), dtype=torch.float16, device="cuda")
    frow = torch.zeros((B, Hg, cap), dtype=torch.int32)
    fslot = torch.zeros((B, Hg, cap), dtype=torch.int32)
    fcount = torch.from_numpy(rng.integers(0, cap + 1, (B, Hg)).astype(np.int32))
    for b in range(B):
        for h in range(Hg):
            c = int(fcount[b, h])
            frow[b, h, :c] = torch.from_numpy(np.sort(rng.choice(S, c, replace=False)).astype(np.int32))
            fslot[b, h, :c] = torch.from_numpy(rng.permutation(cap)[:c].astype(np.int32))
    fr, fs, fc = frow.cuda(), fslot.cuda(), fcount.cuda()
    _lib.call("ig_fetch_slots", pool_dev, fr.data_ptr(), fs.data_ptr(), fc.data_ptr(), B, Hg, S, cap,
              2 * d * 2, stage.data_ptr(), _lib.stream_handle())
    st = stage.cpu()
    for b in range(B):
        for h in range(Hg):
            for k in range(int(fcount[b, h])):
                assert torch.equal(st[b, h, int(fslot[b, h, k])], pool[b, h, int(frow[b, h, k])])
    # stage_put: f32 rows rounded exactly like the pool append
    kv = torch.from_numpy(rng.standard_normal((B, 3 * Hg * d)).astype(np.float32)).cuda()
    pos = torch.from_numpy(rng.integers(0, cap, (B, Hg)).astype(np.int32)).cuda()
    _lib.call("ig_stage_put", kv.data_ptr() + 4 * Hg * d, kv.data_ptr() + 8 * Hg * d, 3 * Hg * d,
              pos.data_ptr(), stage.data_ptr(), _lib.ELT["f16"], B, Hg, d, cap, _lib.stream_handle())
    st, p = stage.cpu(), pos.cpu()
    for b in range(B):
        for h in range(Hg):
            k = kv[b, Hg * d + h * d:Hg * d + (h + 1) * d].half().cpu()
            v = kv[b, 2 * Hg * d + h * d:2 * Hg * d + (h + 1) * d].half().cpu()
            assert torch.equal(st[b, h, int(p[b, h])], torch.cat([k, v]))


SPEC_RUNS = sorted(r for r in RUNS if RUNS[r]["scheme"] == "speculative")


@pytest.mark.parametrize("rname", SPEC_RUNS)
@pytest.mark.parametrize("mname", ["m64", "m256"])
@pytest.mark.parametrize("dense", ["cublas", "packed"])
def test_resident_engine_matches_oracle(mname, rname, dense):
    """dense="packed" (2xf16-split tensor cores) and IEEE-f32 cuBLAS: every
    selection identical to the oracle's (f32-level x_a)."""
    from paper_2406_19707_b200 import DecodeEngine
    _, sk = models(mname)
    ocfg = run_config(rname, record_selection=True)
    sessions = oracle_sessions(sk, ocfg)
    eng = DecodeEngine.from_sessions(sk, engine_cfg(ocfg), copy.deepcopy(sessions), pool_dtype="f32",
                                     resident=True, dense=dense)
    try:
        ref_out, ref_recs = oracle_decode(sessions, ocfg.gen_len)
        got = np.stack([eng.x.cpu().numpy()] + [eng.decode_step().cpu().numpy()
                                                for _ in range(ocfg.gen_len)], axis=1)
        assert _scaled_err(got, ref_out) < 1e-4
        _cmp_records(eng.records, ref_recs, ocfg.batch, exact=True)
        # the slot tables hold exactly the last selection of every layer
        for li in range(1, sk.spec.layers):
            ids, used = eng.slot_id[li - 1].cpu().numpy(), eng.slot_used[li - 1].cpu().numpy()
            n = eng.n[li].cpu().numpy()
            idx = eng.idx[li].cpu().numpy()
            for b in range(ocfg.batch):
                for h in range(eng.Hg):
                    live = ids[b, h, :used[b, h]]
                    assert sorted(live[live >= 0].tolist()) == sorted(idx[b, h, :n[b]].tolist())
    finally:
        eng.close()


@pytest.mark.parametrize("policy", ["counter", "lru", "fifo"])
def test_resident_long_run_eviction(policy):
    from paper_2406_19707_b200 import DecodeEngine
    _, sk = models("m64")
    ocfg = O.RunConfig(scheme="speculative", prompt_len=24, gen_len=300, batch=1,
                       pool_limit=20, pool_policy=O.Policy(policy), record_selection=True)
    sessions = oracle_sessions(sk, ocfg)
    eng = DecodeEngine.from_sessions(sk, engine_cfg(ocfg), copy.deepcopy(sessions), pool_dtype="f32",
                                     resident=True)
    try:
        ref_out, ref_recs = oracle_decode(sessions, ocfg.gen_len)
        got = np.stack([eng.x.cpu().numpy()] + [eng.decode_step().cpu().numpy()
                                                for _ in range(ocfg.gen_len)], axis=1)
        assert _scaled_err(got, ref_out) < 1e-3
        _cmp_records(eng.records, ref_recs, 1, exact=True)
    finally:
        eng.close()


def test_resident_f16_pool_and_fewer_link_rows():
    from paper_2406_19707_b200 import DecodeEngine
    _, sk = models("m256")
    ocfg = run_config("spec", record_selection=True, gen_len=8)
    sessions = oracle_sessions(sk, ocfg)
    eng = DecodeEngine.from_sessions(sk, engine_cfg(ocfg), copy.deepcopy(sessions), pool_dtype="f16",
                                     resident=True)
    try:
        ref_out, ref_recs = oracle_decode(sessions, ocfg.gen_len)
        got = np.stack([eng.x.cpu().numpy()] + [eng.decode_step().cpu().numpy()
                                                for _ in range(ocfg.gen_len)], axis=1)
        assert _scaled_err(got, ref_out) < 5e-3
        assert _cmp_records(eng.records, ref_recs, ocfg.batch, exact=False) >= 0.97
        accounted = sum(r["n_selected"] for it in eng.records for per_b in it for r in per_b[1:]) * eng.Hg
        moved = int(eng.moved_rows[1:].sum())
        assert 0 < moved < accounted
    finally:
        eng.close()


@pytest.mark.parametrize("rname,pool", [("spec", "f16"), ("spec_counter", "f32")])
def test_resident_cuda_graph_is_identical(rname, pool):
    from paper_2406_19707_b200 import DecodeEngine
    _, sk = models("m256")
    ocfg = run_config(rname, gen_len=6)
    sessions = oracle_sessions(sk, ocfg)
    outs = []
    for graph in (False, True):
        eng = DecodeEngine.from_sessions(sk, engine_cfg(ocfg, record_selection=False),
                                         copy.deepcopy(sessions), pool_dtype=pool, cuda_graph=graph,
                                         resident=True)
        try:
            outs.append(np.stack([eng.decode_step().cpu().numpy() for _ in range(ocfg.gen_len)]))
        finally:
            eng.close()
    np.testing.assert_array_equal(outs[0], outs[1])


def test_resident_rejects_bad_combinations():
    from paper_2406_19707_b200 import DecodeEngine
    plain, sk = models("m64")
    with pytest.raises(ValueError):
        DecodeEngine(plain, engine_cfg(run_config("full")), resident=True)
    with pytest.raises(ValueError):
        DecodeEngine(sk, engine_cfg(run_config("spec")), resident=True, hbm_layers=1)


def test_graph_replay_interleaved_with_eager_steps():
    """bench.py replays the captured step, then runs eager (instrumented) steps,
    then replays again: with an odd layer count the eager steps leave x in the
    second buffer, and the replays must still continue from it."""
    from paper_2406_19707_b200 import DecodeEngine
    _, sk = models("m256")                      # 3 layers
    ocfg = run_config("spec", gen_len=9)
    sessions = oracle_sessions(sk, ocfg)
    outs = []
    for mode in ("eager", "mixed"):
        eng = DecodeEngine.from_sessions(sk, engine_cfg(ocfg, record_selection=False),
                                         copy.deepcopy(sessions), pool_dtype="f16", resident=True,
                                         cuda_graph=(mode == "mixed"))
        try:
            o = []
            for i in range(ocfg.gen_len):
                if mode == "mixed":
                    eng.cuda_graph = i not in (3, 4, 6)
                o.append(eng.decode_step().cpu().numpy())
            outs.append(np.stack(o))
        finally:
            eng.close()
    np.testing.assert_array_equal(outs[0], outs[1])


def test_set_resident_toggles_mid_run():
    """bench.py's refetch variant switches a resident engine to refetch mode and
    back mid-run: the decode must equal an engine that never switched."""
    from paper_2406_19707_b200 import DecodeEngine
    _, sk = models("m256")
    ocfg = run_config("spec_counter", gen_len=10)
    sessions = oracle_sessions(sk, ocfg)
    outs = []
    for toggle in (False, True):
        eng = DecodeEngine.from_sessions(sk, engine_cfg(ocfg, record_selection=False),
                                         copy.deepcopy(sessions), pool_dtype="f32", resident=True)
        try:
            o = []
            for i in range(ocfg.gen_len):
                if toggle and i in (3, 6):
                    eng.set_resident(i == 6)
                o.append(eng.decode_step().cpu().numpy())
            outs.append(np.stack(o))
        finally:
            eng.close()
    np.testing.assert_allclose(outs[0], outs[1], rtol=1e-5, atol=1e-5)


def test_spec_stream_matches_single_stream():
    """The speculation chain on its own stream gives the decode of the
    single-stream schedule, bit for bit."""
    from paper_2406_19707_b200 import DecodeEngine
    _, sk = models("m256")
    ocfg = run_config("spec_lru", gen_len=8)
    sessions = oracle_sessions(sk, ocfg)
    outs = []
    for sp in (False, True):
        eng = DecodeEngine.from_sessions(sk, engine_cfg(ocfg, record_selection=False),
                                         copy.deepcopy(sessions), pool_dtype="f16", resident=True,
                                         spec_stream=sp)
        try:
            outs.append(np.stack([eng.decode_step().cpu().numpy() for _ in range(ocfg.gen_len)]))
        finally:
            eng.close()
    np.testing.assert_array_equal(outs[0], outs[1])


def test_llama_like_ffn_narrower_than_fused_qkv():
    """ffn_dim < 4 * model_dim (Llama-2 shape: 11008 vs 16384): the fused
    [W_QKV | W_Q(next)] GEMM is the widest projection and sizes the split-K
    workspace.  Selections identical to the oracle's, outputs within 1e-4."""
    from paper_2406_19707_b200 import DecodeEngine
    spec = O.ModelSpec(layers=3, model_dim=256, heads=2, ffn_dim=640, outlier_channels=8,
                       outlier_scale=2.0, seed=5)
    sk = O.skew_model(O.generate_synthetic(spec), calib_seed=0)
    ocfg = O.RunConfig(scheme="speculative", prompt_len=40, gen_len=5, batch=2, record_selection=True)
    sessions = oracle_sessions(sk, ocfg)
    eng = DecodeEngine.from_sessions(sk, engine_cfg(ocfg), copy.deepcopy(sessions), pool_dtype="f32",
                                     resident=True)
    try:
        ref_out, ref_recs = oracle_decode(sessions, ocfg.gen_len)
        got = np.stack([eng.x.cpu().numpy()] + [eng.decode_step().cpu().numpy()
                                                for _ in range(ocfg.gen_len)], axis=1)
        assert _scaled_err(got, ref_out) < 1e-4
        _cmp_records(eng.records, ref_recs, ocfg.batch, exact=True)
    finally:
        eng.close()


@pytest.mark.parametrize("batch", [12, 20])
def test_wide_batch_engine_matches_oracle(batch):
    """Batches above 8 and above 16 take the packed GEMM's 2-tile (M <= 16) and
    4-tile (M <= 32, one CTA per SM) paths -- C3 runs B = 16, C5 B = 32: every
    selection, n and output row still matches the oracle (f32 pool, eviction)."""
    from paper_2406_19707_b200 import DecodeEngine
    _, sk = models("m256")
    ocfg = run_config("spec_counter", batch=batch, gen_len=4, record_selection=True)
    sessions = oracle_sessions(sk, ocfg)
    eng = DecodeEngine.from_sessions(sk, engine_cfg(ocfg), copy.deepcopy(sessions), pool_dtype="f32")
    try:
        ref_out, ref_recs = oracle_decode(sessions, ocfg.gen_len)
        got = np.stack([eng.x.cpu().numpy()] + [eng.decode_step().cpu().numpy()
                                                for _ in range(ocfg.gen_len)], axis=1)
        assert _scaled_err(got, ref_out) < 1e-4
        _cmp_records(eng.records, ref_recs, ocfg.batch, exact=True)
    finally:
        eng.close()


@pytest.mark.parametrize("S,cap,B,Hg", [(4100, 820, 3, 5), (600, 600, 2, 3), (33000, 6600, 1, 2)])
def test_select_plan_fused_equals_two_launches(S, cap, B, Hg):
    """ig_select_plan (the resident plan in the select's CTA) == ig_select
    followed by ig_resident_plan: idx, n, slot tables, slot counts, fetch lists
    and the moved-rows counter bit-identical, on random scores with ties,
    partly filled slot tables with holes and a previous append position."""
    import torch
    from paper_2406_19707_b200 import _lib
    g = torch.Generator(device="cuda")
    g.manual_seed(S + cap)
    s_len = S - 7
    scores = torch.randint(-40, 40, (B, Hg, S), generator=g, device="cuda").float() / 8
    count_sum = torch.randint(1, cap // 2, (B,), generator=g, device="cuda", dtype=torch.int32) * Hg
    st = torch.zeros(8, dtype=torch.int32, device="cuda")
    st[0] = s_len
    slot0 = torch.full((B, Hg, cap), -1, dtype=torch.int32, device="cuda")
    used0 = torch.randint(0, cap, (B, Hg), generator=g, device="cuda", dtype=torch.int32)
    for b in range(B):
        for h in range(Hg):
            u = min(int(used0[b, h]), s_len)
            used0[b, h] = u
            rows = torch.randperm(s_len, generator=g, device="cuda")[:u].int()
            rows[::5] = -1
            slot0[b, h, :u] = rows
    pos = torch.randint(0, s_len, (B, Hg), generator=g, device="cuda", dtype=torch.int32)
    outs = []
    for fused in (False, True):
        idx = torch.full((B, Hg, cap), -7, dtype=torch.int32, device="cuda")
        n = torch.zeros(B, dtype=torch.int32, device="cuda")
        err = torch.zeros(1, dtype=torch.int32, device="cuda")
        slot, used = slot0.clone(), used0.clone()
        frow = torch.full((B, Hg, cap), -7, dtype=torch.int32, device="cuda")
        fslot = torch.full((B, Hg, cap), -7, dtype=torch.int32, device="cuda")
        fcount = torch.zeros((B, Hg), dtype=torch.int32, device="cuda")
        moved = torch.zeros(1, dtype=torch.int64, device="cuda")
        args = (scores.data_ptr(), count_sum.data_ptr(), st.data_ptr(), B, Hg, Hg, S, cap, 0.2, 1,
                idx.data_ptr(), n.data_ptr(), err.data_ptr())
        if fused:
            _lib.call("ig_select_plan", *args, pos.data_ptr(), slot.data_ptr(), used.data_ptr(), frow.data_ptr(),
                      fslot.data_ptr(), fcount.data_ptr(), moved.data_ptr(), None, _lib.stream_handle())
        else:
            _lib.call("ig_select", *args, None, _lib.stream_handle())
            _lib.call("ig_resident_plan", idx.data_ptr(), n.data_ptr(), pos.data_ptr(), slot.data_ptr(),
                      used.data_ptr(), B, Hg, cap, frow.data_ptr(), fslot.data_ptr(), fcount.data_ptr(),
                      moved.data_ptr(), _lib.stream_handle())
        torch.cuda.synchronize()
        nn = n.cpu()
        sel = [idx[b, :, :int(nn[b])].cpu() for b in range(B)]
        fl = [(frow[b, h, :int(fcount[b, h])].cpu(), fslot[b, h, :int(fcount[b, h])].cpu())
              for b in range(B) for h in range(Hg)]
        outs.append((nn, sel, slot.cpu(), used.cpu(), fcount.cpu(), fl, moved.cpu(), err.cpu()))
    a, b_ = outs
    assert torch.equal(a[0], b_[0])
    for x, y in zip(a[1], b_[1]):
        assert torch.equal(x, y)
    for k in (2, 3, 4, 6, 7):
        assert torch.equal(a[k], b_[k]), k
    for (r1, s1), (r2, s2) in zip(a[5], b_[5]):
        assert torch.equal(r1, r2) and torch.equal(s1, s2)
