"""Operator-level parity on the GPU: each drop-in shim (reference signature) vs
the oracle and the reference's golden vectors.

Bars: indices / n / pool metadata bit-exact; rehearsal scores rtol 1e-5;
attention (f32) rtol 1e-5; layernorm rtol 1e-6.
"""

import numpy as np
import pytest

from oracle import speckv_port as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2406_19707_b200 as pk  # noqa: F401  (raises if the library is missing)
    from paper_2406_19707_b200 import _lib
    _lib.load()


def test_select_tokens_golden_bit_exact(golden):
    from paper_2406_19707_b200 import SpeculationConfig, select_tokens
    for case in golden["ops"]["select"]:
        if "case" not in case:
            continue
        c = case["case"]
        sc = golden["arrays"][f"sel.{c}.scores"]
        cfg = SpeculationConfig(0.3, case["alpha"], case["cap_ratio"], case["min_select"])
        picks, n = select_tokens([sc[h] for h in range(sc.shape[0])], cfg)
        assert n == case["n"], c
        # full list equality: same set AND the reference's stable score order
        np.testing.assert_array_equal(np.stack(picks), golden["arrays"][f"sel.{c}.picks"])


@pytest.mark.parametrize("seed", range(6))
def test_select_tokens_random_with_ties(seed):
    from paper_2406_19707_b200 import SpeculationConfig, select_tokens
    rng = np.random.default_rng(100 + seed)
    for _ in range(8):
        H = int(rng.integers(1, 9))
        s = int(rng.choice([1, 2, 5, 63, 64, 65, 511, 1500, 4097]))
        q = float(rng.choice([0.0, 0.5, 0.01]))
        sc = rng.standard_normal((H, s)).astype(np.float32) * np.float32(rng.choice([0.1, 3.0, 50.0]))
        if q:
            sc = (np.round(sc / q) * q).astype(np.float32)
        sc[:, rng.integers(0, s, size=max(1, s // 10))] = 0.0
        if s > 3:
            sc[0, :2] = -0.0                       # -0.0 and +0.0 tie (linalg.py:184)
        cfg = O.SpeculationConfig(0.3, float(rng.choice([0.25, 1.0, 4.0, 1e9])),
                                  float(rng.choice([0.01, 0.2, 1.0])), int(rng.choice([1, 3])))
        ref_p, ref_n = O.select_tokens([sc[h] for h in range(H)], cfg)
        got_p, got_n = select_tokens([sc[h] for h in range(H)],
                                     SpeculationConfig(*[getattr(cfg, f) for f in
                                                         ("partial_ratio", "alpha", "cap_ratio", "min_select")]))
        assert got_n == ref_n
        for h in range(H):
            np.testing.assert_array_equal(got_p[h], ref_p[h])


def _order_keys(x: np.ndarray) -> np.ndarray:
    """The kernels' order-preserving u32 keys (-0.0 keyed as +0.0)."""
    u = np.where(x == 0, np.float32(0), x).astype(np.float32).view(np.uint32)
    return np.where(u & 0x80000000, ~u, u | 0x80000000).astype(np.uint32)


def _select_direct(sc: np.ndarray, cfg):
    """ig_select on [H, s] scores with the reference's head counts: (n, [H] ascending rows)."""
    import math
    import torch
    from paper_2406_19707_b200 import _lib
    H, s = sc.shape
    S = (s + 3) // 4 * 4
    dsc = torch.zeros((1, H, S), dtype=torch.float32, device="cuda")
    dsc[0, :, :s] = torch.from_numpy(sc).cuda()
    counts = [int(np.sum(v > np.float32(float(np.max(v)) - cfg.alpha))) for v in sc]
    csum = torch.tensor([sum(counts)], dtype=torch.int32, device="cuda")
    st = torch.zeros(8, dtype=torch.int32, device="cuda")
    st[0] = s
    cap = max(int(math.floor(cfg.cap_ratio * s)), cfg.min_select, 1)
    idx = torch.full((1, H, cap), -7, dtype=torch.int32, device="cuda")
    n = torch.zeros(1, dtype=torch.int32, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    _lib.call("ig_select", dsc.data_ptr(), csum.data_ptr(), st.data_ptr(), 1, H, H, S, cap,
              float(cfg.cap_ratio), int(cfg.min_select), idx.data_ptr(), n.data_ptr(), err.data_ptr(),
              None, _lib.stream_handle())
    assert int(err.item()) == 0
    nn = int(n.item())
    got = idx[0].cpu().numpy()
    assert (got[:, nn:] == -7).all()            # nothing written past n
    return nn, [got[h, :nn] for h in range(H)]


@pytest.mark.parametrize("s", [4096, 8193, 32768, 65536, 131072])
@pytest.mark.parametrize("kind", ["normal", "outlier", "flat", "ties", "zeros"])
def test_select_long_rows_and_adversarial(s, kind):
    """ig_select (value bins -> exact rank of the boundary bin, or a radix select
    inside it when it overflows the candidate buffer) vs the reference's stable
    argsort at long contexts (no row-length ceiling below 1M): a huge outlier
    squeezes every other score into one bin (radix path), a flat row is one bin,
    rounded scores tie massively, and +-0.0 tie with each other."""
    rng = np.random.default_rng(s + len(kind))
    H = 3
    sc = rng.standard_normal((H, s)).astype(np.float32) * np.float32(2.5)
    if kind == "outlier":
        sc[:, rng.integers(0, s, 2)] = np.float32(1e6)
        sc[1, 5] = np.float32(-1e7)
    elif kind == "flat":
        sc[:] = np.float32(0.75)
    elif kind == "ties":
        sc = np.round(sc).astype(np.float32)
    elif kind == "zeros":
        sc[:, ::3] = 0.0
        sc[:, 1::3] = -0.0
    for alpha, cap_ratio in ((4.0, 0.2), (1e9, 0.05), (0.5, 1.0)):
        cfg = O.SpeculationConfig(0.3, alpha, cap_ratio, 1)
        ref_p, ref_n = O.select_tokens([sc[h] for h in range(H)], cfg)
        n, got = _select_direct(sc, cfg)
        assert n == ref_n, (kind, alpha)
        for h in range(H):
            np.testing.assert_array_equal(got[h], np.sort(ref_p[h]))


def test_topk_rows_matches_stable_argsort():
    import torch
    from paper_2406_19707_b200 import _lib
    rng = np.random.default_rng(5)
    for rows, length, k in [(1, 10, 3), (7, 128, 39), (40, 64, 20), (3, 5000, 1000), (2, 33, 33)]:
        v = np.round(rng.standard_normal((rows, length)) * 4).astype(np.float32)  # many ties
        dv = torch.from_numpy(v).cuda()
        out = torch.empty((rows, k), dtype=torch.int32, device="cuda")
        _lib.call("ig_topk_rows", dv.data_ptr(), rows, length, k, out.data_ptr(), _lib.stream_handle())
        for r in range(rows):
            np.testing.assert_array_equal(out[r].cpu().numpy(), np.sort(O.topk_indices(v[r], k)))


def test_build_partial_golden(golden):
    from paper_2406_19707_b200 import build_partial
    a = golden["arrays"]
    for case in golden["ops"]["select"]:
        if "bp_case" not in case:
            continue
        c = case["bp_case"]
        np.testing.assert_array_equal(build_partial(a[f"bp.{c}.qt"], a[f"bp.{c}.kt"], case["ratio"]),
                                      a[f"bp.{c}.cols"])


@pytest.mark.parametrize("s", [1, 3, 4, 1000, 4097])
def test_speculate_scores_vs_oracle(s):
    from paper_2406_19707_b200 import speculate_scores
    rng = np.random.default_rng(s)
    H, D, d = 4, 64, 16
    k = 5
    arts = O.Partials(3, H)
    for h in range(H):
        arts.set_head(2, h, O.HeadPartial(np.sort(rng.choice(d, k, replace=False)),
                                          rng.standard_normal((D, k)).astype(np.float32),
                                          rng.standard_normal((s, k)).astype(np.float32) * 3))
    x = rng.standard_normal(D).astype(np.float32)
    ref = O.speculate_scores(x, arts, 2, d)
    got = speculate_scores(x, arts, 2, d)
    for h in range(H):
        np.testing.assert_allclose(got[h], ref[h], rtol=1e-5, atol=1e-5)
    with pytest.raises(ValueError):
        speculate_scores(x, arts, 0, d)


def test_attention_head_golden(golden):
    from paper_2406_19707_b200 import attention_head
    a = golden["arrays"]
    for c in range(12):
        o, w = attention_head(a[f"attn.{c}.q"], a[f"attn.{c}.k"], a[f"attn.{c}.v"])
        np.testing.assert_allclose(o, a[f"attn.{c}.out"], rtol=1e-5, atol=1e-5)
        np.testing.assert_allclose(w, a[f"attn.{c}.w"], rtol=1e-5, atol=1e-6)
    with pytest.raises(ValueError):
        attention_head(np.zeros((1, 4)), np.zeros((0, 4)), np.zeros((0, 4)))


def test_kvpool_golden_logs(golden):
    from paper_2406_19707_b200 import EvictionPolicy, KvPool
    for log in golden["ops"]["pool"]:
        events = []
        p = KvPool(4, limit=log["limit"], policy=EvictionPolicy(log["policy"]),
                   on_overwrite=lambda v, a: events.append((v, a)))
        ref = O.Pool(4, limit=log["limit"], policy=O.Policy(log["policy"]),
                     on_overwrite=None)
        for op in log["ops"]:
            if op[0] == "a":
                k = np.array(op[1], np.float32)
                if len(ref) == ref.limit:
                    assert p.evict_select() == ref.evict_select()
                assert p.append(k, -k) == op[2]
                ref.append(k, -k)
            else:
                K, V = p.fetch(op[1])
                assert float(K.sum()) == pytest.approx(op[2], rel=1e-5, abs=1e-5)
                np.testing.assert_array_equal(V, -K)
                ref.fetch(op[1])
        fin = log["final"]
        np.testing.assert_array_equal(p.arrival_seq, fin["arrival_seq"])
        np.testing.assert_array_equal(p.last_fetch_seq, fin["last_fetch_seq"])
        np.testing.assert_array_equal(p.fetch_counter, fin["fetch_counter"])
        np.testing.assert_array_equal(p.keys, np.array(fin["keys"], np.float32))
        assert len(events) == max(0, sum(op[0] == "a" for op in log["ops"]) - log["limit"])
        with pytest.raises(IndexError):
            p.fetch([len(p)])
        p.close()


def test_layernorm_vs_oracle():
    import torch
    from paper_2406_19707_b200.prefill import layernorm
    rng = np.random.default_rng(9)
    for rows, D in [(1, 64), (16, 5120), (3, 7168)]:
        x = (rng.standard_normal((rows, D)) * 3 + 1).astype(np.float32)
        g = (1 + 0.02 * rng.standard_normal(D)).astype(np.float32)
        b = (0.02 * rng.standard_normal(D)).astype(np.float32)
        ref = O.layernorm(x, g, b, 1e-5)
        got = layernorm(torch.from_numpy(x).cuda(), torch.from_numpy(g).cuda(),
                        torch.from_numpy(b).cuda(), 1e-5).cpu().numpy()
        np.testing.assert_allclose(got, ref, rtol=1e-6, atol=2e-6)


@pytest.mark.parametrize("s", [1, 5, 1023, 1024, 1025, 4101, 9000])
def test_rehearse_count_fused_matches_oracle(s):
    """ig_rehearse_count (tile max + last-tile count) == oracle speculate_scores
    + the count half of select_tokens, per (b, h)."""
    import torch
    from paper_2406_19707_b200 import _lib
    rng = np.random.default_rng(s)
    B, Hg, d, k, D = 3, 4, 32, 10, 96
    S = (s + 3) // 4 * 4
    alpha = 2.0
    x = rng.standard_normal((B, D)).astype(np.float32)
    wq = rng.standard_normal((D, Hg * d)).astype(np.float32)
    cols = np.stack([[np.sort(rng.choice(d, k, replace=False)) for _ in range(Hg)] for _ in range(B)])
    pkey = rng.standard_normal((B, Hg, s, k)).astype(np.float32) * 2
    qspec = (x @ wq).astype(np.float32)
    dev = "cuda"
    pk = torch.zeros((B, Hg, k, S), dtype=torch.float32, device=dev)
    pk[..., :s] = torch.from_numpy(np.ascontiguousarray(pkey.transpose(0, 1, 3, 2))).to(dev)
    scores = torch.empty((B, Hg, S), dtype=torch.float32, device=dev)
    counts = torch.zeros((B, Hg), dtype=torch.int32, device=dev)
    csum = torch.zeros(B, dtype=torch.int32, device=dev)
    mk = torch.zeros((B, Hg), dtype=torch.int32, device=dev)
    tk = torch.zeros((B, Hg), dtype=torch.int32, device=dev)
    st = torch.zeros(8, dtype=torch.int32, device=dev)
    st[0] = s
    tq = torch.from_numpy(qspec).to(dev)
    tc = torch.from_numpy(cols.astype(np.int32)).to(dev)
    scale = float(np.float32(1.0 / np.sqrt(d)))
    rr = torch.zeros((B, Hg, 2), dtype=torch.int32, device=dev)
    _lib.call("ig_rehearse_count", tq.data_ptr(), Hg * d, tc.data_ptr(), pk.data_ptr(), st.data_ptr(),
              B, Hg, d, k, S, scale, alpha, scores.data_ptr(), mk.data_ptr(), tk.data_ptr(),
              counts.data_ptr(), csum.data_ptr(), rr.data_ptr(), _lib.stream_handle())
    assert not mk.any() and not tk.any()          # scratch left zeroed
    got_s = scores.cpu().numpy()[..., :s]
    # row_range: the (max, min) order keys of each row's s scores
    keys = _order_keys(got_s)
    np.testing.assert_array_equal(rr.cpu().numpy().view(np.uint32),
                                  np.stack([keys.max(-1), keys.min(-1)], -1))
    got_c = counts.cpu().numpy()
    for b in range(B):
        arts = O.Partials(2, Hg)
        for h in range(Hg):
            arts.set_head(1, h, O.HeadPartial(cols[b, h], wq[:, h * d:(h + 1) * d][:, cols[b, h]],
                                              pkey[b, h]))
        ref = O.speculate_scores(x[b], arts, 1, d)
        for h in range(Hg):
            np.testing.assert_allclose(got_s[b, h], ref[h], rtol=1e-5, atol=1e-5)
            # the count on the GPU's own scores must follow the reference rule exactly
            v = got_s[b, h]
            assert got_c[b, h] == int(np.sum(v > (float(np.max(v)) - alpha)))
        assert int(csum[b]) == int(got_c[b].sum())


def test_blocked_causal_prefill_attention_matches_oracle():
    """The query-blocked causal attention used for long prompts == model.py:156-180."""
    import torch
    from paper_2406_19707_b200.prefill import causal_attention
    rng = np.random.default_rng(4)
    H, N, d = 3, 300, 16
    q, k, v = (rng.standard_normal((H, N, d)).astype(np.float32) for _ in range(3))
    got = causal_attention(*(torch.from_numpy(a).cuda() for a in (q, k, v)), block=64).cpu().numpy()
    for h in range(H):
        ref, _ = O.attention_head(q[h], k[h], v[h], causal=True)
        np.testing.assert_allclose(got[h], ref, rtol=1e-4, atol=1e-5)


@pytest.mark.parametrize("M,N,K", [(1, 128, 64), (5, 260, 100), (8, 512, 5120), (16, 5120, 5120),
                                   (17, 1024, 2048), (32, 384, 4096), (16, 20480, 512),
                                   (16, 20480, 5120), (4, 4096, 11008), (12, 200, 36)])
@pytest.mark.parametrize("epilogue", [0, 1, 2])
def test_sgemm_packed_vs_float64(M, N, K, epilogue):
    """ig_sgemm_pack + ig_sgemm_packed (persistent stream-K 3xTF32 over packed
    weights) vs float64: every M template, ragged column tiles and row blocks,
    tile segments split over several CTAs, fused epilogues, strided X/Y;
    bit-identical on repeat; tickets left zeroed."""
    import ctypes
    import torch
    from paper_2406_19707_b200 import _lib
    g = torch.Generator(device="cuda")
    g.manual_seed(M * 1000 + N + K + 7)
    X = torch.randn(M, K + 4, device="cuda", generator=g)[:, :K]        # ldx > K
    W = torch.randn(K, N + 8, device="cuda", generator=g)[:, :N]        # ld > N
    R = torch.randn(M, N, device="cuda", generator=g)
    pf, wf, tf = ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_size_t()
    _lib.call("ig_sgemm_packed_sizes", M, N, K, ctypes.byref(pf), ctypes.byref(wf), ctypes.byref(tf),
              kernels=0)
    P = torch.full((pf.value,), float("nan"), device="cuda")
    _lib.call("ig_sgemm_pack", W.data_ptr(), W.stride(0), N, K, P.data_ptr(), _lib.stream_handle())
    ws = torch.empty(wf.value, device="cuda")
    tk = torch.zeros(tf.value, dtype=torch.int32, device="cuda")
    outs = []
    for _ in range(2):
        Yb = torch.full((M, N + 3), float("nan"), device="cuda")
        Y = Yb[:, :N]
        _lib.call("ig_sgemm_packed", X.data_ptr(), X.stride(0), P.data_ptr(), N, K, Y.data_ptr(),
                  Yb.stride(0), R.data_ptr() if epilogue == 2 else None, N if epilogue == 2 else 0, M,
                  epilogue, ws.data_ptr(), ws.numel(), tk.data_ptr(), tk.numel(), _lib.stream_handle())
        outs.append(Y.clone())
        assert torch.isnan(Yb[:, N:]).all()                 # nothing written past N
    ref = X.double() @ W.double()
    if epilogue == 1:
        ref = ref.clamp_min(0)
    elif epilogue == 2:
        ref = ref + R.double()
    torch.testing.assert_close(outs[0].double(), ref, rtol=1e-5, atol=2e-4 * max(1.0, K ** 0.5 / 8))
    assert torch.equal(outs[0], outs[1])
    assert not tk.any()


@pytest.mark.parametrize("elt", ["f16", "bf16"])
def test_attend_512b_row_variants_match(elt):
    """The two 512-B-row attention kernels -- mma.sync (default) and tcgen05
    (IG_ATTEND_IMPL=c) -- each in a subprocess (the switch is read once per
    process), vs float64 attention over the same rows:
    ragged row counts, an excluded row (pos), resident slot tables with empty
    slots (ig_attend_slots)."""
    import os
    import subprocess
    import sys
    import tempfile
    code = (
        "import numpy as np, torch, ctypes, sys\n"
        "from paper_2406_19707_b200 import _lib\n"
        "rng = np.random.default_rng(3)\n"
        "B, Hg, d, cap = 2, 3, 128, 700\n"
        "q = torch.from_numpy(rng.standard_normal((B, 3*Hg*d)).astype(np.float32)).cuda()\n"
        "T = torch.float16 if sys.argv[2] == 'f16' else torch.bfloat16\n"
        "stage = torch.from_numpy((2*rng.standard_normal((B, Hg, cap, 2*d))).astype(np.float32)).to(T).cuda()\n"
        "n = torch.tensor([700, 37], dtype=torch.int32, device='cuda')\n"
        "idx = torch.from_numpy(np.tile(np.arange(cap, dtype=np.int32), (B, Hg, 1))).cuda()\n"
        "pos = torch.full((B, Hg), 5, dtype=torch.int32, device='cuda')\n"
        "st = torch.zeros(8, dtype=torch.int32, device='cuda')\n"
        "pf, tk = ctypes.c_size_t(), ctypes.c_size_t()\n"
        "_lib.call('ig_attend_scratch', B, Hg, d, cap, ctypes.byref(pf), ctypes.byref(tk), kernels=0)\n"
        "part = torch.empty(pf.value, device='cuda'); tick = torch.zeros(tk.value, dtype=torch.int32, device='cuda')\n"
        "out = torch.empty((B, Hg*d), device='cuda')\n"
        "_lib.call('ig_attend', q.data_ptr(), 3*Hg*d, q.data_ptr()+4*Hg*d, q.data_ptr()+8*Hg*d, 3*Hg*d, stage.data_ptr(),"
        " _lib.ELT[sys.argv[2]], idx.data_ptr(), n.data_ptr(), pos.data_ptr(), st.data_ptr(), B, Hg, d, cap, part.data_ptr(),"
        " tick.data_ptr(), out.data_ptr(), Hg*d, _lib.stream_handle())\n"
        "slot = idx.clone(); slot[:, :, 1::7] = -1\n"
        "used = torch.tensor([[700, 650, 9], [1, 0, 300]], dtype=torch.int32, device='cuda')\n"
        "out2 = torch.empty((B, Hg*d), device='cuda')\n"
        "_lib.call('ig_attend_slots', q.data_ptr(), 3*Hg*d, q.data_ptr()+4*Hg*d, q.data_ptr()+8*Hg*d, 3*Hg*d,"
        " stage.data_ptr(), _lib.ELT[sys.argv[2]], slot.data_ptr(), used.data_ptr(), pos.data_ptr(), st.data_ptr(),"
        " B, Hg, d, cap, part.data_ptr(), tick.data_ptr(), out2.data_ptr(), Hg*d, _lib.stream_handle())\n"
        "np.savez(sys.argv[1], out=out.cpu().numpy(), out2=out2.cpu().numpy(), q=q.cpu().numpy(),"
        " stage=stage.float().cpu().numpy(), slot=slot.cpu().numpy(), used=used.cpu().numpy())\n")
    res = {}
    for impl in ("c", "mma"):                   # tcgen05 (opt-in), mma.sync (default)
        f = os.path.join(tempfile.mkdtemp(), "o.npz")
        env = dict(os.environ, IG_ATTEND_IMPL=impl)
        r = subprocess.run([sys.executable, "-c", code, f, elt], env=env, capture_output=True, text=True,
                           cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        assert r.returncode == 0, r.stderr[-2000:]
        res[impl] = np.load(f)
    z = res["c"]
    qn, stg = z["q"].astype(np.float64), z["stage"].astype(np.float64)
    B, Hg, d = 2, 3, 128

    def ref(b, h, rows):
        K = np.concatenate([stg[b, h, rows, :d], qn[b, Hg * d + h * d:Hg * d + (h + 1) * d][None]])
        V = np.concatenate([stg[b, h, rows, d:], qn[b, 2 * Hg * d + h * d:2 * Hg * d + (h + 1) * d][None]])
        lg = K @ qn[b, h * d:(h + 1) * d] / np.sqrt(d)
        w = np.exp(lg - lg.max())
        return (w / w.sum()) @ V

    for impl, o in res.items():
        for b, nb in enumerate((700, 37)):
            for h in range(Hg):
                exp = ref(b, h, [i for i in range(nb) if i != 5])
                np.testing.assert_allclose(o["out"][b, h * d:(h + 1) * d], exp, rtol=2e-5, atol=2e-5,
                                           err_msg=impl)
                used = int(z["used"][b, h])
                rows = [i for i in range(used) if z["slot"][b, h, i] >= 0 and z["slot"][b, h, i] != 5]
                exp2 = ref(b, h, rows)
                np.testing.assert_allclose(o["out2"][b, h * d:(h + 1) * d], exp2, rtol=2e-5, atol=2e-5,
                                           err_msg=impl + " slots")


def test_shim_error_paths_match_reference():
    """The reference's exception behaviour at the boundary (speculation.py:51-54,
    107-114, 124-132, 149-153; pool.py:32-33, 61-64, 91-92; model.py:167-170)."""
    import paper_2406_19707_b200 as G
    cfg = G.SpeculationConfig()
    with pytest.raises(ValueError):
        G.select_tokens([], cfg)
    with pytest.raises(ValueError):
        G.select_tokens([np.zeros(0, np.float32)], cfg)
    with pytest.raises(ValueError):
        G.select_tokens([np.zeros(4, np.float32), np.zeros(5, np.float32)], cfg)
    with pytest.raises(ValueError):
        G.select_tokens([np.zeros(4, np.float32)], G.SpeculationConfig(alpha=0.0))
    with pytest.raises(ValueError):
        G.build_partial(np.zeros((3, 4)), np.zeros((3, 5)), 0.3)
    with pytest.raises(ValueError):
        G.build_partial(np.zeros((3, 4)), np.zeros((3, 4)), 0.0)
    arts = G.PartialArtifacts(3, 1)
    arts.set_head(1, 0, G.HeadArtifacts(np.array([0, 2]), np.zeros((8, 2), np.float32),
                                        np.zeros((0, 2), np.float32)))
    with pytest.raises(ValueError):                     # empty partial key cache
        G.speculate_scores(np.zeros(8, np.float32), arts, 1, 4)
    with pytest.raises(ValueError):
        arts.set_head(0, 0, arts.head(1, 0))            # layer 0 never speculates
    arts.append_partial_key(1, 0, np.arange(4, dtype=np.float32), 0, 1)
    np.testing.assert_array_equal(arts.head(1, 0).partial_k, [[0.0, 2.0]])
    with pytest.raises(G.ArtifactConsistencyError):
        arts.append_partial_key(1, 0, np.arange(4, dtype=np.float32), 5, 2)
    with pytest.raises(G.ArtifactConsistencyError):
        arts.append_partial_key(1, 0, np.arange(4, dtype=np.float32), 1, 7)
    with pytest.raises(ValueError):
        G.KvPool(4, limit=0)
    p = G.KvPool(4, limit=2)
    with pytest.raises(ValueError):
        p.append(np.zeros(3), np.zeros(4))
    with pytest.raises(ValueError):
        p.evict_select()                                # empty pool
    assert p.append(np.ones(4), np.ones(4)) == 0
    with pytest.raises(IndexError):
        p.fetch([1])
    with pytest.raises(IndexError):
        p.fetch([-1])
    K, V = p.fetch([])                                  # empty fetch is legal
    assert K.shape == (0, 4)
    p.close()
    with pytest.raises(ValueError):
        G.attention_head(np.zeros((1, 4)), np.zeros((2, 4)), np.zeros((3, 4)))


def test_select_all_rows_and_single_row():
    """n == s (alpha huge, cap 1.0) selects every row; s == 1 selects row 0."""
    import paper_2406_19707_b200 as G
    sc = [np.random.default_rng(0).standard_normal(37).astype(np.float32) for _ in range(3)]
    picks, n = G.select_tokens(sc, G.SpeculationConfig(0.3, 1e9, 1.0, 1))
    assert n == 37
    for h in range(3):
        np.testing.assert_array_equal(picks[h], O.topk_indices(sc[h], 37))
    picks, n = G.select_tokens([np.array([2.5], np.float32)], G.SpeculationConfig())
    assert n == 1 and list(picks[0]) == [0]


@pytest.mark.parametrize("env", [{"IG_PDL": "0"}, {"IG_PACKED_CTA": "16"}])
def test_sgemm_packed_launch_variants(env):
    """A chained pair of packed GEMMs (FFN-in with ReLU -> FFN-out with residual,
    the decode step's pattern) in a subprocess per launch variant: with PDL off
    the bits equal the default (PDL on) run -- the programmatic overlap never
    lets a GEMM read its input early; the one-CTA-per-SM grid (other stream-K
    segmentation) agrees within f32 summation-order noise."""
    import os
    import subprocess
    import sys
    import tempfile
    code = (
        "import numpy as np, torch, ctypes, sys\n"
        "from paper_2406_19707_b200 import _lib\n"
        "g = torch.Generator(device='cuda'); g.manual_seed(11)\n"
        "M, D, F = 16, 1024, 4096\n"
        "x = torch.randn(M, D, device='cuda', generator=g)\n"
        "w1 = torch.randn(D, F, device='cuda', generator=g) * 0.03\n"
        "w2 = torch.randn(F, D, device='cuda', generator=g) * 0.03\n"
        "def pack(W):\n"
        "    K, N = W.shape\n"
        "    pf, wf, tf = ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_size_t()\n"
        "    _lib.call('ig_sgemm_packed_sizes', M, N, K, ctypes.byref(pf), ctypes.byref(wf), ctypes.byref(tf), kernels=0)\n"
        "    P = torch.empty(pf.value, device='cuda')\n"
        "    _lib.call('ig_sgemm_pack', W.data_ptr(), N, N, K, P.data_ptr(), _lib.stream_handle())\n"
        "    return P, wf.value, tf.value\n"
        "(p1, w1f, t1), (p2, w2f, t2) = pack(w1), pack(w2)\n"
        "ws = torch.empty(max(w1f, w2f), device='cuda'); tk = torch.zeros(max(t1, t2), dtype=torch.int32, device='cuda')\n"
        "h = torch.empty(M, F, device='cuda'); y = torch.empty(M, D, device='cuda')\n"
        "outs = []\n"
        "for _ in range(3):\n"
        "    _lib.call('ig_sgemm_packed', x.data_ptr(), D, p1.data_ptr(), F, D, h.data_ptr(), F, None, 0, M, 1, ws.data_ptr(), ws.numel(), tk.data_ptr(), tk.numel(), _lib.stream_handle())\n"
        "    _lib.call('ig_sgemm_packed', h.data_ptr(), F, p2.data_ptr(), D, F, y.data_ptr(), D, x.data_ptr(), D, M, 2, ws.data_ptr(), ws.numel(), tk.data_ptr(), tk.numel(), _lib.stream_handle())\n"
        "    outs.append(y.cpu().numpy().copy())\n"
        "assert all((o == outs[0]).all() for o in outs)\n"
        "ref = (torch.relu(x.double() @ w1.double()) @ w2.double() + x.double()).cpu().numpy()\n"
        "np.save(sys.argv[1], outs[0]); np.save(sys.argv[1] + '.ref.npy', ref)\n")
    res = {}
    with tempfile.TemporaryDirectory() as td:
        for name, e in (("default", {}), ("variant", env)):
            f = os.path.join(td, name + ".npy")
            r = subprocess.run([sys.executable, "-c", code, f], env=dict(os.environ, **e),
                               capture_output=True, text=True, timeout=300)
            assert r.returncode == 0, r.stderr[-2000:]
            res[name] = np.load(f)
        ref = np.load(os.path.join(td, "default.npy") + ".ref.npy")
    np.testing.assert_allclose(res["default"], ref, rtol=1e-5, atol=1e-4)
    if "IG_PDL" in env:
        np.testing.assert_array_equal(res["variant"], res["default"])
    else:
        np.testing.assert_allclose(res["variant"], res["default"], rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("env", [{"IG_WP_RING": "3"}, {"IG_WP_SEG": "256"}])
def test_attend_wp_variants_match_default(env):
    """The warp-persistent attention's opt-in ring depth / item size (per-process
    switches, so each in a subprocess) produce the default kernel's outputs over
    ragged slot tables (fixed-order merges: bit-identical per item size; the
    256-row items merge fewer segments, so f32 rounding may differ)."""
    import os
    import subprocess
    import sys
    import tempfile
    code = (
        "import numpy as np, torch, ctypes, sys\n"
        "from paper_2406_19707_b200 import _lib\n"
        "g = torch.Generator(device='cuda'); g.manual_seed(5)\n"
        "B, Hg, d, cap = 4, 5, 128, 900\n"
        "q = torch.randn(B, 3 * Hg * d, device='cuda', generator=g)\n"
        "stage = torch.randn(B, Hg, cap, 2 * d, device='cuda', generator=g).half()\n"
        "slot = torch.arange(cap, device='cuda', dtype=torch.int32).repeat(B, Hg, 1).contiguous()\n"
        "slot[:, :, 7] = -1\n"
        "used = torch.tensor([[cap, 819, 300, 1, 640]] * B, dtype=torch.int32, device='cuda')\n"
        "pos = torch.full((B, Hg), 5, dtype=torch.int32, device='cuda')\n"
        "st = torch.zeros(8, dtype=torch.int32, device='cuda')\n"
        "pf, tk = ctypes.c_size_t(), ctypes.c_size_t()\n"
        "_lib.call('ig_attend_scratch', B, Hg, d, cap, ctypes.byref(pf), ctypes.byref(tk), kernels=0)\n"
        "part = torch.empty(pf.value, device='cuda'); tick = torch.zeros(tk.value, dtype=torch.int32, device='cuda')\n"
        "out = torch.empty(B, Hg * d, device='cuda')\n"
        "ld = q.stride(0); Hgd = Hg * d\n"
        "_lib.call('ig_attend_slots', q.data_ptr(), ld, q.data_ptr() + 4 * Hgd, q.data_ptr() + 8 * Hgd, ld, stage.data_ptr(), 1, slot.data_ptr(), used.data_ptr(), pos.data_ptr(), st.data_ptr(), B, Hg, d, cap, part.data_ptr(), tick.data_ptr(), out.data_ptr(), Hgd, _lib.stream_handle())\n"
        "np.save(sys.argv[1], out.cpu().numpy())\n")
    res = {}
    with tempfile.TemporaryDirectory() as td:
        for name, e in (("default", {}), ("variant", env)):
            f = os.path.join(td, name + ".npy")
            e = dict(e, IG_ATTEND_IMPL="mma")          # the warp-persistent mma.sync kernel
            r = subprocess.run([sys.executable, "-c", code, f], env=dict(os.environ, **e),
                               capture_output=True, text=True, timeout=300)
            assert r.returncode == 0, r.stderr[-2000:]
            res[name] = np.load(f)
    if "IG_WP_RING" in env:
        np.testing.assert_array_equal(res["variant"], res["default"])
    else:
        np.testing.assert_allclose(res["variant"], res["default"], rtol=1e-5, atol=1e-6)


_LONG_ROWS_CODE = """
import sys, ctypes, numpy as np, torch
from paper_2406_19707_b200 import _lib
elt = sys.argv[2]
B, Hg, d, cap = 2, 3, 128, 4100
g = torch.Generator(device="cuda"); g.manual_seed(21)
T = torch.float16 if elt == "f16" else torch.bfloat16
q = torch.randn(B, 3 * Hg * d, device="cuda", generator=g)
stage = torch.full((B, Hg, cap, 2 * d), float("nan"), device="cuda").to(T)
used = torch.tensor([[4100, 2049, 0], [3000, 129, 4096]], dtype=torch.int32, device="cuda")
for b in range(B):
    for h in range(Hg):
        n = int(used[b, h])
        stage[b, h, :n] = (2 * torch.randn(n, 2 * d, device="cuda", generator=g)).to(T)
slot = torch.arange(cap, device="cuda", dtype=torch.int32).repeat(B, Hg, 1).contiguous()
slot[:, :, 3::11] = -1
pos = torch.full((B, Hg), 7, dtype=torch.int32, device="cuda")
st = torch.zeros(8, dtype=torch.int32, device="cuda")
pf, tk = ctypes.c_size_t(), ctypes.c_size_t()
_lib.call("ig_attend_scratch", B, Hg, d, cap, ctypes.byref(pf), ctypes.byref(tk), kernels=0)
part = torch.empty(pf.value, device="cuda")
tick = torch.zeros(tk.value, dtype=torch.int32, device="cuda")
outs = []
for _ in range(2):
    out = torch.empty(B, Hg * d, device="cuda")
    _lib.call("ig_attend_slots", q.data_ptr(), 3 * Hg * d, q.data_ptr() + 4 * Hg * d, q.data_ptr() + 8 * Hg * d,
              3 * Hg * d, stage.data_ptr(), _lib.ELT[elt], slot.data_ptr(), used.data_ptr(), pos.data_ptr(),
              st.data_ptr(), B, Hg, d, cap, part.data_ptr(), tick.data_ptr(), out.data_ptr(), Hg * d,
              _lib.stream_handle())
    outs.append(out.cpu().numpy())
assert not tick.any()
np.savez(sys.argv[1], o0=outs[0], o1=outs[1], q=q.double().cpu().numpy(), stage=stage.double().cpu().numpy(),
         used=used.cpu().numpy(), slot=slot.cpu().numpy())
"""


@pytest.mark.parametrize("impl", ["c", "mma"])
@pytest.mark.parametrize("elt", ["f16", "bf16"])
def test_attend_long_rows_vs_float64(elt, impl):
    """Long slot tables (4K rows per (b, h)) through the tcgen05 attention
    (IG_ATTEND_IMPL=c: csrc/attend_tc05.cu -- (b, h) row sets split over
    several CTAs with partial slots + ticket merges) and the default mma.sync
    kernel: an empty set (output = the current row's v), excluded rows (empty
    slots, pos), NaN rows past each count; tickets left zeroed, bit-identical
    on repeat, vs float64."""
    import os
    import subprocess
    import sys
    import tempfile
    f = os.path.join(tempfile.mkdtemp(), "o.npz")
    r = subprocess.run([sys.executable, "-c", _LONG_ROWS_CODE, f, elt], env=dict(os.environ, IG_ATTEND_IMPL=impl),
                       capture_output=True, text=True, timeout=300,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0, r.stderr[-2000:]
    z = np.load(f)
    np.testing.assert_array_equal(z["o0"], z["o1"])        # deterministic merges
    B, Hg, d = 2, 3, 128
    qn, stg, used, slot = z["q"], z["stage"], z["used"], z["slot"]
    for b in range(B):
        for h in range(Hg):
            n = int(used[b, h])
            rows = [i for i in range(n) if int(slot[b, h, i]) >= 0 and int(slot[b, h, i]) != 7]
            K = np.concatenate([stg[b, h, rows, :d], qn[b, Hg * d + h * d:Hg * d + (h + 1) * d][None]])
            V = np.concatenate([stg[b, h, rows, d:], qn[b, 2 * Hg * d + h * d:2 * Hg * d + (h + 1) * d][None]])
            lg = K @ qn[b, h * d:(h + 1) * d] / np.sqrt(d)
            w = np.exp(lg - lg.max())
            np.testing.assert_allclose(z["o0"][b, h * d:(h + 1) * d], (w / w.sum()) @ V, rtol=2e-5, atol=2e-5,
                                       err_msg=f"b{b} h{h} n{n}")
