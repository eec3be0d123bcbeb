"""Full-size parity (BASELINE.json configs C2-C5, one layer each) through
size-independent properties -- the CPU oracle cannot run these sizes, so each
kernel's output is checked against the rule it implements, on the GPU's own
inputs:

* ig_rehearse_count: scores vs a float64 recomputation (rtol 1e-5); counts are
  exactly #(score > float32(max - alpha)) of the GPU scores (speculation.py:156-157);
* ig_select: n is exactly the reference formula (speculation.py:158-161); the
  rows are ascending, unique, < s, and equal to the stable top-n of the GPU scores
  (linalg.py:184) -- bit-exact;
* ig_fetch: every staged row equals the host-pool row it names (bit-exact);
* ig_attend: vs float64 attention over the same rows + the current row;
* ig_append: the new row lands at s (or the policy victim at the limit), partial-K
  mirror, metadata, and the fetch-metadata update (pool.py:53-99).
"""

import ctypes
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

# (name, B, Hg, s): C2 OPT-6.7B B8 2K; C3 OPT-13B B16 4K; C4 Llama-2-7B B4 32K;
# C5 OPT-30B B32 8K as the rank-0 shard of 8 GPUs (56 heads / 8 = 7)
CONFIGS = [("C2", 8, 32, 2048 + 7), ("C3", 16, 40, 4096 + 3), ("C4", 4, 32, 32768 + 1),
           ("C5_rank0_of_8", 32, 7, 8192 + 5)]
D_HEAD, KCOLS, ALPHA, CAP_RATIO = 128, 39, 4.0, 0.2


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2406_19707_b200 import _lib
    _lib.load()


@pytest.mark.parametrize("name,B,Hg,s", CONFIGS)
def test_layer_pipeline_full_size(name, B, Hg, s):
    import torch
    from paper_2406_19707_b200 import _lib
    from paper_2406_19707_b200.engine import HostPool
    dev = torch.device("cuda")
    g = torch.Generator(device=dev)
    g.manual_seed(sum(map(ord, name)))
    d, k = D_HEAD, KCOLS
    S = (s + 1 + 3) // 4 * 4                      # room for the append at row s
    H_total = Hg * (8 if name.startswith("C5") else 1)
    hs = _lib.stream_handle()
    row_bytes = 2 * d * 2
    # ---- inputs: outlier-ish partial keys so the alpha rule selects a realistic n
    qspec = torch.randn(B, Hg * d, device=dev, generator=g)
    pk = torch.randn(B, Hg, k, S, device=dev, generator=g)
    pk[:, :, :4] *= 4.0
    cols = torch.sort(torch.rand(B, Hg, d, device=dev, generator=g).argsort(-1)[..., :k], -1).values.int().contiguous()
    st = torch.zeros(8, dtype=torch.int32, device=dev)
    st[0] = s
    # ---- K1+K2a
    scores = torch.empty(B, Hg, S, device=dev)
    counts = torch.zeros(B, Hg, dtype=torch.int32, device=dev)
    csum = torch.zeros(B, dtype=torch.int32, device=dev)
    mk = torch.zeros((B, Hg), dtype=torch.int32, device=dev)
    tk0 = torch.zeros((B, Hg), dtype=torch.int32, device=dev)
    scale = float(np.float32(1.0 / np.sqrt(d)))
    rr = torch.zeros((B, Hg, 2), dtype=torch.int32, device=dev)
    _lib.call("ig_rehearse_count", qspec.data_ptr(), Hg * d, cols.data_ptr(), pk.data_ptr(),
              st.data_ptr(), B, Hg, d, k, S, scale, ALPHA, scores.data_ptr(), mk.data_ptr(),
              tk0.data_ptr(), counts.data_ptr(), csum.data_ptr(), rr.data_ptr(), hs)
    assert not mk.any() and not tk0.any()      # scratch left zeroed
    qsel = torch.gather(qspec.view(B, Hg, d).double(), 2, cols.long())           # [B, Hg, k]
    ref = torch.einsum("bhj,bhjt->bht", qsel, pk[..., :s].double()) * scale
    sc = scores[..., :s]
    torch.testing.assert_close(sc.double(), ref, rtol=1e-5, atol=1e-5)
    sc_np = sc.cpu().numpy()
    cnt = counts.cpu().numpy()
    for b in range(B):
        for h in range(Hg):
            v = sc_np[b, h]
            assert cnt[b, h] == int(np.sum(v > np.float32(float(v.max()) - ALPHA)))
    # ---- K2b (single GPU: H_total = Hg except the C5 shard, whose sum we scale up)
    if H_total != Hg:
        csum.mul_(H_total // Hg)
    cap = max(int(math.floor(CAP_RATIO * S)), 1)
    idx = torch.zeros(B, Hg, cap, dtype=torch.int32, device=dev)
    n = torch.zeros(B, dtype=torch.int32, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    # with the rehearsal's row ranges, and computing them itself: identical
    idx2 = torch.full_like(idx, -7)
    n2 = torch.zeros_like(n)
    _lib.call("ig_select", scores.data_ptr(), csum.data_ptr(), st.data_ptr(), B, Hg, H_total, S,
              cap, CAP_RATIO, 1, idx.data_ptr(), n.data_ptr(), err.data_ptr(), rr.data_ptr(), hs)
    _lib.call("ig_select", scores.data_ptr(), csum.data_ptr(), st.data_ptr(), B, Hg, H_total, S,
              cap, CAP_RATIO, 1, idx2.data_ptr(), n2.data_ptr(), err.data_ptr(), None, hs)
    assert torch.equal(n, n2)
    for b in range(B):
        assert torch.equal(idx[b, :, :int(n[b])], idx2[b, :, :int(n[b])])
    n_np, idx_np, cs = n.cpu().numpy(), idx.cpu().numpy(), csum.cpu().numpy()
    assert int(err.item()) == 0
    for b in range(B):
        nn = int(math.floor(int(cs[b]) / H_total + 0.5))
        nn = min(min(max(nn, 1), max(int(math.floor(CAP_RATIO * s)), 1)), s)
        assert n_np[b] == nn, (b, n_np[b], nn)
        for h in range(Hg):
            got = idx_np[b, h, :nn]
            assert np.all(np.diff(got) > 0) and got[0] >= 0 and got[-1] < s
            want = np.sort(np.argsort(-sc_np[b, h], kind="stable")[:nn])
            np.testing.assert_array_equal(got, want)
    # ---- K3: host pool (one layer) with random rows, gather, compare bit-exact
    pool = HostPool(B * Hg * S * row_bytes)
    try:
        rows_dev = (torch.randn(B, Hg, S, 2 * d, device=dev, generator=g) * 2).half()
        _lib.call("ig_memcpy2d", pool.host, rows_dev.numel() * 2, rows_dev.data_ptr(),
                  rows_dev.numel() * 2, rows_dev.numel() * 2, 1, hs, kernels=0)
        stage = torch.empty(B, Hg, cap, 2 * d, dtype=torch.float16, device=dev)
        _lib.call("ig_fetch", pool.dev, idx.data_ptr(), n.data_ptr(), B, Hg, S, cap, row_bytes,
                  stage.data_ptr(), 32, 1024, hs)
        stage_tma = torch.empty_like(stage)
        _lib.call("ig_fetch_tma", pool.dev, idx.data_ptr(), n.data_ptr(), None, B, Hg, S, cap,
                  row_bytes, stage_tma.data_ptr(), 16, 1, 32, hs)
        stage_tma2 = torch.empty_like(stage)
        _lib.call("ig_fetch_tma", pool.dev, idx.data_ptr(), n.data_ptr(), None, B, Hg, S, cap,
                  row_bytes, stage_tma2.data_ptr(), 40, 2, 7, hs)
        full = torch.empty(B, Hg, S, 2 * d, dtype=torch.float16, device=dev)   # identity mode
        _lib.call("ig_fetch_tma", pool.dev, None, None, st.data_ptr(), B, Hg, S, S, row_bytes,
                  full.data_ptr(), 32, 1, 16, hs)
        assert torch.equal(full[:, :, :s], rows_dev[:, :, :s])
        for b in range(B):
            nn = int(n_np[b])
            want = torch.gather(rows_dev[b], 1, idx[b, :, :nn].long()[..., None].expand(Hg, nn, 2 * d))
            assert torch.equal(stage[b, :, :nn], want)
            assert torch.equal(stage_tma[b, :, :nn], want)
            assert torch.equal(stage_tma2[b, :, :nn], want)
        # ---- K4: attention over the fetched rows + the current row
        kv_cur = torch.randn(B, 3 * Hg * d, device=dev, generator=g)
        q, kc, vc = (kv_cur[:, i * Hg * d:(i + 1) * Hg * d] for i in range(3))
        pos = torch.full((B, Hg), s, dtype=torch.int32, device=dev)   # no limit: new row at s
        pf, tk = ctypes.c_size_t(), ctypes.c_size_t()
        _lib.call("ig_attend_scratch", B, Hg, d, cap, ctypes.byref(pf), ctypes.byref(tk), kernels=0)
        part = torch.empty(pf.value, device=dev)
        tick = torch.zeros(tk.value, dtype=torch.int32, device=dev)
        out = torch.empty(B, Hg * d, device=dev)
        _lib.call("ig_attend", kv_cur.data_ptr(), 3 * Hg * d, kv_cur.data_ptr() + 4 * Hg * d,
                  kv_cur.data_ptr() + 8 * Hg * d, 3 * Hg * d, stage.data_ptr(), _lib.ELT["f16"],
                  idx.data_ptr(), n.data_ptr(), pos.data_ptr(), st.data_ptr(), B, Hg, d, cap,
                  part.data_ptr(), tick.data_ptr(), out.data_ptr(), Hg * d, hs)
        for b in range(0, B, max(1, B // 4)):
            nn = int(n_np[b])
            Kr = torch.cat([stage[b, :, :nn, :d].double(), kc[b].view(Hg, 1, d).double()], 1)
            Vr = torch.cat([stage[b, :, :nn, d:].double(), vc[b].view(Hg, 1, d).double()], 1)
            lg = torch.einsum("hd,hnd->hn", q[b].view(Hg, d).double(), Kr) / math.sqrt(d)
            o = torch.einsum("hn,hnd->hd", torch.softmax(lg, -1), Vr)
            torch.testing.assert_close(out[b].view(Hg, d).double(), o, rtol=1e-4, atol=1e-4)
        # ---- K5: append + partial-K mirror + fetch metadata (no limit: row s)
        arrival = torch.zeros(B, Hg, S, dtype=torch.int64, device=dev)
        arrival[..., :s] = torch.arange(1, s + 1, device=dev)
        lastf = arrival.clone()
        ctr = torch.randint(0, 255, (B, Hg, S), dtype=torch.uint8, device=dev, generator=g)
        ctr_before = ctr.clone()
        st[2] = s      # seq (low word): s prior appends
        pos_out = torch.zeros(B, Hg, dtype=torch.int32, device=dev)
        events = torch.zeros(B, Hg, 2, dtype=torch.int64, device=dev)
        _lib.call("ig_append", kc.data_ptr(), vc.data_ptr(), 3 * Hg * d, pool.dev, _lib.ELT["f16"],
                  pk.data_ptr(), cols.data_ptr(), k, arrival.data_ptr(), lastf.data_ptr(),
                  ctr.data_ptr(), _lib.POLICY["counter"], 2, idx.data_ptr(), n.data_ptr(), cap,
                  st.data_ptr(), B, Hg, d, S, pos_out.data_ptr(), events.data_ptr(), hs)
        torch.cuda.synchronize()
        assert torch.all(pos_out == s) and torch.all(events[..., 0] == -1)
        host = np.frombuffer((ctypes.c_uint8 * pool.nbytes).from_address(pool.host),
                             dtype=np.float16).reshape(B, Hg, S, 2 * d)
        np.testing.assert_array_equal(host[:, :, s, :d], kc.view(B, Hg, d).half().cpu().numpy())
        np.testing.assert_array_equal(host[:, :, s, d:], vc.view(B, Hg, d).half().cpu().numpy())
        kcur = kc.view(B, Hg, d)
        assert torch.equal(pk[..., s], torch.gather(kcur, 2, cols.long()))
        assert torch.all(arrival[..., s] == s + 1)
        assert torch.all(lastf[..., s] == s + 2)       # the new row is in the fetch set
        # fetch-metadata rule on the selected rows (saturate at 255, halve all on a hit)
        c0, c1 = ctr_before.cpu().numpy(), ctr.cpu().numpy()
        for b in range(0, B, max(1, B // 4)):
            for h in range(Hg):
                exp = c0[b, h, :s + 1].astype(np.int64)
                exp[s] = 0
                sel = list(idx_np[b, h, :n_np[b]]) + [s]
                exp[sel] = np.minimum(exp[sel] + 1, 255)
                if np.any(exp[sel] == 255):
                    exp //= 2
                np.testing.assert_array_equal(c1[b, h, :s + 1], exp)
    finally:
        pool.close()


@pytest.mark.parametrize("policy", ["fifo", "lru", "counter"])
def test_eviction_at_full_size(policy):
    """C3-sized pools at their limit: ig_append's victim is np.argmin of the
    policy key (lowest index on ties), its old arrival is reported, and the row
    is overwritten in place (pool.py:74-81)."""
    import torch
    from paper_2406_19707_b200 import _lib
    from paper_2406_19707_b200.engine import HostPool
    dev = torch.device("cuda")
    g = torch.Generator(device=dev)
    g.manual_seed(7)
    B, Hg, d, s = 16, 40, 128, 4096
    S = s
    hs = _lib.stream_handle()
    arrival = torch.randperm(10 * s, device=dev, generator=g)[:s].repeat(B, Hg, 1).contiguous()
    lastf = torch.randint(0, 50, (B, Hg, S), device=dev, generator=g)   # many ties
    ctr = torch.randint(0, 4, (B, Hg, S), dtype=torch.uint8, device=dev, generator=g)
    st = torch.zeros(8, dtype=torch.int32, device=dev)
    st[0], st[1] = s, s          # at the limit
    kv = torch.randn(B, 2 * Hg * d, device=dev, generator=g)
    pool = HostPool(B * Hg * S * 2 * d * 2)
    try:
        keys = {"fifo": arrival, "lru": lastf, "counter": ctr.long()}[policy].cpu().numpy()
        old_arrival = arrival.cpu().numpy()
        pos = torch.zeros(B, Hg, dtype=torch.int32, device=dev)
        ev = torch.zeros(B, Hg, 2, dtype=torch.int64, device=dev)
        _lib.call("ig_append", kv.data_ptr(), kv.data_ptr() + 4 * Hg * d, 2 * Hg * d, pool.dev,
                  _lib.ELT["f16"], None, None, 1, arrival.data_ptr(), lastf.data_ptr(),
                  ctr.data_ptr(), _lib.POLICY[policy], 0, None, None, 1, st.data_ptr(), B, Hg, d,
                  S, pos.data_ptr(), ev.data_ptr(), hs)
        p, e = pos.cpu().numpy(), ev.cpu().numpy()
        want = keys.argmin(axis=-1)
        np.testing.assert_array_equal(p, want)
        np.testing.assert_array_equal(e[..., 0], want)
        np.testing.assert_array_equal(e[..., 1], np.take_along_axis(old_arrival, want[..., None], -1)[..., 0])
        ar = arrival.cpu().numpy()
        assert np.all(np.take_along_axis(ar, want[..., None], -1) == 1)   # seq 0 + 1
    finally:
        pool.close()
