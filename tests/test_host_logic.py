"""Host-side logic of the engine (CPU): pool sizing, prefill row placement,
head sharding and the two per-layer reductions of tensor parallelism
(world_size-2 gloo), checked against the oracle."""

import math
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import speckv_port as O


@pytest.mark.parametrize("policy", ["fifo", "lru", "counter"])
@pytest.mark.parametrize("n,limit", [(10, None), (10, 10), (10, 4), (33, 7), (5, 1)])
def test_prefill_row_simulation_matches_pool(policy, n, limit):
    from paper_2406_19707_b200.engine import _simulate_prefill_rows
    from paper_2406_19707_b200.pool import EvictionPolicy
    row_of, arr, lf, ct, ovw = _simulate_prefill_rows(n, limit, EvictionPolicy(policy))
    p = O.Pool(2, limit=limit, policy=O.Policy(policy))
    rows = [p.append(np.full(2, t, np.float32), np.zeros(2, np.float32)) for t in range(n)]
    assert list(row_of) == rows
    np.testing.assert_array_equal(arr, p.arrival_seq)
    np.testing.assert_array_equal(lf, p.last_fetch_seq)
    np.testing.assert_array_equal(ct, p.fetch_counter)
    assert ovw == max(0, n - (limit or n))


def test_selection_cap_bounds_every_step():
    """The index buffer (cap rows) holds n for every s <= S_max."""
    for ratio in (0.05, 0.2, 0.5, 1.0):
        for mins in (1, 3):
            for S in (4, 17, 2048, 4100):
                cap = max(int(math.floor(ratio * S)), mins, 1)
                for s in range(1, S + 1, max(1, S // 50)):
                    n_max = min(max(int(math.floor(ratio * s)), mins), s)
                    assert n_max <= cap


def test_integer_rounding_of_shared_n():
    """floor(sum/H + 0.5) in float64 == (2*sum + H) // (2*H) (the kernel form)."""
    rng = np.random.default_rng(0)
    for _ in range(20000):
        H = int(rng.integers(1, 128))
        total = int(rng.integers(0, 40000 * H))
        assert math.floor(total / H + 0.5) == (2 * total + H) // (2 * H)


def test_threshold_cast_matches_numpy_weak_scalar():
    """count uses float32(double(max) - alpha): NumPy 2 casts the Python-float
    threshold to float32 before the compare (speculation.py:156-157)."""
    rng = np.random.default_rng(1)
    for _ in range(2000):
        v = (rng.standard_normal(64) * rng.choice([1e-3, 1, 1e4])).astype(np.float32)
        alpha = float(rng.choice([1e-7, 0.5, 4.0, 5.0, 3.999999]))
        mx = float(np.max(v))
        ref = int(np.sum(v > (mx - alpha)))
        thr32 = np.float32(mx - alpha)
        assert ref == int(np.sum(v > thr32))


def _tp_worker(rank, world, port, H, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(7)
        B, s, d, D = 3, 50, 8, H * 8
        scores = rng.standard_normal((B, H, s)).astype(np.float32) * 3
        heads = np.arange(H).reshape(world, -1)[rank]          # engine: h0 = rank * Hg
        cfg = O.SpeculationConfig(0.3, 2.0, 0.3, 1)
        # per-rank counts for its heads, then the B-int all-reduce (engine.py decode_step)
        local = torch.tensor([sum(int(np.sum(scores[b, h] > np.float32(float(scores[b, h].max()) - cfg.alpha)))
                                  for h in heads) for b in range(B)], dtype=torch.int32)
        dist.all_reduce(local)
        n_tp = [min(min(max((2 * int(local[b]) + H) // (2 * H), cfg.min_select),
                        max(int(math.floor(cfg.cap_ratio * s)), cfg.min_select)), s) for b in range(B)]
        n_ref = [O.select_tokens([scores[b, h] for h in range(H)], cfg)[1] for b in range(B)]
        # row-parallel W_O: sum over ranks of heads_r @ W_O[rows_r] == full product
        att = rng.standard_normal((B, H * d)).astype(np.float32)
        wo = rng.standard_normal((H * d, D)).astype(np.float32)
        r0, r1 = heads[0] * d, (heads[-1] + 1) * d
        part = torch.from_numpy(att[:, r0:r1] @ wo[r0:r1]).double()
        dist.all_reduce(part)
        full = att.astype(np.float64) @ wo.astype(np.float64)
        q.put((rank, n_tp == n_ref, float(np.abs(part.numpy() - full).max())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("H", [4, 6])
def test_head_sharding_two_ranks_gloo(H):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + int.from_bytes(os.urandom(2), "little") % 2000
    procs = [ctx.Process(target=_tp_worker, args=(r, 2, port, H, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, n_ok, err in res:
        assert n_ok, rank
        assert err < 1e-2
