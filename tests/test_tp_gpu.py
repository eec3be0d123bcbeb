"""Head tensor parallelism of the engine, end to end on one GPU: two ranks
(gloo, which handles CUDA tensors) each own H/2 heads, their pool shard and
partial keys; the per-layer head-count sums and W_O outputs are all-reduced.
Outputs must match the unsharded oracle and each rank's selections must be
the oracle's for its heads (NCCL replaces gloo on a multi-GPU box; the
engine code path is the same)."""

import copy
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, q, ffn=None):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import speckv_port as O
        from tests.golden_cfg import MODELS, models, run_config
        from tests.test_engine_gpu import engine_cfg, oracle_sessions, oracle_decode
        from paper_2406_19707_b200 import DecodeEngine
        torch.cuda.set_device(0)
        if ffn is None:
            _, sk = models("m64")
        else:       # an FFN width that does not shard (replicated FFN, one all-reduce per layer)
            import dataclasses
            sk = O.skew_model(O.generate_synthetic(dataclasses.replace(MODELS["m64"], ffn_dim=ffn)),
                              calib_seed=0)
        for rname in ("spec", "spec_counter"):
            ocfg = run_config(rname, record_selection=True)
            sessions = oracle_sessions(sk, ocfg)
            eng = DecodeEngine.from_sessions(sk, engine_cfg(ocfg), copy.deepcopy(sessions),
                                             pool_dtype="f32", group=dist.group.WORLD)
            ref_out, ref_recs = oracle_decode(sessions, ocfg.gen_len)
            got = np.stack([eng.x.cpu().numpy()] + [eng.decode_step().cpu().numpy()
                                                    for _ in range(ocfg.gen_len)], axis=1)
            err = float(np.abs(got - ref_out).max() / max(1.0, np.abs(ref_out).max()))
            mism = 0
            for it, per_b in enumerate(eng.records):
                for b in range(ocfg.batch):
                    for li, r in enumerate(per_b[b]):
                        rr = ref_recs[b][it][li]
                        mism += r["n_selected"] != rr["n_selected"]
                        for hl, sel in enumerate(r["selected"]):
                            mism += set(sel) != set(rr["selected"][eng.h0 + hl])
            peer = eng.peer_ar is not None
            eng.close()
            q.put((rank, rname, err, mism, (eng.Hg, peer, eng.Fg == eng.F)))
    except Exception as e:  # surface the failure to the parent
        q.put((rank, "error", repr(e), -1, 0))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,peer,ffn", [(2, "1", None), (2, "0", None), (4, "1", None),
                                            (2, "1", 260), (4, "1", 260)])
def test_head_parallel_matches_oracle(world, peer, ffn, monkeypatch):
    """peer = 1 (default): the W_O / FFN-out all-reduces run over peer memory
    (ig_allreduce_peer, buffers mapped by CUDA IPC between the processes);
    peer = 0: through the process group (gloo here, NCCL on a multi-GPU box).
    world = 4 (one head per rank) exercises the G > 2 flag / slot logic;
    ffn = 260 does not split into 16-B shards, so the FFN is replicated and
    the step has one output all-reduce per layer (dense call numbering)."""
    monkeypatch.setenv("IG_PEER_AR", peer)
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 31000 + int.from_bytes(os.urandom(2), "little") % 2000
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, ffn)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=900) for _ in range(2 * world)]
    for p in procs:
        p.join(timeout=120)
    for rank, rname, err, mism, info in res:
        assert rname != "error", err
        assert info == (4 // world, peer == "1", ffn is not None)
        assert err < 1e-4, (rank, rname, err)
        assert mism == 0, (rank, rname, mism)


def _nccl_graph_worker(port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        from tests.golden_cfg import models, run_config
        from tests.test_engine_gpu import engine_cfg, oracle_sessions
        from paper_2406_19707_b200 import DecodeEngine
        _, sk = models("m64")
        ocfg = run_config("spec_counter", gen_len=6)
        sessions = oracle_sessions(sk, ocfg)
        outs = {}
        for name, kw in (("eager", dict(group=dist.group.WORLD)),
                         ("graph", dict(group=dist.group.WORLD, cuda_graph=True)),
                         ("plain", {})):
            eng = DecodeEngine.from_sessions(sk, engine_cfg(ocfg, record_selection=False),
                                             copy.deepcopy(sessions), pool_dtype="f32", **kw)
            outs[name] = np.stack([eng.decode_step().cpu().numpy().copy()
                                   for _ in range(ocfg.gen_len)])
            eng.close()
        q.put(("ok", outs))
    except Exception as e:  # surface the failure to the parent
        q.put(("error", repr(e)))
    finally:
        dist.destroy_process_group()


def test_nccl_group_graph_capture_matches_eager():
    """The N > 1 code path (NCCL all-reduces of the head-count sums on the
    speculation stream and of the W_O / FFN-out partials on the compute stream)
    captured into a CUDA graph and replayed: on a one-rank NCCL group (the only
    NCCL group one GPU can host) the replayed steps equal the eager steps of the
    same group and of the group-less engine bit for bit."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_graph_worker, args=(port, q))
    p.start()
    status, res = q.get(timeout=600)
    p.join(timeout=120)
    assert status == "ok", res
    np.testing.assert_array_equal(res["graph"], res["eager"])
    np.testing.assert_array_equal(res["eager"], res["plain"])


def _peer_ar_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2406_19707_b200.engine import PeerAllReduce
        n = 4 * 1024 + 12
        ar = PeerAllReduce(n, dist.group.WORLD, torch.device("cuda", 0))
        st = torch.zeros(8, dtype=torch.int32, device="cuda")
        outs = []
        for step in range(3):                    # epochs from the device step counter
            st[4] = step                         # ig_step_state.step (int32 at byte 16)
            for call in range(4):
                g = torch.Generator(device="cuda")
                g.manual_seed(1000 * step + 10 * call + rank)
                src = torch.randn(n, device="cuda", generator=g)
                res = torch.full((n,), float(call), device="cuda")
                out = torch.empty(n, device="cuda")
                ar(src, out, res if call % 2 else None, st, call, 4, torch.cuda.current_stream().cuda_stream)
                outs.append(out.cpu().numpy())
        ar.close()
        q.put((rank, outs))
    except Exception as e:  # surface the failure to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_peer_allreduce_sums_in_rank_order():
    """ig_allreduce_peer between two processes (IPC-mapped buffers on one GPU):
    out = p0 + p1 (+ residual) bit-identical on both ranks, across calls whose
    slots alternate by parity and epochs that come from the device step
    counter; ragged n (not a multiple of the grid)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 33000 + int.from_bytes(os.urandom(2), "little") % 2000
    procs = [ctx.Process(target=_peer_ar_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
    assert not isinstance(res[0], str), res[0]
    assert not isinstance(res[1], str), res[1]
    n = 4 * 1024 + 12
    k = 0
    for step in range(3):
        for call in range(4):
            parts = []
            for r in range(2):
                g = torch.Generator(device="cuda")
                g.manual_seed(1000 * step + 10 * call + r)
                parts.append(torch.randn(n, device="cuda", generator=g).cpu().numpy())
            exp = parts[0] + parts[1]
            if call % 2:
                exp = exp + np.float32(call)
            np.testing.assert_array_equal(res[0][k], exp)
            np.testing.assert_array_equal(res[1][k], res[0][k])
            k += 1


def _graph_peer_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from tests.golden_cfg import models, run_config
        from tests.test_engine_gpu import engine_cfg, oracle_sessions, oracle_decode
        from paper_2406_19707_b200 import DecodeEngine
        _, sk = models("m64")
        ocfg = run_config("spec_counter", gen_len=6)
        sessions = oracle_sessions(sk, ocfg)
        ref_out, _ = oracle_decode(copy.deepcopy(sessions), ocfg.gen_len)
        outs = {}
        for graph in (False, True):
            eng = DecodeEngine.from_sessions(sk, engine_cfg(ocfg, record_selection=False),
                                             copy.deepcopy(sessions), pool_dtype="f32",
                                             group=dist.group.WORLD, cuda_graph=graph)
            assert eng.peer_ar is not None and eng.peer_cnt is not None
            outs[graph] = np.stack([eng.decode_step().cpu().numpy().copy()
                                    for _ in range(ocfg.gen_len)], axis=1)
            eng.close()
        err = float(np.abs(outs[True] - ref_out[:, 1:]).max() / max(1.0, np.abs(ref_out).max()))
        q.put((rank, bool((outs[True] == outs[False]).all()), err))
    except Exception as e:  # surface the failure to the parent
        q.put((rank, repr(e), -1.0))
    finally:
        dist.destroy_process_group()


def test_two_rank_graph_replay_over_peer_memory():
    """With every collective of the step on peer memory (head-count sums and
    W_O / FFN-out partials), the two-rank head-parallel step is captured into a
    CUDA graph even over gloo: replayed steps equal eager steps bit for bit and
    stay within 1e-4 of the unsharded oracle."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 35000 + int.from_bytes(os.urandom(2), "little") % 2000
    procs = [ctx.Process(target=_graph_peer_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
    for rank, same, err in res:
        assert same is True, (rank, same)
        assert err < 1e-4, (rank, err)
