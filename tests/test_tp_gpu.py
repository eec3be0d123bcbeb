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


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import speckv_port as O
        from tests.golden_cfg import models, run_config
        from tests.test_engine_gpu import engine_cfg, oracle_sessions, oracle_decode
        from paper_2406_19707_b200 import DecodeEngine
        torch.cuda.set_device(0)
        _, sk = models("m64")
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
            eng.close()
            q.put((rank, rname, err, mism, eng.Hg))
    except Exception as e:  # surface the failure to the parent
        q.put((rank, "error", repr(e), -1, 0))
    finally:
        dist.destroy_process_group()


def test_two_rank_head_parallel_matches_oracle():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 31000 + int.from_bytes(os.urandom(2), "little") % 2000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(4)]
    for p in procs:
        p.join(timeout=120)
    for rank, rname, err, mism, hg in res:
        assert rname != "error", err
        assert hg == 2
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
