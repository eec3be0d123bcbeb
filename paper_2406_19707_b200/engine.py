"""B200 decode engine: the batched, stream-overlapped InfiniGen decode path.

Mirrors the reference inference controller (engine.py:199-477): the same
RunConfig fields, the same per-layer order as DecodeSession.decode_step
(engine.py:309-375), and a schema-v1 Trace (engine.py:83-196).  Differences
are in HOW, not WHAT:

  * all B sequences advance together (the reference loops over them,
    engine.py:468-476); every hot op is one launch over (b, h);
  * the KV pool is one pinned host allocation T[L][B][Hg][S_max][2][d]
    (fp16 by default: the reference's 2-byte accounting, engine.py:63) and
    its metadata lives in HBM;
  * three CUDA streams: the compute stream runs LN / QKV (+ the next layer's
    speculation query) / append / attention / W_O / FFN, the speculation
    stream runs layer i+1's rehearse -> select -> resident plan while layer i
    computes, the fetch stream moves the rows that entered a selection from
    the host pool into the HBM slot tables (the overlap the reference models
    analytically in costmodel.py:102-139); one step replays as a CUDA graph;
  * with tensor parallelism over heads (and Megatron-style FFN columns), each
    rank owns H/G heads, their pools and partial keys; per layer it all-reduces
    the B head-count sums (n averages over ALL heads, speculation.py:154-158)
    and the W_O / FFN-out outputs over peer memory.

Hot ops are the library kernels (ig_rehearse_count, ig_select,
ig_resident_plan, ig_fetch_slots, ig_append, ig_attend_slots, ig_layernorm);
the dense projections are ig_sgemm_packed over weights packed once (f16 hi/lo,
f32-accurate tensor-core GEMMs), the prefill's on ig_gemm_tc05 (tcgen05).
No CPU fallback exists.
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .prefill import causal_attention, layernorm, partial_columns
from .speculation import SpeculationConfig, selection_bytes
from .pool import EvictionPolicy

TRACE_SCHEMA_VERSION = 1
PACKED_MAX_M = 32          # rows per ig_sgemm_packed launch
_TORCH_ELT = {"f32": torch.float32, "f16": torch.float16, "bf16": torch.bfloat16}


@dataclass(frozen=True)
class RunConfig:
    """Reference RunConfig (engine.py:51-80) for the schemes on the path."""
    scheme: str = "speculative"            # "speculative" | "full"
    prompt_len: int = 32
    gen_len: int = 8
    batch: int = 1
    speculation: SpeculationConfig = field(default_factory=SpeculationConfig)
    pool_limit: int | None = None
    pool_policy: EvictionPolicy = EvictionPolicy.COUNTER
    prompt_seed: int = 0
    kv_bytes_per_element: int = 2
    record_scores: bool = False
    record_selection: bool = False

    def validate(self) -> None:
        if getattr(self.scheme, "value", self.scheme) not in ("speculative", "full"):
            raise ValueError(f"scheme {self.scheme!r} is not on the B200 path")
        if self.prompt_len < 1:
            raise ValueError("prompt_len must be >= 1")
        if self.gen_len < 0:
            raise ValueError("gen_len must be >= 0")
        if self.batch < 1:
            raise ValueError("batch must be >= 1")
        self.speculation.validate()
        if self.pool_limit is not None and self.pool_limit < 1:
            raise ValueError("pool_limit must be >= 1 when set")


def _f32(a, device):
    if isinstance(a, torch.Tensor):
        return a.to(device=device, dtype=torch.float32).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(device)


def _enable_ieee_fp32():
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    try:
        torch.backends.cuda.matmul.fp32_precision = "ieee"
    except (AttributeError, RuntimeError):
        pass


class _Weight:
    """One decode-step weight matrix [K, N] of this rank: its row-major f32 copy
    (dense="cublas") or its ig_sgemm_packed blocks
    (dense="packed": the row-major copy is dropped once packed)."""

    def __init__(self, rm: torch.Tensor | None, packed: bool, device, *, _shape=None):
        self.is_view = rm is None
        self.K, self.N = (rm.shape if rm is not None else _shape)
        self.rm = None if packed else rm
        self.packed = None
        if packed and rm is not None:
            K, N = rm.shape
            pf = ctypes.c_size_t()
            _lib.call("ig_sgemm_packed_sizes", 1, N, K, ctypes.byref(pf), None, None, kernels=0)
            self.packed = torch.empty(pf.value, dtype=torch.float32, device=device)
            _lib.call("ig_sgemm_pack", rm.data_ptr(), rm.stride(0), N, K, self.packed.data_ptr(),
                      torch.cuda.current_stream(device).cuda_stream, kernels=2)

    @property
    def shape(self):
        return (self.K, self.N)

    def narrow(self, n: int) -> "_Weight":
        """The first n columns (the q/k/v part of the fused [QKV | Q(li+1)]
        matrix): a row-major view; packed blocks are not sliceable."""
        w = _Weight(None, False, None, _shape=(self.K, n))
        w.rm = self.rm[:, :n] if self.rm is not None else None
        return w

    def nbytes(self) -> int:
        t = self.packed if self.packed is not None else self.rm
        return 0 if t is None else t.numel() * t.element_size()


class HostPool:
    """Pinned, mapped, portable host memory for the KV rows (ig_host_alloc: on
    the current GPU's NUMA node when the machine has several)."""

    def __init__(self, nbytes: int):
        host, dev = ctypes.c_void_p(), ctypes.c_void_p()
        _lib.call("ig_host_alloc", nbytes, ctypes.byref(host), ctypes.byref(dev), kernels=0)
        self.host, self.dev, self.nbytes = host.value, dev.value, nbytes
        node = ctypes.c_int(-1)
        _lib.call("ig_host_numa_node", self.host, ctypes.byref(node), kernels=0)
        self.numa_node = node.value

    def numpy(self, dtype, shape) -> np.ndarray:
        """Host view (no copy) -- inspection and tests."""
        buf = (ctypes.c_uint8 * self.nbytes).from_address(self.host)
        return np.frombuffer(buf, dtype=dtype).reshape(shape)

    def close(self) -> None:
        if self.host:
            _lib.call("ig_host_free", self.host, kernels=0)
            self.host = self.dev = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class PeerAllReduce:
    """The head-parallel output all-reduce over peer memory (csrc/collective.cu):
    every rank's receive buffer and flags are mapped into every other rank by
    CUDA IPC (handles exchanged once through the process group); one kernel per
    call pushes this rank's partial into every rank, waits for all of them and
    sums in rank order (+ residual).  Replaces the NCCL all-reduce of the W_O /
    FFN-out partials (engine.py:360-364).

    Calls must be numbered densely (seqno = step * calls + call, call in
    [0, calls)): the receive slots alternate by seqno parity, and a slot is
    safe to overwrite only because call c + 2 is pushed after the sum of c + 1.

    connect=False allocates locally only; peer_collectives() then exchanges the
    handles of several objects with one fixed sequence of collectives."""

    def __init__(self, n: int, group, device, dtype=torch.float32, connect: bool = True):
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        self.n, self.device = n, device
        self.fn = {torch.float32: "ig_allreduce_peer", torch.int32: "ig_allreduce_peer_i32"}[dtype]
        self.recv = self.flags = None
        self._opened = []
        recv, flags = ctypes.c_void_p(), ctypes.c_void_p()
        _lib.call("ig_peer_alloc", n, self.world, ctypes.byref(recv), ctypes.byref(flags), kernels=0)
        self.recv, self.flags = recv.value, flags.value
        self.ticket = self.flags + 4 * 2 * self.world
        try:
            hr, hf = (ctypes.c_char * 64)(), (ctypes.c_char * 64)()
            _lib.call("ig_ipc_get_handle", self.recv, hr, kernels=0)
            _lib.call("ig_ipc_get_handle", self.flags, hf, kernels=0)
            self.handles = (bytes(hr), bytes(hf))
            if connect:
                objs = [None] * self.world
                dist.all_gather_object(objs, self.handles, group=group)
                self.open(objs)
        except Exception:
            self.close()
            raise

    def open(self, handles) -> None:
        """Map every other rank's (recv, flags) pair; handles[r] from rank r."""
        pr, pf = [], []
        for r, (h_r, h_f) in enumerate(handles):
            if r == self.rank:
                pr.append(self.recv)
                pf.append(self.flags)
                continue
            for h, lst in ((h_r, pr), (h_f, pf)):
                ptr = ctypes.c_void_p()
                buf = (ctypes.c_char * 64).from_buffer_copy(h)
                _lib.call("ig_ipc_open_handle", buf, ctypes.byref(ptr), kernels=0)
                self._opened.append(ptr.value)
                lst.append(ptr.value)
        self.peer_recv = torch.tensor(pr, dtype=torch.int64, device=self.device)
        self.peer_flags = torch.tensor(pf, dtype=torch.int64, device=self.device)

    def __call__(self, src, out, residual, st, call: int, calls: int, stream: int) -> None:
        if self.fn == "ig_allreduce_peer_i32":
            _lib.call(self.fn, src.data_ptr(), self.n, self.peer_recv.data_ptr(),
                      self.peer_flags.data_ptr(), self.rank, self.world, st.data_ptr(), call, calls,
                      out.data_ptr(), self.ticket, stream)
            return
        _lib.call(self.fn, src.data_ptr(), self.n, self.peer_recv.data_ptr(),
                  self.peer_flags.data_ptr(), self.rank, self.world, st.data_ptr(), call, calls,
                  _lib.ptr(residual), out.data_ptr(), self.ticket, stream)

    def gemm_push(self, X, P, N: int, K: int, st, call: int, calls: int, ws, tickets, stream) -> None:
        """The packed GEMM whose epilogue pushes X . W into every rank's slot."""
        _lib.call("ig_sgemm_packed_peer", X.data_ptr(), X.stride(0), P.data_ptr(), N, K, X.shape[0],
                  self.peer_recv.data_ptr(), self.peer_flags.data_ptr(), self.rank, self.world,
                  st.data_ptr(), call, calls, self.ticket + 4, ws.data_ptr(), ws.numel(),
                  tickets.data_ptr(), tickets.numel(), stream)

    def sum(self, out, residual, st, call: int, calls: int, stream: int) -> None:
        """Wait for every rank's push of `call`; out = sum over ranks + residual."""
        _lib.call("ig_allreduce_peer_sum", self.n, self.peer_recv.data_ptr(),
                  self.peer_flags.data_ptr(), self.rank, self.world, st.data_ptr(), call, calls,
                  _lib.ptr(residual), out.data_ptr(), stream)

    def close(self) -> None:
        for p in getattr(self, "_opened", []):
            _lib.call("ig_ipc_close", p, kernels=0)
        self._opened = []
        if getattr(self, "recv", None):
            _lib.call("ig_peer_free", self.recv, self.flags, kernels=0)
            self.recv = self.flags = None


def _vote(ok: bool, group, device) -> bool:
    """True iff every rank of the group says ok (one all-reduce)."""
    t = torch.tensor([1 if ok else 0], dtype=torch.int32,
                     device=device if dist.get_backend(group) == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    return bool(int(t.item()))


def peer_collectives(specs, group, device):
    """PeerAllReduce objects for [(n, dtype), ...], or None on every rank if any
    rank cannot allocate, export or map them.  Every rank issues the same
    collectives whatever fails where (vote, gather, vote), so a local failure
    falls back instead of leaving the ranks in mismatched collectives."""
    import sys
    objs, ok = [], True
    try:
        for n, dt in specs:
            objs.append(PeerAllReduce(n, group, device, dt, connect=False))
    except Exception as e:  # noqa: BLE001 -- no IPC on this box
        sys.stderr.write(f"peer all-reduce: local setup failed ({e!r})\n")
        ok = False
    if _vote(ok, group, device):
        gathered = [None] * dist.get_world_size(group)
        dist.all_gather_object(gathered, [o.handles for o in objs], group=group)
        try:
            for i, o in enumerate(objs):
                o.open([g[i] for g in gathered])
        except Exception as e:  # noqa: BLE001 -- no peer mapping between these GPUs
            sys.stderr.write(f"peer all-reduce: mapping failed ({e!r})\n")
            ok = False
        if _vote(ok, group, device):
            return objs
    for o in objs:
        o.close()
    return None


def _simulate_prefill_rows(n: int, limit: int | None, policy: EvictionPolicy):
    """Row of each prompt token and the resulting metadata when N prompt rows
    are appended to an empty pool (engine.py:265-266 -> pool.py:53-81).  All
    pools see the same appends and no fetches during prefill, so one
    simulation serves every (layer, head, sequence)."""
    rows = min(n, limit) if limit else n
    arrival = np.zeros(rows, np.int64)
    lastf = np.zeros(rows, np.int64)
    ctr = np.zeros(rows, np.uint8)
    row_of = np.empty(n, np.int64)
    overwrites = 0
    for t in range(n):
        seq = t + 1
        if limit is None or t < limit:
            r = t
        else:
            key = {EvictionPolicy.FIFO: arrival, EvictionPolicy.LRU: lastf,
                   EvictionPolicy.COUNTER: ctr}[EvictionPolicy(policy)]
            r = int(np.argmin(key))
            overwrites += 1
        row_of[t] = r
        arrival[r] = lastf[r] = seq
        ctr[r] = 0
    return row_of, arrival, lastf, ctr, overwrites


class SelectionOverflowError(RuntimeError):
    """A selection larger than the engine's index buffer (flagged by ig_select)."""


def _jsonable(rec: dict) -> dict:
    """A layer record with array fields as lists (schema-v1 JSON)."""
    return {k: (v.tolist() if isinstance(v, np.ndarray) else v) for k, v in rec.items()}


_LAYER_POS = object()     # _attend default: the layer's ig_append positions


class DecodeEngine:
    """Batched InfiniGen decode on one GPU (or one head shard of a TP group).

    Parameters
    ----------
    model : object shaped like the reference Model (see model.py)
    config : RunConfig
    max_steps : decode steps to size the pool for (default config.gen_len)
    pool_dtype : "f16" (default, e = 2 bytes), "bf16" or "f32"
    group : torch.distributed process group for head tensor parallelism
    fetch_ctas, fetch_threads : gather grid (the rest of the GPU computes)
    fetch_priority : CUDA priority of the fetch stream (lower = more urgent),
        so gather CTAs win free SM slots over compute-stream CTAs
    fetch_impl : "tma" (default: bulk async copies through shared memory,
        fetch_threads/32 warps per CTA, fetch_rows rows per warp batch) or
        "ldg" (16-B vector loads through registers, fetch_threads per CTA).
        Defaults (32 CTAs x 1 warp x 16 rows) come from tools/sweep_fetch.sh on
        C2 and C3 (profiles/r01_fetch_sweep.md).
    hbm_layers : 0 (default: every layer's KV in the pinned host pool) or 1:
        keep layer 0's rows -- which every step reads in full (engine.py:393-396)
        -- resident in HBM, so they never cross the host link.  Traces keep the
        reference byte accounting; bench.py reports moved bytes separately.
    resident : (default: on for the speculative scheme without hbm_layers)
        keep each speculative layer's fetched set in HBM across steps
        (a slot table of at most `cap` rows per (layer, seq, head)) and fetch
        only the rows that enter the selection; layer 0's rows are mirrored in
        HBM and the appended row is written to the mirror in the same step.
        The host pool stays authoritative (every append still goes to it) and
        the attended rows, selections and traces are those of the default path
        (csrc/resident.cu).
    spec_stream : run layer l+1's speculation chain (rehearse -> [count all-reduce]
        -> select -> resident plan) on its own high-priority stream, overlapping
        layer l's append/attention/W_O/FFN (traces recorded with scores use the
        compute stream).
    append_stream : without a pool limit, run ig_append beside the attention on
        its own stream (the attention takes the append position from st.s_len).
        Measured neutral at C3 (803.9 vs 803.8 tok/s), so off by default.
    """

    def __init__(self, model, config: RunConfig, *, max_steps: int | None = None,
                 pool_dtype: str = "f16", device=None, group=None, fetch_ctas: int = 32,
                 fetch_threads: int = 32, fetch_priority: int = 0, hbm_layers: int = 0,
                 fetch_impl: str = "tma", fetch_rows: int = 16, dense: str = "packed",
                 cuda_graph: bool = False, resident: bool | None = None, spec_stream: bool = True,
                 append_stream: bool = False, shard: tuple[int, int] | None = None,
                 record_trace: bool = False):
        config.validate()
        _lib.load()
        _enable_ieee_fp32()
        scheme = getattr(config.scheme, "value", config.scheme)
        if scheme == "speculative" and not getattr(model, "skewed", False):
            raise ValueError("the speculative scheme requires a skewed model")
        spec = model.spec
        self.model, self.config, self.spec, self.scheme = model, config, spec, scheme
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.group = group
        self.world = dist.get_world_size(group) if group is not None else 1
        self.rank = dist.get_rank(group) if group is not None else 0
        if shard is not None:
            # rank r's slice of a G-way head split without a process group: the
            # per-rank state and kernels only (speculate() hook calls, parity at a
            # shard's shapes); decode_step / prefill need the group's collectives
            if group is not None:
                raise ValueError("shard and group are exclusive")
            self.rank, self.world = int(shard[0]), int(shard[1])
            if not 0 <= self.rank < self.world:
                raise ValueError(f"bad shard {shard}")
        H, D, d, L = spec.heads, spec.model_dim, spec.head_dim, spec.layers
        if H % self.world:
            raise ValueError(f"{H} heads do not shard over {self.world} ranks")
        self.H, self.D, self.d, self.L, self.F = H, D, d, L, spec.ffn_dim
        self.Hg = H // self.world
        self.h0 = self.rank * self.Hg
        # FFN tensor parallelism (Megatron MLP: FFN-in column-parallel, FFN-out
        # row-parallel, one all-reduce), so every rank streams 1/G of all weights;
        # replicated if the hidden width does not split into 16-B multiples
        F = spec.ffn_dim
        self.Fg = F // self.world if (F % self.world == 0 and (F // self.world) % 4 == 0) else F
        self.f0 = self.rank * self.Fg if self.Fg != F else 0
        self.B = config.batch
        self.elt = pool_dtype
        self.row_bytes = 2 * d * _lib.ELT_BYTES[pool_dtype]
        if self.row_bytes % 16:
            raise ValueError("2*head_dim*element bytes must be a multiple of 16")
        steps = config.gen_len if max_steps is None else max_steps
        rows = config.prompt_len + steps
        if config.pool_limit is not None:
            rows = min(rows, config.pool_limit)
        self.S_max = (rows + 3) // 4 * 4
        sc = config.speculation
        self.kcols = int(math.ceil(sc.partial_ratio * d))
        self.cap = max(int(math.floor(sc.cap_ratio * self.S_max)), sc.min_select, 1)
        self.policy = EvictionPolicy(config.pool_policy)
        self.fetch_ctas = fetch_ctas
        self.fetch_threads = fetch_threads
        self.fetch_priority = fetch_priority
        if fetch_impl not in ("ldg", "tma"):
            raise ValueError("fetch_impl must be 'ldg' or 'tma'")
        self.fetch_impl = fetch_impl
        self.fetch_rows = fetch_rows
        if dense not in ("cublas", "packed"):
            raise ValueError("dense must be 'packed' or 'cublas'")
        self.dense = dense
        self.cuda_graph = cuda_graph
        if cuda_graph and (config.record_selection or config.record_scores):
            raise ValueError("cuda_graph cannot record traces (host reads every layer)")
        # N > 1: the step's collectives over peer memory (IG_PEER_AR=0: the process group)
        self.use_peer = (group is not None and dist.get_world_size(group) > 1
                         and os.environ.get("IG_PEER_AR", "1") != "0")
        if (cuda_graph and group is not None and not self.use_peer
                and dist.get_backend(group) != "nccl"):
            raise ValueError("cuda_graph needs NCCL for the collectives")
        self._graph = None
        self._graph_mode = False
        self.graph_launches = 0
        if hbm_layers not in (0, 1) or hbm_layers > spec.layers:
            raise ValueError("hbm_layers must be 0 or 1")
        self.hbm_layers = hbm_layers
        if resident is None:
            resident = scheme == "speculative" and not hbm_layers
        if resident and (scheme != "speculative" or hbm_layers):
            raise ValueError("resident needs the speculative scheme and hbm_layers=0")
        self.resident = bool(resident)
        self._res_valid = False
        self.spec_stream_on = bool(spec_stream)
        self.append_stream_on = bool(append_stream)
        # per-layer LayerRecords (bytes, n, pool events; engine.py:420-437) even
        # without record_selection / record_scores -- what the reference's run()
        # always keeps (one host sync per layer: a trace mode, not the perf path)
        self.record_trace = bool(record_trace)
        self._out_host = None           # step_host's pinned output rows
        # IG_FUSE_PLAN=1: the resident plan fused into the select (ig_select_plan) --
        # measured 967 vs 989 tok/s at C3 (profiles/r02aa_*), so two launches by default
        self.fuse_plan = os.environ.get("IG_FUSE_PLAN", "0") == "1"
        # IG_APPEND_FIRST=1: launch ig_append(li) before releasing the speculation
        # chain of li+1 (measured at C3: 952 vs 984 tok/s -- off)
        self.append_first = os.environ.get("IG_APPEND_FIRST", "0") == "1"
        # IG_SELECT_AFTER_ATTEND=1: the select / plan / fetch of layer li+1 wait for
        # attend(li), so the latency-bound select does not hold SM slots the
        # attention needs -- measured 946 vs 998 tok/s at C3 (profiles/r02saa_*): off
        self.select_after_attend = os.environ.get("IG_SELECT_AFTER_ATTEND", "0") == "1"
        self.scale = float(np.float32(1.0 / np.sqrt(d)))   # speculation.py:127
        self._load_weights(model)
        self._alloc()
        # N > 1: the W_O / FFN-out all-reduces over peer memory (IG_PEER_AR=0: NCCL)
        self.peer_ar = self.peer_cnt = None
        # the W_O / FFN-out push folded into the packed GEMM's epilogue (IG_PEER_FUSE=0: a
        # separate push + sum kernel after a plain GEMM)
        self.peer_fuse = (self.dense == "packed" and self.B <= PACKED_MAX_M
                          and os.environ.get("IG_PEER_FUSE", "1") != "0")
        if self.use_peer:
            pc = peer_collectives([(self.B * self.D, torch.float32), (self.B, torch.int32)],
                                  group, self.device)
            if pc is not None:
                self.peer_ar, self.peer_cnt = pc
            else:
                import sys
                sys.stderr.write("DecodeEngine: peer-memory all-reduce unavailable; "
                                 "using the process group\n")
                self.use_peer = False
                if cuda_graph and dist.get_backend(group) != "nccl":
                    raise ValueError("cuda_graph needs NCCL or the peer-memory all-reduce")
        # dense peer-call numbering per step (PeerAllReduce): W_O (+ FFN-out) per layer
        self._ar_per_layer = 2 if self.Fg != self.F else 1
        self.s_host = 0
        self._inst = None
        self.iteration = 0
        self.records: list = []       # per iteration: [B][L] record dicts
        self.prefill_info: dict = {}
        self._prefetched0 = False
        self._res_valid = False

    # ------------------------------------------------------------------ setup
    def _layer_rowmajor(self, li: int, model=None) -> dict:
        """Row-major f32 weights of layer li over this rank's heads / FFN slice
        (views of the model's tensors where no slicing copy is needed)."""
        model = self.model if model is None else model
        if model is None:
            raise RuntimeError("the engine's model was released (release_model); "
                               "row-major weights are gone")
        dev, d, Hg, h0 = self.device, self.d, self.Hg, self.h0
        c0, c1 = h0 * d, (h0 + Hg) * d
        layers = model.layers
        lw = layers[li]
        q, k, v = (_f32(getattr(lw, f), dev) for f in ("w_q", "w_k", "w_v"))
        parts = [q[:, c0:c1], k[:, c0:c1], v[:, c0:c1]]
        if self.scheme == "speculative" and li + 1 < len(layers):
            parts.append(_f32(layers[li + 1].w_q, dev)[:, c0:c1])
        f0, f1 = self.f0, self.f0 + self.Fg
        return {"qkvq": torch.cat(parts, dim=1).contiguous(),
                "wo": _f32(lw.w_o, dev)[c0:c1].contiguous(),
                "ffn_in": _f32(lw.ffn_in, dev)[:, f0:f1].contiguous(),
                "ffn_out": _f32(lw.ffn_out, dev)[f0:f1].contiguous()}

    def _load_weights(self, model) -> None:
        """Per layer: [W_Q | W_K | W_V](li) | W_Q(li+1) over this rank's heads
        (the projections of layer li and the speculation query of layer li+1
        read the same input x_a(li), engine.py:311-327 / speculation.py:133, so
        one GEMM launch streams both), W_O rows, FFN slices, LN vectors.

        dense="packed": each matrix is packed (ig_sgemm_pack) as soon as its
        row-major copy is built and that copy is dropped, so HBM holds ONE copy
        of the decode weights; the prefill re-derives row-major layers from the
        model (self.model) one layer at a time."""
        dev = self.device
        self.wqkv, self.wo, self.ffn_in, self.ffn_out, self.ln = [], [], [], [], []
        self.wfused = []
        Hgd = self.Hg * self.d
        packed = self.dense == "packed"
        for li, lw in enumerate(model.layers):
            rm = self._layer_rowmajor(li, model)
            fused = rm["qkvq"].shape[1] == 4 * Hgd
            wf = _Weight(rm["qkvq"], packed, self.device)
            self.wfused.append(wf if fused else None)
            self.wqkv.append(wf.narrow(3 * Hgd) if fused else wf)
            self.wo.append(_Weight(rm["wo"], packed, dev))
            self.ffn_in.append(_Weight(rm["ffn_in"], packed, dev))
            self.ffn_out.append(_Weight(rm["ffn_out"], packed, dev))
            del rm
            self.ln.append(tuple(_f32(getattr(lw, f), dev) for f in
                                 ("ln1_gain", "ln1_bias", "ln2_gain", "ln2_bias")))
        if packed:
            torch.cuda.synchronize(dev)

    def release_model(self) -> None:
        """Drop the engine's reference to the model (its row-major weights):
        decode needs only the packed copies; a later prefill() raises."""
        if self.dense != "packed":
            raise ValueError("release_model needs dense='packed' (the other paths "
                             "read the row-major weights every step)")
        self.model = None

    def hbm_footprint(self) -> dict:
        """Bytes this engine holds in HBM, by object (torch allocations)."""
        def nb(t):
            return t.numel() * t.element_size() if isinstance(t, torch.Tensor) else 0
        w = 0
        for lst in (self.wfused, self.wqkv, self.wo, self.ffn_in, self.ffn_out):
            for W in lst:
                if W is not None and not W.is_view:
                    w += W.nbytes()
        out = {"weights": w,
               "partial_keys": nb(self.pk),
               "pool_metadata": nb(self.arrival) + nb(self.lastf) + nb(self.counter),
               "resident_slots": (nb(getattr(self, "stage_res", None)) +
                                  nb(getattr(self, "slot_id", None))),
               "layer0_stage": sum(nb(t) for t in self.stage_full) + sum(nb(t) for t in self.stage_sel),
               "model_rowmajor": 0}
        if self.model is not None:
            seen = set()
            for lw in self.model.layers:
                for f in ("w_q", "w_k", "w_v", "w_o", "ffn_in", "ffn_out"):
                    t = getattr(lw, f)
                    if isinstance(t, torch.Tensor) and t.is_cuda and t.data_ptr() not in seen:
                        seen.add(t.data_ptr())
                        out["model_rowmajor"] += nb(t)
        out["torch_allocated"] = int(torch.cuda.memory_allocated(self.device))
        out["host_pool"] = int(self.pool.nbytes) if hasattr(self.pool, "nbytes") else None
        return out

    def _alloc(self) -> None:
        dev, B, L, Hg, d, S, cap = self.device, self.B, self.L, self.Hg, self.d, self.S_max, self.cap
        D, F, kc = self.D, self.F, self.kcols
        i32, i64, f32 = torch.int32, torch.int64, torch.float32
        self.layer_bytes = B * Hg * S * self.row_bytes
        self.pool = HostPool(L * self.layer_bytes)
        T = _TORCH_ELT[self.elt]
        self.pool_hbm = (torch.zeros((self.hbm_layers, B, Hg, S, 2 * d), dtype=T, device=dev)
                         if self.hbm_layers else None)
        spec_ = self.scheme == "speculative"
        self.pk = torch.zeros((max(L - 1, 1), B, Hg, kc, S), dtype=f32, device=dev) if spec_ else None
        self.cols = torch.zeros((L, B, Hg, kc), dtype=i32, device=dev)
        self.arrival = torch.zeros((L, B, Hg, S), dtype=i64, device=dev)
        self.lastf = torch.zeros((L, B, Hg, S), dtype=i64, device=dev)
        self.counter = torch.zeros((L, B, Hg, S), dtype=torch.uint8, device=dev)
        self.st = torch.zeros(8, dtype=i32, device=dev)           # ig_step_state (24 B used)
        self.xbuf = [torch.zeros((B, D), dtype=f32, device=dev) for _ in range(2)]
        self.x = self.xbuf[0]
        self.x_a = torch.empty((B, D), dtype=f32, device=dev)
        self.x_f = torch.empty((B, D), dtype=f32, device=dev)
        # [q | k | v | qspec(next layer)] per sequence, one row of the fused GEMM
        # two [q | k | v | qspec] buffers by layer parity (IG_QKV_DB=1; default one): layer
        # li's GEMM then only waits for the speculation chain of li before its
        # append, not before the GEMM (which overwrites the other parity's qspec)
        self.qkv_db = os.environ.get("IG_QKV_DB", "0") == "1"    # measured neutral (987 vs 990)
        self.qkvq_buf = [torch.empty((B, 4 * Hg * d), dtype=f32, device=dev)
                         for _ in range(2 if self.qkv_db else 1)]
        self._use_qkv(0)
        self.attn = torch.empty((B, Hg * d), dtype=f32, device=dev)
        self.o = torch.empty((B, D), dtype=f32, device=dev)
        self.hidden = torch.empty((B, self.Fg), dtype=f32, device=dev)
        self.scores = torch.empty((B, Hg, S), dtype=f32, device=dev)
        self.maxkey = torch.zeros((B, Hg), dtype=i32, device=dev)      # rehearse scratch
        # each row's (max, min) score order keys, written by ig_rehearse_count's
        # last-tile pass and read by ig_select (no min/max pass of its own)
        self.row_range = torch.zeros((B, Hg, 2), dtype=i32, device=dev)
        self.rtickets = torch.zeros((B, Hg), dtype=i32, device=dev)    # (left zeroed)
        self.counts = torch.zeros((B, Hg), dtype=i32, device=dev)
        self.count_sum = torch.zeros((L, B), dtype=i32, device=dev)
        self.idx = torch.zeros((L, B, Hg, cap), dtype=i32, device=dev)
        self.n = torch.zeros((L, B), dtype=i32, device=dev)
        # device-side error flags in mapped pinned memory, readable by the host at
        # any time without a sync (graph replays included): [0] = ig_select overflow
        self._err_mem = HostPool(64)
        self.err_flags = self._err_mem.numpy(np.int32, (16,))
        self.err_flags[:] = 0
        self.err_ptr = self._err_mem.dev
        self.pos = torch.zeros((L, B, Hg), dtype=i32, device=dev)
        self.events = torch.zeros((L, B, Hg, 2), dtype=i64, device=dev)
        self.stage_full = [torch.empty((B, Hg, S, 2 * d), dtype=T, device=dev)
                           for _ in range(1 if spec_ else 2)]
        self.stage_sel = [torch.empty((B, Hg, cap, 2 * d), dtype=T, device=dev)
                          for _ in range(2 if spec_ and not self.resident else 0)]
        if self.resident:
            self._alloc_resident()
        # packed-GEMM stream-K workspace: the largest over the projections
        Fg = self.Fg
        shapes = [(4 * Hg * d, D), (3 * Hg * d, D), (Hg * d, D), (D, Hg * d), (Fg, D), (D, Fg)]   # (N, K)
        ws = 1
        if self.dense == "packed":
            ws = 0
            for N_, K_ in shapes:
                wf = ctypes.c_size_t()
                _lib.call("ig_sgemm_packed_sizes", min(B, PACKED_MAX_M), N_, K_, None, ctypes.byref(wf),
                          None, kernels=0)
                ws = max(ws, wf.value)
        self.gemm_ws = torch.empty(ws, dtype=f32, device=dev)
        self.gemm_tickets = torch.zeros(max((N_ + 127) // 128 for N_, _ in shapes), dtype=i32, device=dev)
        pf, tk = ctypes.c_size_t(), ctypes.c_size_t()
        _lib.call("ig_attend_scratch", B, Hg, d, S, ctypes.byref(pf), ctypes.byref(tk), kernels=0)
        self.att_partial = torch.empty(pf.value, dtype=f32, device=dev)
        self.att_tickets = torch.zeros(tk.value, dtype=i32, device=dev)
        # stream priorities (IG_STREAM_PRIO = "compute,spec"; tuning A/B only)
        cprio, sprio = (int(v) for v in os.environ.get("IG_STREAM_PRIO", "0,-1").split(","))
        self.compute = torch.cuda.Stream(device=dev, priority=cprio)
        self.fetch_stream = torch.cuda.Stream(device=dev, priority=self.fetch_priority)
        self.spec_stream = torch.cuda.Stream(device=dev, priority=sprio)
        self.append_stream = torch.cuda.Stream(device=dev)
        self.ev_q = [torch.cuda.Event() for _ in range(L)]
        self.ev_qkv = [torch.cuda.Event() for _ in range(L)]
        self.ev_app = [torch.cuda.Event() for _ in range(L)]
        self.ev_sel = [torch.cuda.Event() for _ in range(L)]
        self.ev_fetch = [torch.cuda.Event() for _ in range(L)]
        self.ev_att = [torch.cuda.Event() for _ in range(L)]
        self.ev_step = torch.cuda.Event()

    def _use_qkv(self, li: int) -> None:
        """Bind qkvq / qkv / qspec to layer li's buffer."""
        Hgd = self.Hg * self.d
        self.qkvq = self.qkvq_buf[li % len(self.qkvq_buf)]
        self.qkv = self.qkvq[:, :3 * Hgd]
        self.qspec = self.qkvq[:, 3 * Hgd:]

    def _alloc_resident(self) -> None:
        dev, B, L, Hg, d, cap = self.device, self.B, self.L, self.Hg, self.d, self.cap
        i32 = torch.int32
        Lr = max(L - 1, 1)
        # zero-filled: a slot never written must not hold NaN bits
        self.stage_res = torch.zeros((Lr, B, Hg, cap, 2 * d), dtype=_TORCH_ELT[self.elt], device=dev)
        self.slot_id = torch.full((Lr, B, Hg, cap), -1, dtype=i32, device=dev)
        self.slot_used = torch.zeros((Lr, B, Hg), dtype=i32, device=dev)
        self.frow = torch.zeros((2, B, Hg, cap), dtype=i32, device=dev)
        self.fslot = torch.zeros((2, B, Hg, cap), dtype=i32, device=dev)
        self.fcount = torch.zeros((2, B, Hg), dtype=i32, device=dev)
        self.moved_rows = torch.zeros(L, dtype=torch.int64, device=dev)

    def set_resident(self, on: bool) -> None:
        """Switch between resident selection and refetching every selected row
        each step (the reference's data movement); decode state is kept."""
        on = bool(on)
        torch.cuda.synchronize(self.device)
        if on == self.resident:
            return
        if on and (self.scheme != "speculative" or self.hbm_layers):
            raise ValueError("resident needs the speculative scheme and hbm_layers=0")
        if on:
            self.stage_sel = []
            torch.cuda.empty_cache()
            self._alloc_resident()
        else:
            for name in ("stage_res", "slot_id", "slot_used", "frow", "fslot", "fcount", "moved_rows"):
                delattr(self, name)
            torch.cuda.empty_cache()
            self.stage_sel = [torch.empty((self.B, self.Hg, self.cap, 2 * self.d),
                                          dtype=_TORCH_ELT[self.elt], device=self.device)
                              for _ in range(2)]
        self.resident = on
        self._res_valid = False
        self._prefetched0 = False
        self._graph = None

    def _set_state(self, s_len: int, seq: int) -> None:
        limit = self.config.pool_limit or 0
        st = np.zeros(8, np.int32)
        st[0], st[1] = s_len, limit
        st[2:4] = np.array([seq], np.int64).view(np.int32)
        # the step counter never goes back: the peer all-reduce epochs (step * calls
        # + call + 1) must not repeat a value a stale flag may still hold
        st[4] = int(self.st[4].item())
        self.st.copy_(torch.from_numpy(st))
        self.s_host = s_len

    def pool_view(self) -> np.ndarray:
        """Host pool as [L][B][Hg][S_max][2][d] (no copy).  Layers below
        hbm_layers are authoritative in HBM (layer_rows reads either tier)."""
        npdt = {"f32": np.float32, "f16": np.float16, "bf16": np.uint16}[self.elt]
        return self.pool.numpy(npdt, (self.L, self.B, self.Hg, self.S_max, 2, self.d))

    def layer_rows(self, li: int) -> np.ndarray:
        """Layer li's pool rows [B][Hg][S_max][2][d] as a host array (copy)."""
        torch.cuda.synchronize(self.device)
        if li < self.hbm_layers:
            t = self.pool_hbm[li].view(self.B, self.Hg, self.S_max, 2, self.d)
            return (t.view(torch.uint16) if self.elt == "bf16" else t).cpu().numpy()
        return np.array(self.pool_view()[li])

    def set_hbm_layers(self, n: int) -> None:
        """Move layer 0's rows between the host pool and the HBM tier."""
        if n not in (0, 1):
            raise ValueError("hbm_layers must be 0 or 1")
        if n == 1 and self.resident:
            raise ValueError("hbm_layers=1 needs resident=False (resident mode mirrors layer 0)")
        torch.cuda.synchronize(self.device)
        if n == self.hbm_layers:
            return
        T = _TORCH_ELT[self.elt]
        if n == 1:
            self.pool_hbm = torch.empty((1, self.B, self.Hg, self.S_max, 2 * self.d), dtype=T,
                                        device=self.device)
            _lib.call("ig_memcpy2d", self.pool_hbm.data_ptr(), self.layer_bytes, self.pool.host,
                      self.layer_bytes, self.layer_bytes, 1, _lib.stream_handle(), kernels=0)
        else:
            _lib.call("ig_memcpy2d", self.pool.host, self.layer_bytes, self.pool_hbm.data_ptr(),
                      self.layer_bytes, self.layer_bytes, 1, _lib.stream_handle(), kernels=0)
        torch.cuda.synchronize(self.device)
        if n == 0:
            self.pool_hbm = None
        self.hbm_layers = n
        self._prefetched0 = False
        self._res_valid = False
        self._graph = None

    def _pool_layer_dev(self, li: int) -> int:
        """Device address of layer li's rows (HBM tier or the host pool alias)."""
        if li < self.hbm_layers:
            return self.pool_hbm[li].data_ptr()
        return self.pool.dev + li * self.layer_bytes

    def _pool_layer_host(self, li: int) -> int:
        """Copy-engine address of layer li's rows (UVA: host pointer or HBM)."""
        if li < self.hbm_layers:
            return self.pool_hbm[li].data_ptr()
        return self.pool.host + li * self.layer_bytes

    # ---------------------------------------------------------- state import
    def load_state(self, x, kv, columns=None, meta=None) -> None:
        """Inject decode state without prefill ("state injection").

        x: [B, D]; kv(li, b, h) -> (K [s, d], V [s, d]) for GLOBAL head h;
        columns(li, b, h) -> partial columns for li >= 1; meta(li, b, h) ->
        (arrival, last_fetch, counter, seq) or None for "s plain appends".
        """
        L, B, Hg, d, S = self.L, self.B, self.Hg, self.d, self.S_max
        pv = self.pool_view()
        s_len, seq0 = None, None
        arr = np.zeros((L, B, Hg, S), np.int64)
        lf = np.zeros((L, B, Hg, S), np.int64)
        ct = np.zeros((L, B, Hg, S), np.uint8)
        cols = np.zeros((L, B, Hg, self.kcols), np.int32)
        for li in range(L):
            for b in range(B):
                for hl in range(Hg):
                    h = self.h0 + hl
                    K, V = (np.asarray(a, dtype=np.float32) for a in kv(li, b, h))
                    s = K.shape[0]
                    if s_len is None:
                        s_len = s
                    if s != s_len or s > S:
                        raise ValueError("all pools must hold the same row count <= S_max")
                    if li < self.hbm_layers:
                        rows = torch.from_numpy(np.concatenate([K, V], axis=1)).to(self.device)
                        self.pool_hbm[li, b, hl, :s] = rows.to(self.pool_hbm.dtype)
                    elif self.elt == "bf16":
                        kb = torch.from_numpy(K).to(torch.bfloat16).view(torch.uint16).numpy()
                        vb = torch.from_numpy(V).to(torch.bfloat16).view(torch.uint16).numpy()
                        pv[li, b, hl, :s, 0], pv[li, b, hl, :s, 1] = kb, vb
                    else:
                        pv[li, b, hl, :s, 0], pv[li, b, hl, :s, 1] = K, V
                    if meta is not None and meta(li, b, h) is not None:
                        a_, l_, c_, sq = meta(li, b, h)
                        arr[li, b, hl, :s], lf[li, b, hl, :s], ct[li, b, hl, :s] = a_, l_, c_
                        seq0 = sq
                    else:
                        arr[li, b, hl, :s] = np.arange(1, s + 1)
                        lf[li, b, hl, :s] = np.arange(1, s + 1)
                        seq0 = s
                    if li >= 1 and self.scheme == "speculative":
                        c = np.asarray(columns(li, b, h), dtype=np.int64)
                        if c.shape != (self.kcols,):
                            raise ValueError(f"expected {self.kcols} partial columns, got {c.shape}")
                        cols[li, b, hl] = c
                        self.pk[li - 1, b, hl, :, :s] = torch.from_numpy(
                            np.ascontiguousarray(K[:, c].T)).to(self.device)
        self.arrival.copy_(torch.from_numpy(arr))
        self.lastf.copy_(torch.from_numpy(lf))
        self.counter.copy_(torch.from_numpy(ct))
        self.cols.copy_(torch.from_numpy(cols))
        self.x.copy_(_f32(x, self.device).reshape(self.B, self.D))
        self._set_state(s_len, seq0)
        self._prefetched0 = False
        self._res_valid = False
        self._graph = None
        torch.cuda.synchronize(self.device)

    @classmethod
    def from_sessions(cls, model, config: RunConfig, sessions, **kw) -> "DecodeEngine":
        """Take over reference (or look-alike) DecodeSession objects after their
        prefill: pools[li][h].keys/values/arrival_seq/last_fetch_seq/
        fetch_counter/_seq, artifacts.head(li, h).column_indices, x."""
        eng = cls(model, config, **kw)
        def kv(li, b, h):
            p = sessions[b].pools[li][h]
            return p.keys, p.values
        def cols(li, b, h):
            return sessions[b].artifacts.head(li, h).column_indices
        def meta(li, b, h):
            p = sessions[b].pools[li][h]
            return p.arrival_seq, p.last_fetch_seq, p.fetch_counter, p._seq
        x = np.concatenate([np.asarray(s.x, np.float32).reshape(1, -1) for s in sessions])
        eng.load_state(x, kv, cols if eng.scheme == "speculative" else None, meta)
        eng.iteration = sessions[0].iteration
        return eng

    # ---------------------------------------------------------------- prefill
    @torch.no_grad()
    def prefill(self, prompts, tf32: bool = False, chunk_rows: int = 1 << 16,
                dense: str = "tc05") -> None:
        """GPU prefill of all B prompts (engine.py:245-291).  prompts: [B, N, D].

        Layer-outer and batched over the sequences: layer li's weights are
        split once into tcgen05 operands (dense="tc05", the default:
        csrc/gemm_tc05.cu, f32-level hi/lo split GEMMs with the ReLU and the
        residual adds fused into their epilogues; the causal attention of all
        the group's sequences in one launch of csrc/prefill_attn.cu), every sequence runs through
        the layer in groups of at most `chunk_rows` prompt rows, and the K/V
        rows, partial columns and partial keys of layer li are written without a
        host synchronisation.  dense="torch": cuBLAS GEMMs instead, IEEE fp32, or
        TF32 with tf32=True (A/B only).
        """
        self._need_group()
        if dense not in ("tc05", "torch"):
            raise ValueError("dense must be 'tc05' or 'torch'")
        from . import tcgemm
        cfg, spec = self.config, self.spec
        L, B, Hg, d, S, D = self.L, self.B, self.Hg, self.d, self.S_max, self.D
        N = cfg.prompt_len
        Hgd = Hg * d
        prompts = _f32(prompts, self.device).reshape(B, N, D)
        row_of, arr, lf, ct, ovw = _simulate_prefill_rows(N, cfg.pool_limit, self.policy)
        keep_tok = np.full(len(arr), -1, np.int64)
        for t, r in enumerate(row_of):
            keep_tok[r] = t                       # last token written to each row
        rows = len(arr)
        keep = torch.from_numpy(keep_tok).to(self.device)
        T = _TORCH_ELT[self.elt]
        spec_ = self.scheme == "speculative"
        seqs = max(1, min(B, chunk_rows // max(N, 1)))       # sequences per group
        x_all = prompts.reshape(B * N, D).clone()
        del prompts
        tc = dense == "tc05"
        ws = {}                                   # split-operand buffers, reused per layer

        def mm(X, Wop, Wrm, key, epilogue=0, R=None):
            if tc:
                A = tcgemm.split_rows(X, ws.get(key))
                ws[key] = A
                return tcgemm.gemm(A, Wop, M=X.shape[0], epilogue=epilogue, R=R)
            y = X @ Wrm
            if epilogue == 1:
                y.relu_()
            elif epilogue == 2:
                y += R
            return y

        old = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = bool(tf32)
        try:
            for li in range(L):
                g1, b1, g2, b2 = self.ln[li]
                W = (self._layer_rowmajor(li) if self.dense == "packed" else
                     {"qkvq": (self.wfused[li] or self.wqkv[li]).rm, "wo": self.wo[li].rm,
                      "ffn_in": self.ffn_in[li].rm, "ffn_out": self.ffn_out[li].rm})
                wqkv = W["qkvq"][:, :3 * Hgd]
                if tc:
                    ops = {"qkv": tcgemm.split_weight(wqkv.contiguous()),
                           "wo": tcgemm.split_weight(W["wo"]),
                           "ffn_in": tcgemm.split_weight(W["ffn_in"]),
                           "ffn_out": tcgemm.split_weight(W["ffn_out"])}
                    del W, wqkv
                    W, wqkv = None, None
                else:
                    ops = {"qkv": None, "wo": None, "ffn_in": None, "ffn_out": None}
                    W = dict(W, qkv=wqkv)
                rm = W or {"qkv": None, "wo": None, "ffn_in": None, "ffn_out": None}
                for b0 in range(0, B, seqs):
                    nb = min(seqs, B - b0)
                    x = x_all[b0 * N:(b0 + nb) * N]
                    x_a = layernorm(x, g1, b1, spec.ln_eps)
                    qkv = mm(x_a, ops["qkv"], rm["qkv"], "x").view(nb, N, 3, Hg, d)
                    del x_a
                    att = torch.empty((nb, N, Hg, d), dtype=torch.float32, device=self.device)
                    tc_att = tc and d in (64, 128)
                    if tc_att:           # causal attention of every sequence on tcgen05, one launch
                        sz = ctypes.c_size_t()
                        _lib.call("ig_prefill_attention_scratch", nb, N, Hg, d, ctypes.byref(sz), kernels=0)
                        if "att_work" not in ws or ws["att_work"].numel() < sz.value:
                            ws["att_work"] = torch.empty(sz.value, dtype=torch.uint8, device=self.device)
                        _lib.call("ig_prefill_attention", qkv.data_ptr(), 3 * Hgd, nb, N, Hg, d,
                                  ws["att_work"].data_ptr(), att.data_ptr(), Hgd, _lib.stream_handle())
                    for j in range(nb):
                        q, k, v = (qkv[j, :, i].transpose(0, 1).contiguous() for i in range(3))
                        if not tc_att:
                            att[j] = causal_attention(q, k, v).transpose(0, 1)
                        b = b0 + j
                        # pool rows (keep_tok: which prompt token survives in each row)
                        kvrows = torch.stack([k[:, keep], v[:, keep]], dim=2).to(T).contiguous()
                        base = self._pool_layer_host(li) + b * Hg * S * self.row_bytes
                        _lib.call("ig_memcpy2d", base, S * self.row_bytes, kvrows.data_ptr(),
                                  rows * self.row_bytes, rows * self.row_bytes, Hg,
                                  _lib.stream_handle(), kernels=0)
                        if li >= 1 and spec_:
                            cols = partial_columns(q, k, cfg.speculation.partial_ratio)
                            self.cols[li, b] = cols
                            ksel = torch.gather(k[:, keep], 2,
                                                cols.long()[:, None, :].expand(Hg, rows, self.kcols))
                            self.pk[li - 1, b, :, :, :rows] = ksel.transpose(1, 2)
                        del q, k, v, kvrows
                    del qkv
                    if self.world > 1:
                        o = mm(att.view(nb * N, Hgd), ops["wo"], rm["wo"], "att")
                        dist.all_reduce(o, group=self.group)
                        mid = o.add_(x)
                    else:                              # x_mid = x + attn @ W_O, fused
                        mid = mm(att.view(nb * N, Hgd), ops["wo"], rm["wo"], "att", 2, x)
                    del att
                    xf = layernorm(mid, g2, b2, spec.ln_eps)
                    hid = mm(xf, ops["ffn_in"], rm["ffn_in"], "x", 1)
                    del xf
                    if self.Fg != self.F:
                        ffn = mm(hid, ops["ffn_out"], rm["ffn_out"], "hid")
                        dist.all_reduce(ffn, group=self.group)   # row-parallel FFN-out
                        x.copy_(mid.add_(ffn))
                        del ffn
                    else:                              # x = x_mid + FFN, fused
                        x.copy_(mm(hid, ops["ffn_out"], rm["ffn_out"], "hid", 2, mid))
                    del hid, mid
                del ops, W, rm
            self.x.copy_(x_all.view(B, N, D)[:, -1])
            del x_all, ws
        finally:
            torch.backends.cuda.matmul.allow_tf32 = old
        self.arrival[..., :rows] = torch.from_numpy(arr).to(self.device)
        self.lastf[..., :rows] = torch.from_numpy(lf).to(self.device)
        self.counter[..., :rows] = torch.from_numpy(ct).to(self.device)
        self._set_state(rows, N)
        self._prefetched0 = False
        self._res_valid = False
        self._graph = None
        self.prefill_info = {"prompt_len": N, "pool_rows": rows,
                             "partial_cols": self.kcols if (self.scheme == "speculative" and L > 1) else None,
                             "pool_overwrites": ovw * L * self.H}
        torch.cuda.synchronize(self.device)

    # -------------------------------------------------------- instrumentation
    def instrument(self, steps: int) -> None:
        """Record CUDA events around every fetch / rehearse / select / attend
        launch (on the stream it runs on) for the next ``steps`` decode steps,
        plus the per-step n; read back with kernel_stats().  Event records
        are asynchronous: no host synchronisation is added."""
        self._inst = {"steps": steps, "k": 0, "ev": [], "s": [],
                      "n": torch.zeros((steps, self.L, self.B), dtype=torch.int32, device=self.device)}
        if self.resident:   # rows actually fetched per (step, layer): moved_rows snapshots
            self._inst["moved0"] = self.moved_rows.clone()
            self._inst["moved"] = torch.zeros((steps, self.L), dtype=torch.int64, device=self.device)

    def _mark(self, kind: str, li: int, stream, start: bool, nbytes: int | None = None):
        inst = self._inst
        if inst is None or self._graph_mode or inst["k"] >= inst["steps"]:
            return
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(stream)
        if start:
            inst["ev"].append([inst["k"], kind, li, ev, None, nbytes])
        else:
            for rec in reversed(inst["ev"]):
                if rec[1] == kind and rec[2] == li and rec[4] is None:
                    rec[4] = ev
                    break

    def kernel_stats(self) -> dict:
        """Per kernel kind: launches, total ms, algorithmic bytes (see DESIGN.md
        "Algorithmic bytes")."""
        inst = self._inst
        torch.cuda.synchronize(self.device)
        n_hist = inst["n"].cpu().numpy()
        B, Hg, d, kc, rb = self.B, self.Hg, self.d, self.kcols, self.row_bytes
        moved = None
        if "moved" in inst:
            snap = np.concatenate([inst["moved0"].cpu().numpy()[None], inst["moved"].cpu().numpy()])
            moved = np.diff(snap, axis=0)                 # [step][layer] rows fetched
        out = {}
        for k, kind, li, e0, e1, nb in inst["ev"]:
            if e1 is None:
                continue
            s = inst["s"][k]
            if nb is not None:
                nbytes = nb                               # dense: 4 (K N + M K + M N)
            elif kind == "fetch" and moved is not None and li >= 1:
                nbytes = int(moved[k, li]) * rb           # resident: rows that entered the set
            elif kind == "fetch":
                rows = B * s if (li == 0 or self.scheme == "full") else int(n_hist[k, li].sum())
                nbytes = rows * Hg * rb
            elif kind == "rehearse":
                nbytes = 4 * B * Hg * s * (kc + 1)            # partial K read + scores write
            elif kind == "select":
                nbytes = 4 * B * Hg * s                       # one pass over the scores
            else:                                             # attend: staged rows read
                rows = B * s if (li == 0 or self.scheme == "full") else int(n_hist[k, li].sum())
                nbytes = rows * Hg * rb
            tag = kind if kind != "fetch" else (
                "fetch_all_ce" if (li == 0 or self.scheme == "full")
                else ("fetch_slots" if moved is not None else "fetch_gather"))
            r = out.setdefault(tag, {"launches": 0, "ms": 0.0, "bytes": 0})
            r["launches"] += 1
            r["ms"] += e0.elapsed_time(e1)
            r["bytes"] += nbytes
        for r in out.values():
            r["gbs"] = r["bytes"] / (r["ms"] * 1e6) if r["ms"] > 0 else None
        out["n_mean_per_layer"] = [float(x) for x in n_hist[:inst["k"]].mean(axis=(0, 2))]
        return out

    @torch.no_grad()
    def isolated_kernel_times(self, li: int = 1, reps: int = 5) -> dict:
        """Time the compute-stream path kernels of layer li one at a time with
        nothing else on the GPU (CUDA events, best of `reps`), on the engine's
        current state: the HBM-bound kernels' own roofline, free of the
        concurrent gather.  Leaves the decode state unchanged (scores,
        count_sum and the attention output are scratch)."""
        if self.scheme != "speculative" or not (1 <= li < self.L):
            raise ValueError("needs a speculative layer >= 1")
        torch.cuda.synchronize(self.device)
        B, Hg, d, S, kc = self.B, self.Hg, self.d, self.S_max, self.kcols
        s = self.s_host
        sc = self.config.speculation
        cs = torch.cuda.current_stream(self.device)
        h = cs.cuda_stream
        Hgd = Hg * d
        n_tot = int(self.n[li].sum().item())

        def best(fn, chain=10):
            # `chain` launches between one event pair: a lone launch's time would
            # include the host's launch latency (~10-20 us at these sizes)
            fn()
            t = []
            for _ in range(reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(cs)
                for _ in range(chain):
                    fn()
                e1.record(cs)
                e1.synchronize()
                t.append(e0.elapsed_time(e1) / chain)
            return min(t)

        def rehearse():
            self.count_sum[li].zero_()
            _lib.call("ig_rehearse_count", self.qspec.data_ptr(), self.qkvq.stride(0), self.cols[li].data_ptr(),
                      self.pk[li - 1].data_ptr(), self.st.data_ptr(), B, Hg, d, kc, S, self.scale,
                      float(sc.alpha), self.scores.data_ptr(), self.maxkey.data_ptr(),
                      self.rtickets.data_ptr(), self.counts.data_ptr(),
                      self.count_sum[li].data_ptr(), self.row_range.data_ptr(), h)

        idx_tmp = torch.empty_like(self.idx[li])
        n_tmp = torch.empty_like(self.n[li])

        def select():
            _lib.call("ig_select", self.scores.data_ptr(), self.count_sum[li].data_ptr(),
                      self.st.data_ptr(), B, Hg, self.H, S, self.cap, float(sc.cap_ratio),
                      int(sc.min_select), idx_tmp.data_ptr(), n_tmp.data_ptr(), self.err_ptr,
                      self.row_range.data_ptr(), h)

        def attend():
            if self.resident:
                self._attend_slots(li, h)
            else:
                self._attend(li, self.stage_sel[li % 2], self.idx[li], self.n[li], self.cap, h)

        hid = torch.empty_like(self.hidden)

        def ffn_in():
            self._gemm(self.x_f, self.ffn_in[li], hid, h, epilogue=1)

        rows = [("rehearse_count", rehearse, 4 * B * Hg * s * (kc + 1)),
                ("select", select, 4 * B * Hg * s),
                ("attend", attend, n_tot * Hg * self.row_bytes),
                ("dense_ffn_in", ffn_in, 4 * (self.D * self.Fg + B * self.D + B * self.Fg))]
        out = {}
        for name, fn, nbytes in rows:
            ms = best(fn)
            out[name] = {"ms": ms, "bytes": nbytes, "gbs": nbytes / (ms * 1e6)}
        torch.cuda.synchronize(self.device)
        return out

    def check_errors(self) -> None:
        """Raise for a device-side error flagged by any step launched so far whose
        flag write has reached the host (call after a synchronize to cover all
        of them).  decode_step polls this before every step, graph replays too."""
        if self.err_flags[0]:
            self.err_flags[0] = 0
            raise SelectionOverflowError("selection exceeded the index buffer (cap): n > "
                                         f"{self.cap} rows for some sequence")

    def _need_group(self) -> None:
        if self.world > 1 and self.group is None:
            raise ValueError("a shard engine without a process group runs speculate() only")

    @torch.no_grad()
    def speculate(self, li: int, x_a=None, qspec=None, extra_counts=None) -> dict:
        """The product speculation chain for layer ``li`` (run at layer li-1 in
        decode_step) as one hook call on the engine's current state: the fused
        packed GEMM x_a(li-1) . [W_QKV(li-1) | W_Q(li)] -> ig_rehearse_count(li)
        -> ig_select(li) -- the launches _step makes, on the compute stream.

        x_a : [B, D] LN1 output of layer li-1 (the reference speculate_scores'
            x_a_prev, engine.py:311-316); default: the engine's x_a buffer.
        qspec : optional [B, Hg, k] partial queries replayed in place of the
            GEMM's (x_a . partial_w_q, speculation.py:133), so the rehearsal and
            selection kernels are checked on identical inputs.
        extra_counts : optional [B] int head counts of the heads other ranks
            own (what the count all-reduce adds on a shard engine).

        Returns host arrays: scores [B, Hg, s], counts [B, Hg], count_sum [B],
        n [B], idx [B, Hg, cap] (ascending, first n valid).  Decode state
        (pool, partial keys, selections, slot tables) is not modified."""
        if self.scheme != "speculative" or not (1 <= li < self.L):
            raise ValueError("speculate needs the speculative scheme and 1 <= layer < L")
        B, Hg, d, S, kc = self.B, self.Hg, self.d, self.S_max, self.kcols
        sc = self.config.speculation
        s = self.s_host
        C = self.compute
        C.wait_stream(torch.cuda.current_stream(self.device))
        cs = C.cuda_stream
        with torch.cuda.stream(C):
            if qspec is None:
                if x_a is not None:
                    self.x_a.copy_(_f32(x_a, self.device).reshape(B, self.D))
                self._gemm(self.x_a, self.wfused[li - 1], self.qkvq, cs)
                q_ptr, ldq, cols, dq = self.qspec.data_ptr(), self.qkvq.stride(0), self.cols[li], d
            else:
                q = _f32(qspec, self.device).reshape(B, Hg * kc)
                q_ptr, ldq, dq = q.data_ptr(), Hg * kc, kc
                cols = torch.arange(kc, dtype=torch.int32, device=self.device).repeat(B, Hg, 1).contiguous()
            csum = torch.zeros(B, dtype=torch.int32, device=self.device)
            counts = torch.zeros((B, Hg), dtype=torch.int32, device=self.device)
            _lib.call("ig_rehearse_count", q_ptr, ldq, cols.data_ptr(), self.pk[li - 1].data_ptr(),
                      self.st.data_ptr(), B, Hg, dq, kc, S, self.scale, float(sc.alpha),
                      self.scores.data_ptr(), self.maxkey.data_ptr(), self.rtickets.data_ptr(),
                      counts.data_ptr(), csum.data_ptr(), self.row_range.data_ptr(), cs)
            if extra_counts is not None:
                csum += torch.as_tensor(np.asarray(extra_counts, np.int32), device=self.device)
            idx = torch.zeros((B, Hg, self.cap), dtype=torch.int32, device=self.device)
            n = torch.zeros(B, dtype=torch.int32, device=self.device)
            err = torch.zeros(1, dtype=torch.int32, device=self.device)
            _lib.call("ig_select", self.scores.data_ptr(), csum.data_ptr(), self.st.data_ptr(), B, Hg,
                      self.H, S, self.cap, float(sc.cap_ratio), int(sc.min_select), idx.data_ptr(),
                      n.data_ptr(), err.data_ptr(), self.row_range.data_ptr(), cs)
            out = {"scores": self.scores[:, :, :s].cpu().numpy(), "counts": counts.cpu().numpy(),
                   "count_sum": csum.cpu().numpy(), "n": n.cpu().numpy(), "idx": idx.cpu().numpy()}
        torch.cuda.current_stream(self.device).wait_stream(C)
        if int(err.item()):
            raise RuntimeError("selection exceeded the index buffer (cap)")
        return out

    # ----------------------------------------------------------------- decode
    def _packed_weight(self, W: "_Weight"):
        return W.packed

    def _gemm(self, X, W, Y, cs, epilogue: int = 0, R=None) -> None:
        """Y = X @ W (+ ReLU / + R) on the compute stream."""
        M, K = X.shape
        N = W.N
        if self.dense == "packed":
            P = W.packed
            if P is None:
                raise RuntimeError("packed weights of this matrix are not built")
            if self._inst is not None:
                self._mark("dense", -1, self.compute, True, 4 * (K * N + M * K + M * N))
            # the packed kernel takes <= 32 rows (its x fragments); larger batches
            # stream the weights once per 32-row chunk
            for m0 in range(0, M, PACKED_MAX_M):
                m = min(PACKED_MAX_M, M - m0)
                _lib.call("ig_sgemm_packed", X[m0:].data_ptr(), X.stride(0), P.data_ptr(), N, K,
                          Y[m0:].data_ptr(), Y.stride(0), _lib.ptr(R[m0:] if R is not None else None),
                          R.stride(0) if R is not None else 0, m, epilogue, self.gemm_ws.data_ptr(),
                          self.gemm_ws.numel(), self.gemm_tickets.data_ptr(),
                          self.gemm_tickets.numel(), cs)
            if self._inst is not None:
                self._mark("dense", -1, self.compute, False)
            return
        # dense="cublas": IEEE-f32 torch GEMMs on the row-major weights (A/B only)
        res = torch.addmm(R, X, W.rm) if epilogue == 2 else torch.matmul(X, W.rm)
        if epilogue == 1:
            res.relu_()
        Y.copy_(res)              # Y may be a strided view (qkv of the fused buffer)

    def _issue_full_fetch(self, li: int, s: int, stage: torch.Tensor) -> None:
        self._mark("fetch", li, self.fetch_stream, True)
        _lib.call("ig_fetch_all", self._pool_layer_host(li), self.B, self.Hg, self.S_max, s,
                  self.row_bytes, stage.data_ptr(), self.S_max,
                  self.fetch_stream.cuda_stream, kernels=0)
        self._mark("fetch", li, self.fetch_stream, False)

    def _issue_full_fetch_dev(self, li: int, stage: torch.Tensor) -> None:
        """Every row [0, st.s_len) of layer li by the TMA gather (graph mode)."""
        _lib.call("ig_fetch_tma", self._pool_layer_dev(li), None, None, self.st.data_ptr(), self.B,
                  self.Hg, self.S_max, self.S_max, self.row_bytes, stage.data_ptr(),
                  self.fetch_ctas, max(1, self.fetch_threads // 32), self.fetch_rows,
                  self.fetch_stream.cuda_stream)

    def _attend(self, li: int, stage, idx, n, stage_rows: int, cs: int, pos=_LAYER_POS) -> None:
        Hgd = self.Hg * self.d
        q, ld = self.qkv, self.qkvq.stride(0)
        _lib.call("ig_attend", q.data_ptr(), ld, q.data_ptr() + 4 * Hgd,
                  q.data_ptr() + 8 * Hgd, ld, stage.data_ptr(), _lib.ELT[self.elt],
                  _lib.ptr(idx), _lib.ptr(n), _lib.ptr(self.pos[li] if pos is _LAYER_POS else pos),
                  self.st.data_ptr(),
                  self.B, self.Hg, self.d, stage_rows, self.att_partial.data_ptr(),
                  self.att_tickets.data_ptr(), self.attn.data_ptr(), Hgd, cs)

    def _attend_slots(self, li: int, cs: int, pos=_LAYER_POS) -> None:
        Hgd = self.Hg * self.d
        q, ld = self.qkv, self.qkvq.stride(0)
        _lib.call("ig_attend_slots", q.data_ptr(), ld, q.data_ptr() + 4 * Hgd,
                  q.data_ptr() + 8 * Hgd, ld, self.stage_res[li - 1].data_ptr(),
                  _lib.ELT[self.elt], self.slot_id[li - 1].data_ptr(),
                  self.slot_used[li - 1].data_ptr(),
                  _lib.ptr(self.pos[li] if pos is _LAYER_POS else pos), self.st.data_ptr(),
                  self.B, self.Hg, self.d, self.cap, self.att_partial.data_ptr(),
                  self.att_tickets.data_ptr(), self.attn.data_ptr(), Hgd, cs)

    @torch.no_grad()
    def decode_step(self) -> torch.Tensor:
        """One decode iteration for all B sequences; returns x [B, D] on the
        device (an engine buffer: valid until the next decode_step)."""
        if self.s_host < 1:
            raise RuntimeError("prefill has not run")
        self._need_group()
        self.check_errors()
        if self.config.pool_limit is None and self.s_host >= self.S_max:
            # the reference grows its pool without bound; this one was sized at
            # construction (prompt_len + max_steps rows) and must not overrun
            raise ValueError(f"pool capacity {self.S_max} rows exhausted after "
                             f"{self.iteration} steps: build the engine with a larger max_steps")
        if not self.cuda_graph:
            return self._step()
        cur = torch.cuda.current_stream(self.device)
        if self._graph is None:
            self._graph_mode = True
            try:
                l0 = _lib.launches
                out = self._step()                      # eager step: warms the allocator
                self.graph_launches = _lib.launches - l0
                torch.cuda.synchronize(self.device)
                g = torch.cuda.CUDAGraph()
                s_keep, it_keep = self.s_host, self.iteration
                with torch.cuda.graph(g, stream=self.compute):
                    self._step()                        # captured, not executed
                self.s_host, self.iteration = s_keep, it_keep
                self._graph = g
            finally:
                self._graph_mode = False
            return out
        if self.x is not self.xbuf[0]:          # replays start from xbuf[0]
            self.xbuf[0].copy_(self.x)
            self.x = self.xbuf[0]
        self.compute.wait_stream(cur)
        with torch.cuda.stream(self.compute):
            self._graph.replay()
        cur.wait_stream(self.compute)
        lim = self.config.pool_limit
        self.s_host = min(self.s_host + 1, lim) if lim else self.s_host + 1
        self.iteration += 1
        return self.xbuf[0]

    def _step(self) -> torch.Tensor:
        cfg, spec = self.config, self.spec
        L, B, Hg, d = self.L, self.B, self.Hg, self.d
        Hgd = Hg * d
        speculative = self.scheme == "speculative"
        sc = cfg.speculation
        C, Fs = self.compute, self.fetch_stream
        cs = C.cuda_stream
        # speculation chain stream: its own (overlapping layer li's tail) unless traces
        # read the scores per layer
        SP = self.spec_stream if (self.spec_stream_on and not cfg.record_scores) else C
        sps = SP.cuda_stream
        s = self.s_host
        graph = self._graph_mode
        recording = (cfg.record_selection or cfg.record_scores or self.record_trace) and not graph
        # append stream: without a pool limit the append position is st.s_len, so the
        # attention does not wait for ig_append, which then runs beside it
        AP = (self.append_stream if (self.append_stream_on and cfg.pool_limit is None and not recording)
              else C)
        aps = AP.cuda_stream
        recs = [[None] * L for _ in range(B)]
        spec_scores = [None] * L
        nar = self._ar_per_layer
        C.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(C):
            self.count_sum.zero_()
            self.ev_step.record(C)
            resident = self.resident
            if resident and self._res_valid:
                self.ev_fetch[0].record(C)          # layer 0 mirrored in HBM: no fetch
            elif resident:                          # (re)start: empty slot tables, full layer 0
                self.slot_id.fill_(-1)
                self.slot_used.zero_()
                Fs.wait_event(self.ev_step)
                if graph:
                    self._issue_full_fetch_dev(0, self.stage_full[0])
                else:
                    self._issue_full_fetch(0, s, self.stage_full[0])
                self.ev_fetch[0].record(Fs)
            elif self.hbm_layers:
                self.ev_fetch[0].record(C)          # layer 0 is HBM-resident: no fetch
            elif graph:                             # in-step, row count read on the device
                Fs.wait_event(self.ev_step)
                self._issue_full_fetch_dev(0, self.stage_full[0])
                self.ev_fetch[0].record(Fs)
            elif not self._prefetched0:
                Fs.wait_event(self.ev_step)
                self._issue_full_fetch(0, s, self.stage_full[0])
                self.ev_fetch[0].record(Fs)
            x = self.x
            for li in range(L):
                self._use_qkv(li)
                g1, b1, g2, b2 = self.ln[li]
                _lib.call("ig_layernorm", x.data_ptr(), g1.data_ptr(), b1.data_ptr(),
                          float(spec.ln_eps), B, self.D, self.x_a.data_ptr(), cs)
                spec_wait = speculative and li >= 1 and SP is not C
                if spec_wait and not self.qkv_db:
                    # spec(li) done: qspec is free for the fused GEMM, idx/n/plan of li ready
                    C.wait_event(self.ev_sel[li])
                if li >= 1 and AP is not C:
                    C.wait_event(self.ev_app[li - 1])   # append(li-1) read qkv: free it
                sel = speculative and li >= 1
                ldq = self.qkvq.stride(0)

                def do_append(li=li, sel=sel, ldq=ldq):
                    if spec_wait and self.qkv_db:
                        # idx / n / slot tables of li (the append's fetch metadata and the
                        # attention read them); the GEMM above wrote the other parity's qspec
                        C.wait_event(self.ev_sel[li])
                    if AP is not C:
                        self.ev_qkv[li].record(C)
                        AP.wait_event(self.ev_qkv[li])
                    _lib.call("ig_append", self.qkv.data_ptr() + 4 * Hgd, self.qkv.data_ptr() + 8 * Hgd,
                              ldq, self._pool_layer_dev(li), _lib.ELT[self.elt],
                              _lib.ptr(self.pk[li - 1]) if sel else None,
                              _lib.ptr(self.cols[li]) if sel else None, self.kcols,
                              self.arrival[li].data_ptr(), self.lastf[li].data_ptr(),
                              self.counter[li].data_ptr(), _lib.POLICY[self.policy.value],
                              2 if sel else 1, _lib.ptr(self.idx[li]) if sel else None,
                              _lib.ptr(self.n[li]) if sel else None, self.cap,
                              self.st.data_ptr(), B, Hg, d, self.S_max, self.pos[li].data_ptr(),
                              self.events[li].data_ptr(), aps)
                    if resident and li == 0:            # keep layer 0's mirror complete
                        _lib.call("ig_stage_put", self.qkv.data_ptr() + 4 * Hgd,
                                  self.qkv.data_ptr() + 8 * Hgd, ldq, self.pos[0].data_ptr(),
                                  self.stage_full[0].data_ptr(), _lib.ELT[self.elt], B, Hg, d,
                                  self.S_max, aps)
                    if AP is not C:
                        self.ev_app[li].record(AP)
                appended = False
                deferred = None
                nxt = li + 1
                if nxt < L:
                    if speculative:
                        # q/k/v of this layer + the speculation query of the next
                        self._gemm(self.x_a, self.wfused[li], self.qkvq, cs)
                        if self.append_first and SP is not C:
                            # the append before the rehearsal is released: both become
                            # ready together and the high-priority rehearsal would take
                            # every SM slot first (measured 49 us of append delay at C3)
                            do_append()
                            appended = True
                        if SP is not C:
                            self.ev_q[li].record(C)
                            SP.wait_event(self.ev_q[li])
                        self._mark("rehearse", nxt, SP, True)
                        _lib.call("ig_rehearse_count", self.qspec.data_ptr(), self.qkvq.stride(0),
                                  self.cols[nxt].data_ptr(), self.pk[nxt - 1].data_ptr(),
                                  self.st.data_ptr(), B, Hg, d, self.kcols, self.S_max,
                                  self.scale, float(sc.alpha), self.scores.data_ptr(),
                                  self.maxkey.data_ptr(), self.rtickets.data_ptr(),
                                  self.counts.data_ptr(), self.count_sum[nxt].data_ptr(),
                                  self.row_range.data_ptr(), sps)
                        self._mark("rehearse", nxt, SP, False)
                        def spec_tail(nxt=nxt):
                            """select / plan / fetch of layer nxt (spec and fetch streams)"""
                            par = nxt % 2
                            self._mark("select", nxt, SP, True)
                            if self.peer_cnt is not None:
                                self.peer_cnt(self.count_sum[nxt], self.count_sum[nxt], None, self.st,
                                              nxt - 1, L - 1, sps)
                            elif self.world > 1:
                                with torch.cuda.stream(SP):
                                    dist.all_reduce(self.count_sum[nxt], group=self.group)
                            par = nxt % 2
                            if resident and self.fuse_plan:
                                # select + resident plan of each (b, h) in one CTA
                                _lib.call("ig_select_plan", self.scores.data_ptr(),
                                          self.count_sum[nxt].data_ptr(), self.st.data_ptr(), B, Hg,
                                          self.H, self.S_max, self.cap, float(sc.cap_ratio),
                                          int(sc.min_select), self.idx[nxt].data_ptr(),
                                          self.n[nxt].data_ptr(), self.err_ptr, self.pos[nxt].data_ptr(),
                                          self.slot_id[nxt - 1].data_ptr(),
                                          self.slot_used[nxt - 1].data_ptr(), self.frow[par].data_ptr(),
                                          self.fslot[par].data_ptr(), self.fcount[par].data_ptr(),
                                          self.moved_rows[nxt].data_ptr(), self.row_range.data_ptr(), sps)
                            else:
                                _lib.call("ig_select", self.scores.data_ptr(),
                                          self.count_sum[nxt].data_ptr(), self.st.data_ptr(), B, Hg,
                                          self.H, self.S_max, self.cap, float(sc.cap_ratio),
                                          int(sc.min_select), self.idx[nxt].data_ptr(),
                                          self.n[nxt].data_ptr(), self.err_ptr, self.row_range.data_ptr(), sps)
                            self._mark("select", nxt, SP, False)
                            if cfg.record_scores:
                                spec_scores[nxt] = self.scores[:, :, :s].cpu()
                            if resident and not self.fuse_plan:
                                _lib.call("ig_resident_plan", self.idx[nxt].data_ptr(),
                                          self.n[nxt].data_ptr(), self.pos[nxt].data_ptr(),
                                          self.slot_id[nxt - 1].data_ptr(),
                                          self.slot_used[nxt - 1].data_ptr(), B, Hg, self.cap,
                                          self.frow[par].data_ptr(), self.fslot[par].data_ptr(),
                                          self.fcount[par].data_ptr(),
                                          self.moved_rows[nxt].data_ptr(), sps)
                            self.ev_sel[nxt].record(SP)
                            Fs.wait_event(self.ev_sel[nxt])
                            self._mark("fetch", nxt, Fs, True)
                            if resident:
                                _lib.call("ig_fetch_slots", self._pool_layer_dev(nxt),
                                          self.frow[par].data_ptr(), self.fslot[par].data_ptr(),
                                          self.fcount[par].data_ptr(), B, Hg, self.S_max, self.cap,
                                          self.row_bytes, self.stage_res[nxt - 1].data_ptr(),
                                          Fs.cuda_stream)
                            elif self.fetch_impl == "tma":
                                _lib.call("ig_fetch_tma", self._pool_layer_dev(nxt),
                                          self.idx[nxt].data_ptr(), self.n[nxt].data_ptr(), None, B,
                                          Hg, self.S_max, self.cap, self.row_bytes,
                                          self.stage_sel[nxt % 2].data_ptr(), self.fetch_ctas,
                                          max(1, self.fetch_threads // 32), self.fetch_rows,
                                          Fs.cuda_stream)
                            else:
                                _lib.call("ig_fetch", self._pool_layer_dev(nxt), self.idx[nxt].data_ptr(),
                                          self.n[nxt].data_ptr(), B, Hg, self.S_max, self.cap,
                                          self.row_bytes, self.stage_sel[nxt % 2].data_ptr(),
                                          self.fetch_ctas, self.fetch_threads, Fs.cuda_stream)
                            self._mark("fetch", nxt, Fs, False)
                            self.ev_fetch[nxt].record(Fs)

                        if self.select_after_attend:
                            deferred = spec_tail     # launched behind attend(li), below
                        else:
                            spec_tail()
                    else:
                        if li >= 1:
                            Fs.wait_event(self.ev_att[li - 1])
                        else:
                            Fs.wait_event(self.ev_step)
                        if graph:
                            self._issue_full_fetch_dev(nxt, self.stage_full[nxt % 2])
                        else:
                            self._issue_full_fetch(nxt, s, self.stage_full[nxt % 2])
                        self.ev_fetch[nxt].record(Fs)
                if not (speculative and nxt < L):      # else computed by the fused GEMM
                    self._gemm(self.x_a, self.wqkv[li], self.qkv, cs)
                if not appended:
                    do_append()
                apos = None if AP is not C else self.pos[li]   # NULL: pos = st.s_len
                C.wait_event(self.ev_fetch[li])
                self._mark("attend", li, C, True)
                if sel and resident:
                    self._attend_slots(li, cs, apos)
                elif sel:
                    self._attend(li, self.stage_sel[li % 2], self.idx[li], self.n[li], self.cap, cs, apos)
                elif li < self.hbm_layers:
                    self._attend(li, self.pool_hbm[li], None, None, self.S_max, cs, apos)
                else:
                    stage = self.stage_full[0] if speculative else self.stage_full[li % 2]
                    self._attend(li, stage, None, None, self.S_max, cs, apos)
                self._mark("attend", li, C, False)
                self.ev_att[li].record(C)
                if deferred is not None:            # IG_SELECT_AFTER_ATTEND
                    SP.wait_event(self.ev_att[li])
                    deferred()
                    deferred = None
                if self.world > 1:
                    if self.peer_ar is not None and self.peer_fuse:
                        # the GEMM epilogue pushes into every rank; x_mid = x + sum
                        self.peer_ar.gemm_push(self.attn, self._packed_weight(self.wo[li]), self.D,
                                               Hg * d, self.st, nar * li, nar * L, self.gemm_ws,
                                               self.gemm_tickets, cs)
                        self.peer_ar.sum(self.o, x, self.st, nar * li, nar * L, cs)
                    elif self.peer_ar is not None:              # x_mid = x + sum of partials
                        self._gemm(self.attn, self.wo[li], self.o, cs)
                        self.peer_ar(self.o, self.o, x, self.st, nar * li, nar * L, cs)
                    else:
                        self._gemm(self.attn, self.wo[li], self.o, cs)
                        dist.all_reduce(self.o, group=self.group)
                        self.o.add_(x)                          # x_mid = x + attn_out
                else:
                    self._gemm(self.attn, self.wo[li], self.o, cs, epilogue=2, R=x)
                _lib.call("ig_layernorm", self.o.data_ptr(), g2.data_ptr(), b2.data_ptr(),
                          float(spec.ln_eps), B, self.D, self.x_f.data_ptr(), cs)
                self._gemm(self.x_f, self.ffn_in[li], self.hidden, cs, epilogue=1)
                x_new = self.xbuf[1] if x is self.xbuf[0] else self.xbuf[0]
                if self.Fg != self.F:               # row-parallel FFN-out: sum the ranks
                    if self.peer_ar is not None and self.peer_fuse:
                        self.peer_ar.gemm_push(self.hidden, self._packed_weight(self.ffn_out[li]),
                                               self.D, self.Fg, self.st, nar * li + 1, nar * L,
                                               self.gemm_ws, self.gemm_tickets, cs)
                        self.peer_ar.sum(x_new, self.o, self.st, nar * li + 1, nar * L, cs)
                    elif self.peer_ar is not None:
                        self._gemm(self.hidden, self.ffn_out[li], x_new, cs)
                        self.peer_ar(x_new, x_new, self.o, self.st, nar * li + 1, nar * L, cs)
                    else:
                        self._gemm(self.hidden, self.ffn_out[li], x_new, cs)
                        dist.all_reduce(x_new, group=self.group)
                        x_new.add_(self.o)
                else:
                    self._gemm(self.hidden, self.ffn_out[li], x_new, cs, epilogue=2, R=self.o)
                if recording:
                    self._record(li, s, recs, spec_scores)
                x = x_new
            if AP is not C:
                C.wait_event(self.ev_app[L - 1])    # every append read this step's state
            _lib.call("ig_step_advance", self.st.data_ptr(), cs)
            inst = self._inst
            if inst is not None and not graph and inst["k"] < inst["steps"]:
                inst["n"][inst["k"]].copy_(self.n)
                if "moved" in inst:
                    inst["moved"][inst["k"]].copy_(self.moved_rows)
                inst["s"].append(s)
                inst["k"] += 1
            s_next = min(s + 1, cfg.pool_limit) if cfg.pool_limit else s + 1
            # next step's layer-0 rows stream in while the tail of this step runs
            # (after the last attend that reads stage_full[0])
            if graph:
                if x is not self.xbuf[0]:           # replays must start from xbuf[0]
                    self.xbuf[0].copy_(x)
                    x = self.xbuf[0]
            elif not self.hbm_layers and not resident:
                last0 = 0 if speculative else (L - 1 if (L - 1) % 2 == 0 else L - 2)
                Fs.wait_event(self.ev_att[last0])
                if AP is not C:
                    Fs.wait_event(self.ev_app[0])   # this step's layer-0 row is in the pool
                self._issue_full_fetch(0, s_next, self.stage_full[0])
                self.ev_fetch[0].record(Fs)
                self._prefetched0 = True
            self.x = x
        if resident:
            self._res_valid = True
        torch.cuda.current_stream(self.device).wait_stream(C)
        self.s_host = s_next
        if recording:
            self.check_errors()
        if recording:
            self.records.append([recs[b] for b in range(B)])
        self.iteration += 1
        return x

    def _record(self, li, s, recs, spec_scores) -> None:
        """LayerRecord fields (engine.py:420-446) for every sequence."""
        torch.cuda.synchronize(self.device)
        cfg, spec = self.config, self.spec
        H, d, bpe = self.H, self.d, cfg.kv_bytes_per_element
        speculative = self.scheme == "speculative"
        pos = self.pos[li].cpu().numpy()
        ev = self.events[li].cpu().numpy()
        n_dev = self.n[li].cpu().numpy()
        idx = self.idx[li].cpu().numpy()
        for b in range(self.B):
            n_sel = int(n_dev[b]) if (speculative and li >= 1) else s
            sflops = 0.0
            if speculative and li + 1 < self.L:
                sflops = float(H * (2 * self.D * self.kcols + 2 * self.kcols * s))
            r = {"iteration": self.iteration, "layer": li, "n_selected": n_sel,
                 "bytes": selection_bytes(n_sel, H, d, bpe),
                 "full_bytes": selection_bytes(s, H, d, bpe),
                 "attention_flops": float(H * 4 * n_sel * d),
                 "ffn_flops": float(2 * self.D * self.F * 2),
                 "speculation_flops": sflops,
                 "pool_events": [{"layer": li, "head": self.h0 + h, "victim": int(ev[b, h, 0]),
                                  "arrival_seq": int(ev[b, h, 1])}
                                 for h in range(self.Hg) if ev[b, h, 0] >= 0]}
            if cfg.record_selection:
                sel = []
                for h in range(self.Hg):
                    if speculative and li >= 1:
                        rows = idx[b, h, :n_sel]
                    else:
                        rows = np.arange(s + (0 if (cfg.pool_limit and s >= cfg.pool_limit) else 1))
                    sel.append(sorted(int(i) for i in rows if i != pos[b, h]))
                r["selected"] = sel
            if cfg.record_scores and speculative and li >= 1 and spec_scores[li] is not None:
                r["spec_scores"] = spec_scores[li][b].numpy()     # [Hg, s]; lists in trace()
            recs[b][li] = r

    def step_host(self, x_host: np.ndarray | None = None, out: np.ndarray | None = None) -> np.ndarray:
        """End-to-end API: optional host input row(s) in, host output rows out
        (the reference decode_step returns the output row, engine.py:380).
        out: optional [B, D] float32 array that receives the rows (a pinned one
        takes one direct DMA; it may be x_host itself -- the copy in is ordered
        before the copy out); else a fresh array is returned."""
        if x_host is not None:
            self.x.copy_(torch.from_numpy(np.ascontiguousarray(x_host, np.float32)).reshape(self.B, self.D),
                         non_blocking=True)
        y = self.decode_step()
        if out is not None:
            if out.shape != (self.B, self.D) or out.dtype != np.float32 or not out.flags.c_contiguous:
                raise ValueError(f"out must be a C-contiguous float32 [{self.B}, {self.D}] array")
            torch.from_numpy(out).copy_(y, non_blocking=True)
            torch.cuda.current_stream(self.device).synchronize()
            self.check_errors()
            return out
        if self._out_host is None:      # pinned: one DMA, no pageable staging per step
            self._out_host = torch.empty(y.shape, dtype=y.dtype).pin_memory()
        self._out_host.copy_(y, non_blocking=True)
        torch.cuda.current_stream(self.device).synchronize()
        self.check_errors()
        return self._out_host.numpy().copy()

    def trace(self) -> dict:
        """Schema-v1 trace (engine.py:83-196; selected lists are ascending)."""
        cfg = self.config
        return {"version": TRACE_SCHEMA_VERSION, "scheme": self.scheme, "layers": self.L,
                "heads": self.H, "head_dim": self.d,
                "config": {"scheme": self.scheme, "prompt_len": cfg.prompt_len,
                           "gen_len": cfg.gen_len, "batch": cfg.batch,
                           "partial_ratio": cfg.speculation.partial_ratio,
                           "alpha": cfg.speculation.alpha, "cap_ratio": cfg.speculation.cap_ratio,
                           "min_select": cfg.speculation.min_select,
                           "pool_limit": cfg.pool_limit, "pool_policy": self.policy.value,
                           "prompt_seed": cfg.prompt_seed,
                           "kv_bytes_per_element": cfg.kv_bytes_per_element},
                "sequences": [{"prefill": dict(self.prefill_info),
                               "iterations": [[_jsonable(r) for r in it[b]] for it in self.records]}
                              for b in range(self.B)]}

    def close(self) -> None:
        self.pool.close()
        self._err_mem.close()
        for name in ("peer_ar", "peer_cnt"):
            if getattr(self, name, None) is not None:
                getattr(self, name).close()
                setattr(self, name, None)


def run(model, config: RunConfig, *, prompts=None, **kw):
    """Reference run() (engine.py:456-477) on the B200 path: prefill + gen_len
    decode steps for the whole batch at once.  prompts defaults to the
    reference's seeded normals random_prompt(N, D, prompt_seed + b)."""
    D = model.spec.model_dim
    if prompts is None:
        prompts = np.stack([np.random.default_rng(config.prompt_seed + b)
                            .standard_normal((config.prompt_len, D)).astype(np.float32)
                            for b in range(config.batch)])
    kw.setdefault("record_trace", True)     # the reference's run() always records its LayerRecords
    eng = DecodeEngine(model, config, **kw)
    try:
        eng.prefill(prompts)
        out = eng.x.cpu().numpy()
        for _ in range(config.gen_len):
            out = eng.decode_step().cpu().numpy()
        return eng.trace(), [out[b].copy() for b in range(config.batch)]
    finally:
        eng.close()
