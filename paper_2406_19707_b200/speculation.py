"""Drop-in speculation operators (reference speculation.py) on the B200 kernels.

Same names, signatures, return types and exceptions as the reference module,
so code written against ``speckv.speculation`` -- including its engine, which
imports these names (engine.py:35-38) -- can call them unchanged.  Each call
runs the library kernels (ig_rehearse / ig_score_max / ig_count / ig_select /
ig_order_by_score / ig_topk_rows) on the current CUDA device; inputs and
outputs are host NumPy arrays, as in the reference.  The batched engine
(engine.py) calls the same kernels without the host round trips.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import ArtifactConsistencyError

__all__ = ["SpeculationConfig", "ArtifactConsistencyError", "build_partial", "HeadArtifacts",
           "PartialArtifacts", "speculate_scores", "select_tokens", "selection_bytes"]


@dataclass(frozen=True)
class SpeculationConfig:
    """speculation.py:19-34 (partial ratio 0.3, alpha 4, cap 20%, min 1)."""
    partial_ratio: float = 0.3
    alpha: float = 4.0
    cap_ratio: float = 0.2
    min_select: int = 1

    def validate(self) -> None:
        if not 0 < self.partial_ratio <= 1:
            raise ValueError("partial_ratio must be in (0, 1]")
        if self.alpha <= 0:
            raise ValueError("alpha must be positive")
        if not 0 < self.cap_ratio <= 1:
            raise ValueError("cap_ratio must be in (0, 1]")
        if self.min_select < 1:
            raise ValueError("min_select must be >= 1")


def selection_bytes(n: int, heads: int, head_dim: int, bytes_per_element: int) -> int:
    """Bytes to fetch n tokens' keys and values across all heads (speculation.py:166-168)."""
    return heads * n * 2 * head_dim * bytes_per_element


@dataclass
class HeadArtifacts:
    """speculation.py:61-65."""
    column_indices: np.ndarray
    partial_w_q: np.ndarray
    partial_k: np.ndarray


class PartialArtifacts:
    """Per-layer (>= 1), per-head partial artifacts (speculation.py:68-114)."""

    def __init__(self, layers: int, heads: int):
        self.layers, self.heads = layers, heads
        self._slots = [[None] * heads for _ in range(layers)]

    def set_head(self, layer: int, head: int, artifacts: HeadArtifacts) -> None:
        if layer < 1:
            raise ValueError("layer 0 never speculates and has no artifacts")
        self._slots[layer][head] = artifacts

    def head(self, layer: int, head: int) -> HeadArtifacts:
        art = self._slots[layer][head]
        if art is None:
            raise ValueError(f"no artifacts built for layer {layer} head {head}")
        return art

    def has_layer(self, layer: int) -> bool:
        return 1 <= layer < self.layers and self._slots[layer][0] is not None

    def append_partial_key(self, layer, head, skewed_key_row, position, pool_rows) -> None:
        art = self.head(layer, head)
        row = np.asarray(skewed_key_row, dtype=np.float32).reshape(-1)[art.column_indices]
        have = art.partial_k.shape[0]
        if position == have:
            art.partial_k = np.concatenate([art.partial_k, row[None, :]], axis=0)
        elif 0 <= position < have:
            art.partial_k[position] = row
        else:
            raise ArtifactConsistencyError(
                f"layer {layer} head {head}: pool append at {position} but partial key cache has {have} rows")
        if art.partial_k.shape[0] != pool_rows:
            raise ArtifactConsistencyError(
                f"layer {layer} head {head}: partial key cache has {art.partial_k.shape[0]} rows, pool has {pool_rows}")


def _torch():
    import torch
    _lib.load()
    return torch


def _state(torch, s: int, dev):
    st = torch.zeros(8, dtype=torch.int32, device=dev)
    st[0] = s
    return st


def build_partial(qt, kt, ratio: float) -> np.ndarray:
    """Top ceil(ratio*d) columns of colsum(|Q~| + |K~|), ascending (speculation.py:41-58)."""
    qt = np.asarray(qt, dtype=np.float32)
    kt = np.asarray(kt, dtype=np.float32)
    if qt.shape != kt.shape or qt.ndim != 2:
        raise ValueError(f"query/key shape mismatch: {qt.shape} vs {kt.shape}")
    if not 0 < ratio <= 1:
        raise ValueError("ratio must be in (0, 1]")
    torch = _torch()
    from .prefill import partial_columns
    dev = torch.device("cuda")
    cols = partial_columns(torch.from_numpy(qt)[None].to(dev), torch.from_numpy(kt)[None].to(dev), ratio)
    return cols[0].cpu().numpy().astype(np.int64)


def speculate_scores(x_a_prev, artifacts, layer: int, head_dim: int) -> list:
    """Rehearse layer ``layer`` with the previous layer's attention input
    (speculation.py:117-135): per head ((x . W_Q_partial) . K_partial^T) * scale."""
    if layer < 1:
        raise ValueError("speculation starts at layer 1")
    torch = _torch()
    dev = torch.device("cuda")
    x = torch.from_numpy(np.asarray(x_a_prev, dtype=np.float32).reshape(1, -1)).to(dev)
    H = artifacts.heads
    arts = [artifacts.head(layer, h) for h in range(H)]
    s = arts[0].partial_k.shape[0]
    k = arts[0].partial_w_q.shape[1]
    for h, a in enumerate(arts):
        if a.partial_k.shape[0] == 0:
            raise ValueError(f"layer {layer} head {h}: empty partial key cache")
        if a.partial_k.shape != (s, k) or a.partial_w_q.shape[1] != k:
            raise ValueError("heads disagree on partial shapes")
    S = (s + 3) // 4 * 4
    pwq = torch.from_numpy(np.concatenate([np.asarray(a.partial_w_q, np.float32) for a in arts], axis=1)).to(dev)
    pk = torch.zeros((1, H, k, S), dtype=torch.float32, device=dev)
    pk[0, :, :, :s] = torch.from_numpy(np.stack([np.asarray(a.partial_k, np.float32).T for a in arts])).to(dev)
    # the partial queries x . partial_w_q (speculation.py:133), accumulated in f64 and
    # rounded once: within an ulp of any f32 summation order of the reference's sgemv
    qpart = (x.double() @ pwq.double()).float().contiguous()      # [1, H*k]
    return _rehearse(torch, qpart, pk, s, k, head_dim)


def rehearse_partial_queries(qpart, artifacts, layer: int, head_dim: int) -> list:
    """The second half of speculate_scores on given partial queries
    (qpart [H, k] = x . partial_w_q per head): parity tests replay the
    reference's own queries through the rehearsal kernel with this."""
    torch = _torch()
    dev = torch.device("cuda")
    H = artifacts.heads
    arts = [artifacts.head(layer, h) for h in range(H)]
    s, k = arts[0].partial_k.shape
    S = (s + 3) // 4 * 4
    pk = torch.zeros((1, H, k, S), dtype=torch.float32, device=dev)
    pk[0, :, :, :s] = torch.from_numpy(np.stack([np.asarray(a.partial_k, np.float32).T for a in arts])).to(dev)
    q = torch.from_numpy(np.ascontiguousarray(qpart, dtype=np.float32).reshape(1, H * k)).to(dev)
    return _rehearse(torch, q, pk, s, k, head_dim)


def _rehearse(torch, qpart, pk, s: int, k: int, head_dim: int) -> list:
    dev = qpart.device
    H = pk.shape[1]
    S = pk.shape[3]
    cols = torch.arange(k, dtype=torch.int32, device=dev).repeat(1, H, 1).contiguous()
    scores = torch.empty((1, H, S), dtype=torch.float32, device=dev)
    maxkey = torch.zeros((1, H), dtype=torch.int32, device=dev)
    st = _state(torch, s, dev)
    scale = float(np.float32(1.0 / np.sqrt(head_dim)))
    _lib.call("ig_rehearse", qpart.data_ptr(), H * k, cols.data_ptr(), pk.data_ptr(), st.data_ptr(),
              1, H, k, k, S, scale, scores.data_ptr(), maxkey.data_ptr(), _lib.stream_handle())
    out = scores[0, :, :s].cpu().numpy()
    return [out[h].copy() for h in range(H)]


def select_tokens(scores: list, cfg: SpeculationConfig):
    """Alpha-threshold selection with a head-shared count (speculation.py:138-163).
    Returns (per-head index arrays in stable descending-score order, n)."""
    cfg.validate()
    if not scores or any(np.asarray(s).size == 0 for s in scores):
        raise ValueError("select_tokens needs nonempty score vectors")
    s = np.asarray(scores[0]).size
    if any(np.asarray(v).size != s for v in scores):
        raise ValueError("all heads must score the same token count")
    torch = _torch()
    dev = torch.device("cuda")
    H = len(scores)
    S = (s + 3) // 4 * 4
    sc = torch.zeros((1, H, S), dtype=torch.float32, device=dev)
    sc[0, :, :s] = torch.from_numpy(np.stack([np.asarray(v, np.float32).reshape(-1) for v in scores])).to(dev)
    st = _state(torch, s, dev)
    maxkey = torch.zeros((1, H), dtype=torch.int32, device=dev)
    counts = torch.zeros((1, H), dtype=torch.int32, device=dev)
    csum = torch.zeros(1, dtype=torch.int32, device=dev)
    cap = max(int(math.floor(cfg.cap_ratio * s)), cfg.min_select, 1)
    idx = torch.zeros((1, H, cap), dtype=torch.int32, device=dev)
    n = torch.zeros(1, dtype=torch.int32, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    hs = _lib.stream_handle()
    _lib.call("ig_score_max", sc.data_ptr(), st.data_ptr(), 1, H, S, maxkey.data_ptr(), hs)
    _lib.call("ig_count", sc.data_ptr(), maxkey.data_ptr(), st.data_ptr(), 1, H, S, float(cfg.alpha),
              counts.data_ptr(), csum.data_ptr(), hs)
    _lib.call("ig_select", sc.data_ptr(), csum.data_ptr(), st.data_ptr(), 1, H, H, S, cap,
              float(cfg.cap_ratio), int(cfg.min_select), idx.data_ptr(), n.data_ptr(),
              err.data_ptr(), None, hs)
    _lib.call("ig_order_by_score", sc.data_ptr(), n.data_ptr(), 1, H, S, cap, idx.data_ptr(), hs)
    if int(err.item()):
        raise RuntimeError("selection exceeded its index buffer")
    nn = int(n.item())
    picks = idx[0, :, :nn].cpu().numpy().astype(np.int64)
    return [picks[h].copy() for h in range(H)], nn
