"""NumPy restatement of the reference decode-time KV path (TEST INFRASTRUCTURE).

Header -- what this file is and is not:
  * A CPU oracle: a restatement, in NumPy, of the reference ``speckv`` package's
    decode path (speculate -> select -> fetch -> attend -> append/evict) and of
    the fixture generators that path needs (synthetic model, prompts, offline
    skew, prefill).  Every function cites the reference file:line it follows
    (paths relative to /root/reference/pkg/src/speckv/).
  * It is the checker for the CUDA path and the timed CPU baseline in
    bench.py.  The product package never imports it.
  * Parity with the reference is PINNED by tests/golden/*.npz, produced by
    tests/golden/make_golden.py from the real reference (test_oracle_golden.py
    checks this module against them).

Numerics follow the reference op-for-op (float32 storage, NumPy/OpenBLAS
arithmetic) so that, on the same CPU, results are bit-identical to the
reference.  On another CPU OpenBLAS may pick different kernels; tests compare
floats with tolerances and indices exactly.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass, field
from enum import Enum
from typing import Callable

import numpy as np

F32 = np.float32

# ---------------------------------------------------------------------------
# L0 numerics -- linalg.py
# ---------------------------------------------------------------------------


def softmax_row(v: np.ndarray) -> np.ndarray:
    """Max-shifted softmax of a 1-D float32 vector (linalg.py:40-47)."""
    v = np.asarray(v, dtype=F32)
    if v.ndim != 1 or v.size == 0:
        raise ValueError("softmax_row expects a nonempty 1-D vector")
    e = np.exp(v - np.max(v))
    return (e / np.sum(e)).astype(F32)


def layernorm(x: np.ndarray, gain: np.ndarray, bias: np.ndarray, eps: float) -> np.ndarray:
    """Row layer norm in float32 (linalg.py:50-69)."""
    if eps <= 0:
        raise ValueError("eps must be positive")
    x = np.asarray(x, dtype=F32)
    gain = np.asarray(gain, dtype=F32)
    bias = np.asarray(bias, dtype=F32)
    width = x.shape[-1]
    if gain.shape != (width,) or bias.shape != (width,):
        raise ValueError("gain/bias shape mismatch")
    mu = x.mean(axis=-1, keepdims=True)
    xc = x - mu
    var = np.mean(xc * xc, axis=-1, keepdims=True)
    return ((xc / np.sqrt(var + F32(eps))) * gain + bias).astype(F32)


def topk_indices(v: np.ndarray, k: int) -> np.ndarray:
    """First k entries of a stable descending argsort (linalg.py:177-185).

    Equal values keep ascending index order, so ties go to the lower index.
    """
    v = np.asarray(v)
    if v.ndim != 1:
        raise ValueError("topk_indices expects a 1-D vector")
    if k < 0 or k > v.size:
        raise ValueError(f"k={k} out of range for vector of length {v.size}")
    return np.argsort(-v, kind="stable")[:k]


# One-sided Jacobi SVD (linalg.py:72-174).  Same rotation rule, same schedule,
# same float64 accumulation; used only to build the skewed fixture models.
_JACOBI_TOL = 1e-10
_JACOBI_SWEEPS = 30


def _tournament(d: int) -> list[tuple[np.ndarray, np.ndarray]]:
    """Circle-method pairing rounds (linalg.py:90-106)."""
    seats = list(range(d)) + ([-1] if d % 2 else [])
    m = len(seats)
    out = []
    for _ in range(m - 1):
        pairs = [(seats[i], seats[m - 1 - i]) for i in range(m // 2)]
        pairs = [(a, b) for a, b in pairs if a >= 0 and b >= 0]
        out.append((np.array([a for a, _ in pairs], dtype=np.intp),
                    np.array([b for _, b in pairs], dtype=np.intp)))
        seats = [seats[0], seats[-1]] + seats[1:-1]
    return out


def _orthonormal_fill(u: np.ndarray, col: int, rows: int) -> np.ndarray:
    """Unit vector orthogonal to u[:, :col] (linalg.py:165-174)."""
    for e in range(rows):
        cand = np.zeros(rows)
        cand[e] = 1.0
        if col > 0:
            cand -= u[:, :col] @ (u[:, :col].T @ cand)
        nrm = np.linalg.norm(cand)
        if nrm > 1e-8:
            return cand / nrm
    raise RuntimeError("could not complete orthonormal basis")


def _jacobi(a: np.ndarray):
    """Tall (n >= d) one-sided Jacobi in float64 (linalg.py:109-162)."""
    n, d = a.shape
    w = a.copy()
    v = np.eye(d)
    rounds = _tournament(d)
    for _ in range(_JACOBI_SWEEPS):
        worst = 0.0
        for ii, jj in rounds:
            ci, cj = w[:, ii], w[:, jj]
            g_ij = np.einsum("ij,ij->j", ci, cj)
            g_ii = np.einsum("ij,ij->j", ci, ci)
            g_jj = np.einsum("ij,ij->j", cj, cj)
            live = np.abs(g_ij) > 1e-30 * np.maximum(np.sqrt(g_ii * g_jj), 1e-300)
            if not np.any(live):
                continue
            tau = (g_ii - g_jj) / (2.0 * np.where(live, g_ij, 1.0))
            t = np.sign(tau) / (np.abs(tau) + np.hypot(1.0, tau))
            t = np.where(tau == 0.0, 1.0, t)
            c = 1.0 / np.sqrt(1.0 + t * t)
            s = np.where(live, c * t, 0.0)
            c = np.where(live, c, 1.0)
            worst = max(worst, float(np.max(np.abs(s[live]))))
            w[:, ii] = ci * c + cj * s
            w[:, jj] = cj * c - ci * s
            vi, vj = v[:, ii], v[:, jj]
            v[:, ii] = vi * c + vj * s
            v[:, jj] = vj * c - vi * s
        if worst < _JACOBI_TOL:
            break
    sig = np.linalg.norm(w, axis=0)
    order = np.argsort(-sig, kind="stable")
    sig, w, v = sig[order], w[:, order], v[:, order]
    u = np.zeros((n, d))
    cut = sig[0] * 1e-9 if d > 0 else 0.0
    for j in range(d):
        u[:, j] = w[:, j] / sig[j] if sig[j] > cut else _orthonormal_fill(u, j, n)
    return u, sig, v


def svd(m: np.ndarray):
    """Thin SVD, float32 in/out (linalg.py:72-87)."""
    m = np.asarray(m, dtype=F32)
    if m.ndim != 2 or not np.all(np.isfinite(m)):
        raise ValueError("svd input must be a finite 2-D matrix")
    n, d = m.shape
    if n == 0 or d == 0:
        raise ValueError("svd input must be nonempty")
    if n < d:
        u, s, v = _jacobi(m.T.astype(np.float64))
        return v.astype(F32), s.astype(F32), u.astype(F32)
    u, s, v = _jacobi(m.astype(np.float64))
    return u.astype(F32), s.astype(F32), v.astype(F32)


# ---------------------------------------------------------------------------
# L1 model -- model.py
# ---------------------------------------------------------------------------

OUTLIER_FEEDBACK = 1.5  # model.py:22


@dataclass(frozen=True)
class ModelSpec:
    """model.py:33-60."""
    layers: int
    model_dim: int
    heads: int
    ffn_dim: int
    ln_eps: float = 1e-5
    outlier_channels: int = 0
    outlier_scale: float = 1.0
    seed: int = 0

    @property
    def head_dim(self) -> int:
        return self.model_dim // self.heads


@dataclass
class Layer:
    """LayerWeights (model.py:63-79); row-major float32, x @ W convention."""
    w_q: np.ndarray
    w_k: np.ndarray
    w_v: np.ndarray
    w_o: np.ndarray
    ffn_in: np.ndarray
    ffn_out: np.ndarray
    ln1_gain: np.ndarray
    ln1_bias: np.ndarray
    ln2_gain: np.ndarray
    ln2_bias: np.ndarray

    def head_cols(self, which: str, h: int, d: int) -> np.ndarray:
        w = {"q": self.w_q, "k": self.w_k, "v": self.w_v}[which]
        return w[:, h * d:(h + 1) * d]


@dataclass
class Model:
    spec: ModelSpec
    layers: list
    outlier_indices: np.ndarray
    skewed: bool = False
    skew_matrices: list | None = None


def generate_synthetic(spec: ModelSpec) -> Model:
    """Seeded synthetic model with planted outlier channels (model.py:108-153).

    The RNG draw order (outlier choice, then per layer Q K V O FFN_in FFN_out
    LN1g LN1b LN2g LN2b) is what makes the weights identical to the reference.
    """
    rng = np.random.default_rng(spec.seed)
    D, f = spec.model_dim, spec.ffn_dim
    picks = np.sort(rng.choice(D, size=spec.outlier_channels, replace=False))
    fb = F32(OUTLIER_FEEDBACK * (spec.outlier_scale - 1.0))

    def dense(rows, cols, fan_in):
        return (rng.standard_normal((rows, cols)) / np.sqrt(fan_in)).astype(F32)

    def jitter(base):
        return (base + 0.02 * rng.standard_normal(D)).astype(F32)

    layers = []
    for _ in range(spec.layers):
        wq, wk, wv, wo = (dense(D, D, D) for _ in range(4))
        fi = dense(D, f, D)
        fo = dense(f, D, f)
        g1, b1, g2, b2 = jitter(1.0), jitter(0.0), jitter(1.0), jitter(0.0)
        g1[picks] *= F32(spec.outlier_scale)
        g2[picks] *= F32(spec.outlier_scale)
        if fb > 0:
            for ch in picks:
                hid = int(ch) % f
                fi[ch, hid] += fb
                fo[hid, ch] += fb
        layers.append(Layer(wq, wk, wv, wo, fi, fo, g1, b1, g2, b2))
    return Model(spec, layers, picks)


def random_prompt(n: int, model_dim: int, seed: int) -> np.ndarray:
    """Seeded standard-normal N x D prompt (model.py:453-456)."""
    return np.random.default_rng(seed).standard_normal((n, model_dim)).astype(F32)


def attention_head(q, k, v, causal: bool = False):
    """softmax(q k^T / sqrt(d)) v for one head (model.py:156-180).

    Note the DIVISION by float32(sqrt(d)) here, versus the multiplication by
    float32(1/sqrt(d)) in speculation (speculation.py:127, :134).
    """
    q = np.atleast_2d(np.asarray(q, dtype=F32))
    k = np.asarray(k, dtype=F32)
    v = np.asarray(v, dtype=F32)
    if k.ndim != 2 or k.shape[0] == 0:
        raise ValueError("attention_head requires a nonempty key matrix")
    if k.shape != v.shape or q.shape[1] != k.shape[1]:
        raise ValueError("inconsistent attention shapes")
    logits = (q @ k.T) / F32(np.sqrt(q.shape[1]))
    rows, cols = logits.shape
    w = np.zeros((rows, cols), dtype=F32)
    for r in range(rows):
        end = r + 1 if causal else cols
        w[r, :end] = softmax_row(logits[r, :end])
    return w @ v, w


@dataclass
class Block:
    """The slice of model.BlockInternals (model.py:183-192) the path uses."""
    x_a: np.ndarray
    q: list
    k: list
    v: list


def forward_block(x, layer: Layer, spec: ModelSpec):
    """Prefill pre-norm block with causal attention (model.py:195-244)."""
    x = np.atleast_2d(np.asarray(x, dtype=F32))
    H, d = spec.heads, spec.head_dim
    x_a = layernorm(x, layer.ln1_gain, layer.ln1_bias, spec.ln_eps)
    qs, ks, vs, outs = [], [], [], []
    for h in range(H):
        q = x_a @ layer.head_cols("q", h, d)
        kk = x_a @ layer.head_cols("k", h, d)
        vv = x_a @ layer.head_cols("v", h, d)
        # model.py:229-230 concatenates onto an empty cache -> the rows as-is
        kc = np.concatenate([np.zeros((0, d), dtype=F32), kk], axis=0)
        vc = np.concatenate([np.zeros((0, d), dtype=F32), vv], axis=0)
        o, _ = attention_head(q, kc, vc, causal=True)
        qs.append(q); ks.append(kk); vs.append(vv); outs.append(o)
    mid = x + np.concatenate(outs, axis=1) @ layer.w_o
    xf = layernorm(mid, layer.ln2_gain, layer.ln2_bias, spec.ln_eps)
    out = mid + np.maximum(xf @ layer.ffn_in, F32(0.0)) @ layer.ffn_out
    return out, Block(x_a, qs, ks, vs)


def forward(model: Model, x):
    """Full stack, collecting per-layer internals (model.py:247-263)."""
    blocks = []
    out = x
    for layer in model.layers:
        out, blk = forward_block(out, layer, model.spec)
        blocks.append(blk)
    return out, blocks


# ---------------------------------------------------------------------------
# L2 offline skew -- skewing.py
# ---------------------------------------------------------------------------


def skew_model(model: Model, calib_seed: int, calib_tokens: int | None = None) -> Model:
    """Calibrate per-head skew by SVD and fold it into W_Q / W_K.

    skewing.py:98-104 (4*d seeded calibration rows) -> calibrate_skew
    :30-56 (A = V of SVD(Q_head)) -> _fix_signs :59-66 (max-|entry| of each V
    column positive) -> apply_skew :69-95 (W_Q, W_K head slices @ A).
    """
    if model.skewed:
        raise ValueError("model is already skewed")
    spec = model.spec
    d = spec.head_dim
    n = calib_tokens if calib_tokens is not None else 4 * d
    _, blocks = forward(model, random_prompt(max(n, 2), spec.model_dim, calib_seed))
    mats = []
    for blk in blocks:
        row = []
        for q in blk.q:
            u, _, v = svd(q)
            for j in range(v.shape[1]):
                if v[int(np.argmax(np.abs(v[:, j]))), j] < 0:
                    v[:, j] = -v[:, j]
                    u[:, j] = -u[:, j]
            row.append(v)
        mats.append(row)
    layers = []
    for li, lw in enumerate(model.layers):
        nl = Layer(*(np.array(getattr(lw, name), copy=True) for name in (
            "w_q", "w_k", "w_v", "w_o", "ffn_in", "ffn_out",
            "ln1_gain", "ln1_bias", "ln2_gain", "ln2_bias")))
        for h in range(spec.heads):
            a = np.asarray(mats[li][h], dtype=F32)
            sl = slice(h * d, (h + 1) * d)
            nl.w_q[:, sl] = nl.w_q[:, sl] @ a
            nl.w_k[:, sl] = nl.w_k[:, sl] @ a
        layers.append(nl)
    return Model(spec, layers, model.outlier_indices.copy(), True,
                 [[a.astype(F32).copy() for a in row] for row in mats])


# ---------------------------------------------------------------------------
# L3 mechanisms -- speculation.py, pool.py
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class SpeculationConfig:
    """speculation.py:19-34."""
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


class ArtifactConsistencyError(RuntimeError):
    """speculation.py:37-38."""


def partial_columns(qt, kt, ratio: float) -> np.ndarray:
    """build_partial (speculation.py:41-58): top ceil(ratio*d) columns of
    colsum(|Q~|+|K~|), returned ascending."""
    qt = np.asarray(qt, dtype=F32)
    kt = np.asarray(kt, dtype=F32)
    if qt.shape != kt.shape or qt.ndim != 2:
        raise ValueError("query/key shape mismatch")
    if not 0 < ratio <= 1:
        raise ValueError("ratio must be in (0, 1]")
    k = int(math.ceil(ratio * qt.shape[1]))
    mass = np.sum(np.abs(qt) + np.abs(kt), axis=0)
    return np.sort(topk_indices(mass, k))


@dataclass
class HeadPartial:
    """HeadArtifacts (speculation.py:61-65)."""
    column_indices: np.ndarray
    partial_w_q: np.ndarray   # D x k
    partial_k: np.ndarray     # s x k, row-aligned with the pool


class Partials:
    """PartialArtifacts (speculation.py:68-114)."""

    def __init__(self, layers: int, heads: int):
        self.layers, self.heads = layers, heads
        self.slots = [[None] * heads for _ in range(layers)]

    def set_head(self, layer: int, head: int, art: HeadPartial) -> None:
        if layer < 1:
            raise ValueError("layer 0 never speculates and has no artifacts")
        self.slots[layer][head] = art

    def head(self, layer: int, head: int) -> HeadPartial:
        art = self.slots[layer][head]
        if art is None:
            raise ValueError(f"no artifacts built for layer {layer} head {head}")
        return art

    def append_partial_key(self, layer, head, key_row, position, pool_rows) -> None:
        """Mirror a pool append/overwrite into partial K (speculation.py:92-114)."""
        art = self.head(layer, head)
        row = np.asarray(key_row, dtype=F32).reshape(-1)[art.column_indices]
        have = art.partial_k.shape[0]
        if position == have:
            art.partial_k = np.concatenate([art.partial_k, row[None, :]], axis=0)
        elif 0 <= position < have:
            art.partial_k[position] = row
        else:
            raise ArtifactConsistencyError(
                f"layer {layer} head {head}: pool append at {position} but "
                f"partial key cache has {have} rows")
        if art.partial_k.shape[0] != pool_rows:
            raise ArtifactConsistencyError(
                f"layer {layer} head {head}: partial key cache has "
                f"{art.partial_k.shape[0]} rows, pool has {pool_rows}")


def speculate_scores(x_a_prev, artifacts: Partials, layer: int, head_dim: int) -> list:
    """Rehearsal (speculation.py:117-135): per head
    ((x . W_Q_partial) . K_partial^T) * float32(1/sqrt(d))."""
    if layer < 1:
        raise ValueError("speculation starts at layer 1")
    x = np.asarray(x_a_prev, dtype=F32).reshape(-1)
    scale = F32(1.0 / np.sqrt(head_dim))
    out = []
    for h in range(artifacts.heads):
        art = artifacts.head(layer, h)
        if art.partial_k.shape[0] == 0:
            raise ValueError(f"layer {layer} head {h}: empty partial key cache")
        out.append(((x @ art.partial_w_q) @ art.partial_k.T) * scale)
    return out


def select_tokens(scores: list, cfg: SpeculationConfig):
    """Alpha-threshold selection with a head-shared count (speculation.py:138-163).

    Semantics the GPU kernel must reproduce bit-for-bit:
      thr_h = float32(float(max_h) - alpha)        (NumPy 2 weak-scalar cast)
      c_h   = #{t : score_h[t] > thr_h}            (float32 compare)
      n     = floor(sum(c)/H + 0.5), clamped to [min_select, cap], cap =
              max(floor(cap_ratio * s), min_select), and n <= s
      pick_h = first n of stable argsort(-score_h)
    """
    cfg.validate()
    if not scores or any(s.size == 0 for s in scores):
        raise ValueError("select_tokens needs nonempty score vectors")
    s = scores[0].size
    if any(vec.size != s for vec in scores):
        raise ValueError("all heads must score the same token count")
    counts = [int(np.sum(vec > (float(np.max(vec)) - cfg.alpha))) for vec in scores]
    n = int(math.floor(sum(counts) / len(counts) + 0.5))
    cap = max(int(math.floor(cfg.cap_ratio * s)), cfg.min_select)
    n = min(min(max(n, cfg.min_select), cap), s)
    return [topk_indices(vec, n) for vec in scores], n


def selection_bytes(n: int, heads: int, head_dim: int, bytes_per_element: int) -> int:
    """speculation.py:166-168."""
    return heads * n * 2 * head_dim * bytes_per_element


COUNTER_MAX = 255  # pool.py:19


class Policy(str, Enum):
    """EvictionPolicy (pool.py:22-25)."""
    FIFO = "fifo"
    LRU = "lru"
    COUNTER = "counter"


class Pool:
    """KvPool (pool.py:28-112): per (layer, head, sequence) host KV rows plus
    arrival / last-fetch sequence numbers and an 8-bit saturating counter."""

    def __init__(self, head_dim: int, limit: int | None = None,
                 policy: Policy = Policy.COUNTER, on_overwrite: Callable | None = None):
        if limit is not None and limit < 1:
            raise ValueError("limit must be >= 1 when set")
        self.head_dim, self.limit, self.policy = head_dim, limit, Policy(policy)
        self.keys = np.zeros((0, head_dim), dtype=F32)
        self.values = np.zeros((0, head_dim), dtype=F32)
        self.arrival_seq = np.zeros(0, dtype=np.int64)
        self.last_fetch_seq = np.zeros(0, dtype=np.int64)
        self.fetch_counter = np.zeros(0, dtype=np.uint8)
        self._seq = 0
        self.on_overwrite = on_overwrite

    def __len__(self) -> int:
        return self.keys.shape[0]

    def _tick(self) -> int:
        self._seq += 1
        return self._seq

    def append(self, k_row, v_row) -> int:
        """Append below the limit, else overwrite the policy victim (pool.py:53-81)."""
        k_row = np.asarray(k_row, dtype=F32).reshape(-1)
        v_row = np.asarray(v_row, dtype=F32).reshape(-1)
        if k_row.shape != (self.head_dim,) or v_row.shape != (self.head_dim,):
            raise ValueError("row dim mismatch")
        seq = self._tick()
        if self.limit is None or len(self) < self.limit:
            # pool.py:67-71 grows every array by concatenation (O(s) per row);
            # kept as-is because bench.py times this module as the reference.
            self.keys = np.concatenate([self.keys, k_row[None, :]])
            self.values = np.concatenate([self.values, v_row[None, :]])
            self.arrival_seq = np.append(self.arrival_seq, seq)
            self.last_fetch_seq = np.append(self.last_fetch_seq, seq)
            self.fetch_counter = np.append(self.fetch_counter, np.uint8(0))
            return len(self) - 1
        victim = self.evict_select()
        if self.on_overwrite is not None:
            self.on_overwrite(victim, int(self.arrival_seq[victim]))
        self.keys[victim] = k_row
        self.values[victim] = v_row
        self.arrival_seq[victim] = seq
        self.last_fetch_seq[victim] = seq
        self.fetch_counter[victim] = 0
        return victim

    def fetch(self, indices):
        """Gather rows in order and update metadata (pool.py:83-99): counters
        saturate at 255 and, if any fetched counter is then 255, every counter
        in the pool is halved."""
        idx = np.asarray(indices, dtype=np.int64)
        if idx.size and (idx.min() < 0 or idx.max() >= len(self)):
            raise IndexError(f"fetch index out of range for pool of {len(self)} rows")
        seq = self._tick()
        self.last_fetch_seq[idx] = seq
        bumped = self.fetch_counter[idx].astype(np.int64) + 1
        self.fetch_counter[idx] = np.minimum(bumped, COUNTER_MAX).astype(np.uint8)
        if np.any(self.fetch_counter[idx] == COUNTER_MAX):
            self.fetch_counter //= 2
        return self.keys[idx].copy(), self.values[idx].copy()

    def evict_select(self) -> int:
        """argmin of the policy key, lowest index on ties (pool.py:101-109)."""
        if len(self) == 0:
            raise ValueError("cannot select a victim from an empty pool")
        key = {Policy.FIFO: self.arrival_seq, Policy.LRU: self.last_fetch_seq,
               Policy.COUNTER: self.fetch_counter}[self.policy]
        return int(np.argmin(key))

    def all_indices(self) -> np.ndarray:
        return np.arange(len(self), dtype=np.int64)


# ---------------------------------------------------------------------------
# L4 orchestration -- engine.py (speculative + full schemes)
# ---------------------------------------------------------------------------

TRACE_SCHEMA_VERSION = 1  # engine.py:40


@dataclass(frozen=True)
class RunConfig:
    """engine.py:51-80, restricted to the schemes on the path."""
    scheme: str = "speculative"            # "speculative" | "full"
    prompt_len: int = 32
    gen_len: int = 8
    batch: int = 1
    speculation: SpeculationConfig = field(default_factory=SpeculationConfig)
    pool_limit: int | None = None
    pool_policy: Policy = Policy.COUNTER
    prompt_seed: int = 0
    kv_bytes_per_element: int = 2
    record_scores: bool = False
    record_selection: bool = False


def speculation_flops(model_dim, partial_cols, pool_rows, heads) -> float:
    """costmodel.py:152-155."""
    return float(heads * (2 * model_dim * partial_cols + 2 * partial_cols * pool_rows))


def attention_flops(per_head, head_dim) -> float:
    """costmodel.py:142-144."""
    return float(sum(4 * n * head_dim for n in per_head))


def ffn_flops(model_dim, ffn_dim) -> float:
    """costmodel.py:147-149."""
    return float(2 * model_dim * ffn_dim * 2)


def with_position(indices, position: int) -> np.ndarray:
    """engine.py:449-453: add the current row unless it is already selected."""
    idx = np.asarray(indices, dtype=np.int64)
    return idx if position in idx else np.concatenate([idx, [position]])


# The decode path calls these four operators by name (engine.py:35-38); tests
# substitute the GPU shims here to prove the drop-in boundary.
DEFAULT_HOOKS = {
    "speculate_scores": speculate_scores,
    "select_tokens": select_tokens,
    "attention_head": attention_head,
}


class Session:
    """DecodeSession (engine.py:199-453) for the speculative and full schemes.

    ``hooks`` maps operator names to callables with the reference signatures.
    """

    def __init__(self, model: Model, config: RunConfig, prompt=None, hooks=None,
                 _skip_prefill: bool = False):
        if config.scheme not in ("speculative", "full"):
            raise ValueError(f"scheme {config.scheme!r} is not on the path")
        if config.scheme == "speculative" and not model.skewed:
            raise ValueError("the speculative scheme requires a skewed model")
        self.model, self.config, self.spec = model, config, model.spec
        self.hooks = dict(DEFAULT_HOOKS, **(hooks or {}))
        self.iteration = 0
        self.x = None
        self.artifacts = None
        self.events: list = []
        self.records: list = []      # per iteration: list of per-layer dicts
        self.prefill_info: dict = {}
        self.pools = [[Pool(self.spec.head_dim, config.pool_limit, config.pool_policy,
                            self._listener(li, h))
                       for h in range(self.spec.heads)] for li in range(self.spec.layers)]
        if not _skip_prefill:
            self._prefill(np.asarray(prompt, dtype=F32))

    def _listener(self, li, h):
        def note(victim, old_arrival):
            self.events.append({"layer": li, "head": h, "victim": victim,
                                "arrival_seq": old_arrival})
        return note

    @classmethod
    def from_state(cls, model, config, x_row, kv, columns=None, hooks=None):
        """State injection without prefill: ``kv[li][h]`` is a
        (K, V) pair of s x d arrays; ``columns[li][h]`` the partial columns for
        li >= 1.  Pool metadata is what s plain appends would leave."""
        sess = cls(model, config, hooks=hooks, _skip_prefill=True)
        spec = model.spec
        d = spec.head_dim
        for li in range(spec.layers):
            for h in range(spec.heads):
                K, V = (np.ascontiguousarray(a, dtype=F32) for a in kv[li][h])
                p = sess.pools[li][h]
                s = K.shape[0]
                p.keys, p.values = K.copy(), V.copy()
                p.arrival_seq = np.arange(1, s + 1, dtype=np.int64)
                p.last_fetch_seq = p.arrival_seq.copy()
                p.fetch_counter = np.zeros(s, dtype=np.uint8)
                p._seq = s
        if config.scheme == "speculative":
            sess.artifacts = Partials(spec.layers, spec.heads)
            for li in range(1, spec.layers):
                lw = model.layers[li]
                for h in range(spec.heads):
                    cols = np.asarray(columns[li][h], dtype=np.int64)
                    sess.artifacts.set_head(li, h, HeadPartial(
                        cols, lw.head_cols("q", h, d)[:, cols].copy(),
                        sess.pools[li][h].keys[:, cols].copy()))
        sess.x = np.asarray(x_row, dtype=F32).reshape(1, -1).copy()
        return sess

    def _prefill(self, prompt) -> None:
        """engine.py:245-291 (speculative / full)."""
        cfg, spec = self.config, self.spec
        d = spec.head_dim
        if prompt.shape != (cfg.prompt_len, spec.model_dim):
            raise ValueError("prompt shape mismatch")
        if cfg.scheme == "speculative":
            self.artifacts = Partials(spec.layers, spec.heads)
        x = prompt
        for li, lw in enumerate(self.model.layers):
            out, blk = forward_block(x, lw, spec)
            for h in range(spec.heads):
                for t in range(cfg.prompt_len):
                    self.pools[li][h].append(blk.k[h][t], blk.v[h][t])
            if cfg.scheme == "speculative" and li >= 1:
                for h in range(spec.heads):
                    cols = partial_columns(blk.q[h], blk.k[h], cfg.speculation.partial_ratio)
                    self.artifacts.set_head(li, h, HeadPartial(
                        cols, lw.head_cols("q", h, d)[:, cols].copy(),
                        self.pools[li][h].keys[:, cols].copy()))
            x = out
        self.x = x[-1:].copy()
        cols = None
        if self.artifacts is not None and spec.layers > 1:
            cols = int(self.artifacts.head(1, 0).column_indices.size)
        self.prefill_info = {"prompt_len": cfg.prompt_len,
                             "pool_rows": len(self.pools[0][0]),
                             "partial_cols": cols,
                             "pool_overwrites": len(self.events)}
        self.events = []

    def decode_step(self) -> np.ndarray:
        """One decode iteration over all layers (engine.py:295-380).

        Per layer li: LN1 -> [speculate + select for li+1] -> per-head q/k/v ->
        append (+ partial K mirror) -> fetch set -> fetch -> attend -> W_O ->
        residual -> LN2 -> ReLU FFN -> residual.
        """
        if self.x is None:
            raise RuntimeError("prefill has not run")
        cfg, spec = self.config, self.spec
        H, d = spec.heads, spec.head_dim
        spec_fn = self.hooks["speculate_scores"]
        sel_fn = self.hooks["select_tokens"]
        attn_fn = self.hooks["attention_head"]
        speculative = cfg.scheme == "speculative"
        x = self.x
        recs = []
        carry = None          # (indices per head, n, scores) for this layer
        for li, lw in enumerate(self.model.layers):
            self.events = []
            x_a = layernorm(x, lw.ln1_gain, lw.ln1_bias, spec.ln_eps)
            nxt, sflops = None, 0.0
            if speculative and li + 1 < spec.layers:
                sc = spec_fn(x_a[0], self.artifacts, li + 1, d)
                picks, n = sel_fn(sc, cfg.speculation)
                nxt = (picks, n, sc)
                kc = self.artifacts.head(li + 1, 0).column_indices.size
                sflops = speculation_flops(spec.model_dim, kc, len(self.pools[li + 1][0]), H)
            qh = [(x_a @ lw.head_cols("q", h, d))[0] for h in range(H)]
            kh = [(x_a @ lw.head_cols("k", h, d))[0] for h in range(H)]
            vh = [(x_a @ lw.head_cols("v", h, d))[0] for h in range(H)]
            s_before = len(self.pools[li][0])
            true_sc = None
            if cfg.record_scores:
                scale = F32(1.0 / np.sqrt(d))
                true_sc = [(qh[h] @ self.pools[li][h].keys[:s_before].T) * scale
                           for h in range(H)]
            pos = []
            for h in range(H):
                p = self.pools[li][h].append(kh[h], vh[h])
                pos.append(p)
                if speculative and li >= 1:
                    self.artifacts.append_partial_key(li, h, kh[h], p,
                                                      len(self.pools[li][h]))
            # engine.py:382-418
            if not speculative or li == 0:
                sets = [self.pools[li][h].all_indices() for h in range(H)]
                n_sel = s_before
            else:
                if carry is None:
                    raise RuntimeError(f"layer {li}: missing carried selection")
                sets = [with_position(carry[0][h], pos[h]) for h in range(H)]
                n_sel = carry[1]
            outs = []
            for h in range(H):
                K, V = self.pools[li][h].fetch(sets[h])
                o, _ = attn_fn(qh[h][None, :], K, V)
                outs.append(o)
            mid = x + np.concatenate(outs, axis=1) @ lw.w_o
            xf = layernorm(mid, lw.ln2_gain, lw.ln2_bias, spec.ln_eps)
            x = mid + np.maximum(xf @ lw.ffn_in, F32(0.0)) @ lw.ffn_out
            bpe = cfg.kv_bytes_per_element
            rec = {"iteration": self.iteration, "layer": li, "n_selected": n_sel,
                   "bytes": selection_bytes(n_sel, H, d, bpe),
                   "full_bytes": selection_bytes(s_before, H, d, bpe),
                   "attention_flops": attention_flops([n_sel] * H, d),
                   "ffn_flops": ffn_flops(spec.model_dim, spec.ffn_dim),
                   "speculation_flops": sflops,
                   "pool_events": list(self.events)}
            if cfg.record_selection:
                rec["selected"] = [[int(i) for i in sets[h] if i != pos[h]] for h in range(H)]
            if cfg.record_scores:
                if speculative and carry is not None:
                    rec["spec_scores"] = [[float(v) for v in s] for s in carry[2]]
                if true_sc is not None:
                    rec["true_scores"] = [[float(v) for v in s] for s in true_sc]
            recs.append(rec)
            carry = nxt
        self.x = x
        self.iteration += 1
        self.records.append(recs)
        return x[0].copy()


def run(model: Model, config: RunConfig, hooks=None):
    """engine.py:456-477: prefill + gen_len steps per sequence, prompts seeded
    prompt_seed + b.  Returns (trace dict in schema v1, final rows)."""
    trace = {"version": TRACE_SCHEMA_VERSION, "scheme": config.scheme,
             "layers": model.spec.layers, "heads": model.spec.heads,
             "head_dim": model.spec.head_dim, "config": config_json(config),
             "sequences": []}
    finals = []
    for b in range(config.batch):
        prompt = random_prompt(config.prompt_len, model.spec.model_dim, config.prompt_seed + b)
        sess = Session(model, config, prompt, hooks=hooks)
        out = sess.x[0].copy()
        for _ in range(config.gen_len):
            out = sess.decode_step()
        trace["sequences"].append({"prefill": sess.prefill_info, "iterations": sess.records})
        finals.append(out)
    return trace, finals


def config_json(config: RunConfig) -> dict:
    """engine.py:480-496 (fields of the schemes on the path)."""
    return {
        "scheme": config.scheme, "prompt_len": config.prompt_len,
        "gen_len": config.gen_len, "batch": config.batch,
        "partial_ratio": config.speculation.partial_ratio,
        "alpha": config.speculation.alpha, "cap_ratio": config.speculation.cap_ratio,
        "min_select": config.speculation.min_select, "pool_limit": config.pool_limit,
        "pool_policy": Policy(config.pool_policy).value,
        "prompt_seed": config.prompt_seed,
        "kv_bytes_per_element": config.kv_bytes_per_element,
    }


def dumps_trace(trace: dict) -> str:
    return json.dumps(trace, sort_keys=True)
