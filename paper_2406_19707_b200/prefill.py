"""GPU prefill: the state the decode path starts from.

Reference: DecodeSession._prefill (engine.py:245-291) -- forward_block per
layer (model.py:195-244), every prompt row appended to the pools
(engine.py:265-266), and for layers >= 1 build_partial over the skewed Q/K
(speculation.py:41-58) with partial W_Q / partial K materialised
(engine.py:269-275).  Here the dense math runs as torch GEMMs on the GPU, the
column choice is the library's radix top-k kernel (ig_topk_rows, ties -> lower
index, so equal to topk_indices + sort), and the K/V rows go to the pinned host
pool with one 2-D copy per (layer, sequence).
"""

from __future__ import annotations

import math

import torch
import torch.nn.functional as F

from . import _lib


def layernorm(x: torch.Tensor, gain: torch.Tensor, bias: torch.Tensor, eps: float,
              out: torch.Tensor | None = None) -> torch.Tensor:
    """Reference layernorm (linalg.py:50-69) via ig_layernorm; f64 inputs (the
    offline skew's optional f64 calibration forward) in f64 torch ops."""
    if x.dtype == torch.float64:
        mean = x.mean(dim=-1, keepdim=True)
        c = x - mean
        var = (c * c).mean(dim=-1, keepdim=True)
        y = c / torch.sqrt(var + eps) * gain.to(x.dtype) + bias.to(x.dtype)
        return y if out is None else out.copy_(y)
    x = x.contiguous()
    rows, D = x.shape
    y = torch.empty_like(x) if out is None else out
    _lib.call("ig_layernorm", _lib.ptr(x), _lib.ptr(gain), _lib.ptr(bias), float(eps), rows, D,
              _lib.ptr(y), _lib.stream_handle())
    return y


def causal_attention(q, k, v, block: int = 2048):
    """softmax(q k^T / sqrt(d)) v with a causal mask; q, k, v: [H, N, d] f32.

    Long prompts go in query blocks: f32 SDPA may fall back to the math path,
    which would materialise H x N x N scores (128 GiB at 32 heads x 32K)."""
    n = q.shape[-2]
    if n <= block:
        return F.scaled_dot_product_attention(q, k, v, is_causal=True)
    out = torch.empty_like(q)
    for r0 in range(0, n, block):
        r1 = min(n, r0 + block)
        mask = torch.ones(r1 - r0, r1, dtype=torch.bool, device=q.device).tril(r0)
        out[..., r0:r1, :] = F.scaled_dot_product_attention(q[..., r0:r1, :], k[..., :r1, :],
                                                             v[..., :r1, :], attn_mask=mask)
    return out


def dense_block_forward(x: torch.Tensor, lw, spec):
    """One full pre-norm block over N rows (model.py:195-244); returns
    (out [N, D], q [N, D]).  Used by the GPU skew calibration."""
    H, d, D = spec.heads, spec.head_dim, spec.model_dim
    x_a = layernorm(x, lw.ln1_gain, lw.ln1_bias, spec.ln_eps)
    q, k, v = x_a @ lw.w_q, x_a @ lw.w_k, x_a @ lw.w_v
    n = x.shape[0]
    att = causal_attention(*(t.view(n, H, d).transpose(0, 1) for t in (q, k, v)))
    mid = x + att.transpose(0, 1).reshape(n, D) @ lw.w_o
    xf = layernorm(mid, lw.ln2_gain, lw.ln2_bias, spec.ln_eps)
    return mid + torch.relu(xf @ lw.ffn_in) @ lw.ffn_out, q


def partial_columns(qt: torch.Tensor, kt: torch.Tensor, ratio: float) -> torch.Tensor:
    """build_partial (speculation.py:41-58) for a stack of heads.

    qt, kt: [Hg, N, d] skewed queries / keys.  Returns int32 [Hg, k],
    k = ceil(ratio * d), the top-k columns of sum_rows(|qt| + |kt|) with ties to
    the lower column, ascending."""
    if qt.shape != kt.shape or qt.dim() != 3:
        raise ValueError(f"query/key shape mismatch: {tuple(qt.shape)} vs {tuple(kt.shape)}")
    if not 0 < ratio <= 1:
        raise ValueError("ratio must be in (0, 1]")
    hg, _, d = qt.shape
    k = int(math.ceil(ratio * d))
    mass = (qt.abs() + kt.abs()).sum(dim=1).contiguous()  # [Hg, d]
    cols = torch.empty(hg, k, dtype=torch.int32, device=qt.device)
    _lib.call("ig_topk_rows", _lib.ptr(mass), hg, d, k, _lib.ptr(cols), _lib.stream_handle())
    return cols
