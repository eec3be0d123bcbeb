"""Drop-in attention_head (reference model.py:156-180) on the B200 kernels.

Decode form (q is 1 x d, causal=False) runs ig_attend: the last key/value row
plays the engine's GPU-resident "current row" and rows 0..m-2 are the staged
fetched rows.  The reference also returns the softmax weight row; it is
recomputed here with the same formula (torch on the GPU) since the decode path
itself never materialises it.  The causal (prefill) form runs the prefill
attention (prefill.causal_attention).
"""

from __future__ import annotations

import numpy as np

from . import _lib


def attention_head(q, k, v, causal: bool = False):
    import torch
    _lib.load()
    q = np.atleast_2d(np.asarray(q, dtype=np.float32))
    k = np.asarray(k, dtype=np.float32)
    v = np.asarray(v, dtype=np.float32)
    if k.ndim != 2 or k.shape[0] == 0:
        raise ValueError("attention_head requires a nonempty key matrix")
    if k.shape != v.shape or q.shape[1] != k.shape[1]:
        raise ValueError(f"inconsistent attention shapes q={q.shape} k={k.shape} v={v.shape}")
    if causal and q.shape[0] != k.shape[0]:
        raise ValueError("causal attention requires len(q) == len(k)")
    dev = torch.device("cuda")
    m, d = k.shape
    tq, tk, tv = (torch.from_numpy(a).to(dev) for a in (q, k, v))
    sqrt_d = float(np.float32(np.sqrt(d)))
    if causal:
        from .prefill import causal_attention
        out = causal_attention(tq[None], tk[None], tv[None])[0]
        logits = (tq @ tk.T) / sqrt_d
        mask = torch.ones(m, m, dtype=torch.bool, device=dev).triu(1)
        w = torch.softmax(logits.masked_fill(mask, float("-inf")), dim=-1)
        return out.cpu().numpy(), w.cpu().numpy()
    if q.shape[0] != 1:
        raise ValueError("non-causal attention_head expects a single query row (decode)")
    rows = m - 1
    stage = torch.zeros((1, 1, max(rows, 1), 2 * d), dtype=torch.float32, device=dev)
    if rows:
        stage[0, 0, :rows, :d] = tk[:rows]
        stage[0, 0, :rows, d:] = tv[:rows]
    cur_k = tk[rows:].contiguous()
    cur_v = tv[rows:].contiguous()
    st = torch.zeros(8, dtype=torch.int32, device=dev)
    st[0] = rows
    pos = torch.full((1,), -1, dtype=torch.int32, device=dev)
    cap = max(rows, 1)
    import ctypes
    pf, tkc = ctypes.c_size_t(), ctypes.c_size_t()
    _lib.call("ig_attend_scratch", 1, 1, d, cap, ctypes.byref(pf), ctypes.byref(tkc), kernels=0)
    part = torch.empty(pf.value, dtype=torch.float32, device=dev)
    tickets = torch.zeros(tkc.value, dtype=torch.int32, device=dev)
    out = torch.empty((1, d), dtype=torch.float32, device=dev)
    _lib.call("ig_attend", tq.data_ptr(), d, cur_k.data_ptr(), cur_v.data_ptr(), d, stage.data_ptr(),
              _lib.ELT["f32"], None, None, pos.data_ptr(), st.data_ptr(), 1, 1, d, cap,
              part.data_ptr(), tickets.data_ptr(), out.data_ptr(), d, _lib.stream_handle())
    w = torch.softmax((tq @ tk.T) / sqrt_d, dim=-1)
    return out.cpu().numpy(), w.cpu().numpy()
