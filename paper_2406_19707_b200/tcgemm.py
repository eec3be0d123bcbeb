"""Prompt-length projections on the tcgen05 tensor cores (prefill, SURVEY.md
s8(f) rank 1): f32-level GEMMs from f16 hi/lo operand pairs.

Reference: forward_block (model.py:195-244) as driven by DecodeSession._prefill
(engine.py:245-291) -- x_a @ W_QKV, attn @ W_O, relu(x_f @ W_in) @ W_out, all
IEEE f32 in NumPy/OpenBLAS.  Here each operand is split once (ig_split_f16:
power-of-two scale per operand row, hi = f16, lo = f16 of the remainder) and
ig_gemm_tc05 accumulates hi.hi + hi.lo + lo.hi in f32 in TMEM
(csrc/gemm_tc05.cu).  No fallback: the library must be loaded.
"""

from __future__ import annotations

import torch

from . import _lib


def kpad(K: int) -> int:
    return (K + 63) // 64 * 64


class SplitOperand:
    """A K-major f16 hi/lo operand: rows x [hi (Kp) | lo (Kp)] plus the
    per-row power-of-two inverse scales."""

    def __init__(self, hl: torch.Tensor, inv_scale: torch.Tensor, K: int):
        self.hl, self.inv_scale, self.K = hl, inv_scale, K
        self.rows = hl.shape[0]
        self.Kp = hl.shape[1] // 2


def split_rows(X: torch.Tensor, out: SplitOperand | None = None) -> SplitOperand:
    """A operand from activations X [M, K] (row stride >= K, f32)."""
    if X.dtype != torch.float32 or X.dim() != 2 or X.stride(1) != 1:
        raise ValueError("X must be a row-major f32 matrix")
    M, K = X.shape
    Kp = kpad(K)
    if out is None or out.rows < M or out.Kp != Kp:
        out = SplitOperand(torch.empty((M, 2 * Kp), dtype=torch.float16, device=X.device),
                           torch.empty(M, dtype=torch.float32, device=X.device), K)
    out.K = K
    _lib.call("ig_split_f16", X.data_ptr(), X.stride(0), M, K, 0, Kp, out.hl.data_ptr(),
              out.inv_scale.data_ptr(), _lib.stream_handle())
    return out


def split_weight(W: torch.Tensor) -> SplitOperand:
    """B operand from a weight W [K, N] (row-major f32): rows are W's columns."""
    if W.dtype != torch.float32 or W.dim() != 2 or W.stride(1) != 1:
        raise ValueError("W must be a row-major f32 matrix")
    K, N = W.shape
    Kp = kpad(K)
    op = SplitOperand(torch.empty((N, 2 * Kp), dtype=torch.float16, device=W.device),
                      torch.empty(N, dtype=torch.float32, device=W.device), K)
    _lib.call("ig_split_f16", W.data_ptr(), W.stride(0), K, N, 1, Kp, op.hl.data_ptr(),
              op.inv_scale.data_ptr(), _lib.stream_handle())
    return op


def gemm(A: SplitOperand, B: SplitOperand, out: torch.Tensor | None = None, *, M: int | None = None,
         epilogue: int = 0, R: torch.Tensor | None = None, max_ctas: int = 0) -> torch.Tensor:
    """out[:M] = A @ B^T (= X @ W), epilogue 1: ReLU, 2: + R."""
    if A.Kp != B.Kp or A.K != B.K:
        raise ValueError("operand K mismatch")
    M = A.rows if M is None else M
    N = B.rows
    if out is None:
        out = torch.empty((M, N), dtype=torch.float32, device=A.hl.device)
    if out.stride(1) != 1 or out.shape[0] < M or out.shape[1] != N:
        raise ValueError("bad output")
    if epilogue == 2 and (R is None or R.stride(1) != 1):
        raise ValueError("epilogue 2 needs a row-major residual")
    _lib.call("ig_gemm_tc05", A.hl.data_ptr(), A.inv_scale.data_ptr(), B.hl.data_ptr(),
              B.inv_scale.data_ptr(), M, N, A.K, A.Kp, out.data_ptr(), out.stride(0),
              _lib.ptr(R) if R is not None else None, R.stride(0) if R is not None else 0, epilogue,
              max_ctas, _lib.stream_handle())
    return out


def matmul(X: torch.Tensor, W: torch.Tensor, epilogue: int = 0, R: torch.Tensor | None = None,
           out: torch.Tensor | None = None) -> torch.Tensor:
    """X @ W (+ epilogue) in f32-level precision on tcgen05."""
    return gemm(split_rows(X), split_weight(W), out, epilogue=epilogue, R=R)
