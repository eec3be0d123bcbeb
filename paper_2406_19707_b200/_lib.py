"""ctypes binding of libinfinigen_b200.so (the C ABI in include/infinigen_b200.h).

There is no fallback: if the library or a CUDA device is missing, every
operator raises.  Statuses map onto the reference's exception classes
(include/infinigen_b200.h, "IG_E*" comments).
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libinfinigen_b200.so")

IG_OK, IG_EINVAL, IG_ERANGE, IG_ECONSISTENCY, IG_ENOMEM, IG_ECUDA = 0, 1, 2, 3, 4, 1000
ELT = {"f32": 0, "f16": 1, "bf16": 2}
ELT_BYTES = {"f32": 4, "f16": 2, "bf16": 2}
POLICY = {"fifo": 0, "lru": 1, "counter": 2}

_P = ctypes.c_void_p
_I = ctypes.c_int
_F = ctypes.c_float
_D = ctypes.c_double
_SZ = ctypes.c_size_t
_I64 = ctypes.c_int64

# name -> argtypes (all return int status)
_SIGS = {
    "ig_abi_version": [],
    "ig_host_alloc": [_SZ, ctypes.POINTER(_P), ctypes.POINTER(_P)],
    "ig_host_free": [_P],
    "ig_host_numa_node": [_P, ctypes.POINTER(_I)],
    "ig_rehearse": [_P, _I, _P, _P, _P, _I, _I, _I, _I, _I, _F, _P, _P, _P],
    "ig_rehearse_count": [_P, _I, _P, _P, _P, _I, _I, _I, _I, _I, _F, _D, _P, _P, _P, _P, _P, _P, _P],
    "ig_count": [_P, _P, _P, _I, _I, _I, _D, _P, _P, _P],
    "ig_select": [_P, _P, _P, _I, _I, _I, _I, _I, _D, _I, _P, _P, _P, _P, _P],
    "ig_select_plan": [_P, _P, _P, _I, _I, _I, _I, _I, _D, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "ig_order_by_score": [_P, _P, _I, _I, _I, _I, _P, _P],
    "ig_topk_rows": [_P, _I, _I, _I, _P, _P],
    "ig_fetch": [_P, _P, _P, _I, _I, _I, _I, _I, _P, _I, _I, _P],
    "ig_fetch_tma": [_P, _P, _P, _P, _I, _I, _I, _I, _I, _P, _I, _I, _I, _P],
    "ig_fetch_all": [_P, _I, _I, _I, _I, _I, _P, _I, _P],
    "ig_append": [_P, _P, _I, _P, _I, _P, _P, _I, _P, _P, _P, _I, _I, _P, _P, _I, _P, _I, _I,
                  _I, _I, _P, _P, _P],
    "ig_evict_select": [_P, _P, _P, _I, _P, _I, _I, _I, _P, _P],
    "ig_touch": [_P, _P, _I, _P, _I, _I, _I, _I64, _P, _P, _P],
    "ig_score_max": [_P, _P, _I, _I, _I, _P, _P],
    "ig_attend_scratch": [_I, _I, _I, _I, ctypes.POINTER(_SZ), ctypes.POINTER(_SZ)],
    "ig_attend": [_P, _I, _P, _P, _I, _P, _I, _P, _P, _P, _P, _I, _I, _I, _I, _P, _P, _P, _I, _P],
    "ig_attend_slots": [_P, _I, _P, _P, _I, _P, _I, _P, _P, _P, _P, _I, _I, _I, _I, _P, _P, _P, _I,
                        _P],
    "ig_resident_plan": [_P, _P, _P, _P, _P, _I, _I, _I, _P, _P, _P, _P, _P],
    "ig_fetch_slots": [_P, _P, _P, _P, _I, _I, _I, _I, _I, _P, _P],
    "ig_stage_put": [_P, _P, _I, _P, _P, _I, _I, _I, _I, _I, _P],
    "ig_memcpy2d": [_P, _SZ, _P, _SZ, _SZ, _SZ, _P],
    "ig_sgemm_packed_sizes": [_I, _I, _I, ctypes.POINTER(_SZ), ctypes.POINTER(_SZ),
                              ctypes.POINTER(_SZ)],
    "ig_sgemm_pack": [_P, _I, _I, _I, _P, _P],
    "ig_peer_alloc": [_I, _I, ctypes.POINTER(_P), ctypes.POINTER(_P)],
    "ig_peer_free": [_P, _P],
    "ig_ipc_get_handle": [_P, _P],
    "ig_ipc_open_handle": [_P, ctypes.POINTER(_P)],
    "ig_ipc_close": [_P],
    "ig_allreduce_peer": [_P, _I, _P, _P, _I, _I, _P, _I, _I, _P, _P, _P, _P],
    "ig_allreduce_peer_i32": [_P, _I, _P, _P, _I, _I, _P, _I, _I, _P, _P, _P],
    "ig_sgemm_packed_peer": [_P, _I, _P, _I, _I, _I, _P, _P, _I, _I, _P, _I, _I, _P, _P, _SZ, _P, _SZ,
                             _P],
    "ig_allreduce_peer_sum": [_I, _P, _P, _I, _I, _P, _I, _I, _P, _P, _P],
    "ig_sgemm_packed": [_P, _I, _P, _I, _I, _P, _I, _P, _I, _I, _I, _P, _SZ, _P, _SZ, _P],
    "ig_step_advance": [_P, _P],
    "ig_layernorm": [_P, _P, _P, _F, _I, _I, _P, _P],
    "ig_split_f16": [_P, _I, _I, _I, _I, _I, _P, _P, _P],
    "ig_debug_attend_trace": [_P],
    "ig_prefill_attention_scratch": [_I, _I, _I, _I, ctypes.POINTER(_SZ)],
    "ig_prefill_attention": [_P, _I, _I, _I, _I, _I, _P, _P, _I, _P],
    "ig_gemm_tc05": [_P, _P, _P, _P, _I, _I, _I, _I, _P, _I, _P, _I, _I, _I, _P],
}
EXPORTS = tuple(_SIGS) + ("ig_status_string",)

_lock = threading.Lock()
_lib = None
launches = 0  # kernels enqueued through this binding (bench.py "gpu_launches")


class ArtifactConsistencyError(RuntimeError):
    """Partial key cache fell out of lock-step with its KV pool
    (reference speculation.py:37-38)."""


def load(require_gpu: bool = True) -> ctypes.CDLL:
    """Load the in-tree library; raise if it is missing (no fallback)."""
    global _lib
    import torch  # noqa: F401  (loads the CUDA runtime the library links against)
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                    "(this package has no CPU fallback)")
            lib = ctypes.CDLL(LIB_PATH)
            for name, args in _SIGS.items():
                fn = getattr(lib, name)
                fn.argtypes = args
                fn.restype = ctypes.c_int
            lib.ig_status_string.argtypes = [ctypes.c_int]
            lib.ig_status_string.restype = ctypes.c_char_p
            _lib = lib
    if require_gpu:
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2406_19707_b200 needs a CUDA device (no CPU fallback)")
    return _lib


def check(status: int, what: str) -> None:
    if status == IG_OK:
        return
    msg = f"{what}: {_lib.ig_status_string(status).decode()}"
    if status == IG_EINVAL:
        raise ValueError(msg)
    if status == IG_ERANGE:
        raise IndexError(msg)
    if status == IG_ECONSISTENCY:
        raise ArtifactConsistencyError(msg)
    if status == IG_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def call(name: str, *args, kernels: int = 1) -> None:
    """Invoke an ig_* entry point and raise on a non-OK status."""
    global launches
    lib = _lib if _lib is not None else load()
    check(getattr(lib, name)(*args), name)
    launches += kernels


def ptr(t) -> int:
    """Raw device pointer of a torch tensor (or None -> NULL)."""
    return None if t is None else t.data_ptr()


def stream_handle(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
