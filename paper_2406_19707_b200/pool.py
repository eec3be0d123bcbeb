"""Drop-in KvPool (reference pool.py:28-112) backed by the B200 pool kernels.

Rows live in pinned, mapped host memory (one fixed-capacity allocation instead
of the reference's grow-by-concatenation arrays); per-row metadata lives in
HBM.  append / fetch / evict_select run ig_append / ig_fetch + ig_touch /
(ig_append's victim scan), so the eviction semantics the engine uses are the
ones exercised here: FIFO / LRU / COUNTER argmin with the lowest index on ties,
8-bit saturating counters, "hit 255 -> halve all".
"""

from __future__ import annotations

from enum import Enum

import numpy as np

from . import _lib

COUNTER_MAX = 255


class EvictionPolicy(str, Enum):
    """pool.py:22-25."""
    FIFO = "fifo"
    LRU = "lru"
    COUNTER = "counter"


class KvPool:
    """One (layer, head, sequence) pool with the reference API.

    ``capacity`` bounds the rows this pool can ever hold (defaults to
    ``limit``, else 4096); the reference grows without bound.
    """

    def __init__(self, head_dim: int, limit: int | None = None,
                 policy: EvictionPolicy = EvictionPolicy.COUNTER, on_overwrite=None,
                 capacity: int | None = None, dtype: str = "f32"):
        if limit is not None and limit < 1:
            raise ValueError("limit must be >= 1 when set")
        import torch
        _lib.load()
        self._torch = torch
        self.head_dim, self.limit, self.policy = head_dim, limit, EvictionPolicy(policy)
        self.on_overwrite = on_overwrite
        self.dtype = dtype
        cap = capacity if capacity is not None else (limit if limit is not None else 4096)
        self.capacity = (cap + 3) // 4 * 4
        self.row_bytes = 2 * head_dim * _lib.ELT_BYTES[dtype]
        from .engine import HostPool
        self._host = HostPool(self.capacity * self.row_bytes)
        dev = torch.device("cuda")
        self._dev = dev
        self._arr = torch.zeros(self.capacity, dtype=torch.int64, device=dev)
        self._lf = torch.zeros(self.capacity, dtype=torch.int64, device=dev)
        self._ctr = torch.zeros(self.capacity, dtype=torch.uint8, device=dev)
        self._st = torch.zeros(8, dtype=torch.int32, device=dev)
        self._len = 0
        self._seq = 0

    def __len__(self) -> int:
        return self._len

    def _sync_state(self) -> None:
        st = np.zeros(8, np.int32)
        st[0], st[1] = self._len, self.limit or 0
        st[2:4] = np.array([self._seq], np.int64).view(np.int32)
        self._st.copy_(self._torch.from_numpy(st))

    # -- reference attributes -------------------------------------------------
    def _rows(self) -> np.ndarray:
        npdt = {"f32": np.float32, "f16": np.float16}[self.dtype]
        return self._host.numpy(npdt, (self.capacity, 2, self.head_dim))[: self._len]

    @property
    def keys(self) -> np.ndarray:
        self._torch.cuda.synchronize()
        return self._rows()[:, 0].astype(np.float32)

    @property
    def values(self) -> np.ndarray:
        self._torch.cuda.synchronize()
        return self._rows()[:, 1].astype(np.float32)

    @property
    def arrival_seq(self) -> np.ndarray:
        return self._arr[: self._len].cpu().numpy()

    @property
    def last_fetch_seq(self) -> np.ndarray:
        return self._lf[: self._len].cpu().numpy()

    @property
    def fetch_counter(self) -> np.ndarray:
        return self._ctr[: self._len].cpu().numpy()

    # -- operations -------------------------------------------------------------
    def append(self, k_row, v_row) -> int:
        """pool.py:53-81 via ig_append (fetch_mode 0)."""
        torch = self._torch
        k_row = np.asarray(k_row, dtype=np.float32).reshape(-1)
        v_row = np.asarray(v_row, dtype=np.float32).reshape(-1)
        if k_row.shape != (self.head_dim,) or v_row.shape != (self.head_dim,):
            raise ValueError(f"row dim mismatch: k={k_row.shape} v={v_row.shape}, "
                             f"expected ({self.head_dim},)")
        if (self.limit is None or self._len < self.limit) and self._len >= self.capacity:
            raise ValueError(f"pool capacity {self.capacity} exhausted")
        self._sync_state()
        kv = torch.from_numpy(np.stack([k_row, v_row])).to(self._dev)
        pos = torch.zeros(1, dtype=torch.int32, device=self._dev)
        ev = torch.zeros(2, dtype=torch.int64, device=self._dev)
        d = self.head_dim
        _lib.call("ig_append", kv.data_ptr(), kv.data_ptr() + 4 * d, d, self._host.dev,
                  _lib.ELT[self.dtype], None, None, 1, self._arr.data_ptr(), self._lf.data_ptr(),
                  self._ctr.data_ptr(), _lib.POLICY[self.policy.value], 0, None, None, 1,
                  self._st.data_ptr(), 1, 1, d, self.capacity, pos.data_ptr(), ev.data_ptr(),
                  _lib.stream_handle())
        p = int(pos.item())
        e = ev.cpu().numpy()
        if e[0] >= 0 and self.on_overwrite is not None:
            self.on_overwrite(int(e[0]), int(e[1]))
        self._seq += 1
        if p == self._len:
            self._len += 1
        return p

    def fetch(self, indices):
        """pool.py:83-99: gather in the given order (ig_fetch) and update the
        metadata of the (distinct) fetched rows (ig_touch)."""
        torch = self._torch
        idx = np.asarray(indices, dtype=np.int64).reshape(-1)
        if idx.size and (idx.min() < 0 or idx.max() >= len(self)):
            raise IndexError(f"fetch index out of range for pool of {len(self)} rows")
        self._seq += 1
        self._sync_state()
        d = self.head_dim
        out = torch.empty((max(idx.size, 1), 2 * d), dtype=torch.float32 if self.dtype == "f32"
                          else torch.float16, device=self._dev)
        hs = _lib.stream_handle()
        if idx.size:
            di = torch.from_numpy(idx.astype(np.int32)).to(self._dev)
            nn = torch.tensor([idx.size], dtype=torch.int32, device=self._dev)
            _lib.call("ig_fetch", self._host.dev, di.data_ptr(), nn.data_ptr(), 1, 1,
                      self.capacity, idx.size, self.row_bytes, out.data_ptr(), 1, 256, hs)
            uniq = np.unique(idx).astype(np.int32)   # numpy fancy-index assignment: once per row
            du = torch.from_numpy(uniq).to(self._dev)
            nu = torch.tensor([uniq.size], dtype=torch.int32, device=self._dev)
            _lib.call("ig_touch", du.data_ptr(), nu.data_ptr(), uniq.size, self._st.data_ptr(), 1, 1,
                      self.capacity, self._seq, self._lf.data_ptr(), self._ctr.data_ptr(), hs)
        rows = out[: idx.size].float().cpu().numpy()
        return rows[:, :d].copy(), rows[:, d:].copy()

    def evict_select(self) -> int:
        """pool.py:101-109: argmin of the policy key, lowest index on ties."""
        if len(self) == 0:
            raise ValueError("cannot select a victim from an empty pool")
        self._sync_state()
        out = self._torch.zeros(1, dtype=self._torch.int32, device=self._dev)
        _lib.call("ig_evict_select", self._arr.data_ptr(), self._lf.data_ptr(), self._ctr.data_ptr(),
                  _lib.POLICY[self.policy.value], self._st.data_ptr(), 1, 1, self.capacity,
                  out.data_ptr(), _lib.stream_handle())
        return int(out.item())

    def all_indices(self) -> np.ndarray:
        return np.arange(len(self), dtype=np.int64)

    def close(self) -> None:
        self._host.close()
