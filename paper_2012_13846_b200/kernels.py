"""Coordinate index on the GPU — the `VOXPIPE_BACKEND` seam of the reference
(kernels.py:21-32 selects `_ACTIVE` from {_kernels, _kernels_py}).

`build_table` / `lookup` keep the exact contract of `_kernels.pyx:24-73`
(int64 keys in, opaque pair out, int64 rows with -1 misses out, first
occurrence of a duplicated key wins), so this module can be dropped in as a
third backend ("cuda"): see INTEGRATION.md for the two-line change to the
reference's kernels.py.  The table lives in device memory; the opaque pair
is (device table tensor, capacity).
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .errors import ValidationError
from .tensor import default_device

_FIELD_BITS = 16
_AXIS_BIAS = 1 << (_FIELD_BITS - 1)
_AXIS_MIN = -_AXIS_BIAS
_AXIS_MAX = _AXIS_BIAS - 1
_BATCH_MAX = (1 << _FIELD_BITS) - 1
MAX_PACKED_DIM = 3


def backend_name() -> str:
    return "cuda"


def _as_device_i64(a, device) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to(device=device, dtype=torch.int64).contiguous()
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.int64)).to(device)


def build_table(keys):
    """_kernels.pyx:24-47 — returns the opaque (table, capacity) pair."""
    device = default_device()
    k = _as_device_i64(keys, device)
    n = k.shape[0]
    cap = int(_lib.query("vp_hash_capacity", n))
    table = torch.empty(int(_lib.query("vp_hash_bytes", cap)), dtype=torch.uint8, device=device)
    _lib.call("vp_hash_build", k.data_ptr() if n else None, None, n, table.data_ptr(), cap, _lib.stream())
    return table, cap


def lookup(table, cap, queries):
    """_kernels.pyx:50-73 — int64 rows per query, -1 where absent.  Returns a
    host numpy array when `queries` is host data (the seam contract), else a
    device tensor."""
    on_host = not isinstance(queries, torch.Tensor) or not queries.is_cuda
    q = _as_device_i64(queries, table.device)
    m = q.shape[0]
    rows = torch.empty(max(m, 1), dtype=torch.int64, device=table.device)
    if m:
        _lib.call("vp_hash_lookup", table.data_ptr(), cap, q.data_ptr(), m, rows.data_ptr(), _lib.stream())
    rows = rows[:m]
    return rows.cpu().numpy() if on_host else rows


def packable_dim(dim: int) -> bool:
    return 1 <= dim <= MAX_PACKED_DIM


def pack_rows(rows):
    """kernels.py:53-79 — (N, 1+D) rows -> int64 keys (device pack for D=3)."""
    on_host = not isinstance(rows, torch.Tensor) or not rows.is_cuda
    r = rows if isinstance(rows, torch.Tensor) else torch.as_tensor(np.asarray(rows, dtype=np.int64))
    if r.dim() != 2:
        raise ValidationError("coordinate rows must be a 2-D array")
    dim = r.shape[1] - 1
    if not packable_dim(dim):
        raise ValidationError(f"packing supports 1..{MAX_PACKED_DIM} axes, got {dim}")
    if r.shape[0] == 0:
        return np.empty(0, dtype=np.int64) if on_host else torch.empty(0, dtype=torch.int64, device=r.device)
    b, ax = r[:, 0], r[:, 1:]
    if int(b.min()) < 0 or int(b.max()) > _BATCH_MAX:
        raise ValidationError(f"batch index out of packable range [0, {_BATCH_MAX}]")
    if int(ax.min()) < _AXIS_MIN or int(ax.max()) > _AXIS_MAX:
        raise ValidationError(f"coordinate axis out of packable range [{_AXIS_MIN}, {_AXIS_MAX}]")
    device = default_device()
    if dim == 3:
        c4 = r.to(device=device, dtype=torch.int32).contiguous()
        keys = torch.empty(c4.shape[0], dtype=torch.int64, device=device)
        _lib.call("vp_pack_coords", c4.data_ptr(), c4.shape[0], keys.data_ptr(), None, _lib.stream())
    else:  # D < 3: same fields, fewer of them (kernels.py:75-78)
        rr = r.to(device=device, dtype=torch.int64)
        keys = rr[:, 0].clone()
        for d in range(dim):
            keys = (keys << _FIELD_BITS) | (rr[:, 1 + d] + _AXIS_BIAS)
    return keys.cpu().numpy() if on_host else keys


class CoordIndex:
    """Row lookup over packed int64 coordinate keys (kernels.py:82-92)."""

    def __init__(self, keys):
        self._a, self._b = build_table(keys)

    def lookup(self, queries):
        return lookup(self._a, self._b, queries)


class _PackedRowIndex:
    """kernels.py:125-148 — packs query rows itself; out-of-range rows miss."""

    def __init__(self, rows):
        self._index = CoordIndex(pack_rows(rows))

    def lookup(self, rows):
        on_host = not isinstance(rows, torch.Tensor) or not rows.is_cuda
        r = rows if isinstance(rows, torch.Tensor) else torch.as_tensor(np.asarray(rows, dtype=np.int64))
        r = r.to(self._index._a.device, torch.int64)
        if r.shape[0] == 0:
            out = torch.empty(0, dtype=torch.int64, device=r.device)
            return out.cpu().numpy() if on_host else out
        ok = ((r[:, 0] >= 0) & (r[:, 0] <= _BATCH_MAX) & (r[:, 1:] >= _AXIS_MIN).all(1)
              & (r[:, 1:] <= _AXIS_MAX).all(1))
        out = torch.full((r.shape[0],), -1, dtype=torch.int64, device=r.device)
        if bool(ok.any()):
            out[ok] = self._index.lookup(pack_rows(r[ok]))
        return out.cpu().numpy() if on_host else out


def coord_index(rows):
    """kernels.py:113-122 — the GPU index requires packable rows."""
    return _PackedRowIndex(rows)
