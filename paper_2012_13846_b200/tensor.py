"""Sparse tensors on the GPU — the reference's `voxpipe.tensor` API
(tensor.py:1-301) with device-resident storage.

Storage (B200 layout): coordinates are int32 rows
[batch, x, y, z] (16 B per row; D < 3 pads the unused axes with 0 so every
kernel sees one layout), features are row-major bf16 (tensor-core path) or
fp32 on the device.  `coords` exposes the (N, 1+D) view the reference
exposes; `coords4` is the padded (N, 4) storage the kernels read.

Every check the reference's constructor performs (tensor.py:49-78) runs on
the GPU (one flag word read back); duplicate detection is a hash insert
instead of np.unique.

Two coordinate storages, chosen per tensor:
  * packed (the fast path): int32 (N, 4), every axis in [-16384, 16383] and
    batch <= 65535 — strided outputs and every neighbour query then stay
    inside the reference's packed 64-bit key (kernels.py:40-78);
  * wide: int64 (N, 1+D) for D > 3 axes or coordinates beyond that range —
    the reference's TupleCoordIndex fallback (kernels.py:95-122), served by
    the vp_wide_* kernels (whole-tuple hash).  `coords4` then holds the
    (N, 1+D) int64 rows.
"""
from __future__ import annotations

import json
import struct
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib
from .errors import StructuralError, ValidationError

_BINARY_MAGIC = b"VXSP"
_BINARY_VERSION = 1


def default_device():
    if not torch.cuda.is_available():
        from .errors import ConfigError

        raise ConfigError("voxpipe_b200 needs a CUDA device (B200, sm_100a); none is visible")
    return torch.device("cuda", torch.cuda.current_device())


PACKED_AXIS_MIN, PACKED_AXIS_MAX, PACKED_BATCH_MAX = -16384, 16383, 65535
MAX_AXES = 7  # wide rows: batch + up to 7 axes


def is_wide(c: torch.Tensor) -> bool:
    """Wide storage = int64 rows (N, 1+D); packed = int32 (N, 4)."""
    return c.dtype == torch.int64


def pad_coords(coords, device=None) -> tuple[torch.Tensor, int]:
    """(N, 1+D) int rows -> (storage on the device, D): packed int32 (N, 4)
    when D <= 3 and every value is inside the packed range, else wide int64
    (N, 1+D) rows (module docstring)."""
    if not isinstance(coords, torch.Tensor):
        a = np.asarray(coords, dtype=np.int64)
        # read-only arrays (the reference's SparseTensor marks its arrays so) are copied
        coords = torch.from_numpy(a if a.flags.writeable else a.copy())
    if coords.dim() != 2 or coords.shape[1] < 2:
        raise StructuralError("coords must have shape (N, 1+D) with D >= 1")
    dim = coords.shape[1] - 1
    if dim > MAX_AXES:
        raise ValidationError(f"at most {MAX_AXES} coordinate axes are supported, got {dim}")
    device = device or (coords.device if coords.is_cuda else default_device())
    if coords.dtype == torch.int32 and coords.shape[1] == 4 and coords.is_cuda:
        return coords.contiguous(), dim  # already packed storage (trusted callers)
    if coords.dtype.is_floating_point:
        raise ValidationError("coordinates must be integers")
    wide = dim > 3
    if not wide and coords.numel():
        c64 = coords.to(torch.int64)
        ax = c64[:, 1:]
        wide = bool(ax.min() < PACKED_AXIS_MIN) or bool(ax.max() > PACKED_AXIS_MAX) or bool(
            c64[:, 0].max() > PACKED_BATCH_MAX)
    if wide:
        return coords.to(device=device, dtype=torch.int64).contiguous(), dim
    coords = coords.to(device=device, dtype=torch.int32)
    if dim == 3:
        return coords.contiguous(), dim
    c4 = torch.zeros((coords.shape[0], 4), dtype=torch.int32, device=device)
    c4[:, : 1 + dim] = coords
    return c4, dim


def widen(c: torch.Tensor, dim: int) -> torch.Tensor:
    """Packed (N, 4) int32 -> wide (N, 1+D) int64 (identity on wide rows)."""
    return c if is_wide(c) else c[:, : 1 + dim].to(torch.int64).contiguous()


def _to_features(features, device) -> torch.Tensor:
    if not isinstance(features, torch.Tensor):
        features = torch.as_tensor(np.asarray(features, dtype=np.float64)).to(torch.float32)
    if features.dtype not in (torch.float32, torch.bfloat16, torch.float64):
        features = features.to(torch.float32)
    return features.to(device).contiguous()


def validate(coords4: torch.Tensor, features: Optional[torch.Tensor], stride: tuple[int, ...], dim: int):
    """tensor.py:49-78 invariants, evaluated on the GPU."""
    n = coords4.shape[0]
    flags = torch.zeros(1, dtype=torch.int32, device=coords4.device)
    st = _lib.stream()
    if n and is_wide(coords4):
        ws = _lib.workspace(_lib.query("vp_wide_ws_bytes", n, 0, dim + 1, 1), coords4.device)
        _lib.call("vp_wide_validate", coords4.data_ptr(), n, dim + 1, _lib.i64_array(stride), flags.data_ptr(),
                  ws.data_ptr(), ws.numel(), st)
    elif n:
        ts = tuple(stride) + (1,) * (3 - dim)
        ws = _lib.workspace(_lib.query("vp_validate_coords_ws_bytes", n), coords4.device)
        _lib.call("vp_validate_coords", coords4.data_ptr(), None, n, _lib.i32_array(ts), flags.data_ptr(),
                  ws.data_ptr(), ws.numel(), st)
    if features is not None and features.numel():
        _lib.call("vp_check_finite", features.data_ptr(), _lib.dtype_code(features), features.numel(),
                  flags.data_ptr(), st)
    f = int(flags.item())
    if f & 8:
        raise ValidationError("coordinate out of packable range (batch [0, 65535], axes [-32768, 32767])")
    if f & 2:
        raise ValidationError("batch indices must be non-negative")
    if f & 4:
        raise ValidationError("coordinate axes must be multiples of the tensor stride")
    if f & 16:
        raise ValidationError("features must be finite")
    if f & 1:
        raise StructuralError("duplicate (batch, coords) rows")


class SparseTensor:
    """Immutable (coords, features) pair with tensor-stride bookkeeping
    (tensor.py:36-100), device resident."""

    __slots__ = ("coords4", "features", "tensor_stride", "dim", "plans")

    def __init__(self, coords, features, tensor_stride, *, _trusted: bool = False, _dim: Optional[int] = None,
                 _plans: Optional[dict] = None):
        # plans: the coordinate bookkeeping derived from these rows (output
        # coordinates, kernel maps, sorted tables per (stride, kernel shape)),
        # shared by every tensor on the same coordinates (nn.py) — the role
        # of MinkowskiEngine's coordinate manager
        self.plans = {} if _plans is None else _plans
        if _trusted:
            self.coords4 = coords
            self.dim = _dim if _dim is not None else 3
            self.features = features
            self.tensor_stride = tuple(int(s) for s in tensor_stride)
            return
        c4, dim = pad_coords(coords)
        feats = _to_features(features, c4.device)
        if feats.dim() != 2:
            raise StructuralError("features must have shape (N, D_f)")
        if c4.shape[0] != feats.shape[0]:
            raise StructuralError("coords and features row counts differ")
        stride = tuple(int(s) for s in tensor_stride)
        if len(stride) != dim:
            raise StructuralError("tensor_stride length must equal D")
        if any(s < 1 for s in stride):
            raise ValidationError("tensor_stride entries must be positive")
        validate(c4, feats, stride, dim)
        self.coords4, self.features, self.tensor_stride, self.dim = c4, feats, stride, dim

    @property
    def coords(self) -> torch.Tensor:
        return self.coords4 if is_wide(self.coords4) else self.coords4[:, : 1 + self.dim]

    @property
    def wide(self) -> bool:
        return is_wide(self.coords4)

    @property
    def feature_width(self) -> int:
        return self.features.shape[1]

    @property
    def device(self):
        return self.coords4.device

    def __len__(self) -> int:
        return self.coords4.shape[0]

    def __eq__(self, other) -> bool:
        if not isinstance(other, SparseTensor):
            return NotImplemented
        return (
            self.tensor_stride == other.tensor_stride
            and self.dim == other.dim
            and tuple(self.coords4.shape) == tuple(other.coords4.shape)
            and tuple(self.features.shape) == tuple(other.features.shape)
            and bool(torch.equal(self.coords4, other.coords4))
            and bool(torch.equal(self.features.float(), other.features.float()))
        )

    __hash__ = None

    def with_features(self, features: torch.Tensor) -> "SparseTensor":
        if features.shape[0] != len(self):
            raise StructuralError("coords and features row counts differ")
        return SparseTensor(self.coords4, features.contiguous(), self.tensor_stride, _trusted=True, _dim=self.dim,
                            _plans=self.plans)

    def to_numpy(self) -> tuple[np.ndarray, np.ndarray]:
        """(coords int64 (N, 1+D), features float64) as the reference stores them."""
        return (self.coords.to(torch.int64).cpu().numpy(), self.features.to(torch.float64).cpu().numpy())

    def __repr__(self):
        return (f"SparseTensor(N={len(self)}, D={self.dim}, D_f={self.feature_width}, "
                f"stride={self.tensor_stride}, dtype={self.features.dtype})")


@dataclass(frozen=True)
class PointCloud:
    """Raw points in world units with optional per-point features (tensor.py:103-129)."""

    points: object
    features: Optional[object] = None
    batch_index: int = 0

    def __post_init__(self):
        pts = self.points
        if not isinstance(pts, torch.Tensor):
            pts = torch.as_tensor(np.ascontiguousarray(pts, dtype=np.float64))
        if pts.dim() != 2 or pts.shape[1] < 1:
            raise StructuralError("points must have shape (N, D) with D >= 1")
        if pts.dtype not in (torch.float32, torch.float64):
            pts = pts.to(torch.float64)
        if pts.numel() and not bool(torch.isfinite(pts).all()):
            raise ValidationError("point components must be finite")
        feats = self.features
        if feats is not None:
            if not isinstance(feats, torch.Tensor):
                feats = torch.as_tensor(np.ascontiguousarray(feats, dtype=np.float64))
            if feats.dim() != 2 or feats.shape[0] != pts.shape[0]:
                raise StructuralError("features must be (N, D_f) matching points")
            if feats.numel() and not bool(torch.isfinite(feats).all()):
                raise ValidationError("point features must be finite")
        if self.batch_index < 0:
            raise ValidationError("batch_index must be non-negative")
        object.__setattr__(self, "points", pts)
        object.__setattr__(self, "features", feats)


def voxelize_batch(points: torch.Tensor, cloud_offsets: torch.Tensor, voxel_size: float,
                   resolution: Sequence[int], feature_dtype=torch.float32,
                   return_point_map: bool = False):
    """Fused voxelize (tensor.py:147-184) + batch (tensor.py:205-229) on the
    GPU: points (n, 3) f32/f64 of B clouds delimited by int64 offsets (B+1),
    occupancy features.  Rows are bit-identical to
    batch([voxelize(PointCloud(p_i), voxel_size, resolution) for i]).
    """
    if voxel_size <= 0:
        raise ValidationError("voxel_size must be positive")
    res = [int(r) for r in resolution]
    if len(res) != 3 or min(res) < 1:
        raise ValidationError("resolution must list D positive integers")
    device = points.device if points.is_cuda else default_device()
    points = points.to(device).contiguous()
    offs = cloud_offsets.to(device=device, dtype=torch.int64).contiguous()
    n = points.shape[0]
    nb = offs.shape[0] - 1
    coords = torch.empty((max(n, 1), 4), dtype=torch.int32, device=device)
    n_out = torch.empty(1, dtype=torch.int32, device=device)
    feats = torch.empty((max(n, 1), 1), dtype=feature_dtype, device=device)
    p2v = torch.empty(max(n, 1), dtype=torch.int32, device=device) if return_point_map else None
    ws = _lib.workspace(_lib.query("vp_voxelize_ws_bytes", n), device)
    _lib.call("vp_voxelize", points.data_ptr(), _lib.dtype_code(points), n, offs.data_ptr(), nb, float(voxel_size),
              _lib.i32_array(res), coords.data_ptr(), n_out.data_ptr(), _lib.ptr(p2v), feats.data_ptr(),
              _lib.dtype_code(feats), ws.data_ptr(), ws.numel(), _lib.stream())
    m = int(n_out.item())
    t = SparseTensor(coords[:m], feats[:m], (1, 1, 1), _trusted=True, _dim=3)
    return (t, p2v) if return_point_map else t


def voxelize(cloud: PointCloud, voxel_size: float, resolution: Sequence[int]) -> SparseTensor:
    """tensor.py:147-184 on the GPU.  Mean-merged features use a deterministic
    point-order f64 sum (vp_voxel_mean), occupancy 1.0 otherwise."""
    if voxel_size <= 0:
        raise ValidationError("voxel_size must be positive")
    dim = cloud.points.shape[1]
    res = [int(r) for r in resolution]
    if len(res) != dim or min(res) < 1:
        raise ValidationError("resolution must list D positive integers")
    if dim > 3:
        raise ValidationError("the GPU path supports 1..3 axes")
    device = default_device()
    pts = cloud.points
    n = pts.shape[0]
    fw = 1 if cloud.features is None else cloud.features.shape[1]
    if n == 0:
        return SparseTensor(torch.empty((0, 4), dtype=torch.int32, device=device),
                            torch.empty((0, fw), dtype=torch.float32, device=device), (1,) * dim,
                            _trusted=True, _dim=dim)
    p3 = torch.zeros((n, 3), dtype=pts.dtype)
    p3[:, :dim] = pts
    res3 = res + [1] * (3 - dim)
    offs = torch.tensor([0, n], dtype=torch.int64)
    t, p2v = voxelize_batch(p3.to(device), offs, voxel_size, res3, return_point_map=True)
    coords4 = t.coords4.clone()
    if cloud.batch_index:
        coords4[:, 0] = int(cloud.batch_index)
    feats = t.features
    if cloud.features is not None:
        f = cloud.features.to(device).contiguous()
        if f.dtype not in (torch.float32, torch.float64):
            f = f.to(torch.float64)
        m = len(t)
        out = torch.empty((m, fw), dtype=torch.float32, device=device)
        n_vox = torch.tensor([m], dtype=torch.int32, device=device)
        ws = _lib.workspace(_lib.query("vp_voxel_mean_ws_bytes", n, m), device)
        _lib.call("vp_voxel_mean", f.data_ptr(), _lib.dtype_code(f), n, fw, p2v.data_ptr(), n_vox.data_ptr(), m,
                  out.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream())
        feats = out
    return SparseTensor(coords4, feats, (1,) * dim, _trusted=True, _dim=dim)


def dropout(t: SparseTensor, keep_ratio: float, seed: int) -> SparseTensor:
    """tensor.py:187-202 — same numpy PCG64 row choice (host), gather on device."""
    if not 0 < keep_ratio <= 1:
        raise ValidationError("keep_ratio must be in (0, 1]")
    n = len(t)
    if n == 0 or keep_ratio == 1:
        return t
    keep = int(np.ceil(keep_ratio * n))
    chosen = np.sort(np.random.default_rng(seed).choice(n, size=keep, replace=False))
    idx = torch.as_tensor(chosen, device=t.device)
    return SparseTensor(t.coords4[idx].contiguous(), t.features[idx].contiguous(), t.tensor_stride,
                        _trusted=True, _dim=t.dim)


def batch(tensors: Sequence[SparseTensor]) -> SparseTensor:
    """tensor.py:205-229 — concatenate, batch index = input position,
    duplicate rows raise StructuralError."""
    if not tensors:
        raise StructuralError("batch() needs at least one tensor")
    t0 = tensors[0]
    for t in tensors[1:]:
        if t.dim != t0.dim or t.feature_width != t0.feature_width or t.tensor_stride != t0.tensor_stride:
            raise StructuralError("batched tensors must share D, D_f and stride")
    wide = any(t.wide for t in tensors) or len(tensors) - 1 > PACKED_BATCH_MAX
    cs = []
    for i, t in enumerate(tensors):
        c = widen(t.coords4, t.dim).clone() if wide else t.coords4.clone()
        c[:, 0] = i
        cs.append(c)
    coords = torch.cat(cs, 0)
    dt = torch.float32 if any(t.features.dtype == torch.float32 for t in tensors) else t0.features.dtype
    feats = torch.cat([t.features.to(dt) for t in tensors], 0)
    try:
        validate(coords, None, t0.tensor_stride, t0.dim)
    except StructuralError as exc:
        raise StructuralError(f"batching produced duplicate rows: {exc}") from exc
    return SparseTensor(coords, feats, t0.tensor_stride, _trusted=True, _dim=t0.dim)


def split_batches(t: SparseTensor) -> list[SparseTensor]:
    """tensor.py:232-242 — one tensor per batch index, rows in stored order."""
    out = []
    if len(t) == 0:
        return out
    b = t.coords4[:, 0]
    for i in range(int(b.max().item()) + 1):
        mask = b == i
        c = t.coords4[mask].clone()
        c[:, 0] = 0
        out.append(SparseTensor(c, t.features[mask].contiguous(), t.tensor_stride, _trusted=True, _dim=t.dim))
    return out


def to_json(t: SparseTensor) -> str:
    """tensor.py:245-254 interchange JSON."""
    c, f = t.to_numpy()
    return json.dumps({"dim": t.dim, "feature_width": t.feature_width, "tensor_stride": list(t.tensor_stride),
                       "coords": c.tolist(), "features": f.tolist()})


def from_json(text: str) -> SparseTensor:
    obj = json.loads(text)
    try:
        dim = int(obj["dim"])
        width = int(obj["feature_width"])
        stride = tuple(int(s) for s in obj["tensor_stride"])
        coords = np.asarray(obj["coords"], dtype=np.int64).reshape(-1, 1 + dim)
        feats = np.asarray(obj["features"], dtype=np.float64).reshape(-1, width)
    except (KeyError, TypeError, ValueError) as exc:
        raise ValidationError(f"malformed sparse tensor JSON: {exc}") from exc
    return SparseTensor(coords, feats, stride)


def to_binary(t: SparseTensor) -> bytes:
    """tensor.py:270-278 little-endian binary (f64 features, int64 coords)."""
    c, f = t.to_numpy()
    header = struct.pack("<4sIIIQ", _BINARY_MAGIC, _BINARY_VERSION, t.dim, t.feature_width, len(t))
    return (header + np.asarray(t.tensor_stride, dtype="<i8").tobytes() + np.ascontiguousarray(c, "<i8").tobytes()
            + np.ascontiguousarray(f, "<f8").tobytes())


def binary_size(n: int, dim: int, width: int) -> int:
    """len(to_binary(t)) without materialising it (activation_bytes,
    profiling.py:450)."""
    return struct.calcsize("<4sIIIQ") + 8 * dim + 8 * n * (1 + dim) + 8 * n * width


def from_binary(blob: bytes) -> SparseTensor:
    head = struct.calcsize("<4sIIIQ")
    if len(blob) < head:
        raise ValidationError("binary sparse tensor truncated")
    magic, version, dim, width, n = struct.unpack("<4sIIIQ", blob[:head])
    if magic != _BINARY_MAGIC or version != _BINARY_VERSION:
        raise ValidationError("unrecognized binary sparse tensor header")
    off = head
    stride = np.frombuffer(blob, dtype="<i8", count=dim, offset=off)
    off += 8 * dim
    coords = np.frombuffer(blob, dtype="<i8", count=n * (1 + dim), offset=off)
    off += 8 * n * (1 + dim)
    feats = np.frombuffer(blob, dtype="<f8", count=n * width, offset=off)
    off += 8 * n * width
    if off != len(blob):
        raise ValidationError("binary sparse tensor has trailing bytes")
    return SparseTensor(coords.reshape(n, 1 + dim).copy(), feats.reshape(n, width).copy(),
                        tuple(int(s) for s in stride))
