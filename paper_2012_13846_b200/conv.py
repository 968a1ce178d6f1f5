"""Generalized sparse convolution on B200 — the reference's `voxpipe.conv`
API (conv.py:1-386) backed by the sm_100a kernels of libvoxpipe_b200.so.

Three steps (conv.py:1-8): output coordinates
(`vp_output_coords`), kernel map through a GPU hash (`vp_kernel_map`), and
the per-offset contraction as an output-stationary implicit GEMM on tcgen05
(`vp_conv_fwd` / `vp_conv_dgrad` / `vp_conv_wgrad`).  Kernel maps and output
coordinates are bit-exact with the reference; features/gradients agree within
the bf16/fp32 tolerances stated in DESIGN.md §6.

Precision: bf16 features take the tensor-core path (bf16 operands, fp32
accumulation, bf16 output); fp32 features take the fp32 SIMT path.  Weights
are fp32 masters ([K, C_out, C_in], conv.py:77-105 layout); the tensor-core
path reads a bf16 copy.
"""
from __future__ import annotations

import itertools
import json
import struct
import time
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from . import _lib
from .errors import StructuralError, ValidationError
from .tensor import SparseTensor, binary_size, is_wide, pad_coords, widen

_WEIGHTS_MAGIC = b"VXCW"
_WEIGHTS_VERSION = 1


@dataclass(frozen=True)
class KernelShape:
    """Set of integer offsets swept by the kernel (conv.py:33-74)."""

    dim: int
    extents: tuple
    offsets: np.ndarray  # (K, dim) int64, host

    def __post_init__(self):
        offsets = np.ascontiguousarray(self.offsets, dtype=np.int64)
        if offsets.ndim != 2 or offsets.shape[1] != self.dim:
            raise StructuralError("offsets must have shape (K, dim)")
        if len(np.unique(offsets, axis=0)) != len(offsets):
            raise StructuralError("kernel offsets must be distinct")
        offsets.setflags(write=False)
        object.__setattr__(self, "offsets", offsets)
        object.__setattr__(self, "extents", tuple(int(e) for e in self.extents))

    @classmethod
    def hypercubic(cls, dim: int, size) -> "KernelShape":
        """Full cross-product of centred per-axis offsets, itertools.product
        order (axis 0 slowest; conv.py:51-61)."""
        extents = (size,) * dim if isinstance(size, int) else tuple(size)
        if len(extents) != dim:
            raise StructuralError("need one extent per axis")
        if any(e < 1 or e % 2 == 0 for e in extents):
            raise ValidationError("hypercubic extents must be odd and positive")
        ranges = [range(-(e // 2), e // 2 + 1) for e in extents]
        return cls(dim, extents, np.array(list(itertools.product(*ranges)), dtype=np.int64).reshape(-1, dim))

    @classmethod
    def custom(cls, dim: int, offsets) -> "KernelShape":
        offsets = np.asarray(offsets, dtype=np.int64).reshape(-1, dim)
        extent = tuple(int(2 * np.abs(offsets[:, d]).max() + 1) if len(offsets) else 1 for d in range(dim))
        return cls(dim, extent, offsets)

    @property
    def num_offsets(self) -> int:
        return len(self.offsets)

    def offsets3(self) -> np.ndarray:
        o = np.zeros((self.num_offsets, 3), dtype=np.int32)
        o[:, : self.dim] = self.offsets
        return o

    def is_symmetric(self) -> bool:
        """offsets[K-1-k] == -offsets[k] (true for hypercubic shapes): the
        stride-1 inverse map is the column-flipped forward map."""
        return bool(np.array_equal(self.offsets[::-1], -self.offsets))


class ConvWeights:
    """One (n_out, n_in) matrix per kernel offset (conv.py:77-105), device
    resident: f64 when given f64 (the reference's precision, e.g. numpy
    arrays), else fp32 masters; `operand(dtype)` is the copy the kernels read
    for features of that dtype (bf16 for the tensor cores), cached until the
    masters change."""

    def __init__(self, matrices, device=None):
        if not isinstance(matrices, torch.Tensor):
            matrices = torch.as_tensor(np.ascontiguousarray(matrices, dtype=np.float64))
        if matrices.dim() != 3:
            raise StructuralError("weights must have shape (K, n_out, n_in)")
        from .tensor import default_device

        dt = torch.float64 if matrices.dtype == torch.float64 else torch.float32
        m = matrices.to(device=device or (matrices.device if matrices.is_cuda else default_device()),
                        dtype=dt).contiguous()
        if m.numel() and not bool(torch.isfinite(m).all()):
            raise ValidationError("weight entries must be finite")
        self.matrices = m
        self._ops: dict = {}

    def operand(self, dtype) -> torch.Tensor:
        """The weight operand for features of `dtype`: bf16 features -> bf16,
        fp32 -> fp32, f64 -> f64 (conversions cached per master version)."""
        dtype = torch.bfloat16 if dtype == torch.bfloat16 else (torch.float64 if dtype == torch.float64
                                                                 else torch.float32)
        if self.matrices.dtype == dtype:
            return self.matrices
        hit = self._ops.get(dtype)
        if hit is None or hit[0] != self.matrices._version:
            hit = (self.matrices._version, self.matrices.to(dtype).contiguous())
            self._ops[dtype] = hit
        return hit[1]

    @property
    def bf16(self) -> torch.Tensor:
        return self.operand(torch.bfloat16)

    @property
    def num_offsets(self) -> int:
        return self.matrices.shape[0]

    @property
    def n_out(self) -> int:
        return self.matrices.shape[1]

    @property
    def n_in(self) -> int:
        return self.matrices.shape[2]

    def nbytes(self) -> int:
        """Bytes of the reference's f64 matrices (conv.py:104-105)."""
        return int(self.matrices.numel() * 8)


@dataclass(eq=False)
class KernelMap:
    """Per-offset (input_row, output_row) links (conv.py:108-121).

    Device layout: `nbr` [N_out, K] int32 neighbour table (-1 = no neighbour)
    feeding the implicit GEMM, plus the pair lists in CSR form
    (`pair_in`/`pair_out` int32, `pair_ptr` [K+1]) in the reference's order:
    offset-major, out rows ascending within an offset.
    """

    offsets: np.ndarray
    nbr: torch.Tensor
    pair_in: torch.Tensor
    pair_out: torch.Tensor
    pair_ptr: torch.Tensor
    n_in: int = 0
    _ptr_host: Optional[np.ndarray] = field(default=None, repr=False)

    @property
    def ptr_host(self) -> np.ndarray:
        if self._ptr_host is None:
            self._ptr_host = self.pair_ptr.cpu().numpy().astype(np.int64)
        return self._ptr_host

    @property
    def pairs(self) -> tuple:
        """tuple of (in_rows, out_rows) int64 device tensors per offset."""
        p = self.ptr_host
        return tuple((self.pair_in[p[k]:p[k + 1]].to(torch.int64), self.pair_out[p[k]:p[k + 1]].to(torch.int64))
                     for k in range(len(p) - 1))

    def total_pairs(self) -> int:
        return int(self.ptr_host[-1])

    def inverse(self) -> torch.Tensor:
        """inv [N_in, K]: inv[v, k] = u for every pair (v, u) of offset k."""
        K = self.nbr.shape[1] if self.nbr.dim() == 2 else len(self.offsets)
        inv = torch.empty((max(self.n_in, 1), K), dtype=torch.int32, device=self.nbr.device)
        _lib.call("vp_kernel_map_inverse", self.nbr.data_ptr(), None, self.nbr.shape[0], K, inv.data_ptr(),
                  self.n_in, _lib.stream())
        return inv[: self.n_in]


def _stride3(stride, dim) -> tuple:
    st = (stride,) * dim if isinstance(stride, int) else tuple(int(s) for s in stride)
    if len(st) != dim or any(s < 1 for s in st):
        raise ValidationError("stride must list D positive integers")
    return st


def _output_coords4(coords4: torch.Tensor, tensor_stride: tuple, stride: tuple, dim: int):
    """generate_output_coords on the storage layout -> (coords_out, new_stride)."""
    new_stride = tuple(int(o) * int(s) for o, s in zip(tensor_stride, stride))
    if all(s == 1 for s in stride):
        return coords4.clone(), new_stride
    n = coords4.shape[0]
    if is_wide(coords4) or max(new_stride) > 16384:  # wide rows (kernels.py:95-122 fallback)
        return _output_coords_wide(coords4, new_stride, dim)
    if n == 0:
        return torch.empty((0, 4), dtype=torch.int32, device=coords4.device), new_stride
    out = torch.empty((n, 4), dtype=torch.int32, device=coords4.device)
    n_out = torch.empty(1, dtype=torch.int32, device=coords4.device)
    ws = _lib.workspace(_lib.query("vp_output_coords_ws_bytes", n), coords4.device)
    step = tuple(new_stride) + (1,) * (3 - dim)
    _lib.call("vp_output_coords", coords4.data_ptr(), None, n, _lib.i32_array(step), out.data_ptr(),
              n_out.data_ptr(), None, ws.data_ptr(), ws.numel(), _lib.stream())
    n_o = int(n_out.item())
    if n_o < 0:  # a floored row left the 16-bit packed range: the wide-row path
        return _output_coords_wide(coords4, new_stride, dim)
    return out[:n_o], new_stride


def _output_coords_wide(coords4: torch.Tensor, new_stride: tuple, dim: int):
    """generate_output_coords over wide int64 rows (vp_wide_output_coords)."""
    n = coords4.shape[0]
    c = widen(coords4, dim)
    if n == 0:
        return c.clone(), new_stride
    out = torch.empty_like(c)
    n_out = torch.empty(1, dtype=torch.int32, device=c.device)
    ws = _lib.workspace(_lib.query("vp_wide_ws_bytes", n, 0, dim + 1, 1), c.device)
    _lib.call("vp_wide_output_coords", c.data_ptr(), n, dim + 1, _lib.i64_array(new_stride), out.data_ptr(),
              n_out.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream())
    return out[: int(n_out.item())], new_stride


def generate_output_coords(t: SparseTensor, stride):
    """conv.py:124-146 — (coords (N_out, 1+D) int32 device, new tensor stride).
    Stride s > 1: floor-div by ts*s, rescale, unique rows in first-seen order."""
    st = _stride3(stride, t.dim)
    c4, ns = _output_coords4(t.coords4, t.tensor_stride, st, t.dim)
    return c4[:, : 1 + t.dim], ns


def _kernel_map4(in4: torch.Tensor, out4: torch.Tensor, shape: KernelShape, in_stride: tuple, dim: int,
                 with_pairs: bool = True) -> KernelMap:
    device = in4.device
    in4, out4 = in4.contiguous(), out4.contiguous()  # the C-ABI reads (N, 4) row-major rows
    K = shape.num_offsets
    if K > _lib.MAX_OFFSETS:
        raise ValidationError(f"at most {_lib.MAX_OFFSETS} kernel offsets are supported")
    n_in, n_out = in4.shape[0], out4.shape[0]
    if is_wide(in4) or is_wide(out4):
        return _kernel_map_wide(widen(in4, dim), widen(out4, dim), shape, in_stride, dim)
    if with_pairs and min(n_in, n_out) >= LATTICE_MIN_ROWS and dim == 3:
        km = _kernel_map_lattice(in4, out4, shape, in_stride)
        if km is not None:
            return km
    nbr = torch.empty((max(n_out, 1), K), dtype=torch.int32, device=device)
    cap_p = max(n_out * K, 1)
    pin = torch.empty(cap_p, dtype=torch.int32, device=device) if with_pairs else None
    pout = torch.empty(cap_p, dtype=torch.int32, device=device) if with_pairs else None
    pptr = torch.empty(K + 1, dtype=torch.int32, device=device)  # written by the map (0s when empty)
    ws = _lib.workspace(_lib.query("vp_kernel_map_ws_bytes", n_in, n_out, K), device)
    st3 = tuple(in_stride) + (1,) * (3 - dim)
    offs = shape.offsets3()
    _lib.call("vp_kernel_map", in4.data_ptr() if n_in else None, None, n_in, out4.data_ptr() if n_out else None, None,
              n_out, _lib.i32_array(offs.ravel()), K, _lib.i32_array(st3), nbr.data_ptr(), _lib.ptr(pin),
              _lib.ptr(pout), pptr.data_ptr() if with_pairs else None, ws.data_ptr(), ws.numel(), _lib.stream())
    if not with_pairs:
        pin = pout = torch.empty(0, dtype=torch.int32, device=device)
    return KernelMap(shape.offsets, nbr[:n_out], pin, pout, pptr, n_in=n_in)


# Large maps whose rows sit on a bounded lattice take the dense-grid index
# (vp_grid_set + vp_kernel_map_grid: occupancy bitmap + cell table, the unit
# cube column probe) instead of the open-addressing hash: 2.6x faster at 1M
# rows (tools/map_breakdown.py).  Deciding needs the rows' bounding box on
# the host (one small reduction + one sync), so small maps keep the hash.
LATTICE_MIN_ROWS = int(__import__("os").environ.get("VP_LATTICE_MIN_ROWS", 1 << 17))
LATTICE_MAX_BYTES = 2 << 30  # cell table + bitmap
_LATTICE_GRIDS: dict = {}


def _kernel_map_lattice(in4: torch.Tensor, out4: torch.Tensor, shape: KernelShape, in_stride: tuple):
    """-> KernelMap through the dense-grid index, or None when the rows do not
    sit on one bounded lattice of spacing in_stride (the hash path then runs).
    One bounding-box reduction (vp_coords_bbox) is read back; the set / probe /
    scan / emit / clear then go out in one C call (vp_kernel_map_lattice).
    Results are identical to the hash path (the same pairs and nbr)."""
    s = int(in_stride[0])
    if s < 1 or any(int(v) != s for v in in_stride[:3]):
        return None
    device = in4.device
    st = _lib.stream()
    n_in, n_out = in4.shape[0], out4.shape[0]
    K = shape.num_offsets
    bb = torch.empty(9, dtype=torch.int32, device=device)
    _lib.call("vp_coords_bbox", in4.data_ptr(), n_in, out4.data_ptr(), n_out, s, bb.data_ptr(), st)
    # outputs and workspace are allocated while the reduction runs
    nbr = torch.empty((n_out, K), dtype=torch.int32, device=device)
    pin = torch.empty(n_out * K, dtype=torch.int32, device=device)
    pout = torch.empty(n_out * K, dtype=torch.int32, device=device)
    pptr = torch.empty(K + 1, dtype=torch.int32, device=device)
    ws = _lib.workspace(_lib.query("vp_kernel_map_grid_ws_bytes", n_out, K), device)
    v = bb.cpu().tolist()
    if v[8] != 1 or v[0] < 0:
        return None
    org = [(lo // s) * s for lo in v[1:4]]
    hi = [-v[5], -v[6], -v[7]]
    B = -v[4] + 1
    R = max((hi[a] - org[a]) // s + 1 for a in range(3))
    words = int(_lib.query("vp_grid_words", B, R))
    if words <= 0 or B * R ** 3 >= (1 << 31) or 4 * words > LATTICE_MAX_BYTES:
        return None
    key = (str(device), B, R)
    grid = _LATTICE_GRIDS.get(key)
    if grid is None:
        _LATTICE_GRIDS.clear()  # one lattice kept per process (the most recent shape)
        grid = torch.zeros(words, dtype=torch.int32, device=device)  # zero bitmap == empty index
        _LATTICE_GRIDS[key] = grid
    _lib.call("vp_kernel_map_lattice", in4.data_ptr(), n_in, out4.data_ptr(), n_out,
              _lib.i32_array(shape.offsets3().ravel()), K, s, _lib.i32_array([B, R] + org), grid.data_ptr(),
              grid.numel(), nbr.data_ptr(), pin.data_ptr(), pout.data_ptr(), pptr.data_ptr(), ws.data_ptr(),
              ws.numel(), st)
    return KernelMap(shape.offsets, nbr, pin, pout, pptr, n_in=n_in)


def _kernel_map_wide(inw: torch.Tensor, outw: torch.Tensor, shape: KernelShape, in_stride: tuple,
                     dim: int) -> KernelMap:
    """Kernel map over wide int64 rows (vp_wide_kernel_map): the reference's
    TupleCoordIndex fallback (kernels.py:95-122) with the same pair order."""
    device = inw.device
    K = shape.num_offsets
    n_in, n_out = inw.shape[0], outw.shape[0]
    nbr = torch.empty((max(n_out, 1), K), dtype=torch.int32, device=device)
    cap_p = max(n_out * K, 1)
    pin = torch.empty(cap_p, dtype=torch.int32, device=device)
    pout = torch.empty(cap_p, dtype=torch.int32, device=device)
    pptr = torch.empty(K + 1, dtype=torch.int32, device=device)  # written by the map (0s when empty)
    ws = _lib.workspace(_lib.query("vp_wide_ws_bytes", n_in, n_out, dim + 1, K), device)
    offs = np.ascontiguousarray(shape.offsets, dtype=np.int64).ravel()
    _lib.call("vp_wide_kernel_map", inw.data_ptr() if n_in else None, n_in, outw.data_ptr() if n_out else None, n_out,
              dim + 1, _lib.i32_array(offs), K, _lib.i64_array(in_stride), nbr.data_ptr(), pin.data_ptr(),
              pout.data_ptr(), pptr.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream())
    return KernelMap(shape.offsets, nbr[:n_out], pin, pout, pptr, n_in=n_in)


def build_kernel_map(in_coords, out_coords, shape: KernelShape, in_stride) -> KernelMap:
    """conv.py:149-183 — pair (v, u) at offset k iff out[u] + off_k*in_stride
    == in[v] (batch equal).  One GPU hash over the input rows per call."""
    in4, dim = pad_coords(in_coords)
    out4, dim_o = pad_coords(out_coords, in4.device)
    if dim != dim_o or shape.dim != dim:
        raise StructuralError("coordinate / kernel dimensions differ")
    return _kernel_map4(in4, out4, shape, tuple(int(s) for s in in_stride), dim)


def _check_weights(t: SparseTensor, w: ConvWeights, shape: KernelShape):
    if w.num_offsets != shape.num_offsets:
        raise StructuralError("weights must supply one matrix per offset")
    if w.n_in != t.feature_width:
        raise StructuralError(f"weight n_in {w.n_in} != input feature width {t.feature_width}")
    if shape.dim != t.dim:
        raise StructuralError("kernel shape dimension != tensor dimension")


def sort_table(table: torch.Tensor, n_rows: int, key_mode: int = 0, sched_grid: int = 0):
    """Neighbour-pattern row grouping (vp_kernel_map_group): -> (perm,
    table[perm]) with rows grouped by a 9-bit key of their hit mask, so each
    128-row tile of the implicit GEMM touches few kernel offsets.  key_mode
    0 (columns) for neighbour tables, 1 (planes) for strided inverse tables.
    sched_grid > 0: whole 128-row tiles are then placed for a conv launched
    with that many CTAs (vp_kernel_map_group_sched; vp_conv_tc_grid gives the
    default config's count).  Results of the conv are unchanged."""
    K = table.shape[1]
    cap = max(n_rows, 1)
    perm = torch.empty(cap, dtype=torch.int32, device=table.device)
    ts = torch.empty((cap, K), dtype=torch.int32, device=table.device)
    if n_rows == 0:
        return perm[:0], ts[:0]
    ws = _lib.workspace(_lib.query("vp_kernel_map_sort_ws_bytes", n_rows, K), table.device)
    if n_rows >= FULL_MASK_ROWS and K <= 27:
        key_mode = 2  # large tables: the full 27-bit mask (three passes) groups best
    _lib.call("vp_kernel_map_group_sched", table.data_ptr(), None, n_rows, K, int(key_mode), int(sched_grid),
              perm.data_ptr(), ts.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream())
    return perm, ts


SORT_MIN_ROWS = 1 << 17  # below this the sort's launches cost more than it saves
FULL_MASK_ROWS = 1 << 18  # from here on the grouping sorts by the whole hit mask (key mode 2)


def _sortable(table: torch.Tensor) -> bool:
    return table.dim() == 2 and 1 <= table.shape[1] <= 30 and table.shape[0] >= SORT_MIN_ROWS


def _math_code(t: torch.Tensor, math: str) -> int:
    """Feature dtype code for the C-ABI: math="tf32" runs fp32 features on
    the tensor cores with tf32 multiplies (VP_TF32); "exact" keeps fp32 SIMT."""
    if math not in ("exact", "tf32"):
        raise ValidationError(f"math must be 'exact' or 'tf32', got {math!r}")
    if math == "tf32" and t.dtype == torch.float32:
        return _lib.VP_TF32
    return _lib.dtype_code(t)


def conv_forward_raw(x: torch.Tensor, w: ConvWeights, nbr: torch.Tensor, n_out: int, out_dtype=None,
                     flip: bool = False, perm: Optional[torch.Tensor] = None, math: str = "exact") -> torch.Tensor:
    """y[u] = sum_k W_k x[nbr[u, k]] for u < n_out (the gather-GEMM of Eq. 3).
    With `perm`, table row i holds the neighbours of output row perm[i]."""
    out_dtype = out_dtype or x.dtype
    K = w.num_offsets
    y = torch.empty((max(n_out, 1), w.n_out), dtype=out_dtype, device=x.device)
    wt = w.operand(x.dtype)
    ws = _lib.workspace(_lib.query("vp_conv_fwd_ws_bytes", w.n_in, w.n_out, K), x.device)
    _lib.call("vp_conv_fwd", x.data_ptr(), _math_code(x, math), max(x.shape[0], 1), w.n_in, wt.data_ptr(),
              _lib.dtype_code(wt), w.n_out,
              K, nbr.data_ptr(), int(flip), _lib.ptr(perm), None, n_out, y.data_ptr(), _lib.dtype_code(y),
              ws.data_ptr(), ws.numel(), _lib.stream())
    return y[:n_out]


def conv_dgrad_raw(g: torch.Tensor, w: ConvWeights, table: torch.Tensor, n_in: int, flip: bool,
                   out_dtype=None, perm: Optional[torch.Tensor] = None, math: str = "exact") -> torch.Tensor:
    """grad_in[v] = sum_k W_k^T g[table[v, k]] (conv.py:240)."""
    out_dtype = out_dtype or g.dtype
    K = w.num_offsets
    gi = torch.empty((max(n_in, 1), w.n_in), dtype=out_dtype, device=g.device)
    wt = w.operand(g.dtype)
    ws = _lib.workspace(_lib.query("vp_conv_dgrad_ws_bytes", w.n_in, w.n_out, K), g.device)
    _lib.call("vp_conv_dgrad", g.data_ptr(), _math_code(g, math), max(g.shape[0], 1), w.n_out, wt.data_ptr(),
              _lib.dtype_code(wt),
              w.n_in, K, table.data_ptr(), int(flip), _lib.ptr(perm), None, n_in, gi.data_ptr(), _lib.dtype_code(gi),
              ws.data_ptr(), ws.numel(), _lib.stream())
    return gi[:n_in]


def conv_wgrad_raw(x: torch.Tensor, g: torch.Tensor, w_shape: tuple, kmap: KernelMap) -> torch.Tensor:
    """grad_w[k] = sum over pairs (v, u) of offset k of g[u] x[v]^T (conv.py:241),
    fp32 (f64 for f64 features)."""
    K, n_out_c, n_in_c = w_shape
    gdt = torch.float64 if x.dtype == torch.float64 else torch.float32
    gw = torch.empty((K, n_out_c, n_in_c), dtype=gdt, device=x.device)
    cap_pairs = max(int(kmap.pair_in.numel()), 1)
    ws = _lib.workspace(_lib.query("vp_conv_wgrad_ws_bytes", n_in_c, n_out_c, K, cap_pairs), x.device)
    _lib.call("vp_conv_wgrad", x.data_ptr(), _lib.dtype_code(x), n_in_c, g.data_ptr(), _lib.dtype_code(g), n_out_c,
              K, kmap.pair_in.data_ptr(), kmap.pair_out.data_ptr(), kmap.pair_ptr.data_ptr(), cap_pairs,
              gw.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream())
    return gw


def sparse_conv_forward(t: SparseTensor, w: ConvWeights, shape: KernelShape, stride=1, *,
                        math: str = "exact") -> SparseTensor:
    """conv.py:186-208 — x_out[u] = sum over offsets i with u+i occupied of
    W_i x_in[u+i]; output rows at generate_output_coords(t, stride).
    math="tf32": fp32 features on the tensor cores (tf32 multiplies)."""
    _check_weights(t, w, shape)
    st = _stride3(stride, t.dim)
    out4, ns = _output_coords4(t.coords4, t.tensor_stride, st, t.dim)
    km = _kernel_map4(t.coords4, out4, shape, t.tensor_stride, t.dim, with_pairs=False)
    n_out = out4.shape[0]
    perm, table = sort_table(km.nbr, n_out) if _sortable(km.nbr) else (None, km.nbr)
    y = conv_forward_raw(t.features, w, table, n_out, perm=perm, math=math)
    return SparseTensor(out4, y, ns, _trusted=True, _dim=t.dim)


def sparse_conv_backward(t: SparseTensor, w: ConvWeights, shape: KernelShape, stride, grad_out, *,
                         math: str = "exact"):
    """conv.py:211-242 — (grad_in (N_in, n_in) in the feature dtype,
    grad_w (K, n_out, n_in) fp32).  Recomputes coords and map as the
    reference does."""
    _check_weights(t, w, shape)
    st = _stride3(stride, t.dim)
    out4, _ = _output_coords4(t.coords4, t.tensor_stride, st, t.dim)
    if not isinstance(grad_out, torch.Tensor):
        grad_out = torch.as_tensor(np.asarray(grad_out, dtype=np.float64))
    g = grad_out.to(device=t.device, dtype=t.features.dtype).contiguous()
    if tuple(g.shape) != (out4.shape[0], w.n_out):
        raise StructuralError(f"grad_out shape {tuple(g.shape)} does not match forward output "
                              f"({out4.shape[0]}, {w.n_out})")
    km = _kernel_map4(t.coords4, out4, shape, t.tensor_stride, t.dim)
    if all(s == 1 for s in st) and shape.is_symmetric():
        table, flip = km.nbr, True  # inv[v, k] == nbr[v, K-1-k] when in == out
    else:
        table, flip = km.inverse(), False
    perm = None
    if _sortable(table):  # the flipped table's hit masks are bit-reversed: same grouping
        perm, table = sort_table(table, len(t), 0 if flip else 1)
    gi = conv_dgrad_raw(g, w, table, len(t), flip, perm=perm, math=math)
    gw = conv_wgrad_raw(t.features, g, tuple(w.matrices.shape), km)
    return gi, gw


def sparse_conv_transposed(t: SparseTensor, w: ConvWeights, shape: KernelShape, stride, out_coords) -> SparseTensor:
    """Transposed (adjoint) sparse conv, coarse -> fine: the
    fine rows `out_coords` (tensor stride t.tensor_stride / stride) are the
    input lattice of the strided conv whose map is reused with (in, out)
    swapped.  w: (K, n_out, n_in) applied as y[v] = sum_k W_k x[u] over the
    strided pairs (v, u) of offset k."""
    if w.num_offsets != shape.num_offsets or w.n_in != t.feature_width:
        raise StructuralError("weights do not match kernel shape / feature width")
    st = _stride3(stride, t.dim)
    fine_stride = tuple(a // b for a, b in zip(t.tensor_stride, st))
    if any(a * b != c for a, b, c in zip(fine_stride, st, t.tensor_stride)):
        raise ValidationError("tensor stride is not divisible by the transposed-conv stride")
    fine4, _ = pad_coords(out_coords, t.device)
    km = _kernel_map4(fine4, t.coords4, shape, fine_stride, t.dim, with_pairs=False)
    inv = km.inverse()  # [N_fine, K] -> coarse row
    # y[v] = sum_k W_k x[inv[v,k]] : a forward conv over the inverse table
    perm, tbl = sort_table(inv, fine4.shape[0], 1) if _sortable(inv) else (None, inv)
    y = conv_forward_raw(t.features, w, tbl, fine4.shape[0], perm=perm)
    return SparseTensor(fine4, y, fine_stride, _trusted=True, _dim=t.dim)


def benchmark_forward_backward(t: SparseTensor, w: ConvWeights, shape: KernelShape, stride=1, warmup_iters: int = 2,
                               profile_iters: int = 5) -> dict:
    """conv.py:280-320 with CUDA-event timing (µs, device time) — the same
    record keys as the reference's LayerProfile-shaped dict."""
    out = sparse_conv_forward(t, w, shape, stride)
    g = torch.ones((len(out), w.n_out), dtype=t.features.dtype, device=t.device)
    for _ in range(warmup_iters):
        sparse_conv_forward(t, w, shape, stride)
        sparse_conv_backward(t, w, shape, stride, g)
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    fwd = bwd = 0.0
    for _ in range(profile_iters):
        e0.record()
        sparse_conv_forward(t, w, shape, stride)
        e1.record()
        sparse_conv_backward(t, w, shape, stride, g)
        e2.record()
        e2.synchronize()
        fwd += e0.elapsed_time(e1) * 1e3
        bwd += e1.elapsed_time(e2) * 1e3
    out4, _ = _output_coords4(t.coords4, t.tensor_stride, _stride3(stride, t.dim), t.dim)
    km = _kernel_map4(t.coords4, out4, shape, t.tensor_stride, t.dim)
    return {
        "fwd_time_us": fwd / profile_iters,
        "bwd_time_us": bwd / profile_iters,
        "activation_bytes": binary_size(len(out), out.dim, out.feature_width),
        "param_bytes": w.nbytes(),
        "kernel_map_pairs": km.total_pairs(),
    }


# ---------------------------------------------------------------- weight I/O
def weights_to_json(w: ConvWeights, shape: KernelShape) -> str:
    """conv.py:323-335 format."""
    m = w.matrices.to(torch.float64).cpu().numpy()
    return json.dumps({"format_version": _WEIGHTS_VERSION, "dim": shape.dim, "n_out": w.n_out, "n_in": w.n_in,
                       "weights": {",".join(str(int(v)) for v in off): m[k].tolist()
                                   for k, off in enumerate(shape.offsets)}})


def weights_from_json(text: str):
    obj = json.loads(text)
    try:
        dim = int(obj["dim"])
        items = [(tuple(int(v) for v in key.split(",")), np.asarray(mat, dtype=np.float64))
                 for key, mat in obj["weights"].items()]
    except (KeyError, TypeError, ValueError) as exc:
        raise ValidationError(f"malformed weights JSON: {exc}") from exc
    if not items:
        raise ValidationError("weights JSON lists no offsets")
    shape = KernelShape.custom(dim, np.asarray([o for o, _ in items], dtype=np.int64))
    return ConvWeights(np.stack([m for _, m in items])), shape


def weights_to_binary(w: ConvWeights, shape: KernelShape) -> bytes:
    """conv.py:356-368 `VXCW` v1."""
    head = struct.pack("<4sIIIII", _WEIGHTS_MAGIC, _WEIGHTS_VERSION, shape.dim, w.num_offsets, w.n_out, w.n_in)
    return (head + np.ascontiguousarray(shape.offsets, "<i8").tobytes()
            + np.ascontiguousarray(w.matrices.to(torch.float64).cpu().numpy(), "<f8").tobytes())


def weights_from_binary(blob: bytes):
    head = struct.calcsize("<4sIIIII")
    if len(blob) < head:
        raise ValidationError("binary weights truncated")
    magic, version, dim, k, n_out, n_in = struct.unpack("<4sIIIII", blob[:head])
    if magic != _WEIGHTS_MAGIC or version != _WEIGHTS_VERSION:
        raise ValidationError("unrecognized binary weights header")
    off = head
    offsets = np.frombuffer(blob, dtype="<i8", count=k * dim, offset=off)
    off += 8 * k * dim
    mats = np.frombuffer(blob, dtype="<f8", count=k * n_out * n_in, offset=off)
    off += 8 * k * n_out * n_in
    if off != len(blob):
        raise ValidationError("binary weights have trailing bytes")
    return ConvWeights(mats.reshape(k, n_out, n_in).copy()), KernelShape.custom(dim, offsets.reshape(k, dim))
