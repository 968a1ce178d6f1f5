"""PyTorch drop-in for the sparse convolution: `torch.autograd.Function`s
over the C-ABI kernels and `nn.Module`s holding the weights in the
reference's (K, n_out, n_in) layout (conv.py:77-105).

The reference has no module API of its own — its functional ops
`sparse_conv_forward` / `sparse_conv_backward` (conv.py:186-242) are the
whole float stage.  This module wraps exactly those two as the forward and
backward of one autograd node, so a model built from `SparseConv3d` layers
trains with `loss.backward()`:

  forward  : vp_conv_fwd   y[u] = sum_k W_k x[nbr[u, k]]            (conv.py:205-207)
  backward : vp_conv_dgrad grad_x[v] = sum_k W_k^T g[inv[v, k]]      (conv.py:240)
             vp_conv_wgrad grad_W_k = sum_{(v,u) in pairs_k} g[u] x[v]^T (conv.py:241)

Coordinate bookkeeping (output coordinates, kernel map, dgrad table, the
neighbour-mask row ordering) is computed once per (coordinates, stride,
kernel shape) and cached in the input tensor's `plans` dict, which every
tensor on the same coordinates shares (stride-1 outputs reuse their input's
rows and cache), so a ResNet block builds its map once.

Precision follows the features: bf16 -> tcgen05 tensor cores (fp32
accumulate, bf16 out; fp32 weight gradient), fp32 -> fp32 SIMT kernels,
f64 -> f64 SIMT kernels (the reference's precision: parity ~1e-12 and a
finite-difference gradient check).  No CPU fallback: the ops raise if the
CUDA library is missing.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _lib
from . import conv as C
from .errors import StructuralError, ValidationError
from .tensor import SparseTensor


@dataclass(eq=False)
class ConvPlan:
    """Everything the three kernels need for one conv on one coordinate set."""

    out4: torch.Tensor  # (N_out, 4) int32 output coordinates
    out_stride: tuple
    n_in: int
    n_out: int
    kmap: C.KernelMap  # nbr [N_out, K] + CSR pairs (wgrad)
    fwd_table: torch.Tensor
    fwd_perm: Optional[torch.Tensor]
    dg_table: torch.Tensor  # [N_in, K]: inverse table (or nbr with flip)
    dg_flip: bool
    dg_perm: Optional[torch.Tensor]


def _key(kind, stride, shape: C.KernelShape):
    return (kind, tuple(stride), shape.offsets.tobytes())


def conv_plan(t: SparseTensor, shape: C.KernelShape, stride) -> ConvPlan:
    """Output coordinates + kernel map + dgrad table for conv(t, shape,
    stride), cached on t.plans (generate_output_coords conv.py:124-146 and
    build_kernel_map conv.py:149-183; the strided dgrad table is the map's
    inverse, the stride-1 symmetric one is nbr read column-flipped)."""
    st = C._stride3(stride, t.dim)
    key = _key("conv", st, shape)
    plan = t.plans.get(key)
    if plan is not None:
        return plan
    if shape.dim != t.dim:
        raise StructuralError("kernel shape dimension != tensor dimension")
    if all(s == 1 for s in st):
        out4, ns = t.coords4, t.tensor_stride  # same rows: the output shares the input's plans
    else:
        out4, ns = C._output_coords4(t.coords4, t.tensor_stride, st, t.dim)
    km = C._kernel_map4(t.coords4, out4, shape, t.tensor_stride, t.dim)
    n_in, n_out = len(t), out4.shape[0]
    fperm, ftab = C.sort_table(km.nbr, n_out) if C._sortable(km.nbr) else (None, km.nbr)
    if all(s == 1 for s in st) and shape.is_symmetric():
        dtab, flip = km.nbr, True
    else:
        dtab, flip = km.inverse(), False
    dperm = None
    if C._sortable(dtab):
        dperm, dtab = C.sort_table(dtab, n_in, 0 if flip else 1)
    plan = ConvPlan(out4, ns, n_in, n_out, km, ftab, fperm, dtab, flip, dperm)
    t.plans[key] = plan
    return plan


def transposed_plan(t: SparseTensor, shape: C.KernelShape, stride, out: SparseTensor) -> ConvPlan:
    """Plan of the transposed conv coarse t -> fine `out`: the strided conv
    fine -> coarse read backwards.  Reuses the strided conv's plan cached on
    the fine tensor when the coarse rows are that conv's output rows."""
    st = C._stride3(stride, t.dim)
    fine_stride = tuple(a // b for a, b in zip(t.tensor_stride, st))
    if any(a * b != c for a, b, c in zip(fine_stride, st, t.tensor_stride)):
        raise ValidationError("tensor stride is not divisible by the transposed-conv stride")
    if tuple(out.tensor_stride) != fine_stride:
        raise StructuralError(f"output tensor stride {out.tensor_stride} != {fine_stride}")
    key = _key("convT", st, shape)
    plan = t.plans.get(key)
    if plan is not None and plan.out4 is out.coords4:
        return plan
    down = out.plans.get(_key("conv", st, shape))
    if down is not None and (down.out4 is t.coords4 or torch.equal(down.out4, t.coords4)):
        km = down.kmap
    else:
        km = C._kernel_map4(out.coords4, t.coords4, shape, fine_stride, t.dim)
    inv = km.inverse()  # [N_fine, K] -> coarse row
    fperm, ftab = C.sort_table(inv, len(out), 1) if C._sortable(inv) else (None, inv)
    # backward: grad_x[u] = sum_k Wt_k^T g[nbr[u, k]]  (nbr of the strided map, no flip)
    swapped = C.KernelMap(km.offsets, km.nbr, km.pair_out, km.pair_in, km.pair_ptr, n_in=len(t))
    plan = ConvPlan(out.coords4, fine_stride, len(t), len(out), swapped, ftab, fperm, km.nbr, False, None)
    t.plans[key] = plan
    return plan


def _weights(w: torch.Tensor, x: torch.Tensor) -> C.ConvWeights:
    """The kernels' weight operand around the parameter (no copy for
    fp32/f64 parameters; bf16 features read a bf16 copy), without
    ConvWeights' host-side finiteness check."""
    cw = C.ConvWeights.__new__(C.ConvWeights)
    m = w.detach()
    cw.matrices = m if m.dtype in (torch.float32, torch.float64) else m.to(torch.float32)
    cw._ops = {}
    return cw


class SparseConvFunction(torch.autograd.Function):
    """y = sparse_conv(x; W) on a fixed plan (conv.py:186-242)."""

    @staticmethod
    def forward(ctx, x: torch.Tensor, w: torch.Tensor, plan: ConvPlan, math: str = "exact"):
        x = x.contiguous()
        cw = _weights(w, x)
        y = C.conv_forward_raw(x, cw, plan.fwd_table, plan.n_out, perm=plan.fwd_perm, math=math)
        ctx.save_for_backward(x, w)
        ctx.plan = plan
        ctx.math = math
        return y

    @staticmethod
    def backward(ctx, g: torch.Tensor):
        x, w = ctx.saved_tensors
        plan = ctx.plan
        g = g.to(x.dtype).contiguous()
        cw = _weights(w, x)
        gx = gw = None
        if ctx.needs_input_grad[0]:
            gx = C.conv_dgrad_raw(g, cw, plan.dg_table, plan.n_in, plan.dg_flip, perm=plan.dg_perm, math=ctx.math)
        if ctx.needs_input_grad[1]:
            gw = C.conv_wgrad_raw(x, g, tuple(w.shape), plan.kmap).to(w.dtype)
        return gx, gw, None, None


def sparse_conv(t: SparseTensor, weight: torch.Tensor, shape: C.KernelShape, stride=1,
                math: str = "exact") -> SparseTensor:
    """Differentiable sparse_conv_forward (conv.py:186-208): features and
    weight (K, n_out, n_in) carry autograd.  math="tf32": fp32 features on
    the tensor cores (forward and dgrad; the weight gradient stays fp32)."""
    if weight.dim() != 3 or weight.shape[0] != shape.num_offsets:
        raise StructuralError("weights must supply one (n_out, n_in) matrix per offset")
    if weight.shape[2] != t.feature_width:
        raise StructuralError(f"weight n_in {weight.shape[2]} != input feature width {t.feature_width}")
    plan = conv_plan(t, shape, stride)
    y = SparseConvFunction.apply(t.features, weight, plan, math)
    plans = t.plans if plan.out4 is t.coords4 else None
    return SparseTensor(plan.out4, y, plan.out_stride, _trusted=True, _dim=t.dim, _plans=plans)


def sparse_conv_transpose(t: SparseTensor, weight: torch.Tensor, shape: C.KernelShape, stride,
                          out: SparseTensor) -> SparseTensor:
    """Differentiable transposed conv coarse t -> the rows of `out` (the
    adjoint of the strided conv)."""
    if weight.dim() != 3 or weight.shape[0] != shape.num_offsets or weight.shape[2] != t.feature_width:
        raise StructuralError("weights do not match kernel shape / feature width")
    plan = transposed_plan(t, shape, stride, out)
    y = SparseConvFunction.apply(t.features, weight, plan)
    return SparseTensor(out.coords4, y, plan.out_stride, _trusted=True, _dim=t.dim, _plans=out.plans)


def _kernel_shape(dim, kernel_size) -> C.KernelShape:
    if isinstance(kernel_size, C.KernelShape):
        return kernel_size
    return C.KernelShape.hypercubic(dim, kernel_size)


class SparseConv3d(torch.nn.Module):
    """Generalized sparse convolution layer (Eq. 3; conv.py:186-242).

    weight: (K, out_channels, in_channels), the reference ConvWeights layout,
    initialised N(0, 1) / sqrt(K * in_channels) from
    `generator` (or torch's default RNG)."""

    def __init__(self, in_channels: int, out_channels: int, kernel_size=3, stride=1, dim: int = 3,
                 device=None, dtype=torch.float32, generator: Optional[torch.Generator] = None,
                 allow_tf32: bool = False):
        super().__init__()
        self.shape = _kernel_shape(dim, kernel_size)
        self.stride = stride
        self.math = "tf32" if allow_tf32 else "exact"  # fp32 features: tf32 tensor cores or exact SIMT
        self.in_channels, self.out_channels = int(in_channels), int(out_channels)
        K = self.shape.num_offsets
        w = torch.randn((K, out_channels, in_channels), generator=generator, dtype=torch.float64)
        w = (w / np.sqrt(K * in_channels)).to(dtype)
        self.weight = torch.nn.Parameter(w.to(device) if device is not None else w)

    def forward(self, t: SparseTensor) -> SparseTensor:
        return sparse_conv(t, self.weight, self.shape, self.stride, self.math)

    def extra_repr(self):
        return (f"{self.in_channels}, {self.out_channels}, offsets={self.shape.num_offsets}, "
                f"extents={self.shape.extents}, stride={self.stride}")


class SparseConvTranspose3d(SparseConv3d):
    """Transposed sparse conv (coarse -> fine): forward(t, out) writes the
    rows of `out` (a finer tensor, e.g. the skip connection of a U-Net)."""

    def forward(self, t: SparseTensor, out: SparseTensor) -> SparseTensor:  # type: ignore[override]
        return sparse_conv_transpose(t, self.weight, self.shape, self.stride, out)


# ---------------------------------------------------------------- conv-adjacent glue
# (batch norm / ReLU / residual / global pool.  The
# reference has none — SPEC.md:185 — so parity is self-defined against the
# oracle's numpy glue restatement in oracle/, used by the tests only.)
def _count(n, device):
    return torch.full((1,), n, dtype=torch.int32, device=device)


class SparseBatchNormFunction(torch.autograd.Function):
    """Training-mode batch norm over the rows (+ residual) (+ ReLU), one
    vp_bn_forward / vp_bn_backward each way (fixed-order reductions)."""

    @staticmethod
    def forward(ctx, x, gamma, beta, res, relu: bool, eps: float):
        if x.dtype not in (torch.float32, torch.bfloat16):
            raise ValidationError("batch norm: features must be fp32 or bf16")
        x = x.contiguous()
        n, ch = x.shape
        dev = x.device
        n_dev = _count(n, dev)
        mean = torch.empty(ch, dtype=torch.float32, device=dev)
        rstd = torch.empty(ch, dtype=torch.float32, device=dev)
        ws = _lib.workspace(_lib.query("vp_bn_stats_ws_bytes", n, ch), dev, zero=True)
        y = torch.empty_like(x)
        r = res.to(x.dtype).contiguous() if res is not None else None
        g32, b32 = gamma.detach().float().contiguous(), beta.detach().float().contiguous()
        _lib.call("vp_bn_forward", x.data_ptr(), _lib.dtype_code(x), n_dev.data_ptr(), n, ch, float(eps),
                  mean.data_ptr(), rstd.data_ptr(), g32.data_ptr(), b32.data_ptr(), _lib.ptr(r),
                  _lib.dtype_code(r) if r is not None else 0, int(relu), y.data_ptr(), _lib.dtype_code(y),
                  ws.data_ptr(), ws.numel(), _lib.stream())
        ctx.save_for_backward(x, y, g32, mean, rstd, n_dev)
        ctx.relu, ctx.has_res, ctx.gdtype = bool(relu), res is not None, gamma.dtype
        return y

    @staticmethod
    def backward(ctx, g):
        x, y, g32, mean, rstd, n_dev = ctx.saved_tensors
        n, ch = x.shape
        g = g.to(x.dtype).contiguous()
        gx = torch.empty_like(x)
        gres = torch.empty_like(x) if ctx.has_res else None
        ggamma = torch.empty(ch, dtype=torch.float32, device=x.device)
        gbeta = torch.empty(ch, dtype=torch.float32, device=x.device)
        ws = _lib.workspace(_lib.query("vp_bn_backward_ws_bytes", n, ch), x.device, zero=True)
        _lib.call("vp_bn_backward", g.data_ptr(), None, _lib.dtype_code(g), y.data_ptr(), _lib.dtype_code(y),
                  x.data_ptr(), _lib.dtype_code(x), n_dev.data_ptr(), n, ch, mean.data_ptr(), rstd.data_ptr(),
                  g32.data_ptr(), int(ctx.relu), gx.data_ptr(), _lib.dtype_code(gx), _lib.ptr(gres),
                  ggamma.data_ptr(), gbeta.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream())
        return gx, ggamma.to(ctx.gdtype), gbeta.to(ctx.gdtype), gres, None, None


class SparseBatchNorm(torch.nn.Module):
    """BatchNorm over the rows of a sparse tensor, optionally fused with a
    residual add and ReLU: y = relu(bn(x) [+ res])."""

    def __init__(self, channels: int, eps: float = 1e-5, relu: bool = False, device=None):
        super().__init__()
        self.eps, self.relu = float(eps), bool(relu)
        self.weight = torch.nn.Parameter(torch.ones(channels, device=device))
        self.bias = torch.nn.Parameter(torch.zeros(channels, device=device))

    def forward(self, t: SparseTensor, residual: Optional[SparseTensor] = None) -> SparseTensor:
        res = residual.features if residual is not None else None
        if res is not None and res.shape != t.features.shape:
            raise StructuralError("residual shape differs from the input")
        y = SparseBatchNormFunction.apply(t.features, self.weight, self.bias, res, self.relu, self.eps)
        return t.with_features(y)


class SparseGlobalPoolFunction(torch.autograd.Function):
    """Mean of the rows of each batch index (rows batch-contiguous):
    (N, C) -> (B, C) fp32 (vp_global_pool / vp_global_pool_backward)."""

    @staticmethod
    def forward(ctx, x, coords4, B: int):
        x = x.contiguous()
        n, ch = x.shape
        dev = x.device
        n_dev = _count(n, dev)
        out = torch.empty((B, ch), dtype=torch.float32, device=dev)
        counts = torch.empty(B, dtype=torch.int32, device=dev)
        ws = _lib.workspace(_lib.query("vp_global_pool_ws_bytes", B), dev)
        _lib.call("vp_global_pool", x.data_ptr(), _lib.dtype_code(x), coords4.data_ptr(), n_dev.data_ptr(), n, ch, B,
                  out.data_ptr(), counts.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream())
        ctx.save_for_backward(coords4, counts, n_dev)
        ctx.xshape, ctx.xdtype = (n, ch), x.dtype
        return out

    @staticmethod
    def backward(ctx, g):
        coords4, counts, n_dev = ctx.saved_tensors
        n, ch = ctx.xshape
        gx = torch.empty((n, ch), dtype=ctx.xdtype, device=g.device)
        gf = g.float().contiguous()
        _lib.call("vp_global_pool_backward", gf.data_ptr(), coords4.data_ptr(), counts.data_ptr(), n_dev.data_ptr(),
                  n, ch, gx.data_ptr(), _lib.dtype_code(gx), _lib.stream())
        return gx, None, None


def global_avg_pool(t: SparseTensor, batch_size: int) -> torch.Tensor:
    """(B, C) fp32 per-cloud mean of the features (rows must be grouped by
    batch index, as batch()/voxelize_batch produce them)."""
    return SparseGlobalPoolFunction.apply(t.features, t.coords4, int(batch_size))
