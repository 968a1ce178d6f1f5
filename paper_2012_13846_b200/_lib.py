"""ctypes binding of the C-ABI library `libvoxpipe_b200.so` (include/voxpipe_b200.h).

This is the ONLY way the package reaches its compute: there is no CPU or
PyTorch fallback.  If the library is missing or no CUDA device is present,
the calls raise loudly (ConfigError at load, InternalError at call).
"""
from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import ConfigError, InternalError, StructuralError, ValidationError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libvoxpipe_b200.so")

VP_OK, VP_EVALIDATION, VP_EINTERNAL = 0, 2, 3
VP_F32, VP_BF16, VP_F64, VP_TF32 = 0, 1, 2, 3
MAX_OFFSETS = 343

P = C.c_void_p
I32 = C.c_int32
I64 = C.c_int64
SZ = C.c_size_t
F32 = C.c_float
F64 = C.c_double

# name -> (restype, argtypes); must match include/voxpipe_b200.h exactly
SIGNATURES = {
    "vp_last_error": (C.c_char_p, []),
    "vp_version": (C.c_char_p, []),
    "vp_kernel_launches": (C.c_longlong, []),
    "vp_debug_conv_trace": (C.c_int, [P]),
    "vp_hash_capacity": (I64, [I64]),
    "vp_hash_bytes": (SZ, [I64]),
    "vp_hash_build": (C.c_int, [P, P, I64, P, I64, P]),
    "vp_hash_lookup": (C.c_int, [P, I64, P, I64, P, P]),
    "vp_pack_coords": (C.c_int, [P, I64, P, P, P]),
    "vp_validate_coords_ws_bytes": (SZ, [I64]),
    "vp_validate_coords": (C.c_int, [P, P, I64, P, P, P, SZ, P]),
    "vp_check_finite": (C.c_int, [P, I32, I64, P, P]),
    "vp_output_coords_ws_bytes": (SZ, [I64]),
    "vp_output_coords": (C.c_int, [P, P, I64, P, P, P, P, P, SZ, P]),
    "vp_voxelize_ws_bytes": (SZ, [I64]),
    "vp_voxelize": (C.c_int, [P, I32, I64, P, I32, F64, P, P, P, P, P, I32, P, SZ, P]),
    "vp_voxel_mean_ws_bytes": (SZ, [I64, I64]),
    "vp_voxel_mean": (C.c_int, [P, I32, I64, I32, P, P, I64, P, P, SZ, P]),
    "vp_kernel_map_ws_bytes": (SZ, [I64, I64, I32]),
    "vp_kernel_map": (C.c_int, [P, P, I64, P, P, I64, P, I32, P, P, P, P, P, P, SZ, P]),
    "vp_kernel_map_sort_ws_bytes": (SZ, [I64, I32]),
    "vp_kernel_map_sort": (C.c_int, [P, P, I64, I32, P, P, P, SZ, P]),
    "vp_kernel_map_group": (C.c_int, [P, P, I64, I32, I32, P, P, P, SZ, P]),
    "vp_kernel_map_group_sched": (C.c_int, [P, P, I64, I32, I32, I32, P, P, P, SZ, P]),
    "vp_conv_tc_grid": (I32, [I64, I64]),
    "vp_brick_pool": (I64, [I64, I32, I32]),
    "vp_brick_bytes": (SZ, [I64, I32, I32]),
    "vp_brick_init": (C.c_int, [P, I64, I32, I32, P]),
    "vp_brick_set": (C.c_int, [P, P, I64, P, I64, I32, I32, I32, I32, P]),
    "vp_kernel_map_brick_ws_bytes": (SZ, [I64, I32]),
    "vp_kernel_map_brick": (C.c_int, [P, I64, I32, I32, I32, P, P, I64, P, I32, P, P, P, P, P, P, SZ, P]),
    "vp_kernel_map_inverse": (C.c_int, [P, P, I64, I32, P, I64, P]),
    "vp_grid_words": (I64, [I32, I32]),
    "vp_coords_bbox": (C.c_int, [P, I64, P, I64, I32, P, P]),
    "vp_kernel_map_lattice": (C.c_int, [P, I64, P, I64, P, I32, I32, P, P, I64, P, P, P, P, P, SZ, P]),
    "vp_grid_init": (C.c_int, [P, I32, I32, P]),
    "vp_grid_set": (C.c_int, [P, P, I64, P, I32, I32, I32, I32, P]),
    "vp_kernel_map_grid_ws_bytes": (SZ, [I64, I32]),
    "vp_kernel_map_grid": (C.c_int, [P, I32, I32, I32, P, P, I64, P, I32, P, P, P, P, P, P, SZ, P]),
    "vp_conv_fwd_ws_bytes": (SZ, [I64, I64, I32]),
    "vp_conv_fwd": (C.c_int, [P, I32, I64, I64, P, I32, I64, I32, P, I32, P, P, I64, P, I32, P, SZ, P]),
    "vp_conv_dgrad_ws_bytes": (SZ, [I64, I64, I32]),
    "vp_conv_dgrad": (C.c_int, [P, I32, I64, I64, P, I32, I64, I32, P, I32, P, P, I64, P, I32, P, SZ, P]),
    "vp_conv_wgrad_ws_bytes": (SZ, [I64, I64, I32, I64]),
    "vp_conv_wgrad": (C.c_int, [P, I32, I64, P, I32, I64, I32, P, P, P, I64, P, P, SZ, P]),  # grad_w: fp32 (f64 for f64 operands)
    "vp_conv_wgrad_side": (C.c_int, [P, I32, I64, P, I32, I64, I32, P, P, P, I64, P, P, SZ, P]),
    "vp_conv_wgrad_sgd": (C.c_int, [P, I32, I64, P, I32, I64, I32, P, P, P, I64, P, P, SZ, P, P, P, F32, F32, I32, P]),
    "vp_batch_segments": (C.c_int, [P, P, I64, I32, P, P]),
    "vp_sparse_head_ws_bytes": (SZ, [I32, I64, I32]),
    "vp_sparse_head": (C.c_int, [P, I32, P, I32, I64, P, P, I32, P, P, P, P, P, P, P, P, P, P, P, P, P, P, P, SZ, P]),
    "vp_bn_part_bytes": (SZ, [I64]),
    "vp_conv_fwd_bn": (C.c_int, [P, I32, I64, I64, P, I32, I64, I32, P, I32, P, P, I64, P, I32, P, SZ,
                                 I32, P, P, P, P, P, F32, P, P, P, P]),
    "vp_conv_dgrad_bn": (C.c_int, [P, I32, I64, I64, P, I32, I64, I32, P, I32, P, P, I64, P, I32, P, SZ,
                                   I32, P, P, P, P, P, F32, P, P, P, P]),
    "vp_bn_backward_apply": (C.c_int, [P, I32, P, I32, P, I64, I64, P, P, P, P, P, P, I32, P]),
    "vp_bn_apply_part": (C.c_int, [P, I32, P, I64, I64, F32, P, P, P, P, P, P, I32, I32, P, I32, P]),
    "vp_bn_backward_part": (C.c_int, [P, I32, P, I32, P, I64, I64, P, P, P, P, P, I32, P, P, P]),
    "vp_bn_stats_ws_bytes": (SZ, [I64, I64]),
    "vp_bn_stats": (C.c_int, [P, I32, P, I64, I64, F32, P, P, P, SZ, P]),
    "vp_bn_apply": (C.c_int, [P, I32, P, I64, I64, P, P, P, P, P, I32, I32, P, I32, P]),
    "vp_bn_forward": (C.c_int, [P, I32, P, I64, I64, F32, P, P, P, P, P, I32, I32, P, I32, P, SZ, P]),
    "vp_bn_backward_ws_bytes": (SZ, [I64, I64]),
    "vp_bn_backward": (C.c_int, [P, P, I32, P, I32, P, I32, P, I64, I64, P, P, P, I32, P, I32, P, P, P, P, SZ, P]),
    "vp_global_pool_ws_bytes": (SZ, [I32]),
    "vp_global_pool": (C.c_int, [P, I32, P, P, I64, I64, I32, P, P, P, SZ, P]),
    "vp_global_pool_backward": (C.c_int, [P, P, P, P, I64, I64, P, I32, P]),
    "vp_linear_xent_ws_bytes": (SZ, [I32, I32]),
    "vp_linear_xent": (C.c_int, [P, I32, I32, P, P, I32, P, P, P, P, P, P, P, SZ, P]),
    "vp_sgd_momentum": (C.c_int, [P, P, P, I64, F32, F32, P, I64, P]),
    "vp_cast": (C.c_int, [P, I32, P, I32, I64, P]),
    "vp_wide_ws_bytes": (SZ, [I64, I64, I32, I32]),
    "vp_wide_validate": (C.c_int, [P, I64, I32, P, P, P, SZ, P]),
    "vp_wide_output_coords": (C.c_int, [P, I64, I32, P, P, P, P, SZ, P]),
    "vp_wide_kernel_map": (C.c_int, [P, I64, P, I64, I32, P, I32, P, P, P, P, P, P, SZ, P]),
}

_lib = None
_lock = threading.Lock()


def load():
    """Load (once) and return the CDLL; raise ConfigError if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ConfigError(
                    f"CUDA library not built: {LIB_PATH} (run __graft_entry__.build() or "
                    "python paper_2012_13846_b200/build_lib.py)")
            lib = C.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def check(status: int, what: str):
    if status == VP_OK:
        return
    msg = load().vp_last_error().decode(errors="replace")
    if status == VP_EVALIDATION:
        raise ValidationError(f"{what}: {msg}")
    raise InternalError(f"{what}: {msg}")


def call(name: str, *args):
    """Invoke a status-returning entry point and raise on failure."""
    check(getattr(load(), name)(*args), name)


def query(name: str, *args):
    return getattr(load(), name)(*args)


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None passes NULL)."""
    return None if t is None else t.data_ptr()


def stream():
    import torch

    return torch.cuda.current_stream().cuda_stream


def i32_array(vals):
    vals = [int(v) for v in vals]
    return (C.c_int32 * max(1, len(vals)))(*vals)


def i64_array(vals):
    vals = [int(v) for v in vals]
    return (C.c_int64 * max(1, len(vals)))(*vals)


def dtype_code(t) -> int:
    import torch

    if t.dtype == torch.bfloat16:
        return VP_BF16
    if t.dtype == torch.float32:
        return VP_F32
    if t.dtype == torch.float64:
        return VP_F64
    raise StructuralError(f"unsupported feature dtype {t.dtype}")


def workspace(nbytes: int, device, zero: bool = False):
    """Caller-owned scratch for a C-ABI call, from torch's stream-ordered
    caching allocator.  Uninitialised: every entry point initialises the
    scratch it reads.  zero=True for the BN statistics, whose workspace ends
    in a self-re-arming ticket word that must start at zero
    (include/voxpipe_b200.h)."""
    import torch

    n = max(int(nbytes), 256)
    if zero:
        return torch.zeros(n, dtype=torch.uint8, device=device)
    return torch.empty(n, dtype=torch.uint8, device=device)
