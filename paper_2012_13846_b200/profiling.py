"""Per-layer cost measurement on the GPU — the reference's
`run_benchmark_profile` (profiling.py:333-455) over this package's kernels.

A model description lists layers of three kinds (profiling.py:343-347):
  * "sparse_conv": executed — forward and backward of the layer through
    conv.sparse_conv_forward / sparse_conv_backward on the GPU (output coords,
    kernel map, tcgen05 / SIMT conv), timed with CUDA events (device µs);
    the output feeds the next sparse_conv layer, as in the reference;
  * "synthetic": the declared costs, not executed;
  * "stub": the declared fwd_ms / bwd_ms (the reference busy-waits them on
    the host; a device profile records them as declared).
The synthetic input is the reference's: `input.num_points` uniform points in
[0, resolution)^dim from default_rng(input.seed), voxel size 1 (occupancy
features, or `feature_width` N(0,1) features averaged per voxel).
Records are partition.LayerProfile (the planner's input format).
"""
from __future__ import annotations

import numpy as np
import torch

from . import conv as C
from .errors import ConfigError
from .partition import LayerProfile
from .tensor import PointCloud, binary_size, voxelize


def run_benchmark_profile(model_desc: dict, processor_label: str = "B200", warmup_iters: int = 3,
                          profile_iters: int = 10, feature_dtype=torch.float32) -> list:
    """profiling.py:333-455 on the GPU; returns one LayerProfile per layer."""
    del processor_label  # bookkeeping for the output header, as in the reference
    if warmup_iters < 0 or profile_iters < 1:
        raise ConfigError("warmup_iters must be >= 0 and profile_iters >= 1")
    layers = model_desc.get("layers")
    if not layers:
        raise ConfigError("model description lists no layers")
    current = None
    if any(layer.get("type") == "sparse_conv" for layer in layers):
        spec = model_desc.get("input")
        if not spec:
            raise ConfigError("sparse_conv layers need an 'input' description")
        rng = np.random.default_rng(int(spec.get("seed", 0)))
        dim = int(spec.get("dim", 3))
        res = int(spec.get("resolution", 16))
        n = int(spec.get("num_points", 512))
        width = int(spec.get("feature_width", 1))
        points = rng.random((n, dim)) * res
        feats = rng.standard_normal((n, width)) if width > 1 else None
        current = voxelize(PointCloud(points, feats), 1.0, (res,) * dim)
        current = current.with_features(current.features.to(feature_dtype))
    records = []
    for layer_id, layer in enumerate(layers):
        kind = layer.get("type")
        if kind == "synthetic":
            try:
                records.append(LayerProfile(layer_id, float(layer["fwd_time_us"]), float(layer["bwd_time_us"]),
                                            float(layer.get("activation_bytes", 0)),
                                            float(layer.get("param_bytes", 0))))
            except KeyError as exc:
                raise ConfigError(f"synthetic layer {layer_id} misses {exc}") from exc
            continue
        if kind == "stub":
            fwd_ms = float(layer.get("fwd_ms", 1.0))
            bwd_ms = float(layer.get("bwd_ms", 2 * fwd_ms))
            records.append(LayerProfile(layer_id, fwd_ms * 1e3, bwd_ms * 1e3, float(layer.get("activation_bytes", 0)),
                                        float(layer.get("param_bytes", 0))))
            continue
        if kind == "sparse_conv":
            if current is None:
                raise ConfigError("sparse_conv layer without model input")
            cout = int(layer.get("out_channels", current.feature_width))
            shape = C.KernelShape.hypercubic(current.dim, int(layer.get("kernel_size", 3)))
            stride = int(layer.get("stride", 1))
            fan_in = shape.num_offsets * current.feature_width
            wrng = np.random.default_rng(layer_id)
            w = C.ConvWeights(wrng.standard_normal((shape.num_offsets, cout, current.feature_width)) / np.sqrt(fan_in),
                              device=current.device)
            rec = C.benchmark_forward_backward(current, w, shape, stride, warmup_iters, profile_iters)
            records.append(LayerProfile(layer_id, rec["fwd_time_us"], rec["bwd_time_us"],
                                        float(rec["activation_bytes"]), float(rec["param_bytes"])))
            current = C.sparse_conv_forward(current, w, shape, stride)
            continue
        raise ConfigError(f"layer {layer_id}: unexecutable type {kind!r} with no synthetic cost")
    return records


__all__ = ["run_benchmark_profile", "binary_size"]
