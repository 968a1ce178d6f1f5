"""CPU BASELINE RUNNER — TEST/BENCH INFRASTRUCTURE ONLY.

Runs one SparseResNet training step on the CPU with the REFERENCE's own hot
path: voxelize + batch (voxpipe/tensor.py:147-229) and every convolution
through voxpipe.conv.sparse_conv_forward / sparse_conv_backward
(conv.py:186-242, hash via the compiled _kernels extension) — the reference
built by oracle/build_ref.sh into oracle/_ref.  The model glue the reference
does not have (BN, ReLU, pool, linear, cross entropy, SGD) is
the numpy restatement in voxpipe_oracle.py.  Used only by bench.py's
`cpu_baseline` and `--impl reference` legs.  When oracle/_ref is absent the
runner falls back to the oracle restatement ("port").
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import voxpipe_oracle as O  # noqa: E402


def load_reference():
    """Return (kind, modules) — kind 'reference' when the built reference imports."""
    ref = os.path.join(HERE, "_ref")
    if os.path.isdir(os.path.join(ref, "voxpipe")):
        if ref not in sys.path:
            sys.path.insert(0, ref)
        try:
            from voxpipe import conv as R  # noqa: F401
            from voxpipe import kernels as RK
            from voxpipe import tensor as RT  # noqa: F401

            return ("reference" if RK.backend_name() == "compiled" else "reference-python"), (R, RT)
        except Exception:  # pragma: no cover - broken copy
            pass
    return "port", None


class CpuStep:
    def __init__(self, B, npts, res, planes=(32, 64, 128, 256), blocks=1, classes=40, seed=2):
        self.B, self.npts, self.res = B, npts, res
        self.planes, self.blocks = planes, blocks
        self.params = O.init_params(1, planes, blocks, classes, seed=seed)
        self.mom = None
        self.kind, mods = load_reference()
        if mods is not None:
            R, RT = mods
            shape = R.KernelShape.hypercubic(3, 3)

            def fwd(coords, x, ts, w, offsets, stride):
                y = R.sparse_conv_forward(R.SparseTensor(coords, x, ts), R.ConvWeights(w), shape, stride)
                return y.coords, y.features, y.tensor_stride

            def bwd(coords, x, ts, w, offsets, stride, g):
                return R.sparse_conv_backward(R.SparseTensor(coords, x, ts), R.ConvWeights(w), shape, stride, g)

            def vox(points, offsets):
                ts = [RT.voxelize(RT.PointCloud(points[offsets[i]:offsets[i + 1]]), 1.0, (res,) * 3)
                      for i in range(len(offsets) - 1)]
                bt = RT.batch(ts)
                return bt.coords, bt.features

            self.conv_impl, self.vox = (fwd, bwd), vox
        else:
            self.conv_impl = None
            self.vox = lambda p, o: O.voxelize_batch(p, o, 1.0, res)

    def step(self, points, offsets, labels) -> float:
        c, f = self.vox(np.asarray(points, np.float64), offsets)
        loss, _, self.params, self.mom = O.resnet_train_step(
            self.params, c, f, np.asarray(labels), len(offsets) - 1, planes=self.planes, blocks=self.blocks,
            mom=self.mom, conv_impl=self.conv_impl)
        return float(loss)


def time_steps(B, npts, res, steps, warmup, seed=0):
    """Clouds/s of the CPU path on `steps` timed steps of B clouds each."""
    pts, offs = O.synthetic_batch(B, npts, res, seed=seed, dtype=np.float32)
    labels = np.arange(B) % 40
    cs = CpuStep(B, npts, res)
    for _ in range(warmup):
        cs.step(pts, offs, labels)
    t0 = time.perf_counter()
    for _ in range(steps):
        cs.step(pts, offs, labels)
    dt = time.perf_counter() - t0
    return {"kind": cs.kind, "clouds_per_s": B * steps / dt, "s_per_step": dt / steps}


def layer_split(B, npts, res, seed=0, reps=1):
    """Per conv layer of the SparseResNet on the reference CPU path: wall
    seconds of the reference's generate_output_coords and build_kernel_map
    (conv.py:124-183) against its full sparse_conv_forward / _backward
    (conv.py:186-242, which rebuild both); the remainder is the
    gather-GEMM-scatter plus SparseTensor validation."""
    kind, mods = load_reference()
    if mods is None:
        raise RuntimeError("oracle/_ref (the reference build) is required for the per-layer split")
    R, RT = mods
    pts, offs = O.synthetic_batch(B, npts, res, seed=seed, dtype=np.float32)
    pts = pts.astype(np.float64)
    t0 = time.perf_counter()
    ts = [RT.voxelize(RT.PointCloud(pts[offs[i]:offs[i + 1]]), 1.0, (res,) * 3) for i in range(B)]
    x = RT.batch(ts)
    vox_s = time.perf_counter() - t0
    shape = R.KernelShape.hypercubic(3, 3)
    params = O.init_params(1, seed=2)
    convs, _ = O.resnet_layout(1)
    rows = []
    rng = np.random.default_rng(1)
    for name, ci, co, stride in convs:
        if x.feature_width != ci:
            x = R.SparseTensor(x.coords, rng.normal(size=(len(x), ci)), x.tensor_stride)
        w = R.ConvWeights(params[name + ".w"])
        rec = {"layer": name, "cin": ci, "cout": co, "stride": stride, "n_in": len(x)}
        best = {}
        for _ in range(reps):
            t0 = time.perf_counter()
            oc, _ns = R.generate_output_coords(x, stride)
            t1 = time.perf_counter()
            km = R.build_kernel_map(x.coords, oc, shape, x.tensor_stride)
            t2 = time.perf_counter()
            y = R.sparse_conv_forward(x, w, shape, stride)
            t3 = time.perf_counter()
            R.sparse_conv_backward(x, w, shape, stride, np.ones((len(y), co)))
            t4 = time.perf_counter()
            for k, v in (("coords_s", t1 - t0), ("map_s", t2 - t1), ("fwd_s", t3 - t2), ("bwd_s", t4 - t3)):
                best[k] = min(best.get(k, 1e30), v)
        rec.update({k: round(v, 4) for k, v in best.items()})
        rec["pairs"] = km.total_pairs()
        # fwd and bwd each rebuild coords + map (conv.py:196-208, 228-242)
        rec["gemm_fwd_s"] = round(max(best["fwd_s"] - best["coords_s"] - best["map_s"], 0.0), 4)
        rec["gemm_bwd_s"] = round(max(best["bwd_s"] - best["coords_s"] - best["map_s"], 0.0), 4)
        rows.append(rec)
        x = R.SparseTensor(y.coords, y.features, y.tensor_stride)
    return {"kind": kind, "voxelize_batch_s": round(vox_s, 4), "layers": rows}


if __name__ == "__main__":
    print(time_steps(int(sys.argv[1]) if len(sys.argv) > 1 else 4, 2048, 64, 1, 1))
