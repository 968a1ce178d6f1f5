"""Generate the golden fixtures under tests/golden/ by running the REFERENCE
itself (voxpipe 0.1.0 built into oracle/_ref/ by oracle/build_ref.sh).

The fixtures pin both the CPU oracle (tests/test_oracle.py) and the CUDA path
(tests/test_gpu_*.py).  Run from the repo root in the build container:

    ./oracle/build_ref.sh && python tests/golden/make_golden.py

Everything is seeded; re-running reproduces the same bytes.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from voxpipe import conv as R  # noqa: E402  (reference)
from voxpipe import kernels as RK  # noqa: E402
from voxpipe import tensor as RT  # noqa: E402
import voxpipe_oracle as O  # noqa: E402  (only for the synthetic generator)

assert RK.backend_name() == "compiled"


def kmap_arrays(km):
    """Flatten a reference KernelMap into CSR (ptr, in, out)."""
    ptr = [0]
    vi, ui = [], []
    for a, b in km.pairs:
        vi.append(a)
        ui.append(b)
        ptr.append(ptr[-1] + len(a))
    cat = lambda xs: np.concatenate(xs).astype(np.int64) if xs else np.empty(0, np.int64)
    return np.asarray(ptr, np.int64), cat(vi), cat(ui)


def save(name, **arrs):
    np.savez_compressed(os.path.join(HERE, name), **arrs)
    print("wrote", name, {k: v.shape for k, v in arrs.items()})


def random_coords(rng, n, lo, hi, batches, stride):
    rows = set()
    out = []
    while len(out) < n:
        r = (int(rng.integers(0, batches)),) + tuple(int(v) * stride for v in rng.integers(lo, hi, 3))
        if r not in rows:
            rows.add(r)
            out.append(r)
    return np.asarray(out, np.int64)


def gen_maps():
    """Random inputs with negative coords, strides 1 -> 2 -> 4 -> 8
    (SURVEY §8(c) restatement check, done against the reference here)."""
    rng = np.random.default_rng(1234)
    shape = R.KernelShape.hypercubic(3, 3)
    arrs = {}
    for trial in range(4):
        c = random_coords(rng, 700 + 150 * trial, -30, 30, 3, 1)
        t = R.SparseTensor(c, np.zeros((len(c), 1)), (1, 1, 1))
        arrs[f"t{trial}_in0"] = c
        for lvl in range(3):
            # stride-1 map at this level
            km = R.build_kernel_map(t.coords, t.coords, shape, t.tensor_stride)
            p, vi, ui = kmap_arrays(km)
            arrs[f"t{trial}_l{lvl}_s1_ptr"], arrs[f"t{trial}_l{lvl}_s1_in"], arrs[f"t{trial}_l{lvl}_s1_out"] = p, vi, ui
            oc, ost = R.generate_output_coords(t, 2)
            km = R.build_kernel_map(t.coords, oc, shape, t.tensor_stride)
            p, vi, ui = kmap_arrays(km)
            arrs[f"t{trial}_l{lvl}_s2_oc"] = oc
            arrs[f"t{trial}_l{lvl}_s2_ptr"], arrs[f"t{trial}_l{lvl}_s2_in"], arrs[f"t{trial}_l{lvl}_s2_out"] = p, vi, ui
            t = R.SparseTensor(oc, np.zeros((len(oc), 1)), ost)
    # stride 3 and anisotropic stride (2,1,3) + kernel 3x1x5 custom extents
    c = random_coords(rng, 900, -20, 20, 2, 1)
    t = R.SparseTensor(c, np.zeros((len(c), 1)), (1, 1, 1))
    arrs["aniso_in"] = c
    for tag, st, ks in (("s3", 3, R.KernelShape.hypercubic(3, 3)),
                        ("s213", (2, 1, 3), R.KernelShape.hypercubic(3, (3, 1, 5))),
                        ("k5", 1, R.KernelShape.hypercubic(3, 5)),
                        ("k1", 1, R.KernelShape.hypercubic(3, 1))):
        oc, ost = R.generate_output_coords(t, st)
        km = R.build_kernel_map(t.coords, oc, ks, t.tensor_stride)
        p, vi, ui = kmap_arrays(km)
        arrs[f"aniso_{tag}_oc"], arrs[f"aniso_{tag}_ptr"] = oc, p
        arrs[f"aniso_{tag}_in"], arrs[f"aniso_{tag}_out"] = vi, ui
        arrs[f"aniso_{tag}_offsets"] = ks.offsets
        arrs[f"aniso_{tag}_stride"] = np.asarray(ost, np.int64)
    # out-of-packable-range queries: coords at the +/- edge of int16
    edge = np.asarray([[0, 32767, 0, 0], [0, -32768, 5, 5], [1, 32766, -32768, 32767],
                       [65535, 0, 0, 0], [65535, 32767, 32767, 32767]], np.int64)
    t = R.SparseTensor(edge, np.zeros((len(edge), 1)), (1, 1, 1))
    km = R.build_kernel_map(t.coords, t.coords, R.KernelShape.hypercubic(3, 3), (1, 1, 1))
    p, vi, ui = kmap_arrays(km)
    arrs["edge_in"], arrs["edge_ptr"], arrs["edge_pin"], arrs["edge_pout"] = edge, p, vi, ui
    save("kmaps.npz", **arrs)


def gen_hash():
    rng = np.random.default_rng(99)
    keys = rng.integers(-(2**40), 2**40, size=3000).astype(np.int64)
    keys[100:150] = keys[0:50]            # duplicates: first occurrence wins
    keys[2000] = -1                        # all-ones key (0xFFFF...F)
    keys[2001] = -1
    keys[2002] = 0
    from voxpipe import _kernels as ck
    a, b = ck.build_table(keys)
    q = np.concatenate([keys, rng.integers(-(2**40), 2**40, size=2000).astype(np.int64), [-1, 0, 2**62]])
    rows = ck.lookup(a, b, q)
    save("hash.npz", keys=keys, queries=q, rows=rows)


def gen_voxelize_and_conv():
    arrs = {}
    # C1-shaped mini batch: 3 clouds x 160 pts at 32^3 (occupancy features)
    B, npts, res = 3, 160, 32
    pts = [O.shape_cloud(i, npts, res, seed=5) for i in range(B)]
    ts = [RT.voxelize(RT.PointCloud(p), 1.0, (res,) * 3) for p in pts]
    bt = RT.batch(ts)
    arrs["vox_points"] = np.concatenate(pts)
    arrs["vox_offsets"] = np.arange(B + 1) * npts
    arrs["vox_coords"], arrs["vox_feats"] = bt.coords, bt.features
    # mean-feature voxelization of one cloud with random features, voxel 0.75
    rng = np.random.default_rng(3)
    p = rng.uniform(-2, 9, size=(500, 3))
    f = rng.normal(size=(500, 3))
    t = RT.voxelize(RT.PointCloud(p, f), 0.75, (10, 10, 10))
    arrs["voxm_points"], arrs["voxm_feats_in"] = p, f
    arrs["voxm_coords"], arrs["voxm_feats"] = t.coords, t.features
    # float stage: conv fwd/bwd at C=32 -> 64 stride 1 and 2 on the batch
    shape = R.KernelShape.hypercubic(3, 3)
    rng = np.random.default_rng(1)
    for tag, cin, cout, st in (("s1", 32, 64, 1), ("s2", 32, 64, 2), ("s1b", 64, 32, 1)):
        # inputs are float32-representable so the fixture stores them as f32
        x = rng.normal(size=(len(bt), cin)).astype(np.float32).astype(np.float64)
        w = (rng.normal(size=(27, cout, cin)) / np.sqrt(27 * cin)).astype(np.float32).astype(np.float64)
        t = RT.SparseTensor(bt.coords, x, (1, 1, 1))
        y = R.sparse_conv_forward(t, R.ConvWeights(w), shape, st)
        g = rng.normal(size=y.features.shape).astype(np.float32).astype(np.float64)
        gi, gw = R.sparse_conv_backward(t, R.ConvWeights(w), shape, st, g)
        arrs[f"conv_{tag}_x"], arrs[f"conv_{tag}_w"] = x.astype(np.float32), w.astype(np.float32)
        arrs[f"conv_{tag}_y"], arrs[f"conv_{tag}_yc"] = y.features, y.coords
        arrs[f"conv_{tag}_g"] = g.astype(np.float32)
        arrs[f"conv_{tag}_gi"], arrs[f"conv_{tag}_gw"] = gi, gw
    save("conv.npz", **arrs)


def gen_kats():
    """SPEC.md sparse_conv / sparse_tensor examples, evaluated by the reference."""
    arrs = {}
    # SPEC.md:124-126 generate_output_coords (D=2)
    t = RT.SparseTensor(np.array([[0, 0, 0], [0, 0, 1], [0, 0, 3]]), np.zeros((3, 1)), (1, 1))
    oc, ost = R.generate_output_coords(t, 2)
    arrs["kat_oc_in"], arrs["kat_oc_out"], arrs["kat_oc_stride"] = t.coords, oc, np.asarray(ost)
    # SPEC.md:142-144 full 3x3 grid (D=2), 3^2 kernel
    g = np.array([[0, x, y] for x in range(3) for y in range(3)])
    km = R.build_kernel_map(g, g, R.KernelShape.hypercubic(2, 3), (1, 1))
    p, vi, ui = kmap_arrays(km)
    arrs["kat_grid_in"], arrs["kat_grid_ptr"], arrs["kat_grid_pin"], arrs["kat_grid_pout"] = g, p, vi, ui
    # SPEC.md:151-153 dense oracle on a fully occupied 5x5 grid
    rng = np.random.default_rng(7)
    grid = rng.normal(size=(5, 5, 2))
    w = rng.normal(size=(9, 3, 2))
    shape = R.KernelShape.hypercubic(2, 3)
    dense = R.dense_conv_forward(grid, R.ConvWeights(w), shape)
    arrs["kat_dense_grid"], arrs["kat_dense_w"], arrs["kat_dense_out"] = grid, w, dense
    # SPEC.md:160-162 [1,2,3] * [1,1,1] -> [3,6,5]
    d1 = R.dense_conv_forward(np.array([[1.0], [2.0], [3.0]]), R.ConvWeights(np.ones((3, 1, 1))),
                              R.KernelShape.hypercubic(1, 3))
    arrs["kat_1d_out"] = d1
    save("kats.npz", **arrs)


if __name__ == "__main__":
    gen_hash()
    gen_maps()
    gen_voxelize_and_conv()
    gen_kats()
