"""The CPU oracle (oracle/voxpipe_oracle.py) pinned against golden vectors the
reference itself produced (tests/golden/make_golden.py)."""
import numpy as np
import pytest

import voxpipe_oracle as O
from conftest import csr_pairs, golden


def test_hash_first_occurrence():
    g = golden("hash.npz")
    sk, rows = O.build_table(g["keys"])
    np.testing.assert_array_equal(O.lookup(sk, rows, g["queries"]), g["rows"])


@pytest.mark.parametrize("trial", range(4))
def test_output_coords_and_maps(trial):
    g = golden("kmaps.npz")
    off = O.hypercubic_offsets(3, 3)
    c, ts = g[f"t{trial}_in0"], (1, 1, 1)
    for lvl in range(3):
        pre = f"t{trial}_l{lvl}"
        km = O.build_kernel_map(c, c, off, ts)
        for (a, b), (ea, eb) in zip(km, csr_pairs(g[pre + "_s1_ptr"], g[pre + "_s1_in"], g[pre + "_s1_out"])):
            np.testing.assert_array_equal(a, ea)
            np.testing.assert_array_equal(b, eb)
        oc, nts = O.generate_output_coords(c, ts, 2)
        np.testing.assert_array_equal(oc, g[pre + "_s2_oc"])
        km = O.build_kernel_map(c, oc, off, ts)
        for (a, b), (ea, eb) in zip(km, csr_pairs(g[pre + "_s2_ptr"], g[pre + "_s2_in"], g[pre + "_s2_out"])):
            np.testing.assert_array_equal(a, ea)
            np.testing.assert_array_equal(b, eb)
        c, ts = oc, nts


@pytest.mark.parametrize("tag,stride", [("s3", 3), ("s213", (2, 1, 3)), ("k5", 1), ("k1", 1)])
def test_aniso_maps(tag, stride):
    g = golden("kmaps.npz")
    c = g["aniso_in"]
    oc, nts = O.generate_output_coords(c, (1, 1, 1), stride)
    np.testing.assert_array_equal(oc, g[f"aniso_{tag}_oc"])
    assert tuple(nts) == tuple(g[f"aniso_{tag}_stride"])
    km = O.build_kernel_map(c, oc, g[f"aniso_{tag}_offsets"], (1, 1, 1))
    exp = csr_pairs(g[f"aniso_{tag}_ptr"], g[f"aniso_{tag}_in"], g[f"aniso_{tag}_out"])
    for (a, b), (ea, eb) in zip(km, exp):
        np.testing.assert_array_equal(a, ea)
        np.testing.assert_array_equal(b, eb)


def test_edge_range_maps():
    g = golden("kmaps.npz")
    km = O.build_kernel_map(g["edge_in"], g["edge_in"], O.hypercubic_offsets(3, 3), (1, 1, 1))
    for (a, b), (ea, eb) in zip(km, csr_pairs(g["edge_ptr"], g["edge_pin"], g["edge_pout"])):
        np.testing.assert_array_equal(a, ea)
        np.testing.assert_array_equal(b, eb)


def test_brute_force_agrees():
    g = golden("kmaps.npz")
    c = g["t0_in0"][:300]
    off = O.hypercubic_offsets(3, 3)
    for (a, b), (ea, eb) in zip(O.build_kernel_map(c, c, off, (1, 1, 1)),
                                O.brute_force_kernel_map(c, c, off, (1, 1, 1))):
        np.testing.assert_array_equal(a, ea)
        np.testing.assert_array_equal(b, eb)


def test_voxelize_batch():
    g = golden("conv.npz")
    c, f = O.voxelize_batch(g["vox_points"], g["vox_offsets"], 1.0, 32)
    np.testing.assert_array_equal(c, g["vox_coords"])
    np.testing.assert_array_equal(f, g["vox_feats"])
    c, f = O.voxelize(g["voxm_points"], 0.75, (10, 10, 10), features=g["voxm_feats_in"])
    np.testing.assert_array_equal(c, g["voxm_coords"])
    np.testing.assert_allclose(f, g["voxm_feats"], rtol=0, atol=1e-12)


@pytest.mark.parametrize("tag,stride", [("s1", 1), ("s2", 2), ("s1b", 1)])
def test_conv_fwd_bwd(tag, stride):
    g = golden("conv.npz")
    off = O.hypercubic_offsets(3, 3)
    x, w = g[f"conv_{tag}_x"].astype(np.float64), g[f"conv_{tag}_w"].astype(np.float64)
    oc, y, _ = O.sparse_conv_forward(g["vox_coords"], x, (1, 1, 1), w, off, stride)
    np.testing.assert_array_equal(oc, g[f"conv_{tag}_yc"])
    np.testing.assert_allclose(y, g[f"conv_{tag}_y"], rtol=0, atol=1e-12)
    gi, gw = O.sparse_conv_backward(g["vox_coords"], x, (1, 1, 1), w, off, stride,
                                    g[f"conv_{tag}_g"].astype(np.float64))
    np.testing.assert_allclose(gi, g[f"conv_{tag}_gi"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(gw, g[f"conv_{tag}_gw"], rtol=0, atol=1e-11)


def test_kats():
    g = golden("kats.npz")
    oc, st = O.generate_output_coords(g["kat_oc_in"], (1, 1), 2)
    np.testing.assert_array_equal(oc, g["kat_oc_out"])
    np.testing.assert_array_equal(oc, [[0, 0, 0], [0, 0, 2]])
    assert st == (2, 2)
    km = O.build_kernel_map(g["kat_grid_in"], g["kat_grid_in"], O.hypercubic_offsets(2, 3), (1, 1))
    for (a, b), (ea, eb) in zip(km, csr_pairs(g["kat_grid_ptr"], g["kat_grid_pin"], g["kat_grid_pout"])):
        np.testing.assert_array_equal(a, ea)
        np.testing.assert_array_equal(b, eb)
    d = O.dense_conv_forward(g["kat_dense_grid"], g["kat_dense_w"], O.hypercubic_offsets(2, 3))
    np.testing.assert_allclose(d, g["kat_dense_out"], atol=1e-12)
    d1 = O.dense_conv_forward(np.array([[1.0], [2.0], [3.0]]), np.ones((3, 1, 1)), O.hypercubic_offsets(1, 3))
    np.testing.assert_allclose(d1[:, 0], [3, 6, 5])
    np.testing.assert_allclose(d1, g["kat_1d_out"])


def test_sparse_equals_dense_on_full_grid():
    """SPEC.md:164 oracle equivalence (acceptance 3) on the restatement."""
    rng = np.random.default_rng(0)
    for _ in range(5):
        sh = tuple(int(v) for v in rng.integers(2, 6, 3))
        grid = rng.normal(size=sh + (3,))
        w = rng.normal(size=(27, 4, 3))
        coords = np.array([[0, *idx] for idx in np.ndindex(*sh)])
        feats = np.array([grid[tuple(c[1:])] for c in coords])
        off = O.hypercubic_offsets(3, 3)
        _, y, _ = O.sparse_conv_forward(coords, feats, (1, 1, 1), w, off, 1)
        d = O.dense_conv_forward(grid, w, off)
        np.testing.assert_allclose(y, np.array([d[tuple(c[1:])] for c in coords]), atol=1e-9)


def test_transposed_is_adjoint():
    rng = np.random.default_rng(4)
    c = np.unique(np.concatenate([np.zeros((200, 1), int), rng.integers(-6, 6, (200, 3))], 1), axis=0)
    off = O.hypercubic_offsets(3, 3)
    oc, _ = O.generate_output_coords(c, (1, 1, 1), 2)
    x = rng.normal(size=(len(c), 3))
    w = rng.normal(size=(27, 5, 3))
    _, y, _ = O.sparse_conv_forward(c, x, (1, 1, 1), w, off, 2)
    z = rng.normal(size=(len(oc), 5))
    # <conv(x), z> == <x, convT(z)>
    xt = O.sparse_conv_transposed(c, (1, 1, 1), z, np.ascontiguousarray(w.transpose(0, 2, 1)), off, 2)
    np.testing.assert_allclose((y * z).sum(), (x * xt).sum(), rtol=1e-10)


def test_resnet_step_finite_difference():
    """Glue restatement sanity: analytic grads of the oracle SparseResNet vs
    central differences on a tiny instance (parity unpinned — self-defined)."""
    pts, offs = O.synthetic_batch(2, 120, 16, seed=1, dtype=np.float64)
    c, f = O.voxelize_batch(pts, offs, 1.0, 16)
    planes = (4, 4, 8, 8)
    p = O.init_params(1, planes, 1, 5)
    labels = np.array([1, 3])
    loss, grads, _, _ = O.resnet_train_step(p, c, f, labels, 2, planes=planes)
    rng = np.random.default_rng(0)
    for name in ["stem.w", "s1.b0.c1.w", "s3.down.gamma", "fc.w"]:
        for _ in range(2):
            idx = tuple(rng.integers(0, s) for s in p[name].shape)
            h = 1e-5
            pp = {k: v.copy() for k, v in p.items()}
            pp[name][idx] += h
            lp = O.resnet_train_step(pp, c, f, labels, 2, planes=planes)[0]
            pp[name][idx] -= 2 * h
            lm = O.resnet_train_step(pp, c, f, labels, 2, planes=planes)[0]
            fd = (lp - lm) / (2 * h)
            assert abs(fd - grads[name][idx]) <= 1e-4 * max(1.0, abs(fd)) + 1e-7, (name, fd, grads[name][idx])
