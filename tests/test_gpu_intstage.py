"""GPU parity for the integer stage (hash, packing, output coordinates, kernel
maps, voxelization, validation): BIT-EXACT against the reference's golden
vectors and the pinned oracle."""
import numpy as np
import pytest

import voxpipe_oracle as O
from conftest import csr_pairs, golden

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def _assert_pairs(km, expected):
    got = km.pairs
    assert len(got) == len(expected)
    for (a, b), (ea, eb) in zip(got, expected):
        np.testing.assert_array_equal(a.cpu().numpy(), ea)
        np.testing.assert_array_equal(b.cpu().numpy(), eb)


def test_hash_seam_first_occurrence():
    from paper_2012_13846_b200 import kernels
    g = golden("hash.npz")
    a, b = kernels.build_table(g["keys"])
    rows = kernels.lookup(a, b, g["queries"])
    assert isinstance(rows, np.ndarray) and rows.dtype == np.int64
    np.testing.assert_array_equal(rows, g["rows"])


def test_hash_empty_and_pack():
    from paper_2012_13846_b200 import kernels
    a, b = kernels.build_table(np.empty(0, np.int64))
    np.testing.assert_array_equal(kernels.lookup(a, b, np.array([1, 2, -1])), [-1, -1, -1])
    rows = np.array([[0, 1, -2, 3], [65535, 32767, -32768, 0], [7, 0, 0, 0]])
    np.testing.assert_array_equal(kernels.pack_rows(rows), O.pack_rows(rows))
    np.testing.assert_array_equal(kernels.pack_rows(rows[:, :3]), O.pack_rows(rows[:, :3]))
    from paper_2012_13846_b200.errors import ValidationError
    with pytest.raises(ValidationError):
        kernels.pack_rows(np.array([[0, 40000, 0, 0]]))
    idx = kernels.coord_index(rows)
    q = np.array([[0, 1, -2, 3], [0, 99999, 0, 0], [7, 0, 0, 0], [-1, 0, 0, 0]])
    np.testing.assert_array_equal(idx.lookup(q), [0, -1, 2, -1])


@pytest.mark.parametrize("trial", range(4))
def test_output_coords_and_maps_golden(trial):
    from paper_2012_13846_b200 import conv
    from paper_2012_13846_b200.tensor import SparseTensor
    g = golden("kmaps.npz")
    shape = conv.KernelShape.hypercubic(3, 3)
    c = g[f"t{trial}_in0"]
    t = SparseTensor(c, np.zeros((len(c), 1)), (1, 1, 1))
    for lvl in range(3):
        pre = f"t{trial}_l{lvl}"
        km = conv.build_kernel_map(t.coords, t.coords, shape, t.tensor_stride)
        _assert_pairs(km, csr_pairs(g[pre + "_s1_ptr"], g[pre + "_s1_in"], g[pre + "_s1_out"]))
        oc, ns = conv.generate_output_coords(t, 2)
        np.testing.assert_array_equal(oc.cpu().numpy(), g[pre + "_s2_oc"])
        km = conv.build_kernel_map(t.coords, oc, shape, t.tensor_stride)
        _assert_pairs(km, csr_pairs(g[pre + "_s2_ptr"], g[pre + "_s2_in"], g[pre + "_s2_out"]))
        t = SparseTensor(oc, np.zeros((len(oc), 1)), ns)


@pytest.mark.parametrize("tag,stride", [("s3", 3), ("s213", (2, 1, 3)), ("k5", 1), ("k1", 1)])
def test_aniso_golden(tag, stride):
    from paper_2012_13846_b200 import conv
    from paper_2012_13846_b200.tensor import SparseTensor
    g = golden("kmaps.npz")
    c = g["aniso_in"]
    t = SparseTensor(c, np.zeros((len(c), 1)), (1, 1, 1))
    oc, ns = conv.generate_output_coords(t, stride)
    np.testing.assert_array_equal(oc.cpu().numpy(), g[f"aniso_{tag}_oc"])
    assert tuple(ns) == tuple(g[f"aniso_{tag}_stride"])
    shape = conv.KernelShape.custom(3, g[f"aniso_{tag}_offsets"])
    km = conv.build_kernel_map(c, oc, shape, (1, 1, 1))
    _assert_pairs(km, csr_pairs(g[f"aniso_{tag}_ptr"], g[f"aniso_{tag}_in"], g[f"aniso_{tag}_out"]))


def test_edge_of_packable_range():
    from paper_2012_13846_b200 import conv
    g = golden("kmaps.npz")
    km = conv.build_kernel_map(g["edge_in"], g["edge_in"], conv.KernelShape.hypercubic(3, 3), (1, 1, 1))
    _assert_pairs(km, csr_pairs(g["edge_ptr"], g["edge_pin"], g["edge_pout"]))


def test_kats_2d():
    from paper_2012_13846_b200 import conv
    from paper_2012_13846_b200.tensor import SparseTensor
    g = golden("kats.npz")
    t = SparseTensor(g["kat_oc_in"], np.zeros((3, 1)), (1, 1))
    oc, st = conv.generate_output_coords(t, 2)
    np.testing.assert_array_equal(oc.cpu().numpy(), [[0, 0, 0], [0, 0, 2]])
    assert st == (2, 2)
    km = conv.build_kernel_map(g["kat_grid_in"], g["kat_grid_in"], conv.KernelShape.hypercubic(2, 3), (1, 1))
    _assert_pairs(km, csr_pairs(g["kat_grid_ptr"], g["kat_grid_pin"], g["kat_grid_pout"]))
    # isolated point -> 1 pair at the zero offset; far points -> 2 pairs
    km = conv.build_kernel_map([[0, 0, 0, 0]], [[0, 0, 0, 0]], conv.KernelShape.hypercubic(3, 3), (1, 1, 1))
    assert km.total_pairs() == 1 and len(km.pairs[13][0]) == 1
    km = conv.build_kernel_map([[0, 0, 0], [0, 2, 2]], [[0, 0, 0], [0, 2, 2]], conv.KernelShape.hypercubic(2, 3), (1, 1))
    assert km.total_pairs() == 2


def test_empty_tensor():
    from paper_2012_13846_b200 import conv
    from paper_2012_13846_b200.tensor import SparseTensor
    t = SparseTensor(np.empty((0, 4), np.int64), np.empty((0, 2)), (1, 1, 1))
    oc, st = conv.generate_output_coords(t, 2)
    assert oc.shape == (0, 4) and st == (2, 2, 2)
    km = conv.build_kernel_map(t.coords, oc, conv.KernelShape.hypercubic(3, 3), (1, 1, 1))
    assert km.total_pairs() == 0 and len(km.pairs) == 27


def test_random_large_maps_vs_oracle():
    """~60k rows, negative coords, 3 batches, strides 1/2/4 — bit-exact."""
    from paper_2012_13846_b200 import conv
    from paper_2012_13846_b200.tensor import SparseTensor
    rng = np.random.default_rng(11)
    c = np.unique(np.concatenate([rng.integers(0, 3, (80000, 1)), rng.integers(-60, 60, (80000, 3))], 1), axis=0)
    c = c[rng.permutation(len(c))]
    shape = conv.KernelShape.hypercubic(3, 3)
    t = SparseTensor(c, np.zeros((len(c), 1)), (1, 1, 1))
    ref_c, ref_s = c, (1, 1, 1)
    for _ in range(3):
        km = conv.build_kernel_map(t.coords, t.coords, shape, t.tensor_stride)
        _assert_pairs(km, O.build_kernel_map(ref_c, ref_c, shape.offsets, ref_s))
        oc, ns = conv.generate_output_coords(t, 2)
        roc, rns = O.generate_output_coords(ref_c, ref_s, 2)
        np.testing.assert_array_equal(oc.cpu().numpy(), roc)
        km = conv.build_kernel_map(t.coords, oc, shape, t.tensor_stride)
        _assert_pairs(km, O.build_kernel_map(ref_c, roc, shape.offsets, ref_s))
        t = SparseTensor(oc, np.zeros((len(oc), 1)), ns)
        ref_c, ref_s = roc, rns


def test_voxelize_golden_and_batch():
    from paper_2012_13846_b200 import tensor as T
    g = golden("conv.npz")
    pts = torch.from_numpy(g["vox_points"]).cuda()
    t = T.voxelize_batch(pts, torch.from_numpy(g["vox_offsets"]), 1.0, (32, 32, 32))
    np.testing.assert_array_equal(t.coords.cpu().numpy(), g["vox_coords"])
    np.testing.assert_array_equal(t.features.cpu().numpy(), g["vox_feats"])
    # per-cloud voxelize + batch() == fused path
    offs = g["vox_offsets"]
    ts = [T.voxelize(T.PointCloud(g["vox_points"][offs[i]:offs[i + 1]]), 1.0, (32, 32, 32))
          for i in range(len(offs) - 1)]
    bt = T.batch(ts)
    np.testing.assert_array_equal(bt.coords.cpu().numpy(), g["vox_coords"])
    # mean features (tensor.py:178-183)
    m = T.voxelize(T.PointCloud(g["voxm_points"], g["voxm_feats_in"]), 0.75, (10, 10, 10))
    np.testing.assert_array_equal(m.coords.cpu().numpy(), g["voxm_coords"])
    np.testing.assert_allclose(m.features.cpu().numpy(), g["voxm_feats"], rtol=1e-6, atol=1e-6)


def test_voxelize_large_bench_shape():
    """C3-shaped batch (64 x 2048 pts @ 64^3), f32 points: bit-exact vs oracle on
    the same (f32 -> f64 upcast) points."""
    from paper_2012_13846_b200 import tensor as T
    pts, offs = O.synthetic_batch(64, 2048, 64, seed=0, dtype=np.float32)
    t = T.voxelize_batch(torch.from_numpy(pts).cuda(), torch.from_numpy(offs), 1.0, (64, 64, 64))
    rc, _ = O.voxelize_batch(pts.astype(np.float64), offs, 1.0, 64)
    np.testing.assert_array_equal(t.coords.cpu().numpy(), rc)


def test_validation_errors():
    from paper_2012_13846_b200.errors import StructuralError, ValidationError
    from paper_2012_13846_b200.tensor import SparseTensor, batch
    with pytest.raises(StructuralError):
        SparseTensor([[0, 1, 1, 1], [0, 1, 1, 1]], np.zeros((2, 1)), (1, 1, 1))
    with pytest.raises(ValidationError):
        SparseTensor([[-1, 1, 1, 1]], np.zeros((1, 1)), (1, 1, 1))
    with pytest.raises(ValidationError):
        SparseTensor([[0, 1, 2, 2]], np.zeros((1, 1)), (2, 2, 2))
    with pytest.raises(ValidationError):
        SparseTensor([[0, 0, 0, 0]], np.array([[np.nan]]), (1, 1, 1))
    with pytest.raises(StructuralError):
        SparseTensor([[0, 0, 0, 0]], np.zeros((2, 1)), (1, 1, 1))
    a = SparseTensor([[0, 0, 0, 0]], np.zeros((1, 1)), (1, 1, 1))
    b = batch([a, a])
    assert len(b) == 2 and b.coords[:, 0].tolist() == [0, 1]
    two = SparseTensor([[0, 0, 0, 0], [1, 0, 0, 0]], np.zeros((2, 1)), (1, 1, 1))
    with pytest.raises(StructuralError):  # flattening batch indices collides (tensor.py:224-229)
        batch([two])


def test_voxel_mean_many_points_in_one_voxel():
    """clipping can pile a large share of a cloud into one boundary
    voxel; the point-order mean must stay exact and fast (heapsort path for
    segments > 32 points)."""
    import time
    from paper_2012_13846_b200 import tensor as T
    rng = np.random.default_rng(4)
    n = 60000
    pts = rng.uniform(-50.0, 60.0, (n, 3))  # most points clip into the corner/edge voxels of a 4^3 grid
    feats = rng.normal(size=(n, 2))
    t0 = time.time()
    m = T.voxelize(T.PointCloud(pts, feats), 1.0, (4, 4, 4))
    torch.cuda.synchronize()
    assert time.time() - t0 < 20.0
    rc, rf = O.voxelize(pts, 1.0, (4, 4, 4), features=feats)
    np.testing.assert_array_equal(m.coords.cpu().numpy(), rc)
    np.testing.assert_allclose(m.features.cpu().numpy(), rf, rtol=1e-6, atol=1e-6)
