"""GPU parity for the float stage: forward / dgrad / wgrad (tcgen05 and SIMT
paths) against the reference's golden vectors and the f64 oracle.

Tolerance model: the oracle runs in f64 on the
SAME bf16-rounded inputs and weights, so only accumulation and output
rounding are measured:
  bf16 storage (tcgen05, fp32 accumulate, bf16 out): |d| <= 1e-2 * sum|W||x| (+ bf16 ulp)
  fp32 path (SIMT, fp32 out):                        |d| <= 1e-5 * sum|W||x|
"""
import numpy as np
import pytest

import voxpipe_oracle as O
from conftest import golden

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def bf16_round(a):
    return torch.from_numpy(np.asarray(a, np.float32)).to(torch.bfloat16).float().numpy().astype(np.float64)


def abs_bound(coords, feats, w, offsets, stride, rel):
    """rel * sum_k |W_k| |x| per output element (the error scale of Eq. 3)."""
    _, s, _ = O.sparse_conv_forward(coords, np.abs(feats), (1, 1, 1), np.abs(w), offsets, stride)
    return rel * s + 1e-6


def run_layer(coords, x, w, stride, dtype):
    from paper_2012_13846_b200 import conv
    from paper_2012_13846_b200.tensor import SparseTensor
    shape = conv.KernelShape.hypercubic(3, 3)
    t = SparseTensor(coords, np.zeros((len(coords), 1)), (1, 1, 1))
    xt = torch.from_numpy(np.asarray(x, np.float32)).cuda().to(dtype)
    t = t.with_features(xt)
    W = conv.ConvWeights(torch.from_numpy(np.asarray(w, np.float32)).cuda())
    y = conv.sparse_conv_forward(t, W, shape, stride)
    return t, W, shape, y


@pytest.mark.parametrize("tag,stride", [("s1", 1), ("s2", 2), ("s1b", 1)])
@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_conv_golden(tag, stride, dtype):
    from paper_2012_13846_b200 import conv
    g = golden("conv.npz")
    coords = g["vox_coords"]
    x, w, gy = g[f"conv_{tag}_x"], g[f"conv_{tag}_w"], g[f"conv_{tag}_g"]
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    rel = 1e-2 if dtype == "bf16" else 1e-5
    xr = bf16_round(x) if dtype == "bf16" else x.astype(np.float64)
    wr = bf16_round(w) if dtype == "bf16" else w.astype(np.float64)
    gr = bf16_round(gy) if dtype == "bf16" else gy.astype(np.float64)
    off = O.hypercubic_offsets(3, 3)
    t, W, shape, y = run_layer(coords, x, w, stride, tdt)
    np.testing.assert_array_equal(y.coords.cpu().numpy(), g[f"conv_{tag}_yc"])
    _, ry, _ = O.sparse_conv_forward(coords, xr, (1, 1, 1), wr, off, stride)
    if dtype == "f32":  # inputs are exactly representable: compare with the reference's own f64 output too
        np.testing.assert_allclose(ry, g[f"conv_{tag}_y"], atol=1e-9)
    err = np.abs(y.features.float().cpu().numpy() - ry)
    assert (err <= abs_bound(coords, xr, wr, off, stride, rel)).all(), err.max()
    gi, gw = conv.sparse_conv_backward(t, W, shape, stride, torch.from_numpy(gy).cuda().to(tdt))
    rgi, rgw = O.sparse_conv_backward(coords, xr, (1, 1, 1), wr, off, stride, gr)
    # dgrad bound: rel * sum |W^T| |g| per input element
    K = 27
    km = O.build_kernel_map(coords, O.generate_output_coords(coords, (1, 1, 1), stride)[0], off, (1, 1, 1))
    bgi = np.zeros_like(rgi)
    bgw = np.zeros_like(rgw)
    for k, (vi, ui) in enumerate(km):
        bgi[vi] += np.abs(gr[ui]) @ np.abs(wr[k])
        bgw[k] = np.abs(gr[ui]).T @ np.abs(xr[vi])
    assert (np.abs(gi.float().cpu().numpy() - rgi) <= rel * bgi + 1e-6).all()
    # wgrad is fp32 in both modes; inputs identical -> only accumulation order differs
    assert (np.abs(gw.cpu().numpy() - rgw) <= 1e-5 * bgw + 1e-6).all(), np.abs(gw.cpu().numpy() - rgw).max()


@pytest.mark.parametrize("cin,cout", [(32, 32), (32, 64), (64, 64), (64, 128), (128, 128), (128, 256),
                                      (256, 256), (256, 128), (64, 32), (128, 32), (256, 32)])
@pytest.mark.parametrize("stride", [1, 2])
def test_tc_widths(cin, cout, stride):
    """Every tcgen05 template instantiation used by the models, bf16."""
    from paper_2012_13846_b200 import conv
    pts, offs = O.synthetic_batch(3, 700, 32, seed=cin + cout, dtype=np.float64)
    coords, _ = O.voxelize_batch(pts, offs, 1.0, 32)
    rng = np.random.default_rng(cin * 7 + cout)
    x = rng.normal(size=(len(coords), cin)).astype(np.float32)
    w = (rng.normal(size=(27, cout, cin)) / np.sqrt(27 * cin)).astype(np.float32)
    xr, wr = bf16_round(x), bf16_round(w)
    off = O.hypercubic_offsets(3, 3)
    t, W, shape, y = run_layer(coords, x, w, stride, torch.bfloat16)
    _, ry, _ = O.sparse_conv_forward(coords, xr, (1, 1, 1), wr, off, stride)
    err = np.abs(y.features.float().cpu().numpy() - ry)
    assert (err <= abs_bound(coords, xr, wr, off, stride, 1e-2)).all(), err.max()
    gy = rng.normal(size=ry.shape).astype(np.float32)
    gr = bf16_round(gy)
    gi, gw = conv.sparse_conv_backward(t, W, shape, stride, torch.from_numpy(gy).cuda().to(torch.bfloat16))
    rgi, rgw = O.sparse_conv_backward(coords, xr, (1, 1, 1), wr, off, stride, gr)
    # per-element bounds: dgrad (bf16 store) 1e-2 * sum|W||g|,
    # wgrad (fp32 store) 1e-5 * sum|g||x| — the backward of the absolute values
    bgi, bgw = O.sparse_conv_backward(coords, np.abs(xr), (1, 1, 1), np.abs(wr), off, stride, np.abs(gr))
    ei = np.abs(gi.float().cpu().numpy() - rgi)
    ew = np.abs(gw.cpu().numpy() - rgw)
    assert (ei <= 1e-2 * bgi + 1e-6).all(), (ei / (bgi + 1e-9)).max()
    assert (ew <= 1e-5 * bgw + 1e-7).all(), (ew / (bgw + 1e-9)).max()


@pytest.mark.parametrize("cout,clouds,npts", [(32, 2, 500), (16, 2, 500), (64, 2, 500), (32, 6, 3000)])
def test_stem_cin1_simt(cout, clouds, npts):
    """C_in = 1 (occupancy stem) goes through the SIMT kernels (wgrad: the
    stem kernel, several pair chunks per offset in the large case)."""
    from paper_2012_13846_b200 import conv
    pts, offs = O.synthetic_batch(clouds, npts, 32 if clouds == 2 else 48, seed=9, dtype=np.float64)
    coords, feats = O.voxelize_batch(pts, offs, 1.0, 32 if clouds == 2 else 48)
    rng = np.random.default_rng(5)
    w = (rng.normal(size=(27, cout, 1)) / np.sqrt(27)).astype(np.float32)
    for dt, rel in ((torch.float32, 1e-5), (torch.bfloat16, 1e-2)):
        t, W, shape, y = run_layer(coords, feats, w, 1, dt)
        wr = w.astype(np.float64) if dt == torch.float32 else bf16_round(w)
        _, ry, _ = O.sparse_conv_forward(coords, feats, (1, 1, 1), w.astype(np.float64), O.hypercubic_offsets(3, 3), 1)
        assert np.abs(y.features.float().cpu().numpy() - ry).max() <= rel * np.abs(ry).max() + 1e-5
        gy = rng.normal(size=ry.shape)
        gi, gw = conv.sparse_conv_backward(t, W, shape, 1, torch.from_numpy(gy).cuda().to(dt))
        gq = gy if dt == torch.float32 else bf16_round(gy)
        rgi, rgw = O.sparse_conv_backward(coords, feats, (1, 1, 1), w.astype(np.float64), O.hypercubic_offsets(3, 3), 1, gq)
        assert np.abs(gw.cpu().numpy() - rgw).max() <= 1e-4 * np.abs(rgw).max()


def test_deterministic():
    from paper_2012_13846_b200 import conv
    pts, offs = O.synthetic_batch(4, 1500, 48, seed=2, dtype=np.float64)
    coords, _ = O.voxelize_batch(pts, offs, 1.0, 48)
    rng = np.random.default_rng(1)
    x = rng.normal(size=(len(coords), 64)).astype(np.float32)
    w = (rng.normal(size=(27, 64, 64)) / 40).astype(np.float32)
    t, W, shape, y1 = run_layer(coords, x, w, 1, torch.bfloat16)
    g = torch.randn_like(y1.features)
    a = conv.sparse_conv_backward(t, W, shape, 1, g)
    y2 = conv.sparse_conv_forward(t, W, shape, 1)
    b = conv.sparse_conv_backward(t, W, shape, 1, g)
    assert torch.equal(y1.features, y2.features)
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])


def test_sparse_equals_dense_full_grid():
    """SPEC.md:164 / acceptance 3: fully occupied grids <= 6^3, fp32 path."""
    from paper_2012_13846_b200 import conv
    rng = np.random.default_rng(0)
    for _ in range(6):
        sh = tuple(int(v) for v in rng.integers(2, 7, 3))
        grid = rng.normal(size=sh + (3,))
        w = rng.normal(size=(27, 4, 3))
        coords = np.array([[0, *idx] for idx in np.ndindex(*sh)])
        feats = np.array([grid[tuple(c[1:])] for c in coords])
        t, W, shape, y = run_layer(coords, feats, w, 1, torch.float32)
        d = O.dense_conv_forward(grid, w.astype(np.float32).astype(np.float64), shape.offsets)
        exp = np.array([d[tuple(c[1:])] for c in coords])
        np.testing.assert_allclose(y.features.cpu().numpy(), exp, atol=1e-4)


def test_transposed_conv_adjoint():
    from paper_2012_13846_b200 import conv
    from paper_2012_13846_b200.tensor import SparseTensor
    rng = np.random.default_rng(4)
    c = np.unique(np.concatenate([np.zeros((400, 1), int), rng.integers(-8, 8, (400, 3))], 1), axis=0)
    off = O.hypercubic_offsets(3, 3)
    oc, _ = O.generate_output_coords(c, (1, 1, 1), 2)
    z = rng.normal(size=(len(oc), 32))
    wt = rng.normal(size=(27, 32, 32)) / 30
    coarse = SparseTensor(oc, z, (2, 2, 2))
    y = conv.sparse_conv_transposed(coarse, conv.ConvWeights(wt), conv.KernelShape.hypercubic(3, 3), 2, c)
    ref = O.sparse_conv_transposed(c, (1, 1, 1), z.astype(np.float32), wt.astype(np.float32), off, 2)
    np.testing.assert_allclose(y.features.cpu().numpy(), ref, atol=1e-4)
    assert y.tensor_stride == (1, 1, 1)


@pytest.mark.parametrize("c", [32, 128, 256])
@pytest.mark.parametrize("stride", [1, 2])
def test_mask_sorted_rows_bitwise_equal(c, stride):
    """vp_kernel_map_group (9-bit key grouping, kmap_sort.cu; column key for
    neighbour tables, plane key for strided inverse tables): perm
    is a permutation of the live rows in stable key order, the sorted table
    is table[perm], and forward / dgrad over (sorted table, perm) equal
    the unsorted launch (bit for bit when no tile splits or offset pairing
    regroups the fp32 sums; within one bf16 rounding otherwise)."""
    from paper_2012_13846_b200 import conv
    from paper_2012_13846_b200.tensor import SparseTensor
    pts, offs = O.synthetic_batch(6, 2048, 64, seed=11, dtype=np.float32)
    c0, _ = O.voxelize_batch(pts.astype(np.float64), offs, 1.0, 64)
    t = SparseTensor(c0, np.zeros((len(c0), 1)), (1, 1, 1))
    shape = conv.KernelShape.hypercubic(3, 3)
    out4, _ = conv._output_coords4(t.coords4, (1, 1, 1), (stride,) * 3, 3)
    km = conv._kernel_map4(t.coords4, out4, shape, (1, 1, 1), 3)
    n_out, n = out4.shape[0], len(t)
    perm, ts = conv.sort_table(km.nbr, n_out)
    p = perm.cpu().numpy()
    assert np.array_equal(np.sort(p), np.arange(n_out))
    assert torch.equal(ts, km.nbr[perm.long()])
    from parity_util import check_grouping
    check_grouping(p, ts.cpu().numpy(), 0, "forward table")
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(n, c, device="cuda", generator=g).to(torch.bfloat16)
    W = conv.ConvWeights(torch.randn(27, c, c, device="cuda", generator=g) / (27 * c) ** 0.5)
    y0 = conv.conv_forward_raw(x, W, km.nbr, n_out)
    y1 = conv.conv_forward_raw(x, W, ts, n_out, perm=perm)
    torch.testing.assert_close(y1.float(), y0.float(), rtol=1e-2, atol=1e-2)
    gy = torch.randn(n_out, c, device="cuda", generator=g).to(torch.bfloat16)
    if stride == 1:
        tab, flip = km.nbr, True
    else:
        tab, flip = km.inverse(), False
    ip, its = conv.sort_table(tab, n, 0 if flip else 1)
    check_grouping(ip.cpu().numpy().astype(np.int64), its.cpu().numpy(), 0 if flip else 1, "dgrad table")
    d0 = conv.conv_dgrad_raw(gy, W, tab, n, flip)
    d1 = conv.conv_dgrad_raw(gy, W, its, n, flip, perm=ip)
    torch.testing.assert_close(d1.float(), d0.float(), rtol=1e-2, atol=1e-2)
    # deterministic: the same sorted launch twice is bitwise identical
    assert torch.equal(d1, conv.conv_dgrad_raw(gy, W, its, n, flip, perm=ip))


@pytest.mark.parametrize("c", [128, 256])
@pytest.mark.parametrize("sort", [False, True])
def test_large_n_two_tile_items_vs_torch(c, sort):
    """N >= 2^17 rows selects the 256-row work items (two tiles share every
    weight stage): forward and dgrad against a torch fp32 gather-matmul of
    the same bf16 operands (|d| <= 1e-2 * sum|W||x| style bound)."""
    from paper_2012_13846_b200 import conv
    from paper_2012_13846_b200.tensor import SparseTensor
    pts, offs = O.synthetic_batch(80, 2048, 64, seed=5, dtype=np.float32)
    c0, _ = O.voxelize_batch(pts.astype(np.float64), offs, 1.0, 64)
    assert len(c0) >= (1 << 17)
    t = SparseTensor(c0, np.zeros((len(c0), 1)), (1, 1, 1))
    shape = conv.KernelShape.hypercubic(3, 3)
    km = conv._kernel_map4(t.coords4, t.coords4, shape, (1, 1, 1), 3, with_pairs=False)
    n = len(t)
    g = torch.Generator(device="cuda").manual_seed(7)
    x = torch.randn(n, c, device="cuda", generator=g).to(torch.bfloat16)
    W = conv.ConvWeights(torch.randn(27, c, c, device="cuda", generator=g) / (27 * c) ** 0.5)
    perm, tbl = conv.sort_table(km.nbr, n) if sort else (None, km.nbr)
    y = conv.conv_forward_raw(x, W, tbl, n, perm=perm).float()
    xf = torch.cat([x.float(), torch.zeros(1, c, device="cuda")])
    wf = W.bf16.float()
    idx = km.nbr.long().clone()
    idx[idx < 0] = n
    ref = torch.zeros(n, c, device="cuda")
    mag = torch.zeros(n, c, device="cuda")
    for k in range(27):
        ref += xf[idx[:, k]] @ wf[k].T
        mag += xf[idx[:, k]].abs() @ wf[k].abs().T
    assert bool(((y - ref).abs() <= 1e-2 * mag + 1e-3).all())
    # dgrad (stride 1: the flipped neighbour table)
    gy = torch.randn(n, c, device="cuda", generator=g).to(torch.bfloat16)
    gi = conv.conv_dgrad_raw(gy, W, tbl, n, True, perm=perm).float()
    gf = torch.cat([gy.float(), torch.zeros(1, c, device="cuda")])
    ref = torch.zeros(n, c, device="cuda")
    mag = torch.zeros(n, c, device="cuda")
    for k in range(27):
        ref += gf[idx[:, 26 - k]] @ wf[k]
        mag += gf[idx[:, 26 - k]].abs() @ wf[k].abs()
    assert bool(((gi - ref).abs() <= 1e-2 * mag + 1e-3).all())


SHAPES = {
    "3d_1": (3, 1, None),                 # 1^3 projection (K = 1)
    "3d_5": (3, 5, None),                 # 5^3 (K = 125 > 30: no mask sort, unstaged table)
    "3d_313": (3, (3, 1, 3), None),       # anisotropic extents (K = 9)
    "2d_3": (2, 3, None),                 # 2-D 3x3 (K = 9)
    "1d_5": (1, 5, None),                 # 1-D (K = 5)
    "custom": (3, None, [[0, 0, 0], [1, 0, 0], [0, -1, 0], [0, 0, 2]]),
}


@pytest.mark.parametrize("name", list(SHAPES))
@pytest.mark.parametrize("stride", [1, 2])
@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_kernel_shapes_dims_and_strides(name, stride, dtype):
    """The operator API beyond the 3^3 / 3-D models: 1-D / 2-D tensors,
    1^3 / 5^3 / anisotropic / custom offset sets, strides 1 and 2 — output
    coordinates and kernel maps bit-exact with the reference restatement,
    forward / dgrad / wgrad within the §8(d) tolerance model."""
    from paper_2012_13846_b200 import conv
    from paper_2012_13846_b200.tensor import SparseTensor
    dim, size, custom = SHAPES[name]
    rng = np.random.default_rng(sum(map(ord, name)) + stride)  # stable across processes
    n = 700
    c = np.concatenate([rng.integers(0, 3, (n, 1)), rng.integers(-12, 12, (n, dim))], 1)
    c = c[np.sort(np.unique(c, axis=0, return_index=True)[1])]  # unique rows, first-seen order
    shape = conv.KernelShape.custom(dim, custom) if custom else conv.KernelShape.hypercubic(dim, size)
    off = shape.offsets
    cin, cout = 32, 64
    x = rng.normal(size=(len(c), cin)).astype(np.float32)
    w = (rng.normal(size=(len(off), cout, cin)) / np.sqrt(len(off) * cin)).astype(np.float32)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    rel = 1e-2 if dtype == "bf16" else 1e-5
    xr = bf16_round(x) if dtype == "bf16" else x.astype(np.float64)
    wr = bf16_round(w) if dtype == "bf16" else w.astype(np.float64)
    t = SparseTensor(c, np.zeros((len(c), 1)), (1,) * dim).with_features(torch.from_numpy(x).cuda().to(tdt))
    W = conv.ConvWeights(torch.from_numpy(w).cuda())
    st = (stride,) * dim
    # integer stage: bit-exact
    oc, _ = conv.generate_output_coords(t, st)
    roc, _ = O.generate_output_coords(c, (1,) * dim, st)
    np.testing.assert_array_equal(oc.cpu().numpy(), roc)
    km = conv.build_kernel_map(t.coords, oc, shape, (1,) * dim)
    ref = O.build_kernel_map(c, roc, off, (1,) * dim)
    for (a, b), (ea, eb) in zip(km.pairs, ref):
        np.testing.assert_array_equal(a.cpu().numpy(), ea)
        np.testing.assert_array_equal(b.cpu().numpy(), eb)
    # float stage
    y = conv.sparse_conv_forward(t, W, shape, st)
    _, ry, _ = O.sparse_conv_forward(c, xr, (1,) * dim, wr, off, st)
    _, mag, _ = O.sparse_conv_forward(c, np.abs(xr), (1,) * dim, np.abs(wr), off, st)
    assert (np.abs(y.features.float().cpu().numpy() - ry) <= rel * mag + 1e-6).all()
    gy = rng.normal(size=ry.shape).astype(np.float32)
    gr = bf16_round(gy) if dtype == "bf16" else gy.astype(np.float64)
    gi, gw = conv.sparse_conv_backward(t, W, shape, st, torch.from_numpy(gy).cuda().to(tdt))
    rgi, rgw = O.sparse_conv_backward(c, xr, (1,) * dim, wr, off, st, gr)
    bgi = np.zeros_like(rgi)
    bgw = np.zeros_like(rgw)
    for k, (vi, ui) in enumerate(ref):
        bgi[vi] += np.abs(gr[ui]) @ np.abs(wr[k])
        bgw[k] = np.abs(gr[ui]).T @ np.abs(xr[vi])
    assert (np.abs(gi.float().cpu().numpy() - rgi) <= rel * bgi + 1e-6).all()
    assert (np.abs(gw.cpu().numpy() - rgw) <= 1e-5 * bgw + 1e-6).all()


def test_rows32_kernel_opt_in():
    """The opt-in row-compacted 32-wide kernel (VP_CONV_ROWS=1, read once per
    process -> a child pytest) passes the same fwd/dgrad/wgrad checks as the
    tcgen05 path for C_in = C_out = 32 at stride 1 and 2."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, VP_CONV_ROWS="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", os.path.join(root, "tests", "test_gpu_conv.py"),
                        "-k", "test_tc_widths and 32-32"], capture_output=True, text=True, timeout=600, cwd=root,
                       env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "2 passed" in r.stdout


@pytest.mark.parametrize("cin,cout", [(16, 48), (40, 24), (8, 8), (96, 200), (256, 136), (24, 256)])
@pytest.mark.parametrize("stride", [1, 2])
def test_tc_general_widths(cin, cout, stride):
    """Widths that are multiples of 8 but not tile widths run on the tensor
    cores padded to 32/64/128/256 (zero chunks, masked stores): bf16 bounds."""
    from paper_2012_13846_b200 import conv
    pts, offs = O.synthetic_batch(3, 600, 32, seed=cin * 3 + cout, dtype=np.float64)
    coords, _ = O.voxelize_batch(pts, offs, 1.0, 32)
    rng = np.random.default_rng(cin * 11 + cout)
    x = rng.normal(size=(len(coords), cin)).astype(np.float32)
    w = (rng.normal(size=(27, cout, cin)) / np.sqrt(27 * cin)).astype(np.float32)
    xr, wr = bf16_round(x), bf16_round(w)
    off = O.hypercubic_offsets(3, 3)
    t, W, shape, y = run_layer(coords, x, w, stride, torch.bfloat16)
    _, ry, _ = O.sparse_conv_forward(coords, xr, (1, 1, 1), wr, off, stride)
    err = np.abs(y.features.float().cpu().numpy() - ry)
    assert (err <= abs_bound(coords, xr, wr, off, stride, 1e-2)).all(), err.max()
    gy = rng.normal(size=ry.shape).astype(np.float32)
    gr = bf16_round(gy)
    gi, gw = conv.sparse_conv_backward(t, W, shape, stride, torch.from_numpy(gy).cuda().to(torch.bfloat16))
    rgi, _ = O.sparse_conv_backward(coords, xr, (1, 1, 1), wr, off, stride, gr)
    bgi, _ = O.sparse_conv_backward(coords, np.abs(xr), (1, 1, 1), np.abs(wr), off, stride, np.abs(gr))
    ei = np.abs(gi.float().cpu().numpy() - rgi)
    assert (ei <= 1e-2 * bgi + 1e-6).all(), (ei / (bgi + 1e-9)).max()


@pytest.mark.parametrize("cin,cout", [(16, 32), (32, 32), (64, 64), (128, 256), (24, 40), (128, 32)])
@pytest.mark.parametrize("stride", [1, 2])
def test_tf32_mode(cin, cout, stride):
    """fp32 features with math="tf32" (kind::tf32 tensor cores, fp32 storage
    and accumulation): |d| <= 2e-3 * sum|W||x| per element
    against the f64 oracle on the same fp32 inputs, forward and dgrad."""
    from paper_2012_13846_b200 import conv
    pts, offs = O.synthetic_batch(3, 600, 32, seed=cin + 5 * cout, dtype=np.float64)
    coords, _ = O.voxelize_batch(pts, offs, 1.0, 32)
    rng = np.random.default_rng(cin * 13 + cout)
    x = rng.normal(size=(len(coords), cin)).astype(np.float32)
    w = (rng.normal(size=(27, cout, cin)) / np.sqrt(27 * cin)).astype(np.float32)
    xr, wr = x.astype(np.float64), w.astype(np.float64)
    off = O.hypercubic_offsets(3, 3)
    from paper_2012_13846_b200.tensor import SparseTensor
    shape = conv.KernelShape.hypercubic(3, 3)
    t = SparseTensor(coords, np.zeros((len(coords), 1)), (1, 1, 1)).with_features(torch.from_numpy(x).cuda())
    W = conv.ConvWeights(torch.from_numpy(w).cuda())
    y = conv.sparse_conv_forward(t, W, shape, stride, math="tf32")
    assert y.features.dtype == torch.float32
    _, ry, _ = O.sparse_conv_forward(coords, xr, (1, 1, 1), wr, off, stride)
    err = np.abs(y.features.cpu().numpy() - ry)
    bound = abs_bound(coords, xr, wr, off, stride, 2e-3)
    assert (err <= bound).all(), (err / bound).max()
    # tf32 is really in use: the exact fp32 path agrees with the oracle ~1000x tighter
    ye = conv.sparse_conv_forward(t, W, shape, stride)
    assert np.abs(ye.features.cpu().numpy() - ry).max() < err.max() or err.max() == 0
    gy = rng.normal(size=ry.shape).astype(np.float32)
    gi, gw = conv.sparse_conv_backward(t, W, shape, stride, torch.from_numpy(gy).cuda(), math="tf32")
    rgi, rgw = O.sparse_conv_backward(coords, xr, (1, 1, 1), wr, off, stride, gy.astype(np.float64))
    bgi, _ = O.sparse_conv_backward(coords, np.abs(xr), (1, 1, 1), np.abs(wr), off, stride, np.abs(gy.astype(np.float64)))
    ei = np.abs(gi.cpu().numpy() - rgi)
    assert (ei <= 2e-3 * bgi + 1e-6).all(), (ei / (bgi + 1e-9)).max()


def test_full_mask_grouping_is_the_stable_mask_sort():
    """key mode 2 (three stable 9-bit LSD passes) orders the live rows
    exactly like a stable argsort by the whole 27-bit hit mask."""
    from paper_2012_13846_b200 import _lib, conv
    from paper_2012_13846_b200.tensor import SparseTensor
    pts, offs = O.synthetic_batch(150, 2048, 64, seed=5, dtype=np.float32)
    c0, _ = O.voxelize_batch(pts.astype(np.float64), offs, 1.0, 64)
    assert len(c0) >= conv.FULL_MASK_ROWS
    t = SparseTensor(c0, np.zeros((len(c0), 1)), (1, 1, 1))
    km = conv._kernel_map4(t.coords4, t.coords4, conv.KernelShape.hypercubic(3, 3), (1, 1, 1), 3, with_pairs=False)
    n = len(c0)
    perm, ts = conv.sort_table(km.nbr, n)  # >= FULL_MASK_ROWS: mode 2
    nb = km.nbr[:n].cpu().numpy()
    mask = ((nb >= 0).astype(np.int64) << np.arange(27, dtype=np.int64)).sum(1)
    np.testing.assert_array_equal(perm.cpu().numpy(), np.argsort(mask, kind="stable"))
    assert torch.equal(ts[:n], km.nbr[perm.long()][:n])
