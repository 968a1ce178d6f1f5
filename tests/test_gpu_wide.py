"""Wide coordinates: the GPU counterpart of the reference's TupleCoordIndex
fallback (kernels.py:95-122) — rows with D > 3 axes or values outside the
packed 16-bit fields.  Output coordinates and kernel maps are bit-exact with
the reference itself (oracle/_ref), which indexes such rows by tuple; the
f64 conv forward/backward matches it to 1e-10."""
import zlib

import numpy as np
import pytest

from parity_util import reference

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def ref():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    mods = reference()
    if mods is None:
        pytest.skip("oracle/_ref not built")
    return mods


def _rows(rng, n, dim, lo, hi, batches=3, ts=1):
    c = np.concatenate([rng.integers(0, batches, (n, 1)), rng.integers(lo, hi, (n, dim)) * ts], 1).astype(np.int64)
    _, first = np.unique(c, axis=0, return_index=True)
    return c[np.sort(first)]


CASES = {
    "4d": (4, -6, 6, 1),                     # D > 3: never packable
    "far": (3, 100000, 100040, 1),           # beyond the 16-bit fields
    "neg_edge": (3, -32768, -32700, 1),      # -32768 // 3 * 3 = -32769
    "mixed": (3, -40000, 40000, 1),
    "2d_far": (2, 70000, 70030, 1),
}


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("stride", [2, 3])
def test_wide_output_coords_and_maps_vs_reference(ref, case, stride):
    R, _ = ref
    from paper_2012_13846_b200 import conv
    from paper_2012_13846_b200.tensor import SparseTensor
    dim, lo, hi, ts = CASES[case]
    rng = np.random.default_rng(zlib.crc32(f"{case}{stride}".encode()))
    n = 3000 if dim <= 3 else 1500
    c = _rows(rng, n, dim, lo, hi)
    t = SparseTensor(c, np.zeros((len(c), 1)), (1,) * dim)
    assert t.wide
    rt = R.SparseTensor(c, np.zeros((len(c), 1)), (1,) * dim)
    oc, ns = conv.generate_output_coords(t, stride)
    roc, rns = R.generate_output_coords(rt, stride)
    assert ns == rns
    np.testing.assert_array_equal(oc.cpu().numpy(), roc)
    shape = conv.KernelShape.hypercubic(dim, 3)
    rshape = R.KernelShape.hypercubic(dim, 3)
    for src, dst, st in ((c, c, (1,) * dim), (c, roc, (1,) * dim)):
        km = conv.build_kernel_map(src, dst, shape, st)
        rk = R.build_kernel_map(src, dst, rshape, st)
        assert km.total_pairs() == rk.total_pairs()
        for (a, b), (ea, eb) in zip(km.pairs, rk.pairs):
            np.testing.assert_array_equal(a.cpu().numpy(), ea)
            np.testing.assert_array_equal(b.cpu().numpy(), eb)


@pytest.mark.parametrize("case", ["4d", "far"])
def test_wide_conv_f64_vs_reference(ref, case):
    R, _ = ref
    from paper_2012_13846_b200 import conv
    from paper_2012_13846_b200.tensor import SparseTensor
    dim, lo, hi, ts = CASES[case]
    rng = np.random.default_rng(9)
    c = _rows(rng, 2000, dim, lo, hi)
    x = rng.normal(size=(len(c), 8))
    shape = conv.KernelShape.hypercubic(dim, 3)
    w = rng.normal(size=(shape.num_offsets, 16, 8)) / np.sqrt(shape.num_offsets * 8)
    t = SparseTensor(c, torch.from_numpy(x).cuda(), (1,) * dim)
    W = conv.ConvWeights(torch.from_numpy(w).cuda())
    rt = R.SparseTensor(c, x, (1,) * dim)
    rw = R.ConvWeights(w)
    rshape = R.KernelShape.hypercubic(dim, 3)
    for stride in (1, 2):
        y = conv.sparse_conv_forward(t, W, shape, stride)
        ry = R.sparse_conv_forward(rt, rw, rshape, stride)
        np.testing.assert_array_equal(y.coords.cpu().numpy(), ry.coords)
        assert np.abs(y.features.cpu().numpy() - ry.features).max() <= 1e-10 * np.abs(ry.features).max()
        g = rng.normal(size=ry.features.shape)
        gi, gw = conv.sparse_conv_backward(t, W, shape, stride, torch.from_numpy(g).cuda())
        rgi, rgw = R.sparse_conv_backward(rt, rw, rshape, stride, g)
        assert np.abs(gi.cpu().numpy() - rgi).max() <= 1e-10 * np.abs(rgi).max()
        assert np.abs(gw.cpu().numpy() - rgw).max() <= 1e-10 * np.abs(rgw).max()


def test_wide_validation_errors():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2012_13846_b200.errors import StructuralError, ValidationError
    from paper_2012_13846_b200.tensor import SparseTensor
    with pytest.raises(StructuralError):
        SparseTensor([[0, 1, 2, 3, 4], [0, 1, 2, 3, 4]], np.zeros((2, 1)), (1, 1, 1, 1))
    with pytest.raises(ValidationError):
        SparseTensor([[-1, 100000, 0, 0]], np.zeros((1, 1)), (1, 1, 1))
    with pytest.raises(ValidationError):
        SparseTensor([[0, 100001, 0, 0]], np.zeros((1, 1)), (2, 2, 2))
    t = SparseTensor([[0, 100000, 0, 0], [1, 100000, 0, 0]], np.zeros((2, 1)), (2, 2, 2))
    assert t.wide and len(t) == 2


def test_abi_output_coords_flags_unpackable_rows():
    """at the C-ABI, a row that is packable before downsampling
    but not after (x = -32768 floored to a multiple of 3 = -32769) is not
    merged silently: vp_output_coords reports n_out = -1 (use the wide path)."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2012_13846_b200 import _lib
    c = torch.tensor([[0, -32768, 0, 0], [0, -32767, 5, 0], [1, 3, 3, 3]], dtype=torch.int32, device="cuda")
    out = torch.empty_like(c)
    n_out = torch.empty(1, dtype=torch.int32, device="cuda")
    ws = _lib.workspace(_lib.query("vp_output_coords_ws_bytes", 3), c.device)
    for step, expect in (((3, 3, 3), -1), ((2, 2, 2), 3)):
        _lib.call("vp_output_coords", c.data_ptr(), None, 3, _lib.i32_array(step), out.data_ptr(), n_out.data_ptr(),
                  None, ws.data_ptr(), ws.numel(), _lib.stream())
        assert int(n_out.item()) == expect, (step, int(n_out.item()))
