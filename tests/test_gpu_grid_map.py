"""Dense-grid kernel map through the C-ABI (vp_grid_init / vp_grid_set /
vp_kernel_map_grid): the unit-cube column probe and the generic probe give
pairs and nbr bit-exact with the oracle's build_kernel_map (conv.py:149-183)
on dense and sparse lattices, at every lattice face, for shuffled offset
orders, strided maps, odd lattice sizes (unaligned bitmap start) and a
non-cube kernel; the occupancy bitmap is empty again after the clear."""
import numpy as np
import pytest

import voxpipe_oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def _lattice_rows(rng, B, R, s, density):
    cells = np.argwhere(rng.random((B, R, R, R)) < density)
    rng.shuffle(cells)
    c = np.ascontiguousarray(cells, dtype=np.int32)  # argwhere is column-major
    c[:, 1:] *= s
    return c


def _grid_map(cin, cout, B, R, s, offsets, in_stride):
    from paper_2012_13846_b200 import _lib
    dev = torch.device("cuda")
    st = _lib.stream()
    K = len(offsets)
    grid = torch.full((int(_lib.query("vp_grid_words", B, R)),), 0x5A5A5A5A, dtype=torch.int32, device=dev)
    _lib.call("vp_grid_init", grid.data_ptr(), B, R, st)  # cell values are don't-care: only the bitmap is reset
    ci = torch.from_numpy(np.ascontiguousarray(cin, np.int32)).to(dev)
    co = torch.from_numpy(np.ascontiguousarray(cout, np.int32)).to(dev)
    n_out = len(cout)
    nbr = torch.empty((max(n_out, 1), K), dtype=torch.int32, device=dev)
    pin = torch.empty(max(n_out * K, 1), dtype=torch.int32, device=dev)
    pout = torch.empty_like(pin)
    ptr = torch.empty(K + 1, dtype=torch.int32, device=dev)
    ws = _lib.workspace(_lib.query("vp_kernel_map_grid_ws_bytes", n_out, K), dev)
    _lib.call("vp_grid_set", ci.data_ptr(), None, len(cin), grid.data_ptr(), B, R, s, 0, st)
    _lib.call("vp_kernel_map_grid", grid.data_ptr(), B, R, s, co.data_ptr(), None, n_out,
              _lib.i32_array(np.asarray(offsets, np.int32).ravel()), K, _lib.i32_array(in_stride), nbr.data_ptr(),
              pin.data_ptr(), pout.data_ptr(), ptr.data_ptr(), ws.data_ptr(), ws.numel(), st)
    _lib.call("vp_grid_set", ci.data_ptr(), None, len(cin), grid.data_ptr(), B, R, s, 1, st)
    torch.cuda.synchronize()
    off_bits = (B * R ** 3 + 7) // 8 * 8
    assert bool((grid[off_bits:] == 0).all()), "the clear must leave the occupancy bitmap empty"
    p = ptr.cpu().numpy()
    pairs = [(pin[p[k]:p[k + 1]].cpu().numpy(), pout[p[k]:p[k + 1]].cpu().numpy()) for k in range(K)]
    return pairs, nbr[:n_out].cpu().numpy()


def _check(cin, cout, B, R, s, offsets, in_stride):
    got, nbr = _grid_map(cin, cout, B, R, s, offsets, in_stride)
    exp = O.build_kernel_map(cin, cout, offsets, in_stride)
    for k, ((gi, go), (ei, eo)) in enumerate(zip(got, exp)):
        np.testing.assert_array_equal(gi, ei, err_msg=f"offset {k} in rows")
        np.testing.assert_array_equal(go, eo, err_msg=f"offset {k} out rows")
        col = np.full(len(cout), -1, np.int64)
        col[eo] = ei
        np.testing.assert_array_equal(nbr[:, k], col, err_msg=f"offset {k} nbr")
    return sum(len(e[0]) for e in exp)


@pytest.mark.parametrize("B,R,density", [(2, 64, 0.05), (3, 5, 0.6), (1, 33, 0.3), (4, 16, 1.0), (2, 128, 0.004)])
def test_grid_unit_cube_submanifold(B, R, density):
    rng = np.random.default_rng(R * 7 + B)
    c = _lattice_rows(rng, B, R, 1, density)
    offs = O.hypercubic_offsets(3, 3)
    assert _check(c, c, B, R, 1, offs, (1, 1, 1)) > 0
    perm = rng.permutation(27)  # the caller's offset order is arbitrary
    _check(c, c, B, R, 1, offs[perm], (1, 1, 1))


def test_grid_faces_and_corners():
    """Rows on every face / edge / corner of the lattice (z = 0 and z = R-1
    runs, 64-bit word crossings of the bitmap)."""
    B, R = 2, 64
    pts = set()
    for b in range(B):
        for x in (0, 1, R - 2, R - 1):
            for y in (0, 1, 31, R - 1):
                for z in (0, 1, 2, 30, 31, 32, 33, 62, 63):
                    pts.add((b, x, y, z))
    c = np.array(sorted(pts), np.int32)
    np.random.default_rng(3).shuffle(c)
    _check(c, c, B, R, 1, O.hypercubic_offsets(3, 3), (1, 1, 1))


def test_grid_strided_map():
    """Stride-2 output rows over a stride-1 input lattice (the engine's
    downsampling maps): the unit cube in input lattice steps."""
    rng = np.random.default_rng(5)
    B, R = 2, 32
    cin = _lattice_rows(rng, B, R, 1, 0.2)
    cout = np.unique(cin // np.array([1, 2, 2, 2], np.int32) * np.array([1, 2, 2, 2], np.int32), axis=0)
    rng.shuffle(cout)
    assert _check(cin, cout, B, R, 1, O.hypercubic_offsets(3, 3), (1, 1, 1)) > 0
    # a coarser input level: spacing 2, stride-2 input
    cin2 = cout
    cout2 = np.unique(cin2 // np.array([1, 4, 4, 4], np.int32) * np.array([1, 4, 4, 4], np.int32), axis=0)
    _check(cin2, cout2, B, R // 2, 2, O.hypercubic_offsets(3, 3), (2, 2, 2))


def test_grid_generic_kernel():
    """A non-cube kernel (5^3) takes the generic bitmap probe."""
    rng = np.random.default_rng(9)
    B, R = 2, 20
    c = _lattice_rows(rng, B, R, 1, 0.3)
    _check(c, c, B, R, 1, O.hypercubic_offsets(3, 5), (1, 1, 1))


@pytest.mark.parametrize("stride,shift", [(1, (0, 0, 0)), (1, (-70, 5, -3)), (2, (-64, 0, 2))])
def test_operator_api_lattice_path_equals_hash(monkeypatch, stride, shift):
    """conv.build_kernel_map (the operator API) on a large map takes the
    dense-grid index when the rows sit on a bounded lattice: pairs and nbr
    identical to the hash path, negative / shifted coordinates included;
    rows off the lattice fall back to the hash."""
    from paper_2012_13846_b200 import conv
    rng = np.random.default_rng(21 + stride)
    B, R = 6, 48
    c = _lattice_rows(rng, B, R, stride, 0.12)
    c[:, 1:] += np.array(shift, np.int32) * stride
    shape = conv.KernelShape.hypercubic(3, 3)
    dev = torch.device("cuda")
    c4 = torch.from_numpy(c).to(dev)
    oc4, _ = conv._output_coords4(c4, (stride,) * 3, (2, 2, 2), 3)
    calls = []
    real = conv._kernel_map_lattice
    monkeypatch.setattr(conv, "_kernel_map_lattice", lambda *a: calls.append(1) or real(*a))
    for cin, cout in ((c4, c4), (c4, oc4)):
        monkeypatch.setattr(conv, "LATTICE_MIN_ROWS", 1)
        got = conv._kernel_map4(cin, cout, shape, (stride,) * 3, 3)
        monkeypatch.setattr(conv, "LATTICE_MIN_ROWS", 1 << 40)
        exp = conv._kernel_map4(cin, cout, shape, (stride,) * 3, 3)
        assert torch.equal(got.nbr, exp.nbr)
        for (a, b), (ea, eb) in zip(got.pairs, exp.pairs):
            assert torch.equal(a, ea) and torch.equal(b, eb)
    assert len(calls) == 2
    # a row off the stride lattice: the lattice path declines, the hash path answers
    bad = c4.clone()
    bad[0, 1] += 1
    monkeypatch.setattr(conv, "LATTICE_MIN_ROWS", 1)
    if stride > 1:
        assert real(bad, bad, shape, (stride,) * 3) is None
    got = conv._kernel_map4(bad, bad, shape, (stride,) * 3, 3)
    exp = O.build_kernel_map(bad.cpu().numpy(), bad.cpu().numpy(), shape.offsets, (stride,) * 3)
    for (a, b), (ea, eb) in zip(got.pairs, exp):
        np.testing.assert_array_equal(a.cpu().numpy(), ea)
        np.testing.assert_array_equal(b.cpu().numpy(), eb)
