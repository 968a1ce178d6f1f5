"""Live differential tests against the REFERENCE ITSELF (voxpipe 0.1.0 built
into oracle/_ref by oracle/build_ref.sh; it travels to the GPU box with the
snapshot): the same inputs through `voxpipe.tensor` / `voxpipe.conv` (f64, CPU,
compiled Cython hash) and through this package's GPU operator API.

  integer stage (voxelize + batch, output coordinates, kernel maps): bit-exact
  float stage: fp32 path within 1e-5 * sum|W||x|; bf16 tcgen05 path within
               1e-2 * sum|W||x| on bf16-rounded inputs."""
import os
import sys

import numpy as np
import pytest

import voxpipe_oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ref():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    path = os.path.join(ROOT, "oracle", "_ref")
    if not os.path.isdir(os.path.join(path, "voxpipe")):
        pytest.skip("reference build (oracle/_ref) not present")
    sys.path.insert(0, path)
    from voxpipe import conv as R
    from voxpipe import kernels as RK
    from voxpipe import tensor as RT
    assert RK.backend_name() == "compiled"
    return R, RT


def bf16_round(a):
    return torch.from_numpy(np.asarray(a, np.float32)).to(torch.bfloat16).float().numpy().astype(np.float64)


def test_voxelize_and_batch_vs_reference(ref):
    R, RT = ref
    from paper_2012_13846_b200 import tensor
    pts, offs = O.synthetic_batch(6, 1500, 48, seed=13, dtype=np.float64)
    ts = [RT.voxelize(RT.PointCloud(pts[offs[i]:offs[i + 1]]), 1.0, (48, 48, 48)) for i in range(6)]
    rb = RT.batch(ts)
    t = tensor.voxelize_batch(torch.from_numpy(pts).cuda(), torch.from_numpy(offs), 1.0, (48, 48, 48),
                              feature_dtype=torch.float32)
    np.testing.assert_array_equal(t.coords.cpu().numpy(), rb.coords)
    np.testing.assert_array_equal(t.features.cpu().numpy(), rb.features)


@pytest.mark.parametrize("stride", [1, 2])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_conv_forward_backward_vs_reference(ref, stride, dtype):
    R, RT = ref
    from paper_2012_13846_b200 import conv
    from paper_2012_13846_b200.tensor import SparseTensor
    rng = np.random.default_rng(stride * 10 + (dtype == "bf16"))
    # negative coordinates, three clouds, duplicates removed in first-seen order
    c = np.concatenate([rng.integers(0, 3, (3000, 1)), rng.integers(-20, 20, (3000, 3))], 1)
    c = c[np.sort(np.unique(c, axis=0, return_index=True)[1])]
    cin, cout = 64, 32
    x = rng.normal(size=(len(c), cin))
    w = rng.normal(size=(27, cout, cin)) / np.sqrt(27 * cin)
    if dtype == "bf16":
        x, w = bf16_round(x), bf16_round(w)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    rel = 1e-2 if dtype == "bf16" else 1e-5
    rshape = R.KernelShape.hypercubic(3, 3)
    rt = R.SparseTensor(c, x, (1, 1, 1))
    ry = R.sparse_conv_forward(rt, R.ConvWeights(w), rshape, stride)
    shape = conv.KernelShape.hypercubic(3, 3)
    t = SparseTensor(c, np.zeros((len(c), 1)), (1, 1, 1)).with_features(torch.tensor(x).cuda().to(tdt))
    W = conv.ConvWeights(torch.tensor(w).cuda())
    y = conv.sparse_conv_forward(t, W, shape, stride)
    # integer stage: output coordinates and kernel map bit-exact with the reference
    np.testing.assert_array_equal(y.coords.cpu().numpy(), ry.coords)
    assert y.tensor_stride == tuple(ry.tensor_stride)
    rkm = R.build_kernel_map(c, ry.coords, rshape, (1, 1, 1))
    km = conv.build_kernel_map(t.coords, y.coords, shape, (1, 1, 1))
    for (a, b), (ea, eb) in zip(km.pairs, rkm.pairs):
        np.testing.assert_array_equal(a.cpu().numpy(), ea)
        np.testing.assert_array_equal(b.cpu().numpy(), eb)
    # float stage
    mag = np.zeros_like(ry.features)
    for k, (vi, ui) in enumerate(rkm.pairs):
        mag[ui] += np.abs(x[vi]) @ np.abs(w[k]).T
    assert (np.abs(y.features.float().cpu().numpy() - ry.features) <= rel * mag + 1e-6).all()
    g = rng.normal(size=ry.features.shape)
    if dtype == "bf16":
        g = bf16_round(g)
    rgi, rgw = R.sparse_conv_backward(rt, R.ConvWeights(w), rshape, stride, g)
    gi, gw = conv.sparse_conv_backward(t, W, shape, stride, torch.tensor(g).cuda().to(tdt))
    bgi = np.zeros_like(rgi)
    bgw = np.zeros_like(rgw)
    for k, (vi, ui) in enumerate(rkm.pairs):
        bgi[vi] += np.abs(g[ui]) @ np.abs(w[k])
        bgw[k] = np.abs(g[ui]).T @ np.abs(x[vi])
    assert (np.abs(gi.float().cpu().numpy() - rgi) <= rel * bgi + 1e-6).all()
    assert (np.abs(gw.cpu().numpy() - rgw) <= 1e-5 * bgw + 1e-6).all()


def test_cuda_hash_backend_drives_the_reference_conv(ref):
    """the reference's own conv.py with its coordinate
    index swapped for this package's GPU hash gives the same kernel maps."""
    R, RT = ref
    from voxpipe import kernels as RK
    from paper_2012_13846_b200 import kernels as GK
    rng = np.random.default_rng(3)
    c = np.concatenate([rng.integers(0, 2, (2000, 1)), rng.integers(-15, 15, (2000, 3))], 1)
    c = c[np.sort(np.unique(c, axis=0, return_index=True)[1])]
    oc, _ = R.generate_output_coords(R.SparseTensor(c, np.zeros((len(c), 1)), (1, 1, 1)), 2)
    shape = R.KernelShape.hypercubic(3, 3)
    expect = R.build_kernel_map(c, oc, shape, (1, 1, 1)).pairs
    saved = RK._ACTIVE
    try:
        RK._ACTIVE = GK  # the VOXPIPE_BACKEND=cuda seam
        got = R.build_kernel_map(c, oc, shape, (1, 1, 1)).pairs
    finally:
        RK._ACTIVE = saved
    for (a, b), (ea, eb) in zip(got, expect):
        np.testing.assert_array_equal(a, ea)
        np.testing.assert_array_equal(b, eb)
