"""The PyTorch drop-in (paper_2012_13846_b200.nn): autograd Functions over
vp_conv_fwd / vp_conv_dgrad / vp_conv_wgrad and the SparseConv3d /
SparseConvTranspose3d / SparseBatchNorm modules.

  * SPEC acceptance 4: the analytic backward matches central
    finite differences within 1e-4 relative on 20 random weight/input
    entries across 10 random instances — in f64, the reference's precision.
  * f64 mode vs the reference itself (oracle/_ref voxpipe.conv, conv.py:186-242)
    and the transposed conv vs the oracle's adjoint: 1e-10 relative.
  * bf16 modules are the same kernels as the functional API: bitwise equal.
  * A SparseResNet assembled from the modules (fp32) trains one step to the
    f64 oracle's loss (rel 1e-5) and gradients (rel-L2 1e-3) — the same
    tolerance as the fp32 engine (tests/test_gpu_model.py).
"""
import numpy as np
import pytest

import voxpipe_oracle as O
from parity_util import reference

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def _tensor(seed, clouds=2, npts=300, res=12, width=3, dtype=torch.float64):
    from paper_2012_13846_b200.tensor import SparseTensor
    pts, offs = O.synthetic_batch(clouds, npts, res, seed=seed, dtype=np.float64)
    coords, _ = O.voxelize_batch(pts, offs, 1.0, res)
    rng = np.random.default_rng(seed)
    x = torch.from_numpy(rng.normal(size=(len(coords), width))).to(dtype).cuda()
    return SparseTensor(coords, x, (1, 1, 1)), coords


@pytest.mark.parametrize("kind", ["s1", "s2", "transposed"])
def test_finite_difference_gradcheck_f64(kind):
    """SPEC acceptance 4: 10 instances x 20 random entries, central
    differences, 1e-4 relative."""
    from paper_2012_13846_b200 import nn
    from paper_2012_13846_b200.conv import KernelShape
    shape = KernelShape.hypercubic(3, 3)
    worst = 0.0
    for inst in range(10):
        t, coords = _tensor(100 + inst, width=3)
        rng = np.random.default_rng(inst)
        cout = 4
        if kind == "transposed":
            coarse = nn.sparse_conv(t, torch.zeros((27, 3, 3), dtype=torch.float64, device="cuda"), shape, 2)
            x = torch.from_numpy(rng.normal(size=(len(coarse), 3))).cuda().requires_grad_(True)
            w = torch.from_numpy(rng.normal(size=(27, cout, 3)) / 9).cuda().requires_grad_(True)

            def f(x_, w_):
                return nn.sparse_conv_transpose(coarse.with_features(x_), w_, shape, 2, t).features
        else:
            stride = 1 if kind == "s1" else 2
            x = t.features.clone().requires_grad_(True)
            w = torch.from_numpy(rng.normal(size=(27, cout, 3)) / 9).cuda().requires_grad_(True)

            def f(x_, w_):
                return nn.sparse_conv(t.with_features(x_), w_, shape, stride).features
        y = f(x, w)
        r = torch.from_numpy(rng.normal(size=tuple(y.shape))).cuda()
        (y * r).sum().backward()
        h = 1e-6
        for _ in range(20):
            which = rng.integers(2)
            p = (x, w)[which]
            flat = p.data.view(-1)
            i = int(rng.integers(flat.numel()))
            old = float(flat[i])
            flat[i] = old + h
            lp = float((f(x.detach(), w.detach()) * r).sum())
            flat[i] = old - h
            lm = float((f(x.detach(), w.detach()) * r).sum())
            flat[i] = old
            fd = (lp - lm) / (2 * h)
            an = float(p.grad.view(-1)[i])
            err = abs(fd - an) / max(abs(fd), abs(an), 1e-8)
            worst = max(worst, err)
            assert err <= 1e-4 or abs(fd - an) < 1e-9, (kind, inst, which, i, fd, an)
    print(f"{kind}: worst FD relative error {worst:.2e}")


@pytest.mark.parametrize("stride", [1, 2])
def test_f64_mode_matches_reference(stride):
    """f64 features run the f64 SIMT kernels: forward, grad_in and grad_w
    equal the reference's own f64 conv (conv.py:186-242) to 1e-10."""
    from paper_2012_13846_b200 import nn
    from paper_2012_13846_b200.conv import KernelShape
    mods = reference()
    if mods is None:
        pytest.skip("oracle/_ref not built")
    R, _ = mods
    t, coords = _tensor(7, clouds=3, npts=800, res=20, width=16)
    rng = np.random.default_rng(3)
    w = torch.from_numpy(rng.normal(size=(27, 24, 16)) / np.sqrt(27 * 16)).cuda().requires_grad_(True)
    x = t.features.clone().requires_grad_(True)
    y = nn.sparse_conv(t.with_features(x), w, KernelShape.hypercubic(3, 3), stride)
    g = rng.normal(size=tuple(y.features.shape))
    y.features.backward(torch.from_numpy(g).cuda())
    rs = R.SparseTensor(coords, x.detach().cpu().numpy(), (1, 1, 1))
    rw = R.ConvWeights(w.detach().cpu().numpy())
    shape = R.KernelShape.hypercubic(3, 3)
    ry = R.sparse_conv_forward(rs, rw, shape, stride)
    np.testing.assert_array_equal(y.coords.cpu().numpy(), ry.coords)
    rgi, rgw = R.sparse_conv_backward(rs, rw, shape, stride, g)
    for got, exp in ((y.features.detach(), ry.features), (x.grad, rgi), (w.grad, rgw)):
        got = got.cpu().numpy()
        assert np.abs(got - exp).max() <= 1e-10 * (np.abs(exp).max() + 1e-30)


def test_transposed_module_is_the_adjoint_f64():
    """SparseConvTranspose3d(coarse -> fine) == the oracle's adjoint of the
    strided conv, f64."""
    from paper_2012_13846_b200 import nn
    t, coords = _tensor(11, clouds=2, npts=600, res=16, width=8)
    down = nn.SparseConv3d(8, 8, 3, stride=2, dtype=torch.float64, device="cuda")
    coarse = down(t)
    up = nn.SparseConvTranspose3d(8, 5, 3, stride=2, dtype=torch.float64, device="cuda")
    xc = coarse.features.detach()
    y = up(coarse.with_features(xc), t)
    ref = O.sparse_conv_transposed(coords, (1, 1, 1), xc.cpu().numpy(), up.weight.detach().cpu().numpy(),
                                   O.hypercubic_offsets(3, 3), 2)
    assert np.abs(y.features.detach().cpu().numpy() - ref).max() <= 1e-10 * np.abs(ref).max()


def test_bf16_module_equals_functional_api():
    """The module path runs the same tcgen05 kernels as conv.sparse_conv_forward /
    sparse_conv_backward: bitwise equal outputs and gradients."""
    from paper_2012_13846_b200 import conv, nn
    t, coords = _tensor(5, clouds=4, npts=1500, res=40, width=32, dtype=torch.bfloat16)
    layer = nn.SparseConv3d(32, 64, 3, stride=2, device="cuda")
    x = t.features.clone().requires_grad_(True)
    y = layer(t.with_features(x))
    g = torch.randn(y.features.shape, device="cuda").to(torch.bfloat16)
    y.features.backward(g)
    W = conv.ConvWeights(layer.weight.detach())
    shape = conv.KernelShape.hypercubic(3, 3)
    ry = conv.sparse_conv_forward(t, W, shape, 2)
    rgi, rgw = conv.sparse_conv_backward(t, W, shape, 2, g)
    assert torch.equal(y.coords, ry.coords)
    assert torch.equal(y.features.detach(), ry.features)
    assert torch.equal(x.grad, rgi)
    assert torch.equal(layer.weight.grad, rgw)


class ModuleResNet(torch.nn.Module):
    """SURVEY §8(d) SparseResNet built from the drop-in modules."""

    def __init__(self, planes=(32, 64, 128, 256), classes=40, cin=1):
        from paper_2012_13846_b200 import nn
        super().__init__()
        self.convs = torch.nn.ModuleDict()
        self.bns = torch.nn.ModuleDict()
        convs, _ = O.resnet_layout(cin, planes, 1, classes)
        for name, ci, co, s in convs:
            key = name.replace(".", "_")
            self.convs[key] = nn.SparseConv3d(ci, co, 3, stride=s, device="cuda")
            self.bns[key] = nn.SparseBatchNorm(co, relu=True, device="cuda")
        self.fc = torch.nn.Linear(planes[-1], classes, device="cuda")
        self.names = [n for n, _, _, _ in convs]

    def load(self, p):
        for name in self.names:
            key = name.replace(".", "_")
            self.convs[key].weight.data.copy_(torch.from_numpy(p[name + ".w"]))
            self.bns[key].weight.data.copy_(torch.from_numpy(p[name + ".gamma"]))
            self.bns[key].bias.data.copy_(torch.from_numpy(p[name + ".beta"]))
        self.fc.weight.data.copy_(torch.from_numpy(p["fc.w"]))
        self.fc.bias.data.copy_(torch.from_numpy(p["fc.b"]))

    def forward(self, t, B):
        from paper_2012_13846_b200 import nn

        def cbr(name, x, res=None):
            key = name.replace(".", "_")
            return self.bns[key](self.convs[key](x), res)

        x = cbr("stem", t)
        for s in range(4):
            x = cbr(f"s{s}.down", x)
            h = cbr(f"s{s}.b0.c1", x)
            x = cbr(f"s{s}.b0.c2", h, x)
        return self.fc(nn.global_avg_pool(x, B))


def test_module_resnet_trains_like_the_oracle_fp32():
    from paper_2012_13846_b200 import tensor
    B, P, res = 4, 1500, 48
    pts, offs = O.synthetic_batch(B, P, res, seed=3, dtype=np.float32)
    labels = (np.arange(B) * 7) % 40
    p0 = O.init_params(1, seed=2)
    net = ModuleResNet()
    net.load(p0)
    t = tensor.voxelize_batch(torch.from_numpy(pts).cuda(), torch.from_numpy(offs), 1.0, (res,) * 3)
    logits = net(t, B)
    loss = torch.nn.functional.cross_entropy(logits, torch.from_numpy(labels).cuda())
    loss.backward()
    c, f = O.voxelize_batch(pts.astype(np.float64), offs, 1.0, res)
    pr = {k: v.astype(np.float32).astype(np.float64) for k, v in p0.items()}
    rloss, rg, _, _ = O.resnet_train_step(pr, c, f, labels, B)
    lv = float(loss.detach())
    assert abs(lv - rloss) <= 1e-5 * abs(rloss), (lv, rloss)
    got = {}
    for name in net.names:
        key = name.replace(".", "_")
        got[name + ".w"] = net.convs[key].weight.grad
        got[name + ".gamma"] = net.bns[key].weight.grad
        got[name + ".beta"] = net.bns[key].bias.grad
    got["fc.w"], got["fc.b"] = net.fc.weight.grad, net.fc.bias.grad
    bad = {}
    for k, r in rg.items():
        e = np.linalg.norm(got[k].double().cpu().numpy() - r) / (np.linalg.norm(r) + 1e-12)
        if e > 1e-3:
            bad[k] = e
    assert not bad, bad


def test_plans_are_cached_per_coordinate_set():
    """A stride-1 output shares its input's rows and plan cache: a
    BasicBlock's two convs build one kernel map."""
    from paper_2012_13846_b200 import nn
    t, _ = _tensor(2, clouds=2, npts=500, res=16, width=8, dtype=torch.float32)
    a = nn.SparseConv3d(8, 8, device="cuda")
    b = nn.SparseConv3d(8, 8, device="cuda")
    h = a(t)
    assert h.coords4 is t.coords4 and h.plans is t.plans
    n = len(t.plans)
    b(h)
    assert len(t.plans) == n


def test_tf32_module_equals_functional_api():
    """SparseConv3d(allow_tf32=True) on fp32 features runs the kind::tf32
    tensor-core kernels: bitwise equal to sparse_conv_forward/backward with
    math="tf32", and within 2e-3 (relative to max) of the exact fp32 module."""
    from paper_2012_13846_b200 import conv, nn
    t, coords = _tensor(6, clouds=3, npts=1200, res=32, width=32, dtype=torch.float32)
    layer = nn.SparseConv3d(32, 64, 3, stride=1, device="cuda", allow_tf32=True)
    x = t.features.clone().requires_grad_(True)
    y = layer(t.with_features(x))
    g = torch.randn(y.features.shape, device="cuda")
    y.features.backward(g)
    W = conv.ConvWeights(layer.weight.detach())
    shape = conv.KernelShape.hypercubic(3, 3)
    ry = conv.sparse_conv_forward(t, W, shape, 1, math="tf32")
    rgi, rgw = conv.sparse_conv_backward(t, W, shape, 1, g, math="tf32")
    assert torch.equal(y.features.detach(), ry.features)
    assert torch.equal(x.grad, rgi)
    assert torch.equal(layer.weight.grad, rgw)
    ye = conv.sparse_conv_forward(t, W, shape, 1)
    d = (ye.features - ry.features).abs().max() / ye.features.abs().max()
    assert 0 < float(d) < 2e-3
