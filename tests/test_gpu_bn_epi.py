"""BN statistics fused into the producing conv (vp_conv_fwd_bn /
vp_conv_dgrad_bn, csrc/bn_epi.cuh) against the plain conv + a torch
reduction of the same rows.  No reference code exists for this glue
(SPEC.md:184-185 non-goal), so parity is self-defined:

  * the stored output is BITWISE what the unfused path produces: mode 1 the
    plain conv output, mode 2 bf16(bf16(y) + add) masked by act > 0;
  * the partial rows (nb from the device header) sum to the per-channel
    statistics within fp32 accumulation error: |d| <= 1e-5 * sum|terms|.

Cases cover the tcgen05 epilogue (no split-K), the split-K reduction
(few tiles), the generic pass (fp32 SIMT path) and both conv directions."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def _table(n_out, n_in, K, gen, density=0.3):
    t = torch.randint(0, n_in, (n_out, K), generator=gen, dtype=torch.int64)
    miss = torch.rand((n_out, K), generator=gen) > density
    t[miss] = -1
    return t.to(torch.int32).cuda()


def _reduce_part(part, C):
    nb = int(part[:4].view(torch.int32).item())
    rows = part[256:256 + nb * 2 * C * 4].view(torch.float32).view(nb, 2, C).double()
    return nb, rows.sum(0).cpu().numpy()


def _run(kind, mode, cin, cout, n, dt, seed=0):
    from paper_2012_13846_b200 import _lib
    gen = torch.Generator().manual_seed(seed)
    K = 27
    kin, kout = (cin, cout) if kind == "fwd" else (cout, cin)  # gathered width, produced width
    n_in = n + 17
    x = torch.randn((n_in, kin), generator=gen).cuda().to(dt)
    w = (torch.randn((K, cout, cin), generator=gen) / np.sqrt(K * kin)).cuda().to(dt)
    table = _table(n, n_in, K, gen)
    n_dev = torch.tensor([n], dtype=torch.int32).cuda()
    code = _lib.dtype_code(x)
    wsq = "vp_conv_fwd_ws_bytes" if kind == "fwd" else "vp_conv_dgrad_ws_bytes"
    ws = _lib.workspace(_lib.query(wsq, cin, cout, K), x.device)
    st = _lib.stream()

    def conv(fn, y, *extra):
        if kind == "fwd":
            args = (x.data_ptr(), code, n_in, cin, w.data_ptr(), code, cout, K, table.data_ptr(), 0, None,
                    n_dev.data_ptr(), n, y.data_ptr(), code, ws.data_ptr(), ws.numel())
        else:
            args = (x.data_ptr(), code, n_in, cout, w.data_ptr(), code, cin, K, table.data_ptr(), 0, None,
                    n_dev.data_ptr(), n, y.data_ptr(), code, ws.data_ptr(), ws.numel())
        _lib.call(fn, *args, *extra, st)

    y0 = torch.zeros((n, kout), dtype=dt, device="cuda")
    conv("vp_conv_fwd" if kind == "fwd" else "vp_conv_dgrad", y0)
    y1 = torch.full((n, kout), 7.0, dtype=dt, device="cuda")
    part = _lib.workspace(_lib.query("vp_bn_part_bytes", kout), x.device, zero=True)
    add = torch.randn((n, kout), generator=gen).cuda().to(dt)
    act = torch.relu(torch.randn((n, kout), generator=gen)).cuda().to(dt)
    pre = torch.randn((n, kout), generator=gen).cuda().to(dt)
    mean = torch.randn(kout, generator=gen).cuda()
    fn = "vp_conv_fwd_bn" if kind == "fwd" else "vp_conv_dgrad_bn"
    # finalize in the producer chain too (mode 1: mean / rstd; mode 2: ggamma / gbeta)
    oa = torch.full((kout,), 3.0, device="cuda")
    ob = torch.full((kout,), 3.0, device="cuda")
    rstd_in = torch.rand(kout, generator=gen).cuda() + 0.5
    eps = 1e-5
    if mode == 1:
        conv(fn, y1, 1, part.data_ptr(), None, None, None, None, eps, oa.data_ptr(), ob.data_ptr(), None)
    else:
        conv(fn, y1, 2, part.data_ptr(), add.data_ptr(), act.data_ptr(), pre.data_ptr(), mean.data_ptr(), 0.0,
             oa.data_ptr(), ob.data_ptr(), rstd_in.data_ptr())
    torch.cuda.synchronize()
    if mode == 1:
        exp = y0
        t1, t2 = y0.double(), y0.double() ** 2
    else:
        g = (y0.float() + add.float()).to(dt)
        exp = torch.where(act.float() > 0, g, torch.zeros_like(g))
        t1 = exp.double()
        t2 = exp.double() * (pre.double() - mean.double())
    assert torch.equal(y1, exp), (y1.float() - exp.float()).abs().max()
    nb, got = _reduce_part(part, kout)
    assert 1 <= nb <= 3 * 148
    ref = torch.stack([t1.sum(0), t2.sum(0)]).cpu().numpy()
    scale = torch.stack([t1.abs().sum(0), t2.abs().sum(0)]).cpu().numpy()
    err = np.abs(got - ref)
    assert (err <= 1e-5 * scale + 1e-6).all(), float((err / (scale + 1e-6)).max())
    # the finalized statistics (fixed-order double sums of the partials)
    if mode == 1:
        mu = ref[0] / n
        var = np.maximum(ref[1] / n - mu * mu, 0.0)
        ea, eb = mu, 1.0 / np.sqrt(var + eps)
        sa = scale[0] / n
    else:
        ea, eb = ref[1] * rstd_in.double().cpu().numpy(), ref[0]
        sa = scale[1] * rstd_in.double().cpu().numpy()
    np.testing.assert_allclose(oa.double().cpu().numpy(), ea, rtol=1e-4, atol=1e-5 * sa.max() + 1e-6)
    np.testing.assert_allclose(ob.double().cpu().numpy(), eb, rtol=1e-4, atol=1e-5 * scale[0].max() / max(n, 1) + 1e-6)


@pytest.mark.parametrize("kind", ["fwd", "dgrad"])
@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("cin,cout,n", [(32, 32, 50000), (64, 64, 3000), (128, 256, 1500), (256, 128, 40000),
                                        (32, 64, 300), (64, 32, 129)])
def test_bn_epilogue_tc(kind, mode, cin, cout, n):
    _run(kind, mode, cin, cout, n, torch.bfloat16)


@pytest.mark.parametrize("kind", ["fwd", "dgrad"])
@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("cin,cout,n", [(32, 32, 2000), (24, 40, 700)])
def test_bn_epilogue_generic_pass(kind, mode, cin, cout, n):
    """fp32 features (SIMT conv) and non-tensor-core widths: one pass after the conv."""
    _run(kind, mode, cin, cout, n, torch.float32 if cin == 32 else torch.bfloat16)


@pytest.mark.parametrize("blocks", [1, 2])
def test_trainer_fused_bn_matches_unfused(blocks):
    """The training step with fused BN statistics against the separate
    statistics passes (VP_BN_EPI=0): fp32 engine to 1e-6 (only summation
    order differs), bf16 loss to 1e-3."""
    import voxpipe_oracle as O
    from paper_2012_13846_b200 import model
    B, P, res = 4, 1500, 48
    pts, offs = O.synthetic_batch(B, P, res, seed=5, dtype=np.float32)
    labels = (np.arange(B) * 7) % 40
    for dt, tol in ((torch.float32, 1e-6), (torch.bfloat16, 1e-3)):
        out = []
        for fuse in (True, False):
            tr = model.SparseResNetTrainer(batch=B, points=P, resolution=res, blocks=blocks, seed=2, feature_dtype=dt)
            tr.bn_fuse = fuse
            loss = tr.train_step_from_host(pts, offs, labels)
            out.append((loss, tr.grads_numpy()))
        (la, ga), (lb, gb) = out
        assert abs(la - lb) <= tol * abs(lb), (dt, la, lb)
        if dt == torch.float32:
            for k in gb:
                d = np.linalg.norm(ga[k] - gb[k]) / (np.linalg.norm(gb[k]) + 1e-12)
                assert d <= 1e-4, (k, d)


@pytest.mark.parametrize("n", [5000, 120000])
def test_bn_epilogue_stem(n):
    """C_in = 1 occupancy stem (conv_stem_kernel): statistics from its tile loop."""
    _run("fwd", 1, 1, 32, n, torch.bfloat16)
