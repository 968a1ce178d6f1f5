"""GPU: the grouping's tile schedule (vp_kernel_map_group_sched,
csrc/kmap_sort.cu).  Whole 128-row tiles of the stable grouping are placed so
the conv's round-robin tile -> CTA assignment approximates LPT; the order is
checked exactly against the numpy restatement (parity_util.tile_schedule),
and the conv over the scheduled table must equal the conv over the
descending grouping without moves bit for bit (every row keeps its tile
mates)."""
import numpy as np
import pytest

import voxpipe_oracle as O
from parity_util import stable_grouping, tile_schedule

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def _map(clouds, seed, stride=1):
    from paper_2012_13846_b200 import conv
    from paper_2012_13846_b200.tensor import SparseTensor
    pts, offs = O.synthetic_batch(clouds, 2048, 64, seed=seed, dtype=np.float32)
    c0, _ = O.voxelize_batch(pts.astype(np.float64), offs, 1.0, 64)
    t = SparseTensor(c0, np.zeros((len(c0), 1)), (1, 1, 1))
    shape = conv.KernelShape.hypercubic(3, 3)
    out4, _ = conv._output_coords4(t.coords4, (1, 1, 1), (stride,) * 3, 3)
    km = conv._kernel_map4(t.coords4, out4, shape, (1, 1, 1), 3)
    return km, len(t), out4.shape[0]


def _makespan(p, table, n, G, ovh=3):
    hit = np.asarray(table)[p] >= 0
    ntiles = (n + 127) // 128
    cost = np.array([hit[t * 128:(t + 1) * 128].any(0).sum() for t in range(ntiles)])
    load = np.zeros(G)
    for t in range(ntiles):
        load[t % G] += cost[t] + ovh
    return load.max()


@pytest.mark.parametrize("clouds,seed,G", [(24, 11, 296), (40, 12, 296), (30, 13, 148), (6, 14, 296)])
def test_tile_schedule_exact_and_bitwise(clouds, seed, G):
    from paper_2012_13846_b200 import conv
    km, n_in, n = _map(clouds, seed)
    tab = km.nbr[:n].cpu().numpy()
    pa_t, _ = conv.sort_table(km.nbr, n, 0)
    assert np.array_equal(pa_t.cpu().numpy(), stable_grouping(tab, n, 0))
    # sched_grid = 1: the descending-key grouping without tile moves
    p0_t, ts0 = conv.sort_table(km.nbr, n, 0, sched_grid=1)
    p1_t, ts1 = conv.sort_table(km.nbr, n, 0, sched_grid=G)
    p0 = p0_t.cpu().numpy().astype(np.int64)
    p1 = p1_t.cpu().numpy().astype(np.int64)
    assert np.array_equal(p0, stable_grouping(tab, n, 0, desc=True))
    exp = tile_schedule(p0, tab, n, G)
    assert np.array_equal(p1, exp), "tile schedule differs from the restatement"
    assert torch.equal(ts1[:n], km.nbr[p1_t[:n].long()])
    ntiles = (n + 127) // 128
    if G < ntiles <= 4 * G:
        assert not np.array_equal(p1, p0)
        assert _makespan(p1, tab, n, G) <= _makespan(p0, tab, n, G)
    else:
        assert np.array_equal(p1, p0)
    # conv forward / dgrad over the scheduled table == over the plain grouping, bitwise
    g = torch.Generator(device="cuda").manual_seed(seed)
    c = 32
    x = torch.randn(n_in, c, device="cuda", generator=g).to(torch.bfloat16)
    W = conv.ConvWeights(torch.randn(27, c, c, device="cuda", generator=g) / (27 * c) ** 0.5)
    y0 = conv.conv_forward_raw(x, W, ts0, n, perm=p0_t)
    y1 = conv.conv_forward_raw(x, W, ts1, n, perm=p1_t)
    assert torch.equal(y0, y1)
    gy = torch.randn(n, c, device="cuda", generator=g).to(torch.bfloat16)
    d0 = conv.conv_dgrad_raw(gy, W, ts0, n, True, perm=p0_t)
    d1 = conv.conv_dgrad_raw(gy, W, ts1, n, True, perm=p1_t)
    assert torch.equal(d0, d1)


def test_conv_tc_grid():
    from paper_2012_13846_b200 import _lib
    assert _lib.query("vp_conv_tc_grid", 32, 131072) == 296
    assert _lib.query("vp_conv_tc_grid", 64, 131072) == 296
    assert _lib.query("vp_conv_tc_grid", 32, 256) == 32  # 2 tiles x 16 splits
    assert _lib.query("vp_conv_tc_grid", 7, 131072) == 0
