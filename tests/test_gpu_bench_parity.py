"""Parity AT THE BENCHMARKED CONFIGURATIONS (the trainer built exactly as
bench.py builds it: dense-grid / brick index, prefetch mode, the two captured
CUDA graphs replayed over the bench's pool of synthetic batches).

  C3 = 64 clouds x 2048 pts @ 64^3, blocks=1 (BASELINE configs[2], the bench line)
  C5 = 256 clouds x 16384 pts @ 128^3, blocks=2 (the one-GPU C5 network; levels 1-3
       stride-1 maps are neighbour-mask sorted)

Integer stage: every level's coordinates and all nine kernel maps (CSR pairs,
pair_ptr, the dense nbr table, the strided inverse tables, the mask-sorted
tables and their permutations) of BOTH prefetch states are compared with
np.array_equal against the reference itself (oracle/_ref voxpipe:
tensor.voxelize/batch, conv.generate_output_coords/build_kernel_map,
conv.py:124-183) run on the points each state was built from.

Float stage (C3), tolerances written here:
  * loss after the first step: relative 1e-3 vs the f64 oracle on the same
    bf16-rounded weights with every engine-stored tensor rounded to bf16;
  * every gradient: rel-L2 <= 2 x the oracle's own accumulation-order
    sensitivity (f64 vs fp32 conv accumulation, same rounding points) + 0.02;
  * teacher-forced per layer (engine inputs -> oracle): conv forward output
    |d| <= 2^-8 |y| + 1e-4 * sum|W||x| (bf16 store of an fp32 accumulation);
    BN forward output |d| <= 2^-8 |a| + 1e-3; weight gradient (fp32)
    |d| <= 1e-5 * sum|g||x| + 1e-7.
"""
import numpy as np
import pytest

import voxpipe_oracle as O
from parity_util import bf16_round, check_trainer_state, noise_calibrated_grad_check

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def bench_trainer(B, P, res, blocks, steps, seed_base=0):
    """bench.py's construction and timed loop: prefetch + capture(warmup=1),
    then `steps` replays over a pool of 4 synthetic batches set before each
    step (bench.py:251-286)."""
    from paper_2012_13846_b200 import model
    tr = model.SparseResNetTrainer(batch=B, points=P, resolution=res, blocks=blocks)
    pool = []
    for i in range(4):
        pts, _ = O.synthetic_batch(B, P, res, seed=seed_base + i, dtype=np.float32)
        pool.append((torch.from_numpy(pts).cuda(), torch.from_numpy(((np.arange(B) + 7 * i) % 40).astype(np.int32)).cuda()))
    tr.enable_prefetch()
    tr.set_batch(*pool[0])
    tr.capture(warmup=1)
    p_last = None
    for i in range(steps):
        tr.set_batch(*pool[i % 4])
        if i == steps - 1:
            p_last = tr.state_numpy()  # weights the last replayed step's forward read
        tr.step()
    torch.cuda.synchronize()
    return tr, pool, p_last


def _assert_state_from_pool(state, pool):
    pts = state["points"]
    assert any(torch.equal(pts, p) for p, _ in pool), "state points are not one of the pool batches"


def test_c3_bench_trainer_integer_stage_bit_exact():
    tr, pool, _ = bench_trainer(64, 2048, 64, 1, steps=5)
    assert tr.index_kind == "grid" and tr.prefetch and tr.graphs[0] is not None
    for s in (0, 1):
        _assert_state_from_pool(tr.states[s], pool)
        summ = check_trainer_state(tr.states[s], 64)
        assert summ["kind"] == "reference", "oracle/_ref missing: the C3 check must run against the reference"
        assert summ["rows"][0] > 100000 and len(summ["pairs"]) == 9
        print(f"C3 state {s}: {summ}")
    for g, r in zip(tr.grids, tr.grid_R):  # the lattice occupancy bitmap is empty again between steps
        assert bool((g[64 * r ** 3:] == 0).all())


@pytest.mark.slow
def test_c5_bench_trainer_integer_stage_bit_exact():
    """C5 network on one GPU (bench.py --batch 256 --points 16384 --res 128
    --blocks 2): 3.3M-row level 0, mask-sorted forward
    tables at levels 1-3 (>= 2^18 rows) and sorted strided inverse tables."""
    tr, pool, p_last = bench_trainer(256, 16384, 128, 2, steps=2)
    assert tr.index_kind in ("grid", "brick")
    sorted_maps = [m for m in tr.states[0]["map_s1"] if m.perm is not None]
    assert len(sorted_maps) >= 2, "C5 must exercise the mask-sorted forward tables"
    summ = check_trainer_state(tr.states[tr._phase], 128)
    assert summ["kind"] == "reference"
    assert summ["rows"][0] > 3_000_000
    print(f"C5 state {tr._phase}: {summ}")
    _assert_state_from_pool(tr.states[tr._phase], pool)
    # the float stage through the sorted tables: teacher-forced forward of
    # the first layer on every mask-sorted map, in the state the last replay
    # trained on, against the oracle
    n = _teacher_forced_forward(tr, tr.states[1 - tr._phase], only_sorted=True, p_before=p_last)
    assert n >= 2


def _first_step(B, P, res, blocks):
    """Bench-built trainer (graphs + prefetch), weights restored to their
    initial values after capture's warm-up, then ONE replayed step."""
    from paper_2012_13846_b200 import model
    tr = model.SparseResNetTrainer(batch=B, points=P, resolution=res, blocks=blocks)
    p_init = tr.params.p.clone()
    pts, offs = O.synthetic_batch(B, P, res, seed=0, dtype=np.float32)
    labels = (np.arange(B) * 7) % 40
    dp, dl = torch.from_numpy(pts).cuda(), torch.from_numpy(labels.astype(np.int32)).cuda()
    tr.enable_prefetch()
    tr.set_batch(dp, dl)
    tr.capture(warmup=1)
    tr.params.p.copy_(p_init)
    tr.params.m.zero_()
    tr.params.pb[: tr.params.n_bf16].copy_(tr.params.p[: tr.params.n_bf16].to(torch.bfloat16))
    tr.prime(dp, dl)
    tr.set_batch(dp, dl)
    p0 = tr.state_numpy()
    cur = tr._phase
    tr.step()
    torch.cuda.synchronize()
    return tr, cur, p0, pts, offs, labels


def _teacher_forced_forward(tr, state, p_before, only_sorted=False):
    """Per layer, the oracle's conv on the ENGINE's own stored inputs (bf16 x,
    the bf16 weights the kernels read) vs the engine's conv output.
    only_sorted: just the first layer on each neighbour-mask sorted map."""
    checked = 0
    seen = set()
    for L in state["layers"]:
        m = L["map"]
        if only_sorted and (m.perm is None or id(m) in seen):
            continue
        seen.add(id(m))
        nd = int(L["dst"].n.item())
        ns = int(L["src"].n.item())
        x = L["x"][:ns].float().cpu().numpy().astype(np.float64)
        w = bf16_round(p_before[L["name"] + ".w"])
        ptr = m.ptr.cpu().numpy().astype(np.int64)
        pin, pout = m.pin.cpu().numpy().astype(np.int64), m.pout.cpu().numpy().astype(np.int64)
        ref = np.zeros((nd, w.shape[1]))
        bnd = np.zeros((nd, w.shape[1]))
        ax, aw = np.abs(x), np.abs(w)
        for k in range(27):
            vi, ui = pin[ptr[k]:ptr[k + 1]], pout[ptr[k]:ptr[k + 1]]
            if len(vi):
                ref[ui] += x[vi] @ w[k].T  # out rows are unique per offset
                bnd[ui] += ax[vi] @ aw[k].T
        y = L["y"][:nd].float().cpu().numpy()
        err = np.abs(y - ref)
        tol = 2.0 ** -8 * np.abs(ref) + 1e-4 * bnd + 1e-6
        assert (err <= tol).all(), f"{L['name']}: conv fwd max err {err.max()} (worst ratio {(err / tol).max():.2f})"
        checked += 1
    assert checked > 0
    return checked


def test_c3_first_step_loss_grads_and_teacher_forced_layers():
    tr, cur, p0, pts, offs, labels = _first_step(64, 2048, 64, 1)
    loss = float(tr.loss.item())
    grads = tr.grads_numpy()
    state = tr.states[cur]
    # ---- teacher-forced forward: conv outputs of every layer
    n = _teacher_forced_forward(tr, state, p0)
    assert n == 13  # the SIMT stem (C_in = 1) and the 12 tensor-core convs
    # BN forward (+ residual + ReLU) per layer
    block_in = None
    for L in state["layers"]:
        nd = int(L["dst"].n.item())
        y = L["y"][:nd].float().cpu().numpy().astype(np.float64)
        mu, var = y.mean(0), y.var(0)
        np.testing.assert_allclose(L["mean"].cpu().numpy(), mu, rtol=1e-4, atol=1e-5 * (np.abs(y).max() + 1))
        rstd = 1.0 / np.sqrt(var + 1e-5)
        np.testing.assert_allclose(L["rstd"].cpu().numpy(), rstd, rtol=1e-3)
        z = (y - mu) * rstd * p0[L["name"] + ".gamma"] + p0[L["name"] + ".beta"]
        if L["kind"] == "c1":
            block_in = L["x"][:nd].float().cpu().numpy().astype(np.float64)
        if L["kind"] == "c2":
            z = z + block_in
        a_ref = np.maximum(z, 0)
        a = L["a"][:nd].float().cpu().numpy()
        err = np.abs(a - a_ref)
        assert (err <= 2.0 ** -8 * np.abs(a_ref) + 1e-3).all(), f"{L['name']}: BN fwd max err {err.max()}"
    # ---- teacher-forced weight gradients (fp32 outputs) on the engine's gy and x
    for L in state["layers"]:
        m = L["map"]
        nd, ns = int(L["dst"].n.item()), int(L["src"].n.item())
        x = L["x"][:ns].float().cpu().numpy().astype(np.float64)
        gy = L["gy"][:nd].float().cpu().numpy().astype(np.float64)
        ptr = m.ptr.cpu().numpy().astype(np.int64)
        pin, pout = m.pin.cpu().numpy().astype(np.int64), m.pout.cpu().numpy().astype(np.int64)
        gw = grads[L["name"] + ".w"]
        for k in range(27):
            vi, ui = pin[ptr[k]:ptr[k + 1]], pout[ptr[k]:ptr[k + 1]]
            r = gy[ui].T @ x[vi]
            b = np.abs(gy[ui]).T @ np.abs(x[vi])
            e = np.abs(gw[k] - r)
            assert (e <= 1e-5 * b + 1e-7).all(), f"{L['name']} wgrad offset {k}: max err {e.max()}"
    # ---- end to end: loss and gradients vs the bf16-emulating oracle
    c, f = O.voxelize_batch(pts.astype(np.float64), offs, 1.0, 64)
    rloss, table = noise_calibrated_grad_check(grads, p0, c, f, labels, 64, 1)
    assert abs(loss - rloss) <= 1e-3 * abs(rloss), (loss, rloss)
    print(f"C3 loss {loss} vs {rloss}; grad (err, oracle noise): {table}")
