"""Shared parity helpers for the GPU tests (test infrastructure only).

* `reference()` — the unmodified reference (voxpipe 0.1.0) built into
  oracle/_ref by oracle/build_ref.sh, or None.
* `ref_integer_stage()` — level coordinates and the nine kernel maps of the
  SparseResNet computed BY THE REFERENCE (`voxpipe.tensor.voxelize/batch`,
  `voxpipe.conv.generate_output_coords/build_kernel_map`, conv.py:124-183).
* `check_trainer_state()` — bit-exact comparison of a trainer's level
  coordinates and maps (pairs, ptr, nbr, strided inverse tables, the
  neighbour-mask sorted tables + permutations) against those.
* `noise_calibrated_grad_check()` — the bf16 training step's gradient
  tolerance: the engine's error against the bf16-emulating f64 oracle must
  stay within a small multiple of the oracle's OWN sensitivity to
  accumulation order (the same oracle with fp32 conv accumulation), so a
  real defect in one layer (>= a few % of its gradient) fails while
  chaotic bf16 rounding flips do not.
"""
from __future__ import annotations

import os
import sys

import numpy as np

import voxpipe_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def bf16_round(a):
    import torch

    return torch.from_numpy(np.asarray(a, np.float32)).to(torch.bfloat16).float().numpy().astype(np.float64)


def reference():
    """(conv, tensor) modules of the reference built in oracle/_ref, or None."""
    path = os.path.join(ROOT, "oracle", "_ref")
    if not os.path.isdir(os.path.join(path, "voxpipe")):
        return None
    if path not in sys.path:
        sys.path.insert(0, path)
    from voxpipe import conv as R
    from voxpipe import kernels as RK
    from voxpipe import tensor as RT

    assert RK.backend_name() == "compiled"
    return R, RT


def ref_integer_stage(points, offsets, res, nlev=5):
    """Reference level coordinates [L0..L4] (int64 (N,4)) and, per level i,
    the stride-1 map (level i -> i) and the strided map (i -> i+1), each as a
    list of per-offset (in_rows, out_rows) — computed by the reference when
    oracle/_ref is present, else by the pinned oracle restatement.
    Returns (kind, levels, maps_s1, maps_dn)."""
    mods = reference()
    pts = np.asarray(points, np.float64)
    if mods is not None:
        R, RT = mods
        ts = [RT.voxelize(RT.PointCloud(pts[offsets[i]:offsets[i + 1]]), 1.0, (res,) * 3)
              for i in range(len(offsets) - 1)]
        t = RT.batch(ts)
        shape = R.KernelShape.hypercubic(3, 3)
        levels, strides = [t.coords], [(1, 1, 1)]
        for i in range(1, nlev):
            oc, ns = R.generate_output_coords(R.SparseTensor(levels[-1], np.zeros((len(levels[-1]), 1)),
                                                             strides[-1]), 2)
            levels.append(oc)
            strides.append(ns)
        s1 = [R.build_kernel_map(levels[i], levels[i], shape, strides[i]).pairs for i in range(nlev)]
        dn = [R.build_kernel_map(levels[i], levels[i + 1], shape, strides[i]).pairs for i in range(nlev - 1)]
        return "reference", levels, s1, dn
    c, _ = O.voxelize_batch(pts, offsets, 1.0, res)
    off = O.hypercubic_offsets(3, 3)
    levels, strides = [c], [(1, 1, 1)]
    for i in range(1, nlev):
        oc, ns = O.generate_output_coords(levels[-1], strides[-1], 2)
        levels.append(oc)
        strides.append(ns)
    s1 = [O.build_kernel_map(levels[i], levels[i], off, strides[i]) for i in range(nlev)]
    dn = [O.build_kernel_map(levels[i], levels[i + 1], off, strides[i]) for i in range(nlev - 1)]
    return "oracle", levels, s1, dn


def group_key(table, mode):
    """The grouping key of csrc/kmap_sort.cu for 3^3 tables: mode 0 = which
    (dx, dy) columns hold a hit, 1 = which dx / dy / dz planes, 2 = the whole
    27-bit mask."""
    hit = np.asarray(table) >= 0
    n = hit.shape[0]
    if mode == 2:  # the whole hit mask
        return (hit.astype(np.int64) << np.arange(hit.shape[1], dtype=np.int64)).sum(1)
    if mode == 0:
        bits = hit.reshape(n, 9, 3).any(2)
    else:
        h = hit.reshape(n, 3, 3, 3)
        bits = np.concatenate([h.any((2, 3)), h.any((1, 3)), h.any((1, 2))], 1)
    return (bits.astype(np.int64) << np.arange(9, dtype=np.int64)).sum(1)


def check_grouping(p, ts, mode, what):
    """Rows in ascending key order, stable (equal keys keep row order)."""
    key = group_key(ts, mode)
    d = np.diff(key)
    assert (d >= 0).all(), f"{what}: rows not grouped by key"
    assert (np.diff(p)[d == 0] > 0).all(), f"{what}: grouping not stable"


def stable_grouping(table, n, mode, desc=False):
    """The row order of vp_kernel_map_group: stable sort of the live rows by
    their grouping key (descending for vp_kernel_map_group_sched)."""
    key = group_key(np.asarray(table)[:n], mode)
    if desc:
        key = ((1 << 27) - 1 if mode == 2 else 511) - key
    return np.argsort(key, kind="stable").astype(np.int64)


def tile_schedule(p0, table, n, G, ovh=3, rounds=4):
    """numpy restatement of the grouping's tile schedule (kmap_sort.cu
    tile_cost_kernel / tile_assign_kernel): whole 128-row tiles of the stable
    grouping p0 placed by round-based LPT over the conv's round-robin slots.
    Returns the composed row order."""
    tab = np.asarray(table)
    K = tab.shape[1]
    ntiles = (n + 127) // 128
    if not (0 < G <= 1024 and G < ntiles <= rounds * G and K <= 27):
        return p0
    hit = tab[p0] >= 0
    cost = np.array([hit[t * 128:(t + 1) * 128].any(0).sum() for t in range(ntiles)], np.int64)
    nfull = n // 128
    R, rem = divmod(ntiles, G)
    slots = np.array([R + (b < rem) for b in range(G)], np.int64)
    used = np.zeros(G, np.int64)
    load = np.zeros(G, np.int64)
    tile_at = np.full(ntiles, -1, np.int64)
    if nfull < ntiles:
        br = (ntiles - 1) % G
        load[br] = cost[-1] + ovh
        slots[br] -= 1
        tile_at[-1] = ntiles - 1
    order = sorted(range(nfull), key=lambda t: (-cost[t], t))
    nxt = 0
    while nxt < nfull:  # LPT by rounds: one tile per CTA with a free slot
        avail = sorted((b for b in range(G) if used[b] < slots[b]),
                       key=lambda b: (load[b], slots[b] - used[b], b))
        take = min(len(avail), nfull - nxt)
        for i in range(take):
            b, t = avail[i], order[nxt + i]
            tile_at[b + used[b] * G] = t
            used[b] += 1
            load[b] += cost[t] + ovh
        nxt += take
    src = tile_at[np.arange(n) // 128] * 128 + np.arange(n) % 128
    return p0[src]


def check_tile_blocks(p, p0, n, what):
    """p is p0 with whole 128-row tiles moved (the tile schedule), the ragged
    last tile in place."""
    ntiles = (n + 127) // 128
    if np.array_equal(p, p0):
        return
    blocks0 = {tuple(p0[t * 128:(t + 1) * 128]): t for t in range(n // 128)}
    seen = set()
    for t in range(n // 128):
        key = tuple(p[t * 128:(t + 1) * 128])
        assert key in blocks0, f"{what}: position tile {t} is not a tile of the grouping"
        seen.add(blocks0[key])
    assert len(seen) == n // 128, f"{what}: tiles repeated"
    if n % 128:
        assert np.array_equal(p[(ntiles - 1) * 128:], p0[(ntiles - 1) * 128:n]), f"{what}: ragged tile moved"


def _check_perm_table(perm, table_s, table, n, what, mode=1):
    """A grouped table (vp_kernel_map_group[_sched]): perm is a permutation
    of 0..n-1, table_s[i] == table[perm[i]] row for row, rows in ascending
    stable key order up to whole-tile moves of the tile schedule."""
    p = perm[:n].cpu().numpy().astype(np.int64)
    assert np.array_equal(np.sort(p), np.arange(n)), f"{what}: perm is not a permutation"
    ts = table_s[:n].cpu().numpy()
    np.testing.assert_array_equal(ts, table[p], err_msg=f"{what}: sorted table != table[perm]")
    asc = stable_grouping(table, n, mode)
    if np.array_equal(p, asc):
        return
    check_tile_blocks(p, stable_grouping(table, n, mode, desc=True), n, what)


def check_map(m, pairs, what):
    """Engine Map vs reference per-offset (in, out) pair lists: CSR pairs,
    ptr, the dense neighbour table, the strided inverse table and the sorted
    tables — all bit-exact."""
    nd, ns = int(m.dst.n.item()), int(m.src.n.item())
    ptr = m.ptr.cpu().numpy().astype(np.int64)
    pin, pout = m.pin.cpu().numpy(), m.pout.cpu().numpy()
    nbr = m.nbr[:nd].cpu().numpy()
    K = len(pairs)
    exp_ptr = np.concatenate([[0], np.cumsum([len(a) for a, _ in pairs])])
    np.testing.assert_array_equal(ptr, exp_ptr, err_msg=f"{what}: pair_ptr")
    exp_nbr = np.full((nd, K), -1, np.int64)
    exp_inv = np.full((ns, K), -1, np.int64) if m.inv is not None else None
    for k, (ei, eo) in enumerate(pairs):
        np.testing.assert_array_equal(pin[ptr[k]:ptr[k + 1]], ei, err_msg=f"{what}: pair_in offset {k}")
        np.testing.assert_array_equal(pout[ptr[k]:ptr[k + 1]], eo, err_msg=f"{what}: pair_out offset {k}")
        exp_nbr[eo, k] = ei
        if exp_inv is not None:
            exp_inv[ei, k] = eo
    np.testing.assert_array_equal(nbr, exp_nbr, err_msg=f"{what}: nbr")
    if exp_inv is not None:
        np.testing.assert_array_equal(m.inv[:ns].cpu().numpy(), exp_inv, err_msg=f"{what}: inverse table")
    if m.perm is not None:
        from paper_2012_13846_b200 import model as _model
        fmode = 2 if m.dst.cap >= _model.SparseResNetTrainer.FULL_MASK_ROWS else 0
        _check_perm_table(m.perm, m.nbr_s, exp_nbr, nd, f"{what} forward", mode=fmode)
    if m.iperm is not None:
        _check_perm_table(m.iperm, m.inv_s, exp_inv, ns, f"{what} inverse", mode=1)
    return int(exp_ptr[-1])


def check_trainer_state(state, res):
    """Every level and map of one prefetch state of the trainer against the
    reference run on that state's own input points.  Returns a summary."""
    B = state["labels"].numel()
    pts = state["points"].cpu().numpy()
    P = pts.shape[0] // B
    offs = np.arange(B + 1, dtype=np.int64) * P
    kind, levels, s1, dn = ref_integer_stage(pts, offs, res, nlev=len(state["levels"]))
    rows = []
    for i, lv in enumerate(state["levels"]):
        n = int(lv.n.item())
        np.testing.assert_array_equal(lv.coords[:n].cpu().numpy(), levels[i], err_msg=f"level {i} coords")
        rows.append(n)
    pairs = []
    for i, m in enumerate(state["map_s1"]):
        pairs.append(check_map(m, s1[i], f"map_s1[{i}]"))
    for i, m in enumerate(state["map_dn"]):
        pairs.append(check_map(m, dn[i], f"map_dn[{i}]"))
    return {"kind": kind, "rows": rows, "pairs": pairs}


# ------------------------------------------------------------------ float stage
def _conv32():
    """The oracle's conv with float32 accumulation (same rounding points):
    used only to measure the oracle's own sensitivity to accumulation order."""

    def fwd(coords, x, ts, w, offsets, stride):
        oc, ost = O.generate_output_coords(coords, ts, stride)
        km = O.build_kernel_map(coords, oc, offsets, ts)
        x32, w32 = np.asarray(x, np.float32), np.asarray(w, np.float32)
        out = np.zeros((len(oc), w.shape[1]), np.float32)
        for k, (vi, ui) in enumerate(km):
            if len(vi):
                out[ui] += x32[vi] @ w32[k].T
        return oc, out.astype(np.float64), ost

    def bwd(coords, x, ts, w, offsets, stride, g):
        oc, _ = O.generate_output_coords(coords, ts, stride)
        km = O.build_kernel_map(coords, oc, offsets, ts)
        x32, w32, g32 = np.asarray(x, np.float32), np.asarray(w, np.float32), np.asarray(g, np.float32)
        gi = np.zeros(x32.shape, np.float32)
        gw = np.zeros(w32.shape, np.float32)
        for k, (vi, ui) in enumerate(km):
            if len(vi):
                gi[vi] += g32[ui] @ w32[k]
                gw[k] = g32[ui].T @ x32[vi]
        return gi.astype(np.float64), gw.astype(np.float64)

    return fwd, bwd


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / (np.linalg.norm(b) + 1e-30))


def oracle_bf16_step(p0, coords, feats, labels, B, blocks, acc32=False):
    """The f64 oracle step on the engine's bf16-rounded conv weights with
    every engine-stored tensor rounded to bf16 (act_round)."""
    pr = {k: (bf16_round(v) if k.endswith(".w") and not k.startswith("fc") else v) for k, v in p0.items()}
    return O.resnet_train_step(pr, coords, feats, labels, B, blocks=blocks, wdtype=bf16_round,
                               act_round=bf16_round, conv_impl=_conv32() if acc32 else None)


def noise_calibrated_grad_check(grads, p0, coords, feats, labels, B, blocks, factor=2.0, floor=0.02):
    """Assert for every parameter: relL2(engine, oracle) <= factor *
    relL2(oracle_fp32acc, oracle) + floor.  Returns (loss_ref, table)."""
    rloss, rg, _, _ = oracle_bf16_step(p0, coords, feats, labels, B, blocks)
    _, ng, _, _ = oracle_bf16_step(p0, coords, feats, labels, B, blocks, acc32=True)
    table, bad = {}, {}
    for k, r in rg.items():
        e, n = rel_l2(grads[k], r), rel_l2(ng[k], r)
        table[k] = (round(e, 5), round(n, 5))
        if e > factor * n + floor:
            bad[k] = table[k]
    assert not bad, f"gradient error beyond {factor}x oracle noise + {floor}: {bad}"
    return rloss, table
