"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference's sparse-convolution hot path
(voxpipe 0.1.0, `/root/reference/pkg/src/voxpipe/`), used ONLY as the checker:
by `tests/`, by `__graft_entry__.smoke()` and by `bench.py`'s `cpu_baseline` /
`--impl reference` legs.  Nothing in the product package
(`paper_2012_13846_b200/`) imports this module; the product path fails loudly
when its CUDA library is missing instead of falling back here.

Parity pinning: the integer stage (packing, output coordinates, kernel maps,
voxelization, batching) is pinned bit-exactly against golden vectors produced
by the reference itself (`tests/golden/make_golden.py`, run against the
reference built by `oracle/build_ref.sh`) and re-checked by
`tests/test_oracle.py`.  The float stage (f64 gather-GEMM-scatter forward and
backward) is pinned against the same fixtures to 1e-12.  The model glue
(batch norm, ReLU, residual, global average pool, linear, cross entropy, SGD
with momentum) has NO reference implementation (`SPEC.md:185` lists it as a
non-goal): for those functions parity is self-defined ("parity unpinned").

Each function cites the reference file:line it restates.
"""

from __future__ import annotations

import itertools
import math

import numpy as np

# ---------------------------------------------------------------- packing
# kernels.py:40-46 — 16-bit fields: batch + up to three biased axes
FIELD_BITS = 16
AXIS_BIAS = 1 << (FIELD_BITS - 1)
AXIS_MIN = -AXIS_BIAS
AXIS_MAX = AXIS_BIAS - 1
BATCH_MAX = (1 << FIELD_BITS) - 1


class OracleError(ValueError):
    """Mirror of the reference's ValidationError/StructuralError (errors.py:14-19)."""


def pack_rows(rows: np.ndarray) -> np.ndarray:
    """kernels.py:53-79 — (N, 1+D) int64 rows -> int64 keys; D <= 3."""
    rows = np.asarray(rows, dtype=np.int64)
    dim = rows.shape[1] - 1
    if not 1 <= dim <= 3:
        raise OracleError("packing supports 1..3 axes")
    if rows.shape[0] == 0:
        return np.empty(0, dtype=np.int64)
    b = rows[:, 0]
    ax = rows[:, 1:]
    if b.min() < 0 or b.max() > BATCH_MAX:
        raise OracleError("batch index out of packable range")
    if ax.min() < AXIS_MIN or ax.max() > AXIS_MAX:
        raise OracleError("coordinate axis out of packable range")
    keys = b.astype(np.uint64)
    for d in range(dim):
        keys = (keys << np.uint64(FIELD_BITS)) | (ax[:, d] + AXIS_BIAS).astype(np.uint64)
    return keys.view(np.int64).copy()


def splitmix64(x: np.ndarray) -> np.ndarray:
    """_kernels.pyx:16-21 — splitmix64 finalizer (uint64 wraparound)."""
    x = np.asarray(x).astype(np.uint64)
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def build_table(keys: np.ndarray):
    """_kernels.pyx:24-47 / _kernels_py.py:13-26 — index over int64 keys,
    first occurrence of a duplicated key wins.  Restated as a stable sort."""
    keys = np.ascontiguousarray(keys, dtype=np.int64)
    order = np.argsort(keys, kind="stable")
    sk = keys[order]
    if len(sk) > 1:
        keep = np.ones(len(sk), dtype=bool)
        keep[1:] = sk[1:] != sk[:-1]
        sk, order = sk[keep], order[keep]
    return sk, order.astype(np.int64)


def lookup(sk: np.ndarray, rows: np.ndarray, queries: np.ndarray) -> np.ndarray:
    """_kernels.pyx:50-73 / _kernels_py.py:29-37 — row per query, -1 on miss."""
    q = np.ascontiguousarray(queries, dtype=np.int64)
    if len(sk) == 0:
        return np.full(len(q), -1, dtype=np.int64)
    pos = np.minimum(np.searchsorted(sk, q), len(sk) - 1)
    return np.where(sk[pos] == q, rows[pos], -1).astype(np.int64)


def _packable_ok(rows: np.ndarray) -> np.ndarray:
    """kernels.py:135-143 — rows whose packed key is representable."""
    return (
        (rows[:, 0] >= 0)
        & (rows[:, 0] <= BATCH_MAX)
        & (rows[:, 1:] >= AXIS_MIN).all(axis=1)
        & (rows[:, 1:] <= AXIS_MAX).all(axis=1)
    )


def coord_lookup(index, rows: np.ndarray) -> np.ndarray:
    """kernels.py:131-148 — out-of-range queries are plain misses."""
    rows = np.asarray(rows, dtype=np.int64)
    out = np.full(len(rows), -1, dtype=np.int64)
    if len(rows) == 0:
        return out
    ok = _packable_ok(rows)
    if ok.any():
        out[ok] = lookup(index[0], index[1], pack_rows(rows[ok]))
    return out


# ---------------------------------------------------------------- kernel shape
def hypercubic_offsets(dim: int, size) -> np.ndarray:
    """conv.py:51-61 — itertools.product order, axis 0 slowest."""
    ext = (size,) * dim if isinstance(size, int) else tuple(size)
    ranges = [range(-(e // 2), e // 2 + 1) for e in ext]
    return np.array(list(itertools.product(*ranges)), dtype=np.int64).reshape(-1, dim)


# ---------------------------------------------------------------- coords
def floor_div(a: np.ndarray, b) -> np.ndarray:
    return np.floor_divide(a, b)


def generate_output_coords(coords: np.ndarray, tensor_stride, stride):
    """conv.py:124-146 — stride 1: copy; stride s: floor-div by ts*s, rescale,
    unique rows in FIRST-SEEN order; new stride = ts*s."""
    coords = np.asarray(coords, dtype=np.int64)
    dim = coords.shape[1] - 1
    st = (stride,) * dim if isinstance(stride, int) else tuple(stride)
    new = tuple(int(o) * int(s) for o, s in zip(tensor_stride, st))
    if all(s == 1 for s in st):
        return coords.copy(), new
    if len(coords) == 0:
        return np.empty((0, 1 + dim), dtype=np.int64), new
    step = np.asarray(new, dtype=np.int64)
    rows = coords.copy()
    rows[:, 1:] = floor_div(rows[:, 1:], step) * step
    _, first = np.unique(rows, axis=0, return_index=True)
    first = np.sort(first)  # first-seen order == ascending first index
    return rows[first], new


def build_kernel_map(in_coords, out_coords, offsets, in_stride):
    """conv.py:149-183 — per offset (shape order): pairs (in_row, out_row),
    out rows ascending; pair iff in[v] == out[u] + off*in_stride, batch equal."""
    in_coords = np.asarray(in_coords, dtype=np.int64)
    out_coords = np.asarray(out_coords, dtype=np.int64)
    index = build_table(pack_rows(in_coords)) if len(in_coords) else (
        np.empty(0, np.int64), np.empty(0, np.int64))
    stride = np.asarray(in_stride, dtype=np.int64)
    pairs = []
    for off in np.asarray(offsets, dtype=np.int64):
        if len(out_coords) == 0:
            pairs.append((np.empty(0, np.int64), np.empty(0, np.int64)))
            continue
        q = out_coords.copy()
        q[:, 1:] += off * stride
        r = coord_lookup(index, q)
        hit = r >= 0
        pairs.append((r[hit].astype(np.int64), np.flatnonzero(hit).astype(np.int64)))
    return pairs


def brute_force_kernel_map(in_coords, out_coords, offsets, in_stride):
    """SPEC.md:167 completeness oracle — O(N*K) dict scan."""
    d = {}
    for i, r in enumerate(np.asarray(in_coords, dtype=np.int64)):
        d.setdefault(tuple(int(v) for v in r), i)
    stride = np.asarray(in_stride, dtype=np.int64)
    pairs = []
    for off in np.asarray(offsets, dtype=np.int64):
        vi, ui = [], []
        for u, r in enumerate(np.asarray(out_coords, dtype=np.int64)):
            q = (int(r[0]),) + tuple(int(v) for v in (r[1:] + off * stride))
            v = d.get(q)
            if v is not None:
                vi.append(v)
                ui.append(u)
        pairs.append((np.asarray(vi, np.int64), np.asarray(ui, np.int64)))
    return pairs


# ---------------------------------------------------------------- float stage
def sparse_conv_forward(coords, feats, tensor_stride, weights, offsets, stride=1):
    """conv.py:186-208 — out[ui] += feats[vi] @ W_k.T per offset, in offset order.
    weights: (K, n_out, n_in) float64.  Returns (out_coords, out_feats, out_stride)."""
    feats = np.asarray(feats, dtype=np.float64)
    w = np.asarray(weights, dtype=np.float64)
    if w.shape[0] != len(offsets) or w.shape[2] != feats.shape[1]:
        raise OracleError("weights do not match kernel shape / feature width")
    oc, ost = generate_output_coords(coords, tensor_stride, stride)
    km = build_kernel_map(coords, oc, offsets, tensor_stride)
    out = np.zeros((len(oc), w.shape[1]), dtype=np.float64)
    for k, (vi, ui) in enumerate(km):
        if len(vi):
            out[ui] += feats[vi] @ w[k].T
    return oc, out, ost


def sparse_conv_backward(coords, feats, tensor_stride, weights, offsets, stride, grad_out):
    """conv.py:211-242 — dgrad grad_in[vi] += g[ui] @ W_k; wgrad g[ui].T @ x[vi]."""
    feats = np.asarray(feats, dtype=np.float64)
    w = np.asarray(weights, dtype=np.float64)
    oc, _ = generate_output_coords(coords, tensor_stride, stride)
    g = np.asarray(grad_out, dtype=np.float64)
    if g.shape != (len(oc), w.shape[1]):
        raise OracleError("grad_out shape mismatch")
    km = build_kernel_map(coords, oc, offsets, tensor_stride)
    gi = np.zeros_like(feats)
    gw = np.zeros_like(w)
    for k, (vi, ui) in enumerate(km):
        if len(vi):
            gi[vi] += g[ui] @ w[k]
            gw[k] = g[ui].T @ feats[vi]
    return gi, gw


def sparse_conv_transposed(fine_coords, fine_stride, coarse_feats, weights_t, offsets, stride):
    """transposed conv = adjoint of the strided conv:
    coarse (N_c, C_in) -> fine rows (N_f, C_out) with weights_t (K, C_out, C_in).
    Restated through conv.py:211-242: backward of the strided conv whose
    weights are weights_t transposed, with grad_out = coarse features."""
    wt = np.asarray(weights_t, dtype=np.float64)
    w = np.ascontiguousarray(wt.transpose(0, 2, 1))  # (K, C_in, C_out)
    dummy = np.zeros((len(fine_coords), w.shape[2]))
    gi, _ = sparse_conv_backward(fine_coords, dummy, fine_stride, w, offsets, stride, coarse_feats)
    return gi


def dense_conv_forward(grid, weights, offsets):
    """conv.py:245-277 — zero-padded cross-correlation oracle."""
    grid = np.asarray(grid, dtype=np.float64)
    w = np.asarray(weights, dtype=np.float64)
    spatial = grid.shape[:-1]
    out = np.zeros(spatial + (w.shape[1],))
    for k, off in enumerate(np.asarray(offsets)):
        dst, src = [], []
        for d, o in enumerate(off):
            o = int(o)
            lo, hi = max(0, -o), min(spatial[d], spatial[d] - o)
            if lo >= hi:
                break
            dst.append(slice(lo, hi))
            src.append(slice(lo + o, hi + o))
        else:
            out[tuple(dst)] += grid[tuple(src)] @ w[k].T
    return out


# ---------------------------------------------------------------- data entry
def voxelize(points, voxel_size, resolution, batch_index=0, features=None):
    """tensor.py:147-184 — floor(p/vs), clip [0,res-1], first-seen dedup,
    mean feature (np.add.at order) or occupancy 1.0."""
    pts = np.asarray(points, dtype=np.float64)
    n, dim = pts.shape
    res = np.asarray(resolution, dtype=np.int64)
    fw = 1 if features is None else np.asarray(features).shape[1]
    if n == 0:
        return np.empty((0, 1 + dim), np.int64), np.empty((0, fw))
    vox = np.floor(pts / voxel_size).astype(np.int64)
    np.clip(vox, 0, res - 1, out=vox)
    rows = np.concatenate([np.full((n, 1), batch_index, np.int64), vox], axis=1)
    uniq, first, inv = np.unique(rows, axis=0, return_index=True, return_inverse=True)
    order = np.argsort(first, kind="stable")
    rank = np.empty(len(order), np.int64)
    rank[order] = np.arange(len(order))
    group = rank[np.asarray(inv).ravel()]
    out = uniq[order]
    if features is None:
        return out, np.ones((len(out), 1))
    f = np.zeros((len(out), fw))
    np.add.at(f, group, np.asarray(features, dtype=np.float64))
    f /= np.bincount(group, minlength=len(out)).astype(np.float64)[:, None]
    return out, f


def batch(coord_list, feat_list):
    """tensor.py:205-229 — concatenate, batch index = input position."""
    cs = []
    for i, c in enumerate(coord_list):
        c = np.asarray(c, dtype=np.int64).copy()
        c[:, 0] = i
        cs.append(c)
    return np.concatenate(cs, axis=0), np.concatenate([np.asarray(f, np.float64) for f in feat_list], axis=0)


def has_duplicate_rows(coords) -> bool:
    """tensor.py:28-33."""
    c = np.asarray(coords)
    return len(c) > 0 and len(np.unique(c, axis=0)) != len(c)


# ---------------------------------------------------------------- synthetic data
def shape_cloud(i: int, npts: int, res: int, seed: int = 0) -> np.ndarray:
    """SURVEY §8(d) ModelNet40-shaped synthetic surface (sphere/box/cylinder).
    World units = voxels (voxel_size 1.0)."""
    rng = np.random.default_rng(seed * 100003 + i)
    kind = i % 3
    r = rng.uniform(0.25, 0.48)
    c = rng.uniform(0.5 - 0.48 + r, 0.5 + 0.48 - r, 3)
    if kind == 0:
        v = rng.normal(size=(npts, 3))
        v /= np.linalg.norm(v, axis=1, keepdims=True)
    elif kind == 1:
        v = rng.uniform(-1, 1, size=(npts, 3))
        ax = rng.integers(0, 3, size=npts)
        v[np.arange(npts), ax] = rng.choice([-1.0, 1.0], size=npts)
    else:
        th = rng.uniform(0, 2 * np.pi, npts)
        v = np.stack([np.cos(th), np.sin(th), rng.uniform(-1, 1, npts)], axis=1)
    return np.clip((v * r + c) * res, 0, res - 1e-9)


def synthetic_batch(B: int, npts: int, res: int, seed: int = 0, dtype=np.float32):
    """Points (B*npts, 3) as `dtype` plus per-cloud offsets (B+1,)."""
    pts = np.concatenate([shape_cloud(i, npts, res, seed) for i in range(B)]).astype(dtype)
    offs = np.arange(B + 1, dtype=np.int64) * npts
    return pts, offs


def voxelize_batch(points, offsets, voxel_size, res):
    """voxelize each cloud (tensor.py:147-184) then batch (tensor.py:205-229)."""
    cl, fl = [], []
    for b in range(len(offsets) - 1):
        c, f = voxelize(np.asarray(points[offsets[b]:offsets[b + 1]], np.float64), voxel_size, (res,) * 3)
        cl.append(c)
        fl.append(f)
    return batch(cl, fl)


# ---------------------------------------------------------------- model glue
# No reference implementation exists for anything below:
# parity for these functions is self-defined ("parity unpinned").
BN_EPS = 1e-5


def bn_forward(x, gamma, beta):
    mu = x.mean(axis=0)
    var = x.var(axis=0)
    rstd = 1.0 / np.sqrt(var + BN_EPS)
    xh = (x - mu) * rstd
    return xh * gamma + beta, (xh, rstd, mu, var)


def bn_backward(gy, cache, gamma):
    xh, rstd, _, _ = cache
    n = gy.shape[0]
    gbeta = gy.sum(axis=0)
    ggamma = (gy * xh).sum(axis=0)
    gx = (gamma * rstd / n) * (n * gy - gbeta - xh * ggamma)
    return gx, ggamma, gbeta


def segment_ids(coords):
    return np.asarray(coords)[:, 0].astype(np.int64)


def global_avg_pool(x, coords, B):
    b = segment_ids(coords)
    cnt = np.bincount(b, minlength=B).astype(np.float64)
    s = np.zeros((B, x.shape[1]))
    np.add.at(s, b, x)
    return s / np.maximum(cnt, 1)[:, None], cnt


def cross_entropy(logits, labels):
    m = logits.max(axis=1, keepdims=True)
    e = np.exp(logits - m)
    p = e / e.sum(axis=1, keepdims=True)
    n = logits.shape[0]
    loss = -np.log(p[np.arange(n), labels]).mean()
    g = p.copy()
    g[np.arange(n), labels] -= 1.0
    return loss, g / n


def resnet_layout(cin=1, planes=(32, 64, 128, 256), blocks=1, classes=40):
    """SURVEY §8(d) SparseResNet: stem conv3 s1 (cin->32); per stage a conv3 s2
    then `blocks` BasicBlocks (2x conv3 s1 + identity); BN+ReLU after each conv;
    global average pool per batch index; linear planes[-1] -> classes.
    Returns list of (name, cin, cout, stride) plus classes."""
    convs = [("stem", cin, planes[0], 1)]
    prev = planes[0]
    for s, p in enumerate(planes):
        convs.append((f"s{s}.down", prev, p, 2))
        for b in range(blocks):
            convs.append((f"s{s}.b{b}.c1", p, p, 1))
            convs.append((f"s{s}.b{b}.c2", p, p, 1))
        prev = p
    return convs, classes


def init_params(cin=1, planes=(32, 64, 128, 256), blocks=1, classes=40, seed=2, K=27):
    """Weights ~ N(0,1)/sqrt(K*Cin) via default_rng(seed), layout (K, Cout, Cin)
    (SURVEY §8(d)); BN gamma=1, beta=0; linear N(0,1)/sqrt(Cin), bias 0."""
    convs, classes = resnet_layout(cin, planes, blocks, classes)
    rng = np.random.default_rng(seed)
    p = {}
    for name, ci, co, _ in convs:
        p[name + ".w"] = rng.normal(size=(K, co, ci)) / math.sqrt(K * ci)
        p[name + ".gamma"] = np.ones(co)
        p[name + ".beta"] = np.zeros(co)
    p["fc.w"] = rng.normal(size=(classes, planes[-1])) / math.sqrt(planes[-1])
    p["fc.b"] = np.zeros(classes)
    return p


def resnet_train_step(params, coords, feats, labels, B, planes=(32, 64, 128, 256), blocks=1,
                      lr=1e-2, momentum=0.9, mom=None, wdtype=None, conv_impl=None, act_round=None,
                      trace=None):
    """One SGD step of the SparseResNet in float64 with the reference's conv
    functions (conv.py:186-242) and the glue above.  `wdtype`, when given
    (e.g. a bf16-rounding function), is applied to conv weights and conv
    inputs before each conv so the comparison measures only accumulation.
    `conv_impl` = (forward, backward) with the signatures of
    sparse_conv_forward / sparse_conv_backward above (default: this module's
    restatement; oracle/ref_runner.py passes the reference's own functions).
    `act_round`, when given, rounds every tensor the GPU engine STORES in
    bf16 (conv outputs, BN/residual/ReLU outputs, activation gradients) so a
    bf16 engine can be compared at accumulation-order tolerance.
    Returns (loss, grads, new_params, new_mom)."""
    rnd = wdtype if wdtype is not None else (lambda a: a)
    ra = act_round if act_round is not None else (lambda a: a)
    cfwd, cbwd = conv_impl if conv_impl is not None else (sparse_conv_forward, sparse_conv_backward)
    offsets = hypercubic_offsets(3, 3)
    convs, _ = resnet_layout(feats.shape[1], planes, blocks, params["fc.w"].shape[0])
    tape = []
    x, c, ts = np.asarray(feats, np.float64), np.asarray(coords, np.int64), (1, 1, 1)

    def conv(name, x, c, ts, stride):
        xw = rnd(x)
        w = rnd(params[name + ".w"])
        oc, y, ost = cfwd(c, xw, ts, w, offsets, stride)
        tape.append(("conv", name, c, xw, ts, w, stride))
        if trace is not None:
            trace[name + ".y"] = ra(y)
        return ra(y), oc, ost

    def bnrelu(name, y, relu=True):
        z, cache = bn_forward(y, params[name + ".gamma"], params[name + ".beta"])
        tape.append(("bn", name, cache))
        if trace is not None:
            trace[name + ".mean"], trace[name + ".rstd"] = cache[2], cache[1]
        if relu:
            tape.append(("relu", z > 0))
            z = np.maximum(z, 0)
        return ra(z) if relu else z

    y, c, ts = conv("stem", x, c, ts, 1)
    x = bnrelu("stem", y)
    for s in range(len(planes)):
        y, c, ts = conv(f"s{s}.down", x, c, ts, 2)
        x = bnrelu(f"s{s}.down", y)
        for b in range(blocks):
            idn = x
            tape.append(("res_begin",))
            y, _, _ = conv(f"s{s}.b{b}.c1", x, c, ts, 1)
            h = bnrelu(f"s{s}.b{b}.c1", y)
            y, _, _ = conv(f"s{s}.b{b}.c2", h, c, ts, 1)
            z = bnrelu(f"s{s}.b{b}.c2", y, relu=False) + idn
            tape.append(("res_end", z > 0))
            x = ra(np.maximum(z, 0))
    pooled, cnt = global_avg_pool(x, c, B)
    logits = pooled @ params["fc.w"].T + params["fc.b"]
    loss, gl = cross_entropy(logits, labels)
    grads = {"fc.w": gl.T @ pooled, "fc.b": gl.sum(axis=0)}
    gp = gl @ params["fc.w"]
    seg = segment_ids(c)
    g = ra(gp[seg] / np.maximum(cnt, 1)[seg][:, None])
    # reverse pass
    res_stack = []
    pending = {}
    for item in reversed(tape):
        kind = item[0]
        if kind == "res_end":
            g = g * item[1]
            res_stack.append(ra(g))  # gradient flowing to identity branch
        elif kind == "res_begin":
            g = g + res_stack.pop()
        elif kind == "relu":
            g = g * item[1]
        elif kind == "bn":
            _, name, cache = item
            g, gg, gb = bn_backward(g, cache, params[name + ".gamma"])
            g = ra(g)
            if trace is not None:
                trace[name + ".gy"] = g
            grads[name + ".gamma"] = gg
            grads[name + ".beta"] = gb
        elif kind == "conv":
            _, name, cc, xw, tss, w, stride = item
            gi, gw = cbwd(cc, xw, tss, w, offsets, stride, g)
            grads[name + ".w"] = gw
            g = ra(gi)
    del pending
    new_mom = {}
    new_p = {}
    for k, v in params.items():
        m = (mom[k] if mom is not None else np.zeros_like(v)) * momentum + grads[k]
        new_mom[k] = m
        new_p[k] = v - lr * m
    return loss, grads, new_p, new_mom
