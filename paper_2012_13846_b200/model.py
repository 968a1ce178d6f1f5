"""SparseResNet classifier training on one B200 (SURVEY §8(d) model; BASELINE
config 3: 64 clouds x 2048 points at 64^3, bf16 features).

The whole training step — GPU voxelization of the raw points, strided output
coordinates, the nine kernel maps, 13 sparse convs forward, BN/ReLU/residual,
global pool, linear + cross entropy, the backward pass (dgrad + deterministic
wgrad), and SGD with momentum — is a fixed sequence of C-ABI calls on one
stream over statically allocated, capacity-sized buffers whose live row
counts stay in device memory.  Nothing reads a size back to the host, so the
step is captured once into a CUDA graph and replayed (launch-bound inner
loop -> one graph launch).

Layer list (blocks=1 -> 13 convs): stem conv3 s1 (C_in -> 32); per stage
s in 0..3 with planes (32, 64, 128, 256): conv3 s2 (prev -> p) then `blocks`
BasicBlocks (conv3 s1 p->p, BN, ReLU, conv3 s1 p->p, BN, + identity, ReLU).
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _lib
from .conv import KernelShape

BF16 = torch.bfloat16


@dataclass(eq=False)
class Level:
    """Coordinates of one tensor-stride level (rows batch-contiguous)."""

    coords: torch.Tensor  # (cap, 4) int32
    n: torch.Tensor  # (1,) int32, live rows
    cap: int
    stride: int
    seg: Optional[torch.Tensor] = None  # (2B,) int32 per-cloud row counts / starts (the head's level)


@dataclass(eq=False)
class Map:
    """Kernel map between two levels (conv.py:149-183 layout, device)."""

    nbr: torch.Tensor  # (cap_out, K)
    pin: torch.Tensor
    pout: torch.Tensor
    ptr: torch.Tensor  # (K+1,)
    inv: Optional[torch.Tensor]  # (cap_in, K) for strided maps (dgrad table)
    src: Level
    dst: Level
    ws: torch.Tensor
    # neighbour-mask row ordering (vp_kernel_map_sort) of the tables the
    # tensor-core convs read: fwd (and stride-1 dgrad, flipped) over
    # (nbr_s, perm); strided dgrad over (inv_s, iperm).  None = unsorted.
    perm: Optional[torch.Tensor] = None
    nbr_s: Optional[torch.Tensor] = None
    iperm: Optional[torch.Tensor] = None
    inv_s: Optional[torch.Tensor] = None
    sort_ws: Optional[torch.Tensor] = None


class ParamBuffer:
    """Flat fp32 parameter / gradient / momentum buffers; conv weights first so
    the bf16 shadow (tensor-core operand) is one contiguous prefix."""

    def __init__(self, device):
        self.device = device
        self.specs: list[tuple[str, tuple]] = []
        self.offsets: dict[str, tuple[int, tuple]] = {}
        self.size = 0
        self.n_bf16 = 0

    def add(self, name, shape, bf16=False):
        n = int(np.prod(shape))
        if bf16:
            assert self.n_bf16 == self.size, "bf16 params must come first"
            self.n_bf16 += n
        self.offsets[name] = (self.size, tuple(shape))
        self.size += n

    def finalize(self):
        self.p = torch.zeros(self.size, dtype=torch.float32, device=self.device)
        self.g = torch.zeros_like(self.p)
        self.m = torch.zeros_like(self.p)
        self.pb = torch.zeros(max(self.n_bf16, 1), dtype=BF16, device=self.device)

    def view(self, buf, name):
        off, shape = self.offsets[name]
        return buf[off: off + int(np.prod(shape))].view(shape)

    def bf16_view(self, name):
        off, shape = self.offsets[name]
        return self.pb[off: off + int(np.prod(shape))].view(shape)


_DBG_SKIP_WGRAD = __import__("os").environ.get("VP_DBG_SKIP_WGRAD", "0") == "1"
_DBG_SKIP_PREFETCH = __import__("os").environ.get("VP_DBG_SKIP_PREFETCH", "0") == "1"


class SparseResNetTrainer:
    """Graph-capturable SparseResNet training engine on one GPU."""

    def __init__(self, batch=64, points=2048, resolution=64, planes=(32, 64, 128, 256), blocks=1, classes=40,
                 in_channels=1, lr=1e-2, momentum=0.9, seed=2, voxel_size=1.0, device=None,
                 points_dtype=torch.float32, grad_allreduce=None, feature_dtype=BF16, index="auto", units=None):
        """feature_dtype: bf16 (tensor-core path, the product) or fp32 (SIMT
        kernels; used to validate the engine's dataflow against the f64
        oracle at fp32 tolerance).  index: coordinate index of the kernel
        maps — "grid" (dense per-level lattice), "hash" (the seam's hash
        table) or "auto" (grid while all levels' lattices fit in 4 GiB).
        units: (first, last) inclusive range of pipeline units this engine
        runs (a SparsePipe stage, pipeline.py); None = the whole model.  A
        unit is a pipeline cut granule with a single activation at each end:
        the stem, a strided conv, or a BasicBlock (the last unit also owns
        the pool + linear + loss head).  A stage that does not start at unit
        0 reads its input level coordinates / row count / features from
        `levels[entry].coords`, `levels[entry].n` and `x_in`; a stage that
        does not end at the last unit reads the gradient of its output from
        `g_out_ext` and produces the gradient of its input in `grad_input`."""
        self.B, self.P, self.res = batch, points, resolution
        self.planes, self.blocks, self.classes, self.cin = tuple(planes), blocks, classes, in_channels
        self.lr, self.momentum, self.voxel_size = lr, momentum, voxel_size
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.grad_allreduce = grad_allreduce  # callable(flat_grad) for data parallel, or None
        self.shape = KernelShape.hypercubic(3, 3)
        self.K = self.shape.num_offsets
        self.offs3 = _lib.i32_array(self.shape.offsets3().ravel())
        self.eps = 1e-5
        self.fdt = feature_dtype
        self.fcode = _lib.VP_BF16 if feature_dtype == BF16 else _lib.VP_F32
        dev = self.device
        cap = batch * points
        self.cap = cap
        # ---- inputs (static; copied into before each replay)
        self.points = torch.zeros((cap, 3), dtype=points_dtype, device=dev)
        self.offsets = torch.arange(batch + 1, dtype=torch.int64, device=dev) * points
        self.labels = torch.zeros(batch, dtype=torch.int32, device=dev)
        # ---- levels
        nlev = len(planes) + 1
        # capacities: level i holds at most min(N_{i-1}, B * ceil(res / 2^i)^3)
        # rows (voxelize clips to [0, res-1]; stride-2^i cells per axis)
        caps = [cap]
        for i in range(1, nlev):
            cells = -(-resolution // (2 ** i))
            caps.append(min(caps[-1], batch * cells ** 3))
        self.levels = [Level(torch.zeros((caps[i], 4), dtype=torch.int32, device=dev),
                             torch.zeros(1, dtype=torch.int32, device=dev), caps[i], 2 ** i) for i in range(nlev)]
        self.levels[-1].seg = torch.zeros(2 * batch, dtype=torch.int32, device=dev)
        self.feat0 = torch.zeros((cap, in_channels), dtype=feature_dtype, device=dev)
        self.vox_ws = _lib.workspace(_lib.query("vp_voxelize_ws_bytes", cap), dev)
        self.oc_ws = _lib.workspace(_lib.query("vp_output_coords_ws_bytes", cap), dev)
        # ---- maps: stride-1 per level, strided between consecutive levels
        self.map_s1 = [self._alloc_map(self.levels[i], self.levels[i], strided=False, sort=i > 0) for i in range(nlev)]
        self.map_dn = [self._alloc_map(self.levels[i], self.levels[i + 1], strided=True) for i in range(nlev - 1)]
        # dense-grid coordinate index per level (cells = B * ceil(res/2^i)^3
        # int32, kept empty between steps: only touched cells are cleared);
        # used instead of a hash table while the lattice stays small
        self.grid_R = [-(-resolution // (2 ** i)) for i in range(nlev)]
        grid_bytes = sum(4 * batch * r ** 3 for r in self.grid_R)
        if index not in ("auto", "grid", "brick", "hash"):
            raise ValueError(f"index must be auto|grid|brick|hash, got {index!r}")
        if index == "auto":
            index = __import__("os").environ.get("VP_MAP_INDEX", "grid" if grid_bytes <= (4 << 30) else "brick")
        self.index_kind = index
        self.use_grid = index in ("grid", "brick")  # a lattice index (dense cells or 4^3 bricks)
        self.grids = None
        if index == "grid":
            # cells + occupancy bitmap (vp_grid_words); zeros = an empty bitmap
            self.grids = [torch.zeros(int(_lib.query("vp_grid_words", batch, r)), dtype=torch.int32, device=dev)
                          for r in self.grid_R]
        elif index == "brick":
            self.grids = []
            for i, r in enumerate(self.grid_R):
                nb = int(_lib.query("vp_brick_bytes", self.levels[i].cap, batch, r))
                buf = torch.empty(nb, dtype=torch.uint8, device=dev)
                _lib.call("vp_brick_init", buf.data_ptr(), self.levels[i].cap, batch, r, _lib.stream())
                self.grids.append(buf)
        # ---- pipeline units and the layers this engine owns
        self.layers_all = self._layer_list()
        self.units = self._unit_list(self.layers_all)
        nu = len(self.units)
        self.unit_range = (0, nu - 1) if units is None else (int(units[0]), int(units[1]))
        u0, u1 = self.unit_range
        if not (0 <= u0 <= u1 < nu):
            raise ValueError(f"unit range {units} outside 0..{nu - 1}")
        self.first, self.last = u0 == 0, u1 == nu - 1
        self.layers = [L for u in self.units[u0:u1 + 1] for L in u["layers"]]
        self.entry_level = self.levels.index(self.layers[0]["src"])
        self.exit_level = self.levels.index(self.layers[-1]["dst"])
        # ---- parameters
        pb = ParamBuffer(dev)
        for L in self.layers:
            pb.add(L["name"] + ".w", (self.K, L["cout"], L["cin"]), bf16=True)
        for L in self.layers:
            pb.add(L["name"] + ".gamma", (L["cout"],))
            pb.add(L["name"] + ".beta", (L["cout"],))
        if self.last:
            pb.add("fc.w", (classes, planes[-1]))
            pb.add("fc.b", (classes,))
        pb.finalize()
        self.params = pb
        self._init_params(seed)
        # ---- activations (capacity sized)
        for L in self.layers:
            n = L["dst"].cap
            L["y"] = torch.zeros((n, L["cout"]), dtype=feature_dtype, device=dev)  # conv output (pre-BN)
            L["a"] = torch.zeros((n, L["cout"]), dtype=feature_dtype, device=dev)  # BN(+res)(+ReLU) output
            L["mean"] = torch.zeros(L["cout"], dtype=torch.float32, device=dev)
            L["rstd"] = torch.zeros(L["cout"], dtype=torch.float32, device=dev)
            L["gy"] = torch.zeros((n, L["cout"]), dtype=feature_dtype, device=dev)  # grad wrt conv output
            L["w"] = pb.view(pb.p, L["name"] + ".w")
            # the conv operand: bf16 shadow on the tensor-core path, fp32 master otherwise
            L["wb"] = pb.bf16_view(L["name"] + ".w") if feature_dtype == BF16 else L["w"]
            L["wcode"] = _lib.VP_BF16 if feature_dtype == BF16 else _lib.VP_F32
            L["gw"] = pb.view(pb.g, L["name"] + ".w")
            for k in ("gamma", "beta"):
                L[k] = pb.view(pb.p, f"{L['name']}.{k}")
                L["g" + k] = pb.view(pb.g, f"{L['name']}.{k}")
            L["fwd_ws"] = _lib.workspace(_lib.query("vp_conv_fwd_ws_bytes", L["cin"], L["cout"], self.K), dev)
            L["dg_ws"] = _lib.workspace(_lib.query("vp_conv_dgrad_ws_bytes", L["cin"], L["cout"], self.K), dev)
            L["wg_ws"] = _lib.workspace(_lib.query("vp_conv_wgrad_ws_bytes", L["cin"], L["cout"], self.K,
                                                   L["map"].pin.numel()), dev)
            # zero-filled: the fused BN kernels' ticket word starts (and stays) zero
            L["bn_ws"] = torch.zeros(int(_lib.query("vp_bn_stats_ws_bytes", n, L["cout"])), dtype=torch.uint8,
                                     device=dev)
            # BN statistics partials written by the producing conv's epilogue
            # (forward: this conv; backward: the dgrad of the next conv)
            L["fpart"] = _lib.workspace(_lib.query("vp_bn_part_bytes", L["cout"]), dev, zero=True)
            L["bpart"] = _lib.workspace(_lib.query("vp_bn_part_bytes", L["cout"]), dev, zero=True)
        # gradient buffers per level for the activation flowing back
        self.gact = [torch.zeros((lv.cap, self._width_at(i)), dtype=feature_dtype, device=dev)
                     for i, lv in enumerate(self.levels)]
        # identity (skip-path) gradients per level, two per level so that
        # consecutive BasicBlocks of one level (blocks >= 2) never read and
        # write the same buffer in one launch (_gid)
        self.gid = [[torch.zeros((lv.cap, self._width_at(i)), dtype=feature_dtype, device=dev)
                     for i, lv in enumerate(self.levels)] for _ in range(2 if blocks > 1 else 1)]
        # stage boundary buffers (pipeline): input features of a non-first
        # stage, gradient of the output of a non-last stage
        ent, ext = self.entry_level, self.exit_level
        self.x_in = (None if self.first else
                     torch.zeros((self.levels[ent].cap, self.layers[0]["cin"]), dtype=feature_dtype, device=dev))
        self.g_out_ext = (None if self.last else
                          torch.zeros((self.levels[ext].cap, self.layers[-1]["cout"]), dtype=feature_dtype,
                                      device=dev))
        self.grad_input = None  # gradient wrt x_in after a backward (non-first stages)
        C = planes[-1]
        self.pooled = torch.zeros((batch, C), dtype=torch.float32, device=dev)
        self.pool_counts = torch.zeros(batch, dtype=torch.int32, device=dev)
        self.pool_ws = _lib.workspace(_lib.query("vp_global_pool_ws_bytes", batch), dev)
        self.logits = torch.zeros((batch, classes), dtype=torch.float32, device=dev)
        self.loss = torch.zeros(1, dtype=torch.float32, device=dev)
        self.g_pooled = torch.zeros((batch, C), dtype=torch.float32, device=dev)
        self.xent_ws = _lib.workspace(_lib.query("vp_linear_xent_ws_bytes", batch, classes), dev)
        self.head_ws = _lib.workspace(_lib.query("vp_sparse_head_ws_bytes", batch, C, classes), dev)
        self.graph: Optional[torch.cuda.CUDAGraph] = None
        self.launch_count = 0
        # side streams: the coordinate chain, kernel maps and weight gradients
        # run off the critical path (parallel branches of the captured graph)
        self.concurrent = True
        self.side = [torch.cuda.Stream(device=dev) for _ in range(4)]
        # the step's critical path (conv -> BN -> conv ...) is captured on a
        # HIGH-priority stream; side streams (coordinate chain, maps, weight
        # gradients, prefetch) keep the default low priority, so when both
        # have blocks waiting the SMs go to the critical path first
        self.main_stream = torch.cuda.Stream(device=dev, priority=torch.cuda.Stream.priority_range()[1])
        self.int_side = self.side[:3]  # the integer stage's chain + two map streams
        self._all_streams = list(self.side)
        self._forked = set()
        self.prefetch = False
        self.states = None
        self._sgd_in_backward = False  # set inside step_body / prefetch_body (single-process training)
        self.layer_sgd = __import__("os").environ.get("VP_LAYER_SGD", "1") != "0"
        # BN statistics from the producing conv's epilogue (vp_conv_fwd_bn /
        # vp_conv_dgrad_bn) instead of a separate statistics pass
        self.bn_fuse = __import__("os").environ.get("VP_BN_EPI", "1") != "0"
        # per-layer momentum SGD inside the weight-gradient reduction
        self.fuse_sgd = __import__("os").environ.get("VP_FUSE_SGD", "1") != "0"

    # ------------------------------------------------------------------ setup
    def _width_at(self, level):
        return self.planes[0] if level == 0 else self.planes[level - 1]

    # maps with at least this many output rows are neighbour-mask sorted
    # (vp_kernel_map_sort): at C5-scale levels the sort pays for itself many
    # times over; at C3 (<= 131k rows, diverse masks) its launches cost more
    # than the 1.3-1.7x fewer active offsets per tile save (tools/sweep_c2.py)
    SORT_MIN_ROWS = int(__import__("os").environ.get("VP_SORT_MIN_ROWS", 1 << 18))
    SORT_INV_MIN_ROWS = int(__import__("os").environ.get("VP_SORT_INV_MIN_ROWS", 0))
    # forward tables of levels with at least this many rows (capacity) group by
    # the full 27-bit mask (three passes) instead of the 9-bit column key
    FULL_MASK_ROWS = int(__import__("os").environ.get("VP_FULL_MASK_ROWS", 1 << 18))
    # levels whose forward tables are sorted regardless of size
    SORT_LEVELS = tuple(int(v) for v in __import__("os").environ.get("VP_SORT_LEVELS", "1,2,3").split(",") if v)
    # prefetch mode: fork the next batch's integer stage at the start of the
    # step, concurrent with the forward too (VP_PREFETCH_EARLY=0: after the
    # forward; measured 42.5k -> 43.8k clouds/s at C3 with the early fork)
    PREFETCH_EARLY = __import__("os").environ.get("VP_PREFETCH_EARLY", "1") == "1"

    def _alloc_map(self, src: Level, dst: Level, strided: bool, sort: bool = True) -> Map:
        dev, K = self.device, self.K
        cap_p = dst.cap * K
        m = Map(
            nbr=torch.zeros((dst.cap, K), dtype=torch.int32, device=dev),
            pin=torch.zeros(cap_p, dtype=torch.int32, device=dev),
            pout=torch.zeros(cap_p, dtype=torch.int32, device=dev),
            ptr=torch.zeros(K + 1, dtype=torch.int32, device=dev),
            inv=torch.zeros((src.cap, K), dtype=torch.int32, device=dev) if strided else None,
            src=src, dst=dst,
            ws=_lib.workspace(max(_lib.query("vp_kernel_map_ws_bytes", src.cap, dst.cap, K),
                                  _lib.query("vp_kernel_map_grid_ws_bytes", dst.cap, K)), dev))
        nws = 0
        lvl = int(dst.stride).bit_length() - 1  # level i has tensor stride 2^i
        if sort and (dst.cap >= self.SORT_MIN_ROWS or lvl in self.SORT_LEVELS):
            m.perm = torch.zeros(dst.cap, dtype=torch.int32, device=dev)
            m.nbr_s = torch.zeros((dst.cap, K), dtype=torch.int32, device=dev)
            nws = _lib.query("vp_kernel_map_sort_ws_bytes", dst.cap, K)
        if strided and src.cap >= self.SORT_INV_MIN_ROWS:
            # the inverse table of a strided map is sparse (~2-3 of 27 offsets
            # per input row): grouped rows cut the strided dgrad 2-2.5x at
            # every size, and the sort runs in the prefetched integer stage
            m.iperm = torch.zeros(src.cap, dtype=torch.int32, device=dev)
            m.inv_s = torch.zeros((src.cap, K), dtype=torch.int32, device=dev)
            nws = max(nws, _lib.query("vp_kernel_map_sort_ws_bytes", src.cap, K))
        if nws:
            m.sort_ws = _lib.workspace(nws, dev)
        return m

    def _layer_list(self):
        L = [dict(name="stem", cin=self.cin, cout=self.planes[0], src=self.levels[0], dst=self.levels[0],
                  map=self.map_s1[0], kind="stem")]
        prev = self.planes[0]
        for s, p in enumerate(self.planes):
            L.append(dict(name=f"s{s}.down", cin=prev, cout=p, src=self.levels[s], dst=self.levels[s + 1],
                          map=self.map_dn[s], kind="down"))
            for b in range(self.blocks):
                L.append(dict(name=f"s{s}.b{b}.c1", cin=p, cout=p, src=self.levels[s + 1], dst=self.levels[s + 1],
                              map=self.map_s1[s + 1], kind="c1", block=b))
                L.append(dict(name=f"s{s}.b{b}.c2", cin=p, cout=p, src=self.levels[s + 1], dst=self.levels[s + 1],
                              map=self.map_s1[s + 1], kind="c2", block=b))
            prev = p
        for i, l in enumerate(L):
            l["index"] = i
            l["level"] = self.levels.index(l["dst"])
        return L

    @staticmethod
    def _unit_list(layers):
        """Pipeline cut granules (stem | strided conv | BasicBlock) in order."""
        units, i = [], 0
        while i < len(layers):
            k = layers[i]["kind"]
            if k == "c1":
                units.append(dict(kind="block", layers=[layers[i], layers[i + 1]]))
                i += 2
            else:
                units.append(dict(kind=k, layers=[layers[i]]))
                i += 1
        for j, u in enumerate(units):
            u["index"] = j
            u["name"] = u["layers"][0]["name"].rsplit(".c1", 1)[0]
        return units

    def _init_params(self, seed):
        """Weights ~ N(0,1)/sqrt(K*C_in) via default_rng(seed), layout (K, C_out,
        C_in) (oracle.init_params / SURVEY §8(d)); BN gamma 1, beta 0; fc
        N(0,1)/sqrt(C)."""
        rng = np.random.default_rng(seed)
        pb = self.params
        for L in self.layers_all:  # draw every layer so a stage's slice equals the full model's
            w = rng.normal(size=(self.K, L["cout"], L["cin"])) / math.sqrt(self.K * L["cin"])
            if L["name"] + ".w" in pb.offsets:
                pb.view(pb.p, L["name"] + ".w").copy_(torch.from_numpy(w))
                pb.view(pb.p, L["name"] + ".gamma").fill_(1.0)
        fcw = rng.normal(size=(self.classes, self.planes[-1])) / math.sqrt(self.planes[-1])
        if "fc.w" in pb.offsets:
            pb.view(pb.p, "fc.w").copy_(torch.from_numpy(fcw))
        pb.pb[: pb.n_bf16].copy_(pb.p[: pb.n_bf16].to(BF16))

    def load_params(self, params: dict):
        pb = self.params
        for k, v in params.items():
            pb.view(pb.p, k).copy_(torch.as_tensor(np.asarray(v), dtype=torch.float32))
        pb.pb[: pb.n_bf16].copy_(pb.p[: pb.n_bf16].to(BF16))

    def state_numpy(self) -> dict:
        pb = self.params
        return {k: pb.view(pb.p, k).cpu().numpy().astype(np.float64) for k in pb.offsets}

    def grads_numpy(self) -> dict:
        pb = self.params
        return {k: pb.view(pb.g, k).cpu().numpy().astype(np.float64) for k in pb.offsets}

    # ------------------------------------------------------------------ step pieces
    def _c(self, name, *args):
        self.launch_count += 1
        _lib.call(name, *args)

    def _grid_set(self, i, st, clear):
        lv = self.levels[i]
        if self.index_kind == "brick":
            self._c("vp_brick_set", lv.coords.data_ptr(), lv.n.data_ptr(), lv.cap, self.grids[i].data_ptr(), lv.cap,
                    self.B, self.grid_R[i], lv.stride, int(clear), st)
            return
        self._c("vp_grid_set", lv.coords.data_ptr(), lv.n.data_ptr(), lv.cap, self.grids[i].data_ptr(), self.B,
                self.grid_R[i], lv.stride, int(clear), st)

    # stride-1 forward tables of these levels are tile-scheduled for the conv
    # grid that consumes them (vp_kernel_map_group_sched: their 4 convs per
    # block; VP_TILE_SCHED=0: plain grouping everywhere)
    TILE_SCHED = __import__("os").environ.get("VP_TILE_SCHED", "1") != "0"
    TILE_SCHED_LEVELS = tuple(int(v) for v in __import__("os").environ.get("VP_TILE_SCHED_LEVELS", "1").split(",") if v)

    def _sched_grid(self, m, level):
        i = self.levels.index(level)
        if not self.TILE_SCHED or m.dst is not m.src or i not in self.TILE_SCHED_LEVELS:
            return 0
        return int(_lib.query("vp_conv_tc_grid", self._width_at(i), level.cap))

    def _build_map(self, m, st):
        ist = _lib.i32_array((m.src.stride,) * 3)
        if self.index_kind == "brick":
            i = self.levels.index(m.src)
            self._c("vp_kernel_map_brick", self.grids[i].data_ptr(), m.src.cap, self.B, self.grid_R[i], m.src.stride,
                    m.dst.coords.data_ptr(), m.dst.n.data_ptr(), m.dst.cap, self.offs3, self.K, ist, m.nbr.data_ptr(),
                    m.pin.data_ptr(), m.pout.data_ptr(), m.ptr.data_ptr(), m.ws.data_ptr(), m.ws.numel(), st)
        elif self.use_grid:
            i = self.levels.index(m.src)
            self._c("vp_kernel_map_grid", self.grids[i].data_ptr(), self.B, self.grid_R[i], m.src.stride,
                    m.dst.coords.data_ptr(), m.dst.n.data_ptr(), m.dst.cap, self.offs3, self.K, ist, m.nbr.data_ptr(),
                    m.pin.data_ptr(), m.pout.data_ptr(), m.ptr.data_ptr(), m.ws.data_ptr(), m.ws.numel(), st)
        else:
            self._c("vp_kernel_map", m.src.coords.data_ptr(), m.src.n.data_ptr(), m.src.cap, m.dst.coords.data_ptr(),
                    m.dst.n.data_ptr(), m.dst.cap, self.offs3, self.K, ist, m.nbr.data_ptr(), m.pin.data_ptr(),
                    m.pout.data_ptr(), m.ptr.data_ptr(), m.ws.data_ptr(), m.ws.numel(), st)
        if m.inv is not None:
            self._c("vp_kernel_map_inverse", m.nbr.data_ptr(), m.dst.n.data_ptr(), m.dst.cap, self.K,
                    m.inv.data_ptr(), m.src.cap, st)
        # tile schedule for the consuming convs' grid (forward table: the
        # convs writing the map's output level; inverse table: the strided
        # dgrad writing its input level)
        if m.perm is not None:
            self._c("vp_kernel_map_group_sched", m.nbr.data_ptr(), m.dst.n.data_ptr(), m.dst.cap, self.K,
                    2 if m.dst.cap >= self.FULL_MASK_ROWS else 0, self._sched_grid(m, m.dst), m.perm.data_ptr(),
                    m.nbr_s.data_ptr(), m.sort_ws.data_ptr(), m.sort_ws.numel(), st)
        if m.iperm is not None:
            self._c("vp_kernel_map_group_sched", m.inv.data_ptr(), m.src.n.data_ptr(), m.src.cap, self.K, 1,
                    self._sched_grid(m, m.src), m.iperm.data_ptr(), m.inv_s.data_ptr(), m.sort_ws.data_ptr(),
                    m.sort_ws.numel(), st)

    @staticmethod
    def fwd_table(L):
        m = L["map"]
        return m.nbr_s if m.perm is not None else m.nbr

    @staticmethod
    def fwd_perm(L):
        return L["map"].perm

    @staticmethod
    def dgrad_table(L):
        """(table, flip, perm) of the layer's dgrad gather."""
        m = L["map"]
        if m.inv is None:  # stride 1, symmetric 3^3: inv[v,k] == nbr[v,K-1-k]
            return (m.nbr_s, 1, m.perm) if m.perm is not None else (m.nbr, 1, None)
        return (m.inv_s, 0, m.iperm) if m.iperm is not None else (m.inv, 0, None)

    def _integer_stage(self, st):
        """Voxelize (first stage) -> strided coordinate chain -> the kernel
        maps this engine's layers use.  With `concurrent`, the coordinate
        chain and every map but the first layer's run on side streams
        (waiting only on the levels they read), overlapping the first map and
        the first convolutions on the main stream."""
        lv = self.levels
        ent, ext = self.entry_level, self.exit_level
        if self.first:
            res3 = _lib.i32_array((self.res,) * 3)
            self._c("vp_voxelize", self.points.data_ptr(), _lib.dtype_code(self.points), self.cap,
                    self.offsets.data_ptr(), self.B, float(self.voxel_size), res3, lv[0].coords.data_ptr(),
                    lv[0].n.data_ptr(), None, self.feat0.data_ptr(), self.fcode, self.vox_ws.data_ptr(),
                    self.vox_ws.numel(), st)
        self.map_events = {}
        # maps used by this engine's layers, grouped by the level they gather from
        by_level = {}
        for L in self.layers:
            i = self.levels.index(L["src"])
            if all(m is not L["map"] for m in by_level.get(i, [])):
                by_level.setdefault(i, []).append(L["map"])
        first_map = self.layers[0]["map"]
        main = torch.cuda.current_stream()
        conc = self.concurrent

        def out_coords(i, stream):
            step = _lib.i32_array((lv[i].stride,) * 3)
            self._c("vp_output_coords", lv[i - 1].coords.data_ptr(), lv[i - 1].n.data_ptr(), lv[i - 1].cap, step,
                    lv[i].coords.data_ptr(), lv[i].n.data_ptr(), None, self.oc_ws.data_ptr(), self.oc_ws.numel(),
                    stream)

        def segments(stream):  # per-cloud row segments of the head's level (vp_sparse_head)
            if self.last:
                lx = lv[ext]
                self._c("vp_batch_segments", lx.coords.data_ptr(), lx.n.data_ptr(), lx.cap, self.B, lx.seg.data_ptr(),
                        stream)

        lev_ev = {}
        self.seg_event = None
        if conc:
            chain = self.int_side[0]
            self._forked.add(id(chain))
            chain.wait_stream(main)
            with torch.cuda.stream(chain):
                for i in range(ent + 1, ext + 1):
                    out_coords(i, chain.cuda_stream)
                    lev_ev[i] = torch.cuda.Event()
                    lev_ev[i].record(chain)
                segments(chain.cuda_stream)
                self.seg_event = torch.cuda.Event()
                self.seg_event.record(chain)
        else:
            for i in range(ent + 1, ext + 1):
                out_coords(i, st)
            segments(st)

        def needs(stream, i, maps):
            if not conc:
                return
            if i in lev_ev:
                stream.wait_event(lev_ev[i])
            if any(m.dst is not m.src for m in maps) and (i + 1) in lev_ev:
                stream.wait_event(lev_ev[i + 1])

        def build(i, maps, stream, set_grid, clear_grid, record):
            ss = stream.cuda_stream if conc else st
            if self.use_grid and set_grid:
                self._grid_set(i, ss, clear=False)
            for m in maps:
                self._build_map(m, ss)
                if record:
                    ev = torch.cuda.Event()
                    ev.record(stream)
                    self.map_events[id(m)] = ev
            if self.use_grid and clear_grid:
                self._grid_set(i, ss, clear=True)

        for i in sorted(by_level):
            maps = by_level[i]
            if not conc:
                build(i, maps, main, True, True, False)
                continue
            side = self.int_side[1 + (i % 2)]
            if first_map in maps:
                # the first layer's map on the critical path; the level's other
                # map (and the index clear) on a side stream after it
                needs(main, i, [first_map])
                rest = [m for m in maps if m is not first_map]
                build(i, [first_map], main, True, not rest, False)
                if rest:
                    ev0 = torch.cuda.Event()
                    ev0.record(main)
                    self._forked.add(id(side))  # joined (so joinable) only when it takes work
                    side.wait_event(ev0)
                    needs(side, i, rest)
                    with torch.cuda.stream(side):
                        build(i, rest, side, False, True, True)
            else:
                self._forked.add(id(side))
                side.wait_stream(main)  # fork from the origin (a no-op dependency when i > entry)
                needs(side, i, maps)
                with torch.cuda.stream(side):
                    build(i, maps, side, True, True, True)

    def _wait_map(self, m):
        ev = getattr(self, "map_events", {}).get(id(m))
        if ev is not None:
            torch.cuda.current_stream().wait_event(ev)

    def _conv_bn(self, L, x, res, relu, st):
        dst = L["dst"]
        fc = self.fcode
        self._wait_map(L["map"])
        conv = (x.data_ptr(), fc, x.shape[0], L["cin"], L["wb"].data_ptr(), L["wcode"], L["cout"], self.K,
                self.fwd_table(L).data_ptr(), 0, _lib.ptr(self.fwd_perm(L)), dst.n.data_ptr(), dst.cap,
                L["y"].data_ptr(), fc, L["fwd_ws"].data_ptr(), L["fwd_ws"].numel())
        if self.bn_fuse:
            # conv with the BN statistics from its epilogue, then normalise
            # (+ residual) (+ ReLU) from those partials: two launches
            self._c("vp_conv_fwd_bn", *conv, 1, L["fpart"].data_ptr(), None, None, None, None, self.eps,
                    L["mean"].data_ptr(), L["rstd"].data_ptr(), None, st)
            self._c("vp_bn_apply", L["y"].data_ptr(), fc, dst.n.data_ptr(), dst.cap, L["cout"], L["mean"].data_ptr(),
                    L["rstd"].data_ptr(), L["gamma"].data_ptr(), L["beta"].data_ptr(), _lib.ptr(res), fc, int(relu),
                    L["a"].data_ptr(), fc, st)
        else:
            self._c("vp_conv_fwd", *conv, st)
            # batch statistics + normalise (+ residual) (+ ReLU)
            self._c("vp_bn_forward", L["y"].data_ptr(), fc, dst.n.data_ptr(), dst.cap, L["cout"], self.eps,
                    L["mean"].data_ptr(), L["rstd"].data_ptr(), L["gamma"].data_ptr(), L["beta"].data_ptr(),
                    _lib.ptr(res), fc, int(relu), L["a"].data_ptr(), fc, L["bn_ws"].data_ptr(),
                    L["bn_ws"].numel(), st)
        L["x"] = x
        return L["a"]

    def _forward(self, st):
        x = self.feat0 if self.first else self.x_in
        for u in self.units[self.unit_range[0]:self.unit_range[1] + 1]:
            Ls = u["layers"]
            if u["kind"] == "block":
                idn = x
                h = self._conv_bn(Ls[0], x, None, True, st)
                x = self._conv_bn(Ls[1], h, idn, True, st)
            else:
                x = self._conv_bn(Ls[0], x, None, True, st)
        self.out_act = x
        if not self.last:
            return x
        last = self.levels[-1]
        C = self.planes[-1]
        if self.bn_fuse:
            # pool + linear + cross entropy + the rows' gradient masked by the
            # last BN's ReLU with that BN's backward statistics, fused
            if getattr(self, "seg_event", None) is not None and not self.prefetch:
                torch.cuda.current_stream().wait_event(self.seg_event)
            pb = self.params
            Ll = self.layers[-1]
            self._c("vp_sparse_head", x.data_ptr(), self.fcode, last.seg.data_ptr(), self.B, C,
                    pb.view(pb.p, "fc.w").data_ptr(), pb.view(pb.p, "fc.b").data_ptr(), self.classes,
                    self.labels.data_ptr(), self.pooled.data_ptr(), self.logits.data_ptr(), self.loss.data_ptr(),
                    pb.view(pb.g, "fc.w").data_ptr(), pb.view(pb.g, "fc.b").data_ptr(), Ll["a"].data_ptr(),
                    Ll["y"].data_ptr(), Ll["mean"].data_ptr(), Ll["rstd"].data_ptr(), self._gm_buf(Ll).data_ptr(),
                    Ll["bpart"].data_ptr(), Ll["ggamma"].data_ptr(), Ll["gbeta"].data_ptr(), self.head_ws.data_ptr(),
                    self.head_ws.numel(), st)
            return x
        self._c("vp_global_pool", x.data_ptr(), self.fcode, last.coords.data_ptr(), last.n.data_ptr(), last.cap, C,
                self.B, self.pooled.data_ptr(), self.pool_counts.data_ptr(), self.pool_ws.data_ptr(),
                self.pool_ws.numel(), st)
        pb = self.params
        self._c("vp_linear_xent", self.pooled.data_ptr(), self.B, C, pb.view(pb.p, "fc.w").data_ptr(),
                pb.view(pb.p, "fc.b").data_ptr(), self.classes, self.labels.data_ptr(), self.logits.data_ptr(),
                self.loss.data_ptr(), self.g_pooled.data_ptr(), pb.view(pb.g, "fc.w").data_ptr(),
                pb.view(pb.g, "fc.b").data_ptr(), self.xent_ws.data_ptr(), self.xent_ws.numel(), st)
        return x

    def _gid(self, c2):
        """The skip-path gradient buffer of the BasicBlock ending in c2."""
        return self.gid[c2["block"] % len(self.gid)][c2["level"]]

    def _gm_buf(self, P):
        """Where the producer stores layer P's masked BN gradient: the
        identity-gradient buffer of P's level when P ends a BasicBlock (that
        gradient is also the block's skip-path gradient), else the level's
        activation-gradient buffer."""
        return self._gid(P) if P["kind"] == "c2" else self.gact[P["level"]]

    def _bn_conv_backward(self, L, g_out, g_out2, g_res, st, need_dgrad=True, prepared=False, prev=None,
                          prev_add=None):
        """BN(+ReLU) backward then conv dgrad/wgrad.  g_out (+g_out2) is the
        gradient wrt L['a']; returns the gradient wrt the conv input.

        prepared: the producer of g_out (the next conv's dgrad epilogue)
        already stored L's masked gradient in g_out and wrote L's BN partials
        (L['bpart']), so only the apply runs here.  prev: the layer whose
        activation is L's input; with BN fusion on, this dgrad's epilogue
        prepares prev's BN backward the same way (prev_add = the skip-path
        gradient that joins prev's output) and the result is prev's masked
        gradient."""
        dst, src, m = L["dst"], L["src"], L["map"]
        fc = self.fcode
        if prepared:  # (ggamma, gbeta) were finalized by the producer chain
            self._c("vp_bn_backward_apply", g_out.data_ptr(), fc, L["y"].data_ptr(), fc, dst.n.data_ptr(), dst.cap,
                    L["cout"], L["mean"].data_ptr(), L["rstd"].data_ptr(), L["gamma"].data_ptr(),
                    L["ggamma"].data_ptr(), L["gbeta"].data_ptr(), L["gy"].data_ptr(), fc, st)
        else:
            self._c("vp_bn_backward", g_out.data_ptr(), _lib.ptr(g_out2), fc, L["a"].data_ptr(), fc,
                    L["y"].data_ptr(), fc, dst.n.data_ptr(), dst.cap, L["cout"], L["mean"].data_ptr(),
                    L["rstd"].data_ptr(), L["gamma"].data_ptr(), 1, L["gy"].data_ptr(), fc, _lib.ptr(g_res),
                    L["ggamma"].data_ptr(), L["gbeta"].data_ptr(), L["bn_ws"].data_ptr(), L["bn_ws"].numel(), st)
        x = L["x"]
        if _DBG_SKIP_WGRAD:  # experiments only: the step without weight gradients (never for results)
            return self._dgrad_only(L, prev, prev_add, need_dgrad, st)
        if self._fuse_sgd():
            return self._wgrad_sgd_after_dgrad(L, prev, prev_add, need_dgrad, st)
        if self.concurrent:  # weight gradient off the critical path
            ws = self.side[3 - (L["index"] % 2)]
            self._forked.add(id(ws))
            ws.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(ws):  # the side-stream variant (SM-capped persistent grid)
                self._c("vp_conv_wgrad_side", x.data_ptr(), fc, L["cin"], L["gy"].data_ptr(), fc, L["cout"],
                        self.K, m.pin.data_ptr(), m.pout.data_ptr(), m.ptr.data_ptr(), m.pin.numel(),
                        L["gw"].data_ptr(), L["wg_ws"].data_ptr(), L["wg_ws"].numel(), ws.cuda_stream)
        else:
            self._c("vp_conv_wgrad", x.data_ptr(), fc, L["cin"], L["gy"].data_ptr(), fc, L["cout"],
                    self.K, m.pin.data_ptr(), m.pout.data_ptr(), m.ptr.data_ptr(), m.pin.numel(), L["gw"].data_ptr(),
                    L["wg_ws"].data_ptr(), L["wg_ws"].numel(), st)
        if not need_dgrad:
            self._layer_sgd(L, ws if self.concurrent else None, None, st)
            return None
        table, flip, perm = self.dgrad_table(L)
        dgrad = (L["gy"].data_ptr(), fc, L["gy"].shape[0], L["cout"], L["wb"].data_ptr(), L["wcode"], L["cin"],
                 self.K, table.data_ptr(), flip, _lib.ptr(perm), src.n.data_ptr(), src.cap)
        if prev is not None and self.bn_fuse:
            gin = self._gm_buf(prev)
            self._c("vp_conv_dgrad_bn", *dgrad, gin.data_ptr(), fc, L["dg_ws"].data_ptr(), L["dg_ws"].numel(), 2,
                    prev["bpart"].data_ptr(), _lib.ptr(prev_add), prev["a"].data_ptr(), prev["y"].data_ptr(),
                    prev["mean"].data_ptr(), 0.0, prev["ggamma"].data_ptr(), prev["gbeta"].data_ptr(),
                    prev["rstd"].data_ptr(), st)
        else:
            gin = self.gact[self.levels.index(src)]
            self._c("vp_conv_dgrad", *dgrad, gin.data_ptr(), fc, L["dg_ws"].data_ptr(), L["dg_ws"].numel(), st)
        if self._sgd_in_backward:
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream())
            self._layer_sgd(L, ws if self.concurrent else None, ev, st)
        return gin

    def _fuse_sgd(self):
        """Per-layer SGD inside the weight-gradient reduction: single-process
        training with side streams (no gradient all-reduce between them)."""
        return self.fuse_sgd and self._sgd_in_backward and self.grad_allreduce is None and self.concurrent

    def _wgrad_sgd_after_dgrad(self, L, prev, prev_add, need_dgrad, st):
        """The layer's weight-gradient partials on a side stream as soon as
        its gradient exists, dgrad on the critical path, then the partial
        reduction with the momentum SGD fused in (vp_conv_wgrad_sgd phases
        1 / 2) once the dgrad — the step's last reader of W — is issued."""
        main = torch.cuda.current_stream()
        ws = self.side[3 - (L["index"] % 2)]
        self._forked.add(id(ws))
        ws.wait_stream(main)
        m, fc, pb = L["map"], self.fcode, self.params
        off, shape = pb.offsets[L["name"] + ".w"]
        x = L["x"]
        args = (x.data_ptr(), fc, L["cin"], L["gy"].data_ptr(), fc, L["cout"], self.K, m.pin.data_ptr(),
                m.pout.data_ptr(), m.ptr.data_ptr(), m.pin.numel(), L["gw"].data_ptr(), L["wg_ws"].data_ptr(),
                L["wg_ws"].numel(), pb.p.data_ptr() + 4 * off, pb.m.data_ptr() + 4 * off, pb.pb.data_ptr() + 2 * off,
                float(self.lr), float(self.momentum))
        with torch.cuda.stream(ws):
            self._c("vp_conv_wgrad_sgd", *args, 1, ws.cuda_stream)
        gin = self._dgrad_only(L, prev, prev_add, need_dgrad, st)
        ws.wait_stream(main)
        with torch.cuda.stream(ws):
            self._c("vp_conv_wgrad_sgd", *args, 2, ws.cuda_stream)
        return gin

    def _dgrad_only(self, L, prev, prev_add, need_dgrad, st):
        if not need_dgrad:
            return None
        src, fc = L["src"], self.fcode
        table, flip, perm = self.dgrad_table(L)
        dgrad = (L["gy"].data_ptr(), fc, L["gy"].shape[0], L["cout"], L["wb"].data_ptr(), L["wcode"], L["cin"],
                 self.K, table.data_ptr(), flip, _lib.ptr(perm), src.n.data_ptr(), src.cap)
        gin = self._gm_buf(prev) if (prev is not None and self.bn_fuse) else self.gact[self.levels.index(src)]
        if prev is not None and self.bn_fuse:
            self._c("vp_conv_dgrad_bn", *dgrad, gin.data_ptr(), fc, L["dg_ws"].data_ptr(), L["dg_ws"].numel(), 2,
                    prev["bpart"].data_ptr(), _lib.ptr(prev_add), prev["a"].data_ptr(), prev["y"].data_ptr(),
                    prev["mean"].data_ptr(), 0.0, prev["ggamma"].data_ptr(), prev["gbeta"].data_ptr(),
                    prev["rstd"].data_ptr(), st)
        else:
            self._c("vp_conv_dgrad", *dgrad, gin.data_ptr(), fc, L["dg_ws"].data_ptr(), L["dg_ws"].numel(), st)
        return gin

    def _layer_sgd(self, L, side, after, st):
        """Momentum SGD of this layer's conv weights as soon as its weight
        gradient exists and its dgrad (the last reader of W this step) has
        been issued: on the weight-gradient side stream, off the critical
        path.  Data parallel: the layer's gradient is all-reduced there first
        (bucket = one layer, overlapping the rest of the backward).  Pipeline
        stages keep the flat update of their stashed masters (sgd_into)."""
        if not self._sgd_in_backward:
            return
        pb = self.params
        off, shape = pb.offsets[L["name"] + ".w"]
        n = int(np.prod(shape))
        args = (pb.p.data_ptr() + 4 * off, pb.m.data_ptr() + 4 * off, pb.g.data_ptr() + 4 * off, n, float(self.lr),
                float(self.momentum), pb.pb.data_ptr() + 2 * off, n)
        if side is None:
            if self.grad_allreduce is not None:
                self.grad_allreduce(pb.g[off:off + n])
            self._c("vp_sgd_momentum", *args, st)
            return
        if after is not None:
            side.wait_event(after)
        with torch.cuda.stream(side):
            if self.grad_allreduce is not None:
                self.grad_allreduce(pb.g[off:off + n])
            self._c("vp_sgd_momentum", *args, side.cuda_stream)

    def _backward(self, st):
        prepared = False  # g already holds the masked gradient + BN statistics (fused producer)
        if self.last and self.bn_fuse:
            g = self._gm_buf(self.layers[-1])  # written by vp_sparse_head in the forward
            prepared = True
        elif self.last:
            last = self.levels[-1]
            C = self.planes[-1]
            g = self.gact[-1]
            self._c("vp_global_pool_backward", self.g_pooled.data_ptr(), last.coords.data_ptr(),
                    self.pool_counts.data_ptr(), last.n.data_ptr(), last.cap, C, g.data_ptr(), self.fcode, st)
        else:
            g = self.g_out_ext  # gradient of this stage's output, received from the next stage
        g2 = None  # pending identity-branch gradient for the current activation
        units = self.units[self.unit_range[0]:self.unit_range[1] + 1]
        # the layer whose activation feeds each layer (None: the engine's input)
        prev_of = {id(L): (self.layers[i - 1] if i > 0 else None) for i, L in enumerate(self.layers)}
        for u in reversed(units):
            Ls = u["layers"]
            if u["kind"] == "block":
                c1, c2 = Ls
                gid = self._gid(c2)
                # out = relu(bn2(conv2(h)) + idn): mask by out, identity grad -> gid
                # (prepared: the producer stored it there already); gh lives in
                # gact[lvl] and c1's dgrad overwrites it after use.  c2's dgrad
                # prepares c1's BN; c1's prepares the previous unit's output
                # layer, whose gradient joins this block's identity gradient.
                gh = self._bn_conv_backward(c2, g, g2, gid, st, prepared=prepared, prev=c1)
                gx = self._bn_conv_backward(c1, gh, None, None, st, prepared=self.bn_fuse, prev=prev_of[id(c1)],
                                            prev_add=gid)
                g, g2 = gx, gid
            elif u["kind"] == "down":
                g = self._bn_conv_backward(Ls[0], g, g2, None, st, prepared=prepared, prev=prev_of[id(Ls[0])])
                g2 = None
            else:  # stem: no input gradient
                self._bn_conv_backward(Ls[0], g, g2, None, st, need_dgrad=False, prepared=prepared)
                g = g2 = None
            # the next (earlier) unit's output layer was prepared by this unit's
            # first dgrad when that layer is inside this engine
            prepared = self.bn_fuse and prev_of[id(Ls[0])] is not None
            if prepared:
                g2 = None  # already folded into the prepared gradient
        if not self.first:
            if g2 is not None:
                g.add_(g2)  # the stage input fed both branches of its first block
            self.grad_input = g

    def _optimizer(self, st):
        pb = self.params
        self.join_side_streams()
        if self._sgd_in_backward:  # conv weights were updated layer by layer; BN + fc here
            rest = pb.size - pb.n_bf16
            if self.grad_allreduce is not None:
                self.grad_allreduce(pb.g[pb.n_bf16:])
            self._c("vp_sgd_momentum", pb.p.data_ptr() + 4 * pb.n_bf16, pb.m.data_ptr() + 4 * pb.n_bf16,
                    pb.g.data_ptr() + 4 * pb.n_bf16, rest, float(self.lr), float(self.momentum), None, 0, st)
            return
        if self.grad_allreduce is not None:
            self.grad_allreduce(pb.g)
        self._c("vp_sgd_momentum", pb.p.data_ptr(), pb.m.data_ptr(), pb.g.data_ptr(), pb.size, float(self.lr),
                float(self.momentum), pb.pb.data_ptr(), pb.n_bf16, st)

    def step_body(self):
        """One full training step on the current stream (graph-capturable)."""
        st = _lib.stream()
        self.launch_count = 0
        self._sgd_in_backward = self.layer_sgd
        try:
            self._integer_stage(st)
            self._forward(st)
            self._backward(st)
            self._optimizer(st)
        finally:
            self._sgd_in_backward = False

    def join_side_streams(self):
        """Join the side streams forked since the last join (a captured body
        may only wait on streams that joined its capture)."""
        if self.concurrent:
            main = torch.cuda.current_stream()
            for sd in self._all_streams:
                if id(sd) in self._forked:
                    main.wait_stream(sd)
        self._forked = set()

    def forward_body(self):
        """Pipeline stage forward (integer stage + this engine's layers [+ head])."""
        st = _lib.stream()
        self.launch_count = 0
        self._integer_stage(st)
        self._forward(st)
        self.join_side_streams()

    def backward_body(self):
        """Pipeline stage backward: gradients into params.g (and grad_input)."""
        st = _lib.stream()
        self.launch_count = 0
        self._backward(st)
        self.join_side_streams()

    def sgd_into(self, p, m, pb_shadow):
        """SGD with momentum of this engine's gradient into external master
        buffers (PipeDream weight stashing: the gradient computed with the
        stashed weights updates the latest weights)."""
        pb = self.params
        self._c("vp_sgd_momentum", p.data_ptr(), m.data_ptr(), pb.g.data_ptr(), pb.size, float(self.lr),
                float(self.momentum), pb_shadow.data_ptr(), pb.n_bf16, _lib.stream())

    # ------------------------------------------------------------------ prefetch
    _STATE_ATTRS = ("points", "labels", "levels", "feat0", "map_s1", "map_dn", "layers_all", "units", "layers")

    def _state(self):
        return {k: getattr(self, k) for k in self._STATE_ATTRS}

    def _use(self, state):
        for k, v in state.items():
            setattr(self, k, v)

    def enable_prefetch(self):
        """Double-buffer the integer stage: the coordinates and kernel maps of
        the NEXT batch (which depend only on its points, not on the weights)
        are built on their own streams while the current batch runs its
        backward pass, taking voxelization, the strided coordinate chain and
        the nine maps off the step's critical path.  Two copies of the
        integer-stage buffers (points, labels, levels, maps); the layer
        records of the second copy share every activation, gradient and
        parameter tensor with the first.  Whole-model engines only."""
        if not (self.first and self.last):
            raise ValueError("prefetch needs a whole-model engine")
        if self.states is not None:
            return
        a = self._state()
        dev = self.device
        levels = [Level(torch.zeros_like(lv.coords), torch.zeros_like(lv.n), lv.cap, lv.stride,
                        None if lv.seg is None else torch.zeros_like(lv.seg)) for lv in self.levels]
        lmap = dict(zip(map(id, self.levels), levels))

        def clone_map(m):
            m2 = self._alloc_map(lmap[id(m.src)], lmap[id(m.dst)], m.inv is not None, sort=m.perm is not None)
            return m2

        map_s1 = [clone_map(m) for m in self.map_s1]
        map_dn = [clone_map(m) for m in self.map_dn]
        mmap = dict(zip(map(id, self.map_s1 + self.map_dn), map_s1 + map_dn))
        layers_all = []
        for L in self.layers_all:
            L2 = dict(L)  # activations / params shared
            L2["src"], L2["dst"], L2["map"] = lmap[id(L["src"])], lmap[id(L["dst"])], mmap[id(L["map"])]
            layers_all.append(L2)
        units = self._unit_list(layers_all)
        b = dict(points=torch.zeros_like(self.points), labels=torch.zeros_like(self.labels), levels=levels,
                 feat0=torch.zeros_like(self.feat0), map_s1=map_s1, map_dn=map_dn, layers_all=layers_all,
                 units=units, layers=[L for u in units for L in u["layers"]])
        self.states = [a, a] if _DBG_SKIP_PREFETCH else [a, b]
        # the prefetched integer stage gets its own streams (the origin P
        # replaces the step's main stream; chain + two map streams)
        self.pf_stream = torch.cuda.Stream(device=dev)
        self.int_side = [torch.cuda.Stream(device=dev) for _ in range(3)]
        self._all_streams = list(self.side) + [self.pf_stream] + self.int_side
        self.prefetch = True
        self._phase = 0  # the state the next step trains on
        self.graphs = [None, None]

    def prefetch_body(self, cur: int):
        """One training step on state `cur` (its integer stage was built by
        the previous step) while the integer stage of state 1-cur is built
        concurrently with the backward pass."""
        st = _lib.stream()
        self.launch_count = 0
        self._use(self.states[cur])
        self.map_events = {}  # cur's maps were completed by the previous step
        main = torch.cuda.current_stream()
        P = self.pf_stream

        def fork():
            if _DBG_SKIP_PREFETCH:  # experiments only: no next-batch integer stage (never for results)
                return
            P.wait_stream(main)
            self._forked.add(id(P))
            self._use(self.states[1 - cur])
            with torch.cuda.stream(P):
                self._integer_stage(P.cuda_stream)
            self._use(self.states[cur])

        if self.PREFETCH_EARLY:  # concurrent with the forward as well
            fork()
        self._forward(st)
        if not self.PREFETCH_EARLY:
            fork()
        self._sgd_in_backward = self.layer_sgd
        try:
            self._backward(st)
            self._optimizer(st)
        finally:
            self._sgd_in_backward = False

    def prefetch_prologue(self):
        """Build the integer stage of the state the next step trains on."""
        self._use(self.states[self._phase])
        self._integer_stage(_lib.stream())
        self.join_side_streams()

    def prime(self, points: torch.Tensor, labels: torch.Tensor):
        """Prefetch mode: load the batch the next step trains on and build its
        integer stage now (the pipeline's fill)."""
        cur = self.states[self._phase]
        cur["points"].copy_(points, non_blocking=True)
        cur["labels"].copy_(labels, non_blocking=True)
        self.prefetch_prologue()

    # ------------------------------------------------------------------ public
    def set_batch(self, points: torch.Tensor, labels: torch.Tensor, non_blocking=True):
        """Stage a batch.  In prefetch mode it is the batch the NEXT step
        prefetches (its coordinates / maps are built during that step and it
        trains on the step after)."""
        if self.prefetch:
            nxt = self.states[1 - self._phase]
            nxt["points"].copy_(points, non_blocking=non_blocking)
            nxt["labels"].copy_(labels, non_blocking=non_blocking)
            return
        self.points.copy_(points, non_blocking=non_blocking)
        self.labels.copy_(labels, non_blocking=non_blocking)

    def capture(self, warmup: int = 1):
        """Record the step into a CUDA graph (after eager warm-up steps that
        populate the kernels' one-time attribute caches).  In prefetch mode
        two graphs (one per buffer phase) are recorded and alternate."""
        if self.prefetch:
            return self._capture_prefetch()
        s = torch.cuda.Stream(device=self.device)
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(warmup):
                self.step_body()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=self.main_stream):
            self.step_body()
        self.graph = g
        return g

    def _capture_prefetch(self):
        """Warm up and record both phases.  Trains two warm-up steps (on the
        primed batch, then on the staged one) and leaves the pipeline primed
        with the staged batch again (phase 0)."""
        s = torch.cuda.Stream(device=self.device)
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self._phase = 0
            self.prefetch_prologue()
            for ph in (0, 1):  # eager warm-up of both phases (ends with state 0 prefetched)
                self.prefetch_body(ph)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        lib = _lib.load()
        for ph in (0, 1):
            k0 = lib.vp_kernel_launches()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=self.main_stream):
                self.prefetch_body(ph)
            self.graphs[ph] = g
            self.kernels_per_step = lib.vp_kernel_launches() - k0
        self._phase = 0
        self.graph = self.graphs[0]
        return self.graphs

    def step(self):
        if self.prefetch:
            if self.graphs[self._phase] is not None:
                self.graphs[self._phase].replay()
            else:
                self.prefetch_body(self._phase)
            self._phase = 1 - self._phase
            return
        if self.graph is not None:
            self.graph.replay()
        else:
            self.step_body()

    def train_step_from_host(self, points_np, offsets_np, labels_np) -> float:
        """End-to-end convenience call: host points -> device, one step, loss."""
        pts = torch.as_tensor(np.ascontiguousarray(points_np)).to(self.points.dtype)
        if pts.shape[0] != self.cap:
            raise ValueError("point count must equal batch * points")
        offs = np.asarray(offsets_np)
        if not np.array_equal(offs, np.arange(self.B + 1) * self.P):
            raise ValueError("fixed-size clouds expected (offsets = arange(B+1) * points)")
        self.set_batch(pts.to(self.device), torch.as_tensor(np.asarray(labels_np), dtype=torch.int32).to(self.device))
        self.step()
        return float(self.loss.item())

    def profile_layers(self, iters: int = 20, warmup: int = 3) -> list[dict]:
        """SmartProfile on the GPU (profiling.py:416-455): per
        conv layer, CUDA-event device time of its forward (conv + BN stats +
        BN apply) and of its backward split into BN backward, dgrad and wgrad,
        each timed alone on one stream (eager, non-concurrent) on the current
        batch.  Also the activation bytes a pipeline cut after the layer sends
        (coords int32 [N,4] + bf16 feats [N,C]) and the fp32
        parameter bytes.  Returns one dict per layer in layer order."""
        conc = self.concurrent
        self.concurrent = False
        try:
            st = _lib.stream()
            self._integer_stage(st)
            self._forward(st)
            self._backward(st)
            torch.cuda.synchronize()
            esz = 2 if self.fdt == BF16 else 4

            def timed(fn):
                for _ in range(warmup):
                    fn()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for _ in range(iters):
                    fn()
                b.record()
                b.synchronize()
                return a.elapsed_time(b) * 1e3 / iters

            out = []
            for L in self.layers:
                x = L["x"]
                res = L["a"] if L["kind"] == "c2" else None  # any same-shape buffer: cost only
                n_out = int(L["dst"].n.item())
                fwd = timed(lambda: self._conv_bn(L, x, res, True, st))
                bn_b = timed(lambda: self._c(
                    "vp_bn_backward", L["gy"].data_ptr(), None, self.fcode, L["a"].data_ptr(), self.fcode,
                    L["y"].data_ptr(), self.fcode, L["dst"].n.data_ptr(), L["dst"].cap, L["cout"],
                    L["mean"].data_ptr(), L["rstd"].data_ptr(), L["gamma"].data_ptr(), 1, L["gy"].data_ptr(),
                    self.fcode, None, L["ggamma"].data_ptr(), L["gbeta"].data_ptr(), L["bn_ws"].data_ptr(),
                    L["bn_ws"].numel(), st))
                m, fc = L["map"], self.fcode
                wg = timed(lambda: self._c(
                    "vp_conv_wgrad", x.data_ptr(), fc, L["cin"], L["gy"].data_ptr(), fc, L["cout"], self.K,
                    m.pin.data_ptr(), m.pout.data_ptr(), m.ptr.data_ptr(), m.pin.numel(), L["gw"].data_ptr(),
                    L["wg_ws"].data_ptr(), L["wg_ws"].numel(), st))
                dg = 0.0
                if L["kind"] != "stem":
                    src = L["src"]
                    gin = self.gact[self.levels.index(src)]
                    table, flip, perm = self.dgrad_table(L)
                    dg = timed(lambda: self._c(
                        "vp_conv_dgrad", L["gy"].data_ptr(), fc, L["gy"].shape[0], L["cout"], L["wb"].data_ptr(),
                        L["wcode"], L["cin"], self.K, table.data_ptr(), flip, _lib.ptr(perm), src.n.data_ptr(), src.cap,
                        gin.data_ptr(), fc, L["dg_ws"].data_ptr(), L["dg_ws"].numel(), st))
                pairs = int(m.ptr[-1].item())
                out.append({"name": L["name"], "cin": L["cin"], "cout": L["cout"], "n_out": n_out, "pairs": pairs,
                            "fwd_us": fwd, "bn_bwd_us": bn_b, "dgrad_us": dg, "wgrad_us": wg,
                            "bwd_us": bn_b + dg + wg, "gflop_fwd": 2.0 * pairs * L["cin"] * L["cout"] / 1e9,
                            "activation_bytes": n_out * (16 + esz * L["cout"]),
                            "param_bytes": 4 * (self.K * L["cin"] * L["cout"] + 2 * L["cout"])})
            return out  # activations/gradients are scratch now: profile on a dedicated trainer
        finally:
            self.concurrent = conc

    def level_sizes(self) -> list[int]:
        return [int(l.n.item()) for l in self.levels]

    def pair_counts(self) -> list[int]:
        return [int(m.ptr[-1].item()) for m in self.map_s1 + self.map_dn]
