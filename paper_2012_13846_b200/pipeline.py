"""SparsePipe pipeline runtime on B200 (schedule
semantics SPEC.md:386-412,433): the SparseResNet cut into contiguous stages by
the partitioner (partition.py, fed by per-unit GPU profiles), one process per
GPU, micro-batches flowing between stages as (coords, features) sparse tensors
over NCCL P2P on NVLink, PipeDream 1F1B with weight stashing, and replicated
stages with round-robin micro-batch routing plus an intra-group all_reduce.

The reference ships none of this as code: the paper ran PipeDream
over Gloo.  Parity is self-defined: tests/test_pipeline.py checks the
schedule's invariants on CPU with the gloo backend, and
tests/test_gpu_pipeline.py checks on the GPU that a pipelined run equals an
emulation of the same weight-version semantics on the single-GPU engine.

Wire format per micro-batch — the analogue of the reference's binary
sparse-tensor format (tensor.py:270-301: header, then coords, then
features), live rows only:
  forward (stage s -> s+1), on the forward-direction communicator:
    header  int32 [4]          (n, C, tensor_stride, B) — sent alone first; the
                               receiver reads it, then posts the payload
    coords  int32 [n, 4]       rows [batch, x, y, z] of the cut level
    feats   bf16  [n, C]       activation of the last unit of stage s
    labels  int32 [B]          class labels travel with the clouds
  backward (s+1 -> s), on the backward-direction communicator:
    grad    bf16  [n, C]       n known to both sides from the forward header
Receivers keep capacity-sized buffers; only 16 + 16 n + 2 n C + 4 B bytes
(forward) and 2 n C bytes (backward) cross NVLink.  Activations and
gradients use separate communicators, so sends are posted and left in flight
(waited only before their buffer is rewritten) while receives are waited in
stream order right before the compute that consumes them: F(mb)'s send never
gates B(mb').
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, Optional

from .errors import StructuralError, ValidationError


# ---------------------------------------------------------------- topology
@dataclass(frozen=True)
class StageSpec:
    """One pipeline stage: inclusive unit range and the ranks replicating it."""

    unit_start: int
    unit_end: int
    ranks: tuple


@dataclass(frozen=True)
class Topology:
    stages: tuple  # of StageSpec

    @classmethod
    def from_plan(cls, plan, rank_of: Optional[dict] = None) -> "Topology":
        """PartitionPlan (partition.py) -> stages over ranks.  Processor ids
        map to ranks through `rank_of` (default: their order in the plan)."""
        stages, nxt = [], 0
        for s in plan.stages:
            if rank_of is None:
                ranks = tuple(range(nxt, nxt + len(s.assigned_processors)))
                nxt += len(ranks)
            else:
                ranks = tuple(rank_of[p] for p in s.assigned_processors)
            stages.append(StageSpec(s.layer_start, s.layer_end, ranks))
        return cls(tuple(stages))

    @classmethod
    def even(cls, n_units: int, cuts: list, replicas: Optional[list] = None) -> "Topology":
        """Stages ending after the given units; replicas[s] ranks each."""
        ends = list(cuts) + [n_units - 1]
        reps = replicas or [1] * len(ends)
        st, start, r = [], 0, 0
        for e, m in zip(ends, reps):
            st.append(StageSpec(start, e, tuple(range(r, r + m))))
            start, r = e + 1, r + m
        return cls(tuple(st))

    @property
    def world(self) -> int:
        return sum(len(s.ranks) for s in self.stages)

    def mb_multiple(self) -> int:
        """Micro-batch counts must be multiples of every stage's replica count:
        replicas all-reduce once per backward round, so a short round would
        leave a collective without partners."""
        m = 1
        for s in self.stages:
            m = m * len(s.ranks) // math.gcd(m, len(s.ranks))
        return m

    def locate(self, rank: int):
        """-> (stage index, replica index) of a rank, or None if idle."""
        for i, s in enumerate(self.stages):
            if rank in s.ranks:
                return i, s.ranks.index(rank)
        return None

    def validate(self, n_units: int) -> None:
        nxt, seen = 0, set()
        for s in self.stages:
            if s.unit_start != nxt or s.unit_end < s.unit_start or not s.ranks:
                raise StructuralError("stages must cover the units contiguously with >= 1 rank each")
            if seen & set(s.ranks):
                raise StructuralError("a rank may serve only one stage")
            seen |= set(s.ranks)
            nxt = s.unit_end + 1
        if nxt != n_units:
            raise StructuralError("stages do not cover every unit")


def route_replica(minibatch_id: int, replica_count: int) -> int:
    """deterministic round robin; backward follows forward."""
    if replica_count < 1:
        raise ValidationError("replica_count must be >= 1")
    return minibatch_id % replica_count


# ---------------------------------------------------------------- schedule
@dataclass(frozen=True)
class Comm:
    kind: str  # "send_fwd" | "recv_fwd" | "send_bwd" | "recv_bwd"
    mb: int
    peer: int  # rank


@dataclass(frozen=True)
class Action:
    """One step of a rank's program: communications posted together (one
    NCCL group) before the compute, then the compute F(mb) / B(mb), or a
    communication-only step (op == "comm")."""

    op: str  # "F" | "B" | "comm"
    mb: int
    comms: tuple = ()


def local_microbatches(n_mb: int, n_replicas: int, replica: int) -> list:
    return [i for i in range(n_mb) if route_replica(i, n_replicas) == replica]


def schedule_1f1b(topo: Topology, rank: int, n_mb: int) -> list:
    """PipeDream 1F1B program of one rank over micro-batches 0..n_mb-1
    (stage s admits S - s forwards before its first
    backward).  Communications are grouped the Megatron way — the send of an
    activation goes out together with the receive of a gradient and vice
    versa — so paired ranks never wait on each other's unposted operation."""
    loc = topo.locate(rank)
    if loc is None:
        return []
    s, r = loc
    S = len(topo.stages)
    st = topo.stages[s]
    mbs = local_microbatches(n_mb, len(st.ranks), r)
    M = len(mbs)
    W = min(S - s - 1, M)

    def peer(stage, mb):
        ranks = topo.stages[stage].ranks
        return ranks[route_replica(mb, len(ranks))]

    def recv_fwd(mb):
        return Comm("recv_fwd", mb, peer(s - 1, mb)) if s > 0 else None

    def send_fwd(mb):
        return Comm("send_fwd", mb, peer(s + 1, mb)) if s < S - 1 else None

    def recv_bwd(mb):
        return Comm("recv_bwd", mb, peer(s + 1, mb)) if s < S - 1 else None

    def send_bwd(mb):
        return Comm("send_bwd", mb, peer(s - 1, mb)) if s > 0 else None

    def grp(*cs):
        return tuple(c for c in cs if c is not None)

    prog = []
    for i in range(W):
        prog.append(Action("F", mbs[i], grp(recv_fwd(mbs[i]))))
        prog.append(Action("comm", mbs[i], grp(send_fwd(mbs[i]))))
    R = M - W
    pending = grp(recv_fwd(mbs[W])) if R > 0 else ()
    for j in range(R):
        f, b = mbs[W + j], mbs[j]
        prog.append(Action("F", f, pending))
        prog.append(Action("B", b, grp(send_fwd(f), recv_bwd(b))))
        pending = grp(send_bwd(b), recv_fwd(mbs[W + j + 1])) if j < R - 1 else grp(send_bwd(b))
    if R > 0:
        prog.append(Action("comm", mbs[M - 1], pending))
    for j in range(R, M):
        b = mbs[j]
        prog.append(Action("B", b, grp(recv_bwd(b))))
        prog.append(Action("comm", b, grp(send_bwd(b))))
    return [a for a in prog if a.op != "comm" or a.comms]


def simulate_versions(topo: Topology, n_mb: int, stash: bool = True) -> list:
    """Weight-version audit without running anything: for
    every (mb, stage) the number of updates the stage's replica had applied
    when F(mb) ran and when B(mb) ran.  With stashing B uses F's weights;
    without it B sees the latest weights.  Replicated stages all-reduce, so
    one update = one backward per replica."""
    out = []
    for s, st in enumerate(topo.stages):
        for r, rank in enumerate(st.ranks):
            version, fwd_v = 0, {}
            for a in schedule_1f1b(topo, rank, n_mb):
                if a.op == "F":
                    fwd_v[a.mb] = version
                elif a.op == "B":
                    out.append((a.mb, s, fwd_v[a.mb], fwd_v[a.mb] if stash else version))
                    version += 1
    return sorted(out)


# ---------------------------------------------------------------- transport
def boundary_tensors(e, kind: str) -> list:
    """Capacity-sized tensors behind one communication of `kind` for engine
    e (LocalTransport moves them whole; DistTransport sends live rows)."""
    if kind == "send_fwd":
        lv = e.levels[e.exit_level]
        return [lv.n, lv.coords, e.out_act, e.labels]
    if kind == "recv_fwd":
        lv = e.levels[e.entry_level]
        return [lv.n, lv.coords, e.x_in, e.labels]
    if kind == "send_bwd":
        return [e.grad_input]
    return [e.g_out_ext]  # recv_bwd


class DistTransport:
    """torch.distributed P2P (NCCL on B200 over NVLink/NVSwitch; gloo for the
    CPU tests) with the header-first live-size wire format of the module
    docstring.  Two extra communicators over the whole world carry the
    forward (activation) and backward (gradient) directions; replica groups
    carry the gradient all_reduce."""

    def __init__(self, dist, topo: Optional["Topology"] = None, host_stage: bool = False):
        """Creating a process group is collective over the whole world, so
        every rank builds the direction communicators and every replica
        group of `topo` up front, in the same order.  host_stage: move device
        tensors through host memory (gloo with several ranks on one GPU — a
        functional test of the runtime where NCCL cannot run two ranks per
        device)."""
        self.dist = dist
        self.host_stage = host_stage
        self._groups = {}
        world = list(range(dist.get_world_size()))
        self.g_fwd = dist.new_group(world)
        self.g_bwd = dist.new_group(world)
        if topo is not None:
            for st in topo.stages:
                if len(st.ranks) > 1:
                    self._groups[tuple(st.ranks)] = dist.new_group(list(st.ranks))
        self.bytes_sent = 0
        self.messages = 0

    # -- point to point ------------------------------------------------------
    def _send(self, runner, slot, t, peer, group):
        keep = t
        if self.host_stage and t.is_cuda:
            keep = t.cpu()
        w = self.dist.isend(keep, peer, group=group)
        runner.pending_sends.setdefault(slot, []).append((w, keep))
        self.bytes_sent += t.numel() * t.element_size()
        self.messages += 1

    def _recv(self, t, peer, group):
        """Blocking-in-stream-order receive into t (a contiguous view)."""
        if self.host_stage and t.is_cuda:
            h = torch_empty_like_host(t)
            self.dist.irecv(h, peer, group=group).wait()
            t.copy_(h)
            return
        self.dist.irecv(t, peer, group=group).wait()

    def exchange(self, runner, comms) -> None:
        import torch

        for c in comms:
            e = runner.engine_of(c.mb)
            slot = runner.slot_of[c.mb]
            if c.kind == "send_fwd":
                lv = e.levels[e.exit_level]
                n = int(lv.n.item())  # the stage's forward has produced the cut level
                C = e.out_act.shape[1]
                runner.wire_rows[(c.mb, "out")] = n
                hdr = torch.tensor([n, C, int(getattr(lv, "stride", 1)), e.labels.numel()], dtype=torch.int32,
                                   device=lv.n.device)
                for t in (hdr, lv.coords[:n], e.out_act[:n], e.labels):
                    self._send(runner, slot, t, c.peer, self.g_fwd)
            elif c.kind == "recv_fwd":
                lv = e.levels[e.entry_level]
                hdr = torch.empty(4, dtype=torch.int32, device=lv.n.device)
                self._recv(hdr, c.peer, self.g_fwd)
                n, C, _ts, B = (int(v) for v in hdr.tolist())
                if n > lv.coords.shape[0] or C != e.x_in.shape[1] or B != e.labels.numel():
                    raise StructuralError(f"pipeline header {(n, C, B)} does not fit the stage input "
                                          f"(cap {lv.coords.shape[0]}, C {e.x_in.shape[1]}, B {e.labels.numel()})")
                runner.wire_rows[(c.mb, "in")] = n
                lv.n.fill_(n)
                for t in (lv.coords[:n], e.x_in[:n], e.labels):
                    self._recv(t, c.peer, self.g_fwd)
            elif c.kind == "send_bwd":
                n = runner.wire_rows[(c.mb, "in")]
                self._send(runner, slot, e.grad_input[:n].contiguous(), c.peer, self.g_bwd)
            else:  # recv_bwd
                n = runner.wire_rows[(c.mb, "out")]
                self._recv(e.g_out_ext[:n], c.peer, self.g_bwd)

    def wait_sends(self, runner, slot=None) -> None:
        """Complete the in-flight sends of one slot (before its buffers are
        rewritten) or of all slots."""
        slots = list(runner.pending_sends) if slot is None else [slot]
        for s in slots:
            for w, _ in runner.pending_sends.pop(s, []):
                w.wait()

    # -- replica groups ------------------------------------------------------
    def group(self, ranks: tuple):
        if len(ranks) <= 1:
            return None
        if tuple(ranks) not in self._groups:
            raise StructuralError("replica group not created: pass the topology to DistTransport on every rank")
        return self._groups[tuple(ranks)]

    def allreduce_mean(self, t, group) -> None:
        if group is None:
            return
        if self.host_stage and t.is_cuda:
            h = t.cpu()
            self.dist.all_reduce(h, group=group)
            t.copy_(h.div_(self.dist.get_world_size(group)))
            return
        self.dist.all_reduce(t, group=group)
        t.div_(self.dist.get_world_size(group))


def torch_empty_like_host(t):
    import torch

    return torch.empty(t.shape, dtype=t.dtype, device="cpu")


class LocalTransport:
    """Every rank in ONE process (single-GPU validation of the stage
    engines and the schedule): a send copies its tensors into a mailbox
    keyed by (src, dst, kind, mb); the matching receive copies them out.
    Replica-group all_reduce averages the gradients of the group's ranks
    once all of them have posted theirs."""

    def __init__(self):
        self.box = {}
        self.posted = set()

    def post_sends(self, runner, comms) -> bool:
        """Post the group's sends (once each); True if anything new was posted."""
        new = False
        for c in comms:
            if c.kind.startswith("send"):
                key = (runner.rank, c.peer, c.kind, c.mb)
                if key not in self.posted:
                    self.posted.add(key)
                    self.box[key] = [t.clone() for t in boundary_tensors(runner.engine_of(c.mb), c.kind)]
                    new = True
        return new

    def recvs_ready(self, runner, comms) -> bool:
        return all((c.peer, runner.rank, c.kind.replace("recv", "send"), c.mb) in self.box
                   for c in comms if c.kind.startswith("recv"))

    def take_recvs(self, runner, comms) -> None:
        for c in comms:
            if c.kind.startswith("recv"):
                src = self.box.pop((c.peer, runner.rank, c.kind.replace("recv", "send"), c.mb))
                for d, t in zip(boundary_tensors(runner.engine_of(c.mb), c.kind), src):
                    d.copy_(t)

    def exchange(self, runner, comms) -> None:
        self.post_sends(runner, comms)
        if not self.recvs_ready(runner, comms):
            raise StructuralError("local transport: receive before its send")
        self.take_recvs(runner, comms)

    def group(self, ranks: tuple):
        return tuple(ranks) if len(ranks) > 1 else None

    def wait_sends(self, runner, slot=None) -> None:  # sends are copies: complete when posted
        return None

    def allreduce_mean(self, t, group) -> None:
        raise StructuralError("replicated stages in LocalPipeline reduce through LocalPipeline")


# ---------------------------------------------------------------- stage runner
@dataclass
class StageStats:
    forwards: int = 0
    backwards: int = 0
    audit: list = field(default_factory=list)  # (mb, stage, fwd_version, bwd_version)
    losses: dict = field(default_factory=dict)


class StageRunner:
    """Executes one rank's 1F1B program on a stage engine.

    Slots: the rank keeps `depth` in-flight micro-batches (its warm-up depth
    + 1); each slot is an engine (SparseResNetTrainer restricted to the
    stage's units) with its own activations, kernel maps and its own copy of
    the weights — the PipeDream weight stash: at F(mb) the slot's weights are
    refreshed from the stage's master weights, B(mb) computes gradients with
    exactly those weights, and the gradient updates the master (SGD with
    momentum) — so fwd_version == bwd_version for every (mb, stage).  With
    stash=False the slot is refreshed again before B (the §III-A staleness
    the stash removes), for the audit test.

    `make_engine(units)` builds an engine; `batch_of(mb)` returns (points,
    labels) device tensors for the first stage."""

    def __init__(self, topo: Topology, rank: int, n_mb: int, make_engine: Callable, batch_of: Callable,
                 transport, stash: bool = True, use_graphs: bool = False):
        import torch

        if n_mb % topo.mb_multiple():
            raise ValidationError(f"{n_mb} micro-batches: must be a multiple of {topo.mb_multiple()} (the replica "
                                  "counts' lcm) so every replica group all-reduces the same number of rounds")
        self.topo, self.rank, self.n_mb = topo, rank, n_mb
        self.stage, self.replica = topo.locate(rank)
        self.S = len(topo.stages)
        st = topo.stages[self.stage]
        self.spec = st
        self.program = schedule_1f1b(topo, rank, n_mb)
        n_local = len(local_microbatches(n_mb, len(st.ranks), self.replica))
        depth = max(1, min(self.S - self.stage, n_local))
        self.slots = [make_engine((st.unit_start, st.unit_end)) for _ in range(depth)]
        e0 = self.slots[0]
        self.first, self.last = e0.first, e0.last
        # master weights (fp32 + bf16 shadow) and momentum
        self.master_p = e0.params.p.clone()
        self.master_pb = e0.params.pb.clone()
        self.master_m = torch.zeros_like(self.master_p)
        self.version = 0
        self.batch_of = batch_of
        self.tr = transport
        self.stash = stash
        self.group = transport.group(st.ranks)
        self.stats = StageStats()
        self.slot_of = {}
        self.slot_version = [None] * depth
        self.use_graphs = use_graphs
        self.graphs = {}
        self._next_slot = 0
        self.pending_sends = {}  # slot -> [(work, buffer)] still in flight
        self.wire_rows = {}  # (mb, "in" | "out") -> live rows of the boundary level

    def engine_of(self, mb):
        return self.slots[self.slot_of[mb]]

    def prepare(self, a: Action):
        """Bind F(mb) to the next slot (round robin over the in-flight depth)."""
        if a.op == "F" and a.mb not in self.slot_of:
            self.slot_of[a.mb] = self._next_slot % len(self.slots)
            self._next_slot += 1

    def _refresh(self, e):
        e.params.p.copy_(self.master_p)
        e.params.pb.copy_(self.master_pb)

    def _run(self, e, which):
        import torch

        body = e.forward_body if which == "F" else e.backward_body
        if not self.use_graphs:
            body()
            return
        key = (id(e), which)
        g = self.graphs.get(key)
        if g is None:
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                body()
            torch.cuda.current_stream().wait_stream(s)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                body()
            self.graphs[key] = g
        g.replay()

    def compute(self, a: Action):
        if a.op == "F":
            self.forward(a)
        elif a.op == "B":
            self.backward_grad(a)
            if self.group is not None:
                self.tr.allreduce_mean(self.engine_of(a.mb).params.g, self.group)
            self.finish_backward(a)

    def forward(self, a: Action):
        e = self.engine_of(a.mb)
        self.tr.wait_sends(self, self.slot_of[a.mb])  # this slot's previous sends read the buffers F rewrites
        self._refresh(e)
        self.slot_version[self.slot_of[a.mb]] = self.version
        if self.first:
            pts, lab = self.batch_of(a.mb)
            e.set_batch(pts, lab)
        self._run(e, "F")
        self.stats.forwards += 1
        if self.last:
            self.stats.losses[a.mb] = e.loss.clone()

    def backward_grad(self, a: Action):
        e = self.engine_of(a.mb)
        self.tr.wait_sends(self, self.slot_of[a.mb])
        if not self.stash:
            self._refresh(e)
        self._run(e, "B")

    def finish_backward(self, a: Action):
        """Apply the (group-averaged) gradient to the master weights."""
        e = self.engine_of(a.mb)
        fwd_v = self.slot_version[self.slot_of[a.mb]]
        e.sgd_into(self.master_p, self.master_m, self.master_pb)
        self.stats.audit.append((a.mb, self.stage, fwd_v, fwd_v if self.stash else self.version))
        self.version += 1
        self.stats.backwards += 1

    def execute(self, a: Action):
        self.prepare(a)
        self.tr.exchange(self, a.comms)
        self.compute(a)

    def run(self):
        for a in self.program:
            self.execute(a)
        self.tr.wait_sends(self)
        return self.stats


class LocalPipeline:
    """All ranks of a topology in one process on one device, each a
    StageRunner over one LocalTransport, interleaved in a dependency
    -respecting order: a rank reaching an action posts the action's sends,
    and runs it once every receive of the group has its matching send.
    Replica groups average their gradients when all members reached the
    same backward.  Executes exactly the per-rank programs the multi-GPU
    runtime executes."""

    def __init__(self, topo: Topology, n_mb: int, make_engine, batch_of, stash=True, use_graphs=False):
        self.tr = LocalTransport()
        self.topo = topo
        ranks = [r for s in topo.stages for r in s.ranks]
        self.runners = {r: StageRunner(topo, r, n_mb, make_engine, batch_of, self.tr, stash, use_graphs)
                        for r in ranks}
        self.pc = {r: 0 for r in ranks}

    def run(self):
        import torch

        waiting = {}  # replicated stage -> {rank: action} whose gradient awaits the group mean
        progress = True
        while progress:
            progress = False
            for r, run in self.runners.items():
                prog = run.program
                while self.pc[r] < len(prog) and r not in waiting.get(run.stage, {}):
                    a = prog[self.pc[r]]
                    run.prepare(a)
                    if self.tr.post_sends(run, a.comms):
                        progress = True
                    if not self.tr.recvs_ready(run, a.comms):
                        break
                    self.tr.take_recvs(run, a.comms)
                    self.pc[r] += 1
                    progress = True
                    if a.op == "F":
                        run.forward(a)
                    elif a.op == "B":
                        run.backward_grad(a)
                        if run.group is None:
                            run.finish_backward(a)
                        else:
                            box = waiting.setdefault(run.stage, {})
                            box[r] = a
                            if len(box) == len(run.group):  # every replica reached this round
                                grads = [self.runners[rr].engine_of(aa.mb).params.g for rr, aa in sorted(box.items())]
                                mean = torch.stack(grads).mean(0)
                                for rr, aa in sorted(box.items()):
                                    self.runners[rr].engine_of(aa.mb).params.g.copy_(mean)
                                    self.runners[rr].finish_backward(aa)
                                waiting[run.stage] = {}
        stuck = {r: self.pc[r] for r, run in self.runners.items() if self.pc[r] < len(run.program)}
        if stuck or any(waiting.values()):
            raise StructuralError(f"pipeline deadlock: ranks stuck at {stuck}")
        return {r: run.stats for r, run in self.runners.items()}


# ---------------------------------------------------------------- planning
def unit_profile(engine, records: list, model_name: str, processor_type: str = "B200"):
    """Per-layer GPU records (SparseResNetTrainer.profile_layers) -> the
    reference's ProfileSet over pipeline units (profiling.py:43-105): times
    and parameter bytes summed over the unit's convs, activation bytes of the
    unit's output (what a cut after it sends: coords + bf16 features)."""
    from .partition import LayerProfile, ProfileSet

    by_name = {r["name"]: r for r in records}
    recs = []
    for u in engine.units:
        rs = [by_name[L["name"]] for L in u["layers"]]
        recs.append(LayerProfile(u["index"], sum(r["fwd_us"] for r in rs), sum(r["bwd_us"] for r in rs),
                                 float(rs[-1]["activation_bytes"]), float(sum(r["param_bytes"] for r in rs))))
    return ProfileSet(model_name, engine.B, {processor_type: recs})


def plan_topology(profiles, n_gpus: int, bandwidth: float, max_stages: Optional[int] = None):
    """SparsePipe partition of the units over n homogeneous GPUs (Eq. 5) ->
    (PartitionPlan, Topology)."""
    from .partition import ClusterSpec, plan

    cluster = ClusterSpec.homogeneous(n_gpus, next(iter(profiles.profiles)), bandwidth)
    p = plan(profiles, cluster, max_stages=max_stages)
    rank_of = {proc.instance_id: i for i, proc in enumerate(cluster.processors)}
    return p, Topology.from_plan(p, rank_of)
