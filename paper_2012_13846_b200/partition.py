"""SparsePipe heterogeneity-aware pipeline partitioner (PAPER.md:252-322,
Eq. 4/5, Algorithm 1/2; behavioural spec SPEC.md:270-362).

The reference ships this module as specification only, so the restatement is
pinned by the SPEC's worked examples and properties (tests/test_partition.py)
and by an exhaustive brute-force oracle over the same search space.

Inputs are the reference's interchange formats (profiling.py:28-323): a
per-processor-type layer profile (fwd/bwd µs, activation/param bytes,
`format_version` 1) and a cluster spec (processors + bandwidth bytes/s).  On
B200 the profile comes from `profile_layers()` in pipeline.py — per-unit CUDA
-event timings of this repo's own kernels — which is the "measured per-layer
GPU cost" the north_star asks the partitioner to be fed with.

Objective (Eq. 5):  C(i, j, S) = min( Q(i, j, S),
    min_{i<=k<j, split of S into prefix S1 / suffix S2}
        max( C(i, k, S1), a_k / BW, Q(k+1, j, S2) ) )
with Eq. 4   Q(i, j, S) = ( max_{a in S} sum_{l=i..j} t_a^l
                            + 2 (m-1) sum_{l=i..j} p^l / BW ) / m.
Processor subsets are contiguous segments of the capability-sorted list
("limited to O(n)"); the last stage takes the suffix
(SPEC.md:361).  Prefix sizes m <= M are all tried (idle processors allowed,
SPEC.md:352), both sort orders are evaluated, and ties prefer
fewer stages, then less inter-stage activation traffic.
"""
from __future__ import annotations

import itertools
import json
import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from .errors import ConfigError, StructuralError, ValidationError

FORMAT_VERSION = 1
_REL_TIE = 1e-12


# ---------------------------------------------------------------- formats
@dataclass(frozen=True)
class LayerProfile:
    """profiling.py:43-66 — one layer's fwd/bwd µs and activation/param bytes."""

    layer_id: int
    fwd_time_us: float
    bwd_time_us: float
    activation_bytes: float
    param_bytes: float

    def __post_init__(self):
        vals = (self.fwd_time_us, self.bwd_time_us, self.activation_bytes, self.param_bytes)
        if any(not math.isfinite(v) or v < 0 for v in vals):
            raise ValidationError("layer profile fields must be finite and >= 0")
        if self.layer_id < 0:
            raise ValidationError("layer_id must be >= 0")

    def total_time_us(self) -> float:
        return self.fwd_time_us + self.bwd_time_us


@dataclass
class ProfileSet:
    """profiling.py:69-157 — per-processor-type profiles of one model; sizes
    must agree across types (they are model properties)."""

    model_name: str
    batch_size: int
    profiles: dict = field(default_factory=dict)

    def __post_init__(self):
        if not self.profiles:
            raise StructuralError("profile set lists no processor types")
        names = list(self.profiles)
        ref = self.profiles[names[0]]
        if not ref:
            raise StructuralError("profile set lists no layers")
        for t in names:
            recs = self.profiles[t]
            if len(recs) != len(ref):
                raise StructuralError(f"processor type {t!r} lists {len(recs)} layers, {names[0]!r} {len(ref)}")
            for i, r in enumerate(recs):
                if r.layer_id != i:
                    raise StructuralError(f"layer ids must be 0..L-1 in order; got {r.layer_id} at {i}")
                if r.activation_bytes != ref[i].activation_bytes or r.param_bytes != ref[i].param_bytes:
                    raise StructuralError(f"layer {i}: sizes differ between {t!r} and {names[0]!r}")

    @property
    def num_layers(self) -> int:
        return len(next(iter(self.profiles.values())))

    def layer_times_s(self, type_name: str) -> np.ndarray:
        if type_name not in self.profiles:
            raise ConfigError(f"processor type {type_name!r} not profiled")
        return np.array([r.total_time_us() * 1e-6 for r in self.profiles[type_name]])

    def activation_bytes(self) -> np.ndarray:
        return np.array([r.activation_bytes for r in next(iter(self.profiles.values()))])

    def param_bytes(self) -> np.ndarray:
        return np.array([r.param_bytes for r in next(iter(self.profiles.values()))])

    def merged_with(self, other: "ProfileSet") -> "ProfileSet":
        if other.model_name != self.model_name or other.batch_size != self.batch_size:
            raise StructuralError("cannot merge profiles of different models or batch sizes")
        if set(self.profiles) & set(other.profiles):
            raise StructuralError("duplicate processor types")
        return ProfileSet(self.model_name, self.batch_size, {**self.profiles, **other.profiles})


def profile_to_json(pset: ProfileSet, type_name: str) -> str:
    """The reference profile file (profiling.py:160-179)."""
    return json.dumps({
        "format_version": FORMAT_VERSION, "model_name": pset.model_name, "batch_size": pset.batch_size,
        "processor_type": type_name,
        "layers": [{"layer_id": r.layer_id, "fwd_time_us": r.fwd_time_us, "bwd_time_us": r.bwd_time_us,
                    "activation_bytes": r.activation_bytes, "param_bytes": r.param_bytes}
                   for r in pset.profiles[type_name]]}, indent=2, sort_keys=True)


def profile_from_json(text: str, bwd_fwd_ratio: float = 2.0) -> ProfileSet:
    """profiling.py:182-231 — a record may carry total_time_us only, split
    by the bwd:fwd ratio (default 2)."""
    try:
        obj = json.loads(text)
    except json.JSONDecodeError as exc:
        raise ValidationError(f"profile file is not valid JSON: {exc}") from exc
    try:
        if int(obj.get("format_version", -1)) != FORMAT_VERSION:
            raise ValidationError("unsupported or missing profile format_version")
        recs = []
        for r in obj["layers"]:
            if "total_time_us" in r and "fwd_time_us" not in r:
                tot = float(r["total_time_us"])
                fwd = tot / (1.0 + bwd_fwd_ratio)
                bwd = tot - fwd
            else:
                fwd, bwd = float(r["fwd_time_us"]), float(r["bwd_time_us"])
            recs.append(LayerProfile(int(r["layer_id"]), fwd, bwd, float(r["activation_bytes"]),
                                     float(r["param_bytes"])))
        return ProfileSet(str(obj["model_name"]), int(obj["batch_size"]), {str(obj["processor_type"]): recs})
    except (KeyError, TypeError, ValueError) as exc:
        raise ValidationError(f"malformed profile file: {exc}") from exc


@dataclass(frozen=True)
class Processor:
    instance_id: str
    type_name: str


@dataclass
class ClusterSpec:
    """profiling.py:242-283 — processors + one bandwidth (bytes/s).  On an
    NVSwitch box every pair sees the same bandwidth, so Eq. 4/5's single BW
    is exact."""

    processors: list
    bandwidth_bytes_per_sec: float
    # optional per-pair overrides {(a, b) sorted: bytes/s} and per-type
    # metadata {type: {field: value}}, kept and round-tripped as the
    # reference's ClusterSpec does (profiling.py:242-323); the planner, like
    # the reference's, uses the single bandwidth
    pair_bandwidth: dict = field(default_factory=dict)
    processor_types: dict = field(default_factory=dict)

    def __post_init__(self):
        if not self.processors:
            raise ValidationError("cluster lists no processors")
        if not (self.bandwidth_bytes_per_sec > 0):
            raise ValidationError("bandwidth must be positive")
        ids = [p.instance_id for p in self.processors]
        if len(set(ids)) != len(ids):
            raise StructuralError("duplicate processor instance ids")

    def bandwidth_between(self, a: str, b: str) -> float:
        key = (a, b) if a <= b else (b, a)
        return self.pair_bandwidth.get(key, self.bandwidth_bytes_per_sec)

    def type_of(self, instance_id: str) -> str:
        for p in self.processors:
            if p.instance_id == instance_id:
                return p.type_name
        raise ConfigError(f"unknown processor instance {instance_id!r}")

    @classmethod
    def homogeneous(cls, n: int, type_name: str, bandwidth: float) -> "ClusterSpec":
        return cls([Processor(f"{type_name}{i}", type_name) for i in range(n)], bandwidth)


def cluster_to_json(c: ClusterSpec) -> str:
    obj = {"format_version": FORMAT_VERSION,
           "processors": [{"id": p.instance_id, "type": p.type_name} for p in c.processors],
           "bandwidth_bytes_per_sec": c.bandwidth_bytes_per_sec}
    if c.pair_bandwidth:
        obj["pair_bandwidth"] = [{"a": a, "b": b, "bandwidth_bytes_per_sec": v}
                                 for (a, b), v in sorted(c.pair_bandwidth.items())]
    if c.processor_types:
        obj["processor_types"] = {k: dict(v) for k, v in sorted(c.processor_types.items())}
    return json.dumps(obj, indent=2, sort_keys=True)


def cluster_from_json(text: str) -> ClusterSpec:
    try:
        obj = json.loads(text)
        if int(obj.get("format_version", -1)) != FORMAT_VERSION:
            raise ValidationError("unsupported or missing cluster format_version")
        pair = {}
        for rec in obj.get("pair_bandwidth", []):
            a, b = str(rec["a"]), str(rec["b"])
            bw = float(rec["bandwidth_bytes_per_sec"])
            if not bw > 0:
                raise ValidationError("pair bandwidth must be positive")
            pair[(a, b) if a <= b else (b, a)] = bw
        types = {str(k): dict(v) for k, v in obj.get("processor_types", {}).items()}
        return ClusterSpec([Processor(str(r["id"]), str(r["type"])) for r in obj["processors"]],
                           float(obj["bandwidth_bytes_per_sec"]), pair, types)
    except (json.JSONDecodeError, KeyError, TypeError, ValueError) as exc:
        raise ValidationError(f"malformed cluster file: {exc}") from exc


# ---------------------------------------------------------------- plan types
@dataclass(frozen=True)
class Stage:
    """inclusive layer range, processors, predicted time."""

    layer_start: int
    layer_end: int
    assigned_processors: tuple
    predicted_stage_time: float


@dataclass(frozen=True)
class PartitionPlan:
    """contiguous stages; objective = slowest stage incl.
    inter-stage transfers; split_config like "7-1"."""

    stages: tuple
    objective: float

    @property
    def split_config(self) -> str:
        return "-".join(str(len(s.assigned_processors)) for s in self.stages)

    def to_json(self) -> str:
        """Plan file."""
        return json.dumps({"format_version": FORMAT_VERSION, "objective_seconds": self.objective,
                           "split_config": self.split_config,
                           "stages": [{"layer_start": s.layer_start, "layer_end": s.layer_end,
                                       "processors": list(s.assigned_processors),
                                       "predicted_stage_time": s.predicted_stage_time} for s in self.stages]},
                          indent=2, sort_keys=True)

    @classmethod
    def from_json(cls, text: str) -> "PartitionPlan":
        try:
            obj = json.loads(text)
            st = tuple(Stage(int(s["layer_start"]), int(s["layer_end"]), tuple(str(p) for p in s["processors"]),
                             float(s["predicted_stage_time"])) for s in obj["stages"])
            return cls(st, float(obj["objective_seconds"]))
        except (json.JSONDecodeError, KeyError, TypeError, ValueError) as exc:
            raise ValidationError(f"malformed plan file: {exc}") from exc

    def validate(self, num_layers: int) -> None:
        """Stages contiguous over [0, L-1], processor sets non-empty and disjoint."""
        if not self.stages:
            raise StructuralError("plan has no stages")
        nxt = 0
        seen = set()
        for s in self.stages:
            if s.layer_start != nxt or s.layer_end < s.layer_start:
                raise StructuralError("stages must partition the layers contiguously")
            if not s.assigned_processors or seen & set(s.assigned_processors):
                raise StructuralError("stage processor lists must be non-empty and disjoint")
            seen |= set(s.assigned_processors)
            nxt = s.layer_end + 1
        if nxt != num_layers:
            raise StructuralError("stages do not cover every layer")


# ---------------------------------------------------------------- cost model
class _Costs:
    """Prefix sums so Eq. 4 is O(m) per (i, j, group)."""

    def __init__(self, profiles: ProfileSet, cluster: ClusterSpec, bw: float):
        if not (bw > 0):
            raise ValidationError("bandwidth must be positive")
        self.bw = float(bw)
        self.L = profiles.num_layers
        self.types = {}
        for p in cluster.processors:
            if p.type_name not in self.types:
                t = profiles.layer_times_s(p.type_name)  # ConfigError if unknown
                self.types[p.type_name] = np.concatenate([[0.0], np.cumsum(t)])
        self.type_of = {p.instance_id: p.type_name for p in cluster.processors}
        self.pcum = np.concatenate([[0.0], np.cumsum(profiles.param_bytes())])
        self.act = profiles.activation_bytes()

    def compute(self, i: int, j: int, type_name: str) -> float:
        c = self.types[type_name]
        return float(c[j + 1] - c[i])

    def q(self, i: int, j: int, group: Sequence[str]) -> float:
        """Eq. 4, verbatim incl. the 1/m on the sync term."""
        m = len(group)
        if m == 0:
            raise ValidationError("processor group must be non-empty")
        slow = max(self.compute(i, j, self.type_of[a]) for a in group)
        sync = 2.0 * (m - 1) * float(self.pcum[j + 1] - self.pcum[i]) / self.bw if m > 1 else 0.0
        return (slow + sync) / m

    def comm(self, k: int) -> float:
        """a_k / BW: activation transfer after layer k (Eq. 5)."""
        return float(self.act[k]) / self.bw


def stage_time_q(i: int, j: int, processor_group: Sequence[str], profiles: ProfileSet, cluster: ClusterSpec,
                 bw: Optional[float] = None) -> float:
    """SPEC.md:291-299 / Eq. 4."""
    if i > j:
        raise ValidationError("stage needs i <= j")
    c = _Costs(profiles, cluster, cluster.bandwidth_bytes_per_sec if bw is None else bw)
    return c.q(i, j, list(processor_group))


def get_comp_time(i: int, j: int, processor_group: Sequence[str], profiles: ProfileSet, cluster: ClusterSpec,
                  bw: Optional[float] = None) -> float:
    """Algorithm 2: data-parallel time of layers i..j on the
    group — the same contract as Eq. 4."""
    return stage_time_q(i, j, processor_group, profiles, cluster, bw)


def sort_processors(cluster: ClusterSpec, profiles: ProfileSet) -> list:
    """slowest first by whole-model single-processor time,
    ties by instance id."""
    tot = {t: float(profiles.layer_times_s(t).sum()) for t in {p.type_name for p in cluster.processors}}
    return [p.instance_id for p in sorted(cluster.processors, key=lambda p: (-tot[p.type_name], p.instance_id))]


def _key(obj: float, nstages: int, traffic: float):
    return (obj, nstages, traffic)


def _better(a, b) -> bool:
    """Lexicographic (objective, stages, traffic) with a relative tie band on
    the float objective."""
    if b is None:
        return True
    tol = _REL_TIE * max(abs(a[0]), abs(b[0]), 1e-300)
    if a[0] < b[0] - tol:
        return True
    if a[0] > b[0] + tol:
        return False
    if a[1] != b[1]:
        return a[1] < b[1]
    return a[2] < b[2] - _REL_TIE * max(abs(a[2]), abs(b[2]), 1e-300)


def _plan_order(costs: _Costs, order: list, max_stages: int):
    """Algorithm 1 over prefixes of `order`: best[j][m] for layers 0..j on
    order[:m] (stages use contiguous segments, last stage the suffix), with
    at most `max_stages` stages (one DP layer per extra stage)."""
    L, M = costs.L, len(order)
    best = [[(_key(costs.q(0, j, order[:m]), 1, 0.0), None) if m else None for m in range(M + 1)]
            for j in range(L)]
    for _ in range(1, min(max_stages, L)):
        prev = best
        best = [row[:] for row in prev]
        for j in range(1, L):
            for m in range(2, M + 1):
                cand = best[j][m]
                for k in range(j):
                    a = costs.comm(k)
                    for m1 in range(1, m):
                        lk = prev[k][m1][0]
                        if max(lk[0], a) > cand[0][0] * (1 + _REL_TIE):
                            continue  # cannot win or tie: skip the Eq. 4 evaluation
                        r = costs.q(k + 1, j, order[m1:m])
                        key = _key(max(lk[0], a, r), lk[1] + 1, lk[2] + float(costs.act[k]))
                        if _better(key, cand[0]):
                            cand = (key, (k, m1, prev))
                best[j][m] = cand
    return best


def _reconstruct(costs: _Costs, order: list, best, j: int, m: int) -> list:
    stages = []
    tbl = best
    while True:
        back = tbl[j][m][1]
        if back is None:
            stages.append((0, j, tuple(order[:m])))
            break
        k, m1, tbl = back
        stages.append((k + 1, j, tuple(order[m1:m])))
        j, m = k, m1
    stages.reverse()
    return stages


def _make_plan(costs: _Costs, stages: list) -> PartitionPlan:
    st = tuple(Stage(a, b, procs, costs.q(a, b, list(procs))) for a, b, procs in stages)
    obj = max(s.predicted_stage_time for s in st)
    for s in st[:-1]:
        obj = max(obj, costs.comm(s.layer_end))
    return PartitionPlan(st, obj)


def _plan_key(costs: _Costs, p: PartitionPlan):
    return _key(p.objective, len(p.stages), sum(float(costs.act[s.layer_end]) for s in p.stages[:-1]))


def plan(profiles: ProfileSet, cluster: ClusterSpec, bw: Optional[float] = None,
         max_stages: Optional[int] = None) -> PartitionPlan:
    """Eq. 5 dynamic program (Algorithm 1) on both sort
    orders and every prefix size; deterministic.  max_stages (default: no
    limit) bounds the pipeline depth, e.g. 2 for Table III's two-stage
    configurations."""
    costs = _Costs(profiles, cluster, cluster.bandwidth_bytes_per_sec if bw is None else bw)
    base = sort_processors(cluster, profiles)
    best_plan, best_key = None, None
    for order in (base, base[::-1]):
        tbl = _plan_order(costs, order, max_stages or costs.L)
        for m in range(1, len(order) + 1):
            p = _make_plan(costs, _reconstruct(costs, order, tbl, costs.L - 1, m))
            k = _plan_key(costs, p)
            if _better(k, best_key):
                best_plan, best_key = p, k
    return best_plan


def data_parallel_plan(profiles: ProfileSet, cluster: ClusterSpec, bw: Optional[float] = None) -> PartitionPlan:
    """Algorithm 2's baseline: one stage replicated on every processor."""
    costs = _Costs(profiles, cluster, cluster.bandwidth_bytes_per_sec if bw is None else bw)
    return _make_plan(costs, [(0, costs.L - 1, tuple(sort_processors(cluster, profiles)))])


def _compositions(L: int):
    """All ways to cut layers 0..L-1 into contiguous stages (as end indices)."""
    for r in range(L):
        for cuts in itertools.combinations(range(L - 1), r):
            ends = list(cuts) + [L - 1]
            starts = [0] + [c + 1 for c in cuts]
            yield list(zip(starts, ends))


def brute_force_plan(profiles: ProfileSet, cluster: ClusterSpec, bw: Optional[float] = None,
                     restrict_to_prefixes: bool = True, max_stages: Optional[int] = None) -> PartitionPlan:
    """exhaustive oracle (L <= 10, M <= 5).  With
    restrict_to_prefixes the processors of S stages are S consecutive
    segments of a prefix of either sort order (the DP's search space);
    otherwise any disjoint non-empty subsets."""
    L, M = profiles.num_layers, len(cluster.processors)
    if L > 10 or M > 5:
        raise ValidationError("brute_force_plan is limited to L <= 10 layers and M <= 5 processors")
    costs = _Costs(profiles, cluster, cluster.bandwidth_bytes_per_sec if bw is None else bw)
    base = sort_processors(cluster, profiles)
    best_plan, best_key = None, None

    def consider(stages):
        nonlocal best_plan, best_key
        p = _make_plan(costs, stages)
        k = _plan_key(costs, p)
        if _better(k, best_key):
            best_plan, best_key = p, k

    for parts in _compositions(L):
        S = len(parts)
        if max_stages is not None and S > max_stages:
            continue
        if restrict_to_prefixes:
            for order in (base, base[::-1]):
                for m in range(S, M + 1):
                    for cuts in itertools.combinations(range(1, m), S - 1):
                        b = [0, *cuts, m]
                        consider([(a, e, tuple(order[b[s]:b[s + 1]])) for s, (a, e) in enumerate(parts)])
        else:
            # assign each processor to one of S stages or to "idle" (S)
            for assign in itertools.product(range(S + 1), repeat=M):
                groups = [tuple(base[i] for i in range(M) if assign[i] == s) for s in range(S)]
                if all(groups):
                    consider([(a, e, groups[s]) for s, (a, e) in enumerate(parts)])
    return best_plan


def plan_with_types_as(profiles: ProfileSet, cluster: ClusterSpec, type_name: str,
                       bw: Optional[float] = None) -> PartitionPlan:
    """PipeDream's homogeneity assumption (SPEC.md:425-431 'MP' row): plan as
    if every processor were `type_name` (normally the slowest)."""
    homo = ClusterSpec([Processor(p.instance_id, type_name) for p in cluster.processors],
                       cluster.bandwidth_bytes_per_sec)
    return plan(profiles, homo, bw)


def evaluate(plan_: PartitionPlan, profiles: ProfileSet, cluster: ClusterSpec, bw: Optional[float] = None) -> float:
    """Objective of an arbitrary plan under the real cluster's costs."""
    costs = _Costs(profiles, cluster, cluster.bandwidth_bytes_per_sec if bw is None else bw)
    return _make_plan(costs, [(s.layer_start, s.layer_end, s.assigned_processors) for s in plan_.stages]).objective
