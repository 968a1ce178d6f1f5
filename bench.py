#!/usr/bin/env python
"""Benchmark: SparseResNet training throughput (point clouds / s) on B200.

Workload (BASELINE.json configs[2], "C3"): 64 synthetic ModelNet40-shaped
clouds x 2048 points at 64^3 voxels per GPU, bf16 features, 13-conv
SparseResNet, SGD momentum 0.9.  A step = one full training step from raw
points: GPU voxelization, strided output coordinates, 9 kernel maps, forward,
backward, optimizer (nothing cached across steps).

  value : whole-job clouds/s with the points already in HBM (device timed,
          CUDA events per step, L2 flushed between steps with a 256 MiB write)
  e2e   : clouds/s through the public trainer API from pinned HOST memory:
          H2D of the step's points + labels, the step, D2H of the loss, all
          inside the timed region
  roofline : dominant conv kernel (largest per-launch device time among every
          layer's tensor-core forward / dgrad / wgrad), re-launched on the
          step's own data and tables with the L2 flushed before each launch;
          SURVEY §8(d) algorithmic bytes / FLOPs (paper_2012_13846_b200/roofline.py)
  cpu_baseline : the reference's own CPU path (oracle/_ref voxpipe, convs via
          voxpipe.conv + numpy glue) on a bounded sample of the same workload

Multi-GPU (torchrun, one process per GPU, NCCL): data parallel, each rank a
full 64-cloud batch (weak scaling), one NCCL all_reduce of the flat gradient
buffer per step; time = max over ranks.

`--impl reference` times the reference CPU path alone (rank 0; other ranks exit).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

# rank 0's stdout carries exactly one JSON line: everything else written to
# fd 1 (NCCL's version banner, library prints) is sent to stderr, and the
# JSON line goes to a private duplicate of the original stdout
_JSON_OUT = os.fdopen(os.dup(1), "w")
os.dup2(2, 1)


def emit(line: dict) -> None:
    _JSON_OUT.write(json.dumps(line) + "\n")
    _JSON_OUT.flush()

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

def metric_config(args):
    """BASELINE.json metric on the workload the flags select: the default is
    configs[2] ("C3"); --batch 256 --points 16384 --res 128 --blocks 2 is the
    C5 network on one GPU."""
    c3 = (args.batch, args.points, args.res, args.blocks) == (64, 2048, 64, 1)
    c5 = (args.res, args.blocks) == (128, 2)
    tag = "C3" if c3 else ("C5" if c5 else "custom")
    global CONFIG_TAG
    CONFIG_TAG = tag
    metric = (f"point clouds/sec train (SparseResNet{'' if args.blocks == 1 else f' blocks={args.blocks}'}, "
              f"{args.batch}x{args.points} pts @ {args.res}^3, bf16)")
    config = {"workload": f"{tag}{' (one GPU)' if tag == 'C5' else ''}: sparse-ResNet classifier, {args.batch} clouds x {args.points} pts/cloud at "
                          f"{args.res}^3 voxels per GPU, {1 + 4 * (1 + 2 * args.blocks)} convs (blocks={args.blocks}), "
                          "bf16 features, SGD momentum",
              "global_batch_per_gpu": args.batch, "points_per_cloud": args.points, "resolution": args.res,
              "planes": [32, 64, 128, 256], "blocks": args.blocks, "classes": 40,
              "l2": "flushed between timed steps (256 MiB memset, outside the events)"}
    return metric, config


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--points", type=int, default=2048)
    ap.add_argument("--res", type=int, default=64)
    ap.add_argument("--blocks", type=int, default=1)
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-roofline", action="store_true", help="skip the per-kernel roofline timing (quick A/B runs)")
    ap.add_argument("--cpu-sample", type=int, default=64,
                    help="clouds per CPU-baseline step (default: the full 64-cloud C3 batch)")
    ap.add_argument("--profile-only", action="store_true", help="warm-up + a few steps, no JSON (for ncu)")
    ap.add_argument("--plan", default="dp",
                    help="N>1: 'dp' (every GPU a replica, gradient all_reduce), 'auto' (SparsePipe partitioner "
                         "on per-unit GPU profiles -> pipeline stages), or unit cuts like '3' / '1,4,6'")
    ap.add_argument("--p2p-gbs", type=float, default=770.0, help="NVLink P2P GB/s per direction for the planner")
    ap.add_argument("--pipeline-test", action="store_true",
                    help="functional test of the multi-process pipeline on ONE GPU: every rank on cuda:0, gloo "
                         "transport through host memory (not a performance number)")
    ap.add_argument("--dp-allreduce", action="store_true",
                    help="run the data-parallel gradient all_reduce even at one GPU (tests its graph capture)")
    return ap.parse_args()


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region (NVML via
    nvidia_ml_py, polled every ~2 ms from a thread, so even a short timed
    region gets samples); falls back to `nvidia-smi -lms` when NVML is absent."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index):
        self.index, self.rows, self.proc, self.nvml = index, [], None, None
        self.stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_sm = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nvml = None

    def _poll(self):
        nv = self.nvml
        bits = [0x8, 0x40, 0x20, 0x4]  # HwSlowdown, HwThermalSlowdown, SwThermalSlowdown, SwPowerCap
        while not self.stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.rows.append([str(sm), str(self.max_sm)] + ["Active" if rs & b else "Not Active" for b in bits])
            except Exception:
                return
            time.sleep(0.002)

    def __enter__(self):
        if self.nvml is not None:
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return self
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([v.strip() for v in line.split(",")])

    def __exit__(self, *a):
        self.stop.set()
        if self.nvml is not None:
            self.t.join(timeout=1)
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({self.NAMES[i] for r in self.rows for i in range(4) if len(r) > 2 + i and r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows), "source": "nvml" if self.nvml else "nvidia-smi"}


def cpu_baseline(args, steps=2, warmup=1, seed=0):
    import ref_runner

    nthreads = os.cpu_count() or 1
    r = ref_runner.time_steps(args.cpu_sample, args.points, args.res, steps, warmup, seed=seed)
    return {"value": round(r["clouds_per_s"], 3), "unit": "clouds/s", "cores": nthreads, "kind":
            "reference" if r["kind"] == "reference" else "port",
            "sample": f"{steps} timed steps (+{warmup} warm-up) of {args.cpu_sample} clouds x {args.points} pts @ "
                      f"{args.res}^3 through voxpipe.tensor.voxelize/batch + voxpipe.conv fwd/bwd (compiled hash) + "
                      f"numpy BN/pool/linear/SGD glue; OpenBLAS threads={nthreads}"}


def run_reference(args, rank):
    if rank != 0:
        return
    import ref_runner

    t0 = time.time()
    # bounded sample: ~0.105 s of reference CPU work per cloud on a 16-thread
    # host (profiles/r1_bench_reference.json), so size each step's cloud count
    # for the whole --steps K --warmup W run to take about two minutes
    per_cloud_s = 0.105
    budget = 120.0 / max(1, args.steps + args.warmup)
    args.cpu_sample = int(max(2, min(args.cpu_sample, round(budget / per_cloud_s))))
    r = ref_runner.time_steps(args.cpu_sample, args.points, args.res, max(1, args.steps), max(0, args.warmup))
    value = r["clouds_per_s"]
    cores = os.cpu_count() or 1
    line = {"metric": METRIC, "value": round(value, 3), "unit": "clouds/s", "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(r["s_per_step"] * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": dict(CONFIG, sample_clouds_per_step=args.cpu_sample),
            "cpu_baseline": {"value": round(value, 3), "unit": "clouds/s", "cores": cores,
                             "kind": "reference" if r["kind"] == "reference" else "port",
                             "sample": f"each step {args.cpu_sample} clouds of the C3 workload (bounded sample)"},
            "e2e": {"value": round(value, 3), "unit": "clouds/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": round(time.time() - t0, 1)}
    emit(line)


def main():
    args = parse()
    global METRIC, CONFIG
    METRIC, CONFIG = metric_config(args)
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank)
        return

    import torch
    import torch.distributed as dist

    import voxpipe_oracle as O
    from paper_2012_13846_b200 import _lib, model

    if args.pipeline_test:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.pipeline_test:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    allreduce = None
    if world > 1 or args.dp_allreduce:
        if not dist.is_initialized():  # --dp-allreduce at world 1 (capture test of the collective)
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)

        def allreduce(flat):  # one NCCL all_reduce of the flat fp32 gradient buffer per step (graph-captured)
            dist.all_reduce(flat)
            flat.div_(dist.get_world_size())

    if world > 1 and args.plan != "dp":
        return run_pipeline(args, rank, world, local, dev)
    tr = model.SparseResNetTrainer(batch=args.batch, points=args.points, resolution=args.res, blocks=args.blocks,
                                   device=dev, grad_allreduce=allreduce)
    # synthetic data pool: 4 distinct batches per rank, resident in HBM and pinned host memory
    pool_n = 4
    host_pts, host_lab, dev_pts, dev_lab = [], [], [], []
    for i in range(pool_n):
        pts, _ = O.synthetic_batch(args.batch, args.points, args.res, seed=1000 * rank + i, dtype=np.float32)
        lab = ((np.arange(args.batch) + 7 * i) % 40).astype(np.int32)
        hp = torch.from_numpy(pts).pin_memory()
        hl = torch.from_numpy(lab).pin_memory()
        host_pts.append(hp)
        host_lab.append(hl)
        dev_pts.append(hp.to(dev))
        dev_lab.append(hl.to(dev))
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)

    use_graph = not args.no_graph
    if use_graph:
        # the next batch's coordinates and kernel maps are built while the
        # current batch runs its backward (model.enable_prefetch)
        tr.enable_prefetch()
    tr.set_batch(dev_pts[0], dev_lab[0])
    k0 = _lib.load().vp_kernel_launches()
    if use_graph:
        tr.capture(warmup=1)
        kern_per_step = tr.kernels_per_step  # library kernels in one captured step graph
    else:
        tr.step_body()
        kern_per_step = _lib.load().vp_kernel_launches() - k0

    def one_step(i):
        tr.set_batch(dev_pts[i % pool_n], dev_lab[i % pool_n])  # D2D into the static input buffers
        tr.step()

    for i in range(args.warmup):
        one_step(i)
    torch.cuda.synchronize()
    if args.profile_only:
        for i in range(3):
            one_step(i)
        torch.cuda.synchronize()
        print(f"profile-only done: levels={tr.level_sizes()} pairs={tr.pair_counts()} kernels/step={kern_per_step}")
        return

    # ---------------- device-resident timed region
    stream = torch.cuda.current_stream()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.zero_()  # L2 flush, outside the events
            evs[i][0].record(stream)
            one_step(i)
            evs[i][1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = sum(a.elapsed_time(b) for a, b in evs)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    value = world * args.batch * args.steps / (ms / 1e3)
    loss = float(tr.loss.item())

    # ---------------- e2e through the public API from pinned host memory
    h2d = int(host_pts[0].numel() * host_pts[0].element_size() + host_lab[0].numel() * 4)
    d2h = 4
    loss_host = torch.empty(1, dtype=torch.float32).pin_memory()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # Each step's pinned-host -> HBM upload runs on a copy stream into a
    # staging buffer while the previous step computes; the step itself only
    # waits for its upload and does a 1.5 MB device copy into the engine's
    # static input buffers.  Every byte still crosses PCIe inside the region.
    h2d_stream = torch.cuda.Stream(device=dev)
    stage = [(torch.empty_like(dev_pts[0]), torch.empty_like(dev_lab[0])) for _ in range(2)]
    ready = [torch.cuda.Event() for _ in range(2)]
    free = [torch.cuda.Event() for _ in range(2)]

    def upload(i):
        b = i % 2
        h2d_stream.wait_event(free[b])
        with torch.cuda.stream(h2d_stream):
            stage[b][0].copy_(host_pts[i % pool_n], non_blocking=True)
            stage[b][1].copy_(host_lab[i % pool_n], non_blocking=True)
        ready[b].record(h2d_stream)

    e0.record(stream)
    upload(0)
    for i in range(args.steps):
        b = i % 2
        stream.wait_event(ready[b])
        tr.set_batch(stage[b][0], stage[b][1])
        free[b].record(stream)
        if i + 1 < args.steps:
            upload(i + 1)
        tr.step()
        loss_host.copy_(tr.loss, non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_value = world * args.batch * args.steps / (e2e_ms / 1e3)

    # ---------------- roofline of the dominant kernel (standalone, same data)
    roof = None if args.no_roofline else roofline(tr, dev, CONFIG_TAG)

    if world > 1:
        dist.barrier()
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            try:
                cpu = cpu_baseline(args)
            except Exception as exc:  # pragma: no cover
                cpu = {"value": None, "unit": "clouds/s", "cores": os.cpu_count(), "kind": "port",
                       "sample": f"failed: {exc}"}
        line = {"metric": METRIC, "value": round(value, 2), "unit": "clouds/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
                "config": dict(CONFIG, parallelism=f"dp{world}", cuda_graph=use_graph,
                               level_rows=tr.level_sizes(), map_pairs=tr.pair_counts()),
                "e2e": {"value": round(e2e_value, 2), "unit": "clouds/s", "h2d_bytes_per_step": h2d,
                        "d2h_bytes_per_step": d2h},
                "gpu_launches": int(kern_per_step * args.steps),
                "gpu_launches_per_step": int(kern_per_step),
                "roofline": roof, "cpu_baseline": cpu, "clocks": clk.summary(), "final_loss": round(loss, 5)}
        emit(line)
    if dist.is_initialized():
        dist.destroy_process_group()


def run_pipeline(args, rank, world, local, dev):
    """SparsePipe on N GPUs: stages from the partitioner fed with this box's
    measured per-unit GPU costs (or explicit cuts), micro-batches of
    `--batch` clouds over NCCL P2P, PipeDream 1F1B with weight stashing.
    A step = `world` micro-batches (the same clouds per GPU as DP, weak
    scaling); the timed region is one continuous 1F1B run of K steps
    (fill and drain included), device-timed, max over ranks."""
    import torch
    import torch.distributed as dist

    import voxpipe_oracle as O
    from paper_2012_13846_b200 import model, partition, pipeline as PL

    def make(units):
        return model.SparseResNetTrainer(batch=args.batch, points=args.points, resolution=args.res,
                                         blocks=args.blocks, device=dev, units=units)

    probe = make(None)
    n_units = len(probe.units)
    if args.plan == "auto":
        prof_json = None
        if rank == 0:
            pts, _ = O.synthetic_batch(args.batch, args.points, args.res, seed=0, dtype=np.float32)
            probe.set_batch(torch.from_numpy(pts).to(dev), torch.zeros(args.batch, dtype=torch.int32, device=dev))
            ps = PL.unit_profile(probe, probe.profile_layers(), "sparse_resnet")
            prof_json = partition.profile_to_json(ps, "B200")
        box = [prof_json]
        dist.broadcast_object_list(box, src=0)
        ps = partition.profile_from_json(box[0])
        plan, topo = PL.plan_topology(ps, world, args.p2p_gbs * 1e9)
        split = plan.split_config
    else:
        cuts = [int(c) for c in args.plan.split(",")]
        topo = PL.Topology.even(n_units, cuts)
        split = "-".join("1" for _ in topo.stages)
    del probe
    topo.validate(n_units)
    tr = PL.DistTransport(dist, topo, host_stage=args.pipeline_test)  # collective: builds the replica groups
    active = topo.locate(rank) is not None  # the plan may leave a GPU idle
    pool = []
    for i in range(4):
        pts, _ = O.synthetic_batch(args.batch, args.points, args.res, seed=1000 + i, dtype=np.float32)
        pool.append((torch.from_numpy(pts).to(dev),
                     torch.tensor([(b + 7 * i) % 40 for b in range(args.batch)], dtype=torch.int32, device=dev)))
    dist.barrier()  # first collective on every rank before any P2P group

    mult = topo.mb_multiple()  # every replica group all-reduces the same number of rounds

    def run(n_mb):
        n_mb = -(-n_mb // mult) * mult
        return PL.StageRunner(topo, rank, n_mb, make, lambda mb: pool[mb % len(pool)], tr,
                              use_graphs=not args.no_graph)

    n_timed = -(-(args.steps * world) // mult) * mult
    if active:
        warm = run(max(1, args.warmup) * world)
        warm.run()
        torch.cuda.synchronize()
        timed = run(n_timed)
        # reuse the warmed engines, graphs and weights
        timed.slots, timed.graphs = warm.slots[:len(timed.slots)], warm.graphs
        timed.master_p, timed.master_pb, timed.master_m = warm.master_p, warm.master_pb, warm.master_m
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dist.barrier()
    torch.cuda.synchronize()
    e0.record(st)
    if active:
        timed.run()
    e1.record(st)
    torch.cuda.synchronize()
    dist.barrier()
    ms = torch.tensor([e0.elapsed_time(e1)], device="cpu" if args.pipeline_test else dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    value = n_timed * args.batch / (ms / 1e3)
    # PipeDream weight-stashing audit: every (micro-batch,
    # stage) backward used the weight version its forward used
    audit = timed.stats.audit if active else []
    audits = [None] * world
    dist.all_gather_object(audits, audit)
    checked = sum(len(a) for a in audits)
    violations = sum(1 for a in audits for _, _, fv, bv in a if fv != bv)
    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 2), "unit": "clouds/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4), "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
                "config": dict(CONFIG, parallelism=f"pipeline {split}", stages=[
                    [s.unit_start, s.unit_end, list(s.ranks)] for s in topo.stages],
                    micro_batch_clouds=args.batch, micro_batches_per_step=world, micro_batches_timed=n_timed,
                    cuda_graph=not args.no_graph,
                    l2="not flushed: one continuous 1F1B stream (fill + drain inside the timed region)"),
                "weight_version_audit": {"checked": checked, "violations": violations},
                "e2e": None, "gpu_launches": None, "roofline": None, "cpu_baseline": None}
        emit(line)
    dist.barrier()
    dist.destroy_process_group()


def roofline(tr, dev, tag, iters=20):
    """Roofline of the dominant conv kernel of the step and of the kernel-map
    builder (paper_2012_13846_b200/roofline.py: SURVEY §8(d) algorithmic
    work; every launch preceded by an L2 flush, CUDA events on the launching
    stream, the step's own data and tables).

    Candidates: each tensor-core layer's forward, dgrad and wgrad launch
    (the C_in = 1 stem runs SIMT kernels).  Dominant = the largest device
    time per launch; all candidates are listed under `kernels`."""
    import torch

    from paper_2012_13846_b200 import _lib
    from paper_2012_13846_b200 import roofline as RL

    hbm, tc_peak, src = RL.peaks()
    flush = RL.Flusher(dev)
    st = torch.cuda.current_stream().cuda_stream
    fc = _lib.VP_BF16
    rows = []
    for L in tr.layers:
        if L["cin"] < 32:
            continue
        src_l, dst, m = L["src"], L["dst"], L["map"]
        P = int(m.ptr[-1].item())
        n_in, n_out = int(src_l.n.item()), int(dst.n.item())
        x = L["x"]

        def fwd(L=L, dst=dst, x=x):
            _lib.call("vp_conv_fwd", x.data_ptr(), fc, x.shape[0], L["cin"], L["wb"].data_ptr(), fc, L["cout"],
                      tr.K, tr.fwd_table(L).data_ptr(), 0, _lib.ptr(tr.fwd_perm(L)), dst.n.data_ptr(), dst.cap,
                      L["y"].data_ptr(), fc, L["fwd_ws"].data_ptr(), L["fwd_ws"].numel(), st)

        table, flip, perm = tr.dgrad_table(L)
        gin = tr.gact[tr.levels.index(src_l)]

        def dgrad(L=L, src_l=src_l, table=table, flip=flip, perm=perm, gin=gin):
            _lib.call("vp_conv_dgrad", L["gy"].data_ptr(), fc, L["gy"].shape[0], L["cout"], L["wb"].data_ptr(), fc,
                      L["cin"], tr.K, table.data_ptr(), flip, _lib.ptr(perm), src_l.n.data_ptr(), src_l.cap,
                      gin.data_ptr(), fc, L["dg_ws"].data_ptr(), L["dg_ws"].numel(), st)

        def wgrad(L=L, m=m, x=x):
            _lib.call("vp_conv_wgrad", x.data_ptr(), fc, L["cin"], L["gy"].data_ptr(), fc, L["cout"], tr.K,
                      m.pin.data_ptr(), m.pout.data_ptr(), m.ptr.data_ptr(), m.pin.numel(), L["gw"].data_ptr(),
                      L["wg_ws"].data_ptr(), L["wg_ws"].numel(), st)

        for mode, fn, key, (a, b, ci, co) in (
                ("fwd", fwd, f"conv_fwd_tc<{L['cin']},{L['cout']}>", (n_in, n_out, L["cin"], L["cout"])),
                ("dgrad", dgrad, f"conv_dgrad_tc<{L['cout']},{L['cin']}>", (n_out, n_in, L["cout"], L["cin"])),
                ("wgrad", wgrad, f"conv_wgrad_tc<{L['cin']},{L['cout']}>", (n_in, n_out, L["cin"], L["cout"]))):
            t = RL.time_cold(fn, flush, iters)
            F, B = RL.conv_work(P, a, b, ci, co, tr.K, mode)
            rec = RL.classify(F, B, t, hbm, tc_peak)
            rows.append((t, key, L["name"], mode, P, n_in, n_out, rec))
    t, key, name, mode, P, n_in, n_out, rec = max(rows, key=lambda r: r[0])
    out = {"kernel": f"{key} {mode} layer {name} (N_in={n_in}, N_out={n_out}, pairs={P})", **rec,
           "traffic": RL.ncu_traffic(tag, key, name), "peak_source": src,
           "timing": "mean of per-launch CUDA events, L2 flushed (256 MiB write) before every launch",
           "kernels": {f"{nm}.{md}": [r["us_per_launch"], r["frac"], r["bound"]] for _, _, nm, md, *_x, r in rows}}
    # kernel-map builder as the step runs it, level 0 stride-1: index insert
    # (dense grid, or hash) + probe + ordered pair compaction (+ grid clear)
    m = tr.map_s1[0]

    def map_launch():
        if tr.use_grid:
            tr._grid_set(0, st, clear=False)
        tr._build_map(m, st)
        if tr.use_grid:
            tr._grid_set(0, st, clear=True)

    tm = RL.time_cold(map_launch, flush, iters)
    nm = int(m.src.n.item())
    pm = int(m.ptr[-1].item())
    name = {"grid": "vp_grid_set + vp_kernel_map_grid", "brick": "vp_brick_set + vp_kernel_map_brick"}.get(
        tr.index_kind, "vp_kernel_map")
    out["map"] = {"kernel": f"{name} level0 stride-1 (N={nm}, pairs={pm})",
                  **RL.classify(0.0, RL.map_bytes(nm, nm, pm), tm, hbm, tc_peak)}
    return out


if __name__ == "__main__":
    main()
