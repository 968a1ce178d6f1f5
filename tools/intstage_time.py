"""GPU: the C3 integer stage alone (voxelize -> coordinates -> 9 kernel maps
-> groupings), event-timed on the trainer's own streams (side streams
joined), with and without the grouping's tile schedule; plus the CUPTI
kernel times of the grouping kernels.  Usage: python tools/intstage_time.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import voxpipe_oracle as O  # noqa: E402
from paper_2012_13846_b200 import _lib, model  # noqa: E402

tr = model.SparseResNetTrainer(batch=64, points=2048, resolution=64)
pts, offs = O.synthetic_batch(64, 2048, 64, seed=1000, dtype=np.float32)
tr.train_step_from_host(pts, offs, np.arange(64) % 40)


def run():
    tr._integer_stage(_lib.stream())
    tr.join_side_streams()


for mode in (False, True, False, True):
    tr.TILE_SCHED = mode
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(30):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    print(f"tile schedule {mode}: integer stage median {np.median(ts):.1f} us (min {np.min(ts):.1f})")
from torch.profiler import ProfilerActivity, profile  # noqa: E402

tr.TILE_SCHED = True
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(5):
        run()
    torch.cuda.synchronize()
agg = {}
for ev in prof.events():
    if ev.device_type.name == "CUDA" and ("tile_" in ev.name or "group_" in ev.name or "permute_rows" in ev.name):
        agg.setdefault(ev.name.split("(")[0], []).append(ev.device_time)
for k, v in sorted(agg.items()):
    print(f"  {k:40s} n={len(v) // 5:3d}/stage  mean {np.mean(v):6.2f} us  max {np.max(v):6.2f} us")
