"""Kernel timeline of the captured C3 training step via torch.profiler
(CUPTI): per-kernel device start/end inside graph replays -> busy/idle
breakdown and the top kernels by total time.  Writes gpurun_out/timeline.json."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import voxpipe_oracle as O  # noqa: E402
from paper_2012_13846_b200 import model  # noqa: E402

tr = model.SparseResNetTrainer(batch=64, points=2048, resolution=64)
tr.enable_prefetch()
pool = []
for i in range(4):
    pts, _ = O.synthetic_batch(64, 2048, 64, seed=1000 + i, dtype=np.float32)
    pool.append((torch.from_numpy(pts).cuda(), torch.arange(64, dtype=torch.int32).cuda() % 40))
tr.set_batch(*pool[0])
tr.capture()
for i in range(6):
    tr.set_batch(*pool[i % 4])
    tr.step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for i in range(4):
        tr.set_batch(*pool[i % 4])
        tr.step()
    torch.cuda.synchronize()
evs = []
for e in prof.events():
    if e.device_type.name == "CUDA" and e.time_range.elapsed_us() > 0:
        evs.append((e.time_range.start, e.time_range.end, e.name))
evs.sort()
# last full step: split on the copy of the staged batch (memcpy) boundaries is fragile; use the last quarter
t0, t1 = evs[0][0], evs[-1][1]
span = (t1 - t0) / 4
a = t1 - span
step = [(s, e, n) for s, e, n in evs if s >= a]
busy = 0.0
cur_s, cur_e = None, None
for s, e, n in step:
    if cur_e is None or s > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
        cur_s, cur_e = s, e
    else:
        cur_e = max(cur_e, e)
busy += cur_e - cur_s
print(f"step span {span:.1f} us, GPU busy (any kernel) {busy:.1f} us, idle {span - busy:.1f} us, kernels {len(step)}")
tot = {}
for s, e, n in step:
    k = n.split("<")[0].split("(")[0]
    tot.setdefault(k, [0.0, 0])
    tot[k][0] += e - s
    tot[k][1] += 1
for k, (t, c) in sorted(tot.items(), key=lambda x: -x[1][0])[:30]:
    print(f"  {t:8.1f} us  {c:3d}x  {k[:80]}")
os.makedirs("gpurun_out", exist_ok=True)
json.dump([(s - a, e - a, n) for s, e, n in step], open("gpurun_out/timeline.json", "w"))
