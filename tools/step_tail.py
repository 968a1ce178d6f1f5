"""Where the full C3 step (prefetch + graphs + side streams) spends the time
after its critical path: CUPTI timeline of replays, one step from stem conv
to stem conv; prints the kernels that END in the last `--tail` microseconds
of the step and the busy-SM picture (how many kernels overlap) over time."""
import argparse
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

ap = argparse.ArgumentParser()
ap.add_argument("--tail", type=float, default=250.0)
a = ap.parse_args()
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
    for i in range(3):
        tr.set_batch(*pool[i % 4])
        tr.step()
    torch.cuda.synchronize()
evs = sorted((e.time_range.start, e.time_range.end, e.name) for e in prof.events()
             if e.device_type.name == "CUDA" and e.time_range.elapsed_us() > 0)
stems = [s for s, _, n in evs if "conv_stem" in n]
t0, t1 = stems[-2], stems[-1]
step = [(s, e, n) for s, e, n in evs if t0 <= s < t1]
print(f"step {t1 - t0:.1f} us, kernels {len(step)}")
# the critical path's last kernel: the head's successors end with the stem's BN backward + sgd
crit_end = max(e for s, e, n in step if "bn_backward_apply" in n)
print(f"last bn_backward_apply ends at {crit_end - t0:.1f} us; step tail after it {t1 - crit_end:.1f} us")
for s, e, n in step:
    if e >= t1 - a.tail:
        short = n.split("(")[0].replace("void ", "")[:60]
        print(f"  {s - t0:8.1f} -> {e - t0:8.1f} ({e - s:6.1f} us)  {short}")
