"""Critical path of the C3 step alone: the captured step with the side-stream
work removed (VP_DBG_SKIP_WGRAD=1 VP_DBG_SKIP_PREFETCH=1 must be set in the
environment: experiments only), replayed under CUPTI; prints every kernel of
one step in start order with its duration and the gap before it, then the
totals (kernel time vs gaps) per kernel family."""
import collections
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

assert os.environ.get("VP_DBG_SKIP_WGRAD") == "1" and os.environ.get("VP_DBG_SKIP_PREFETCH") == "1"
tr = model.SparseResNetTrainer(batch=64, points=2048, resolution=64)
tr.enable_prefetch()
pts, _ = O.synthetic_batch(64, 2048, 64, seed=0, dtype=np.float32)
lab = torch.arange(64, dtype=torch.int32).cuda() % 40
tr.set_batch(torch.from_numpy(pts).cuda(), lab)
tr.capture()
for _ in range(5):
    tr.step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        tr.step()
    torch.cuda.synchronize()
evs = sorted((e.time_range.start, e.time_range.end, e.name) for e in prof.events()
             if e.device_type.name == "CUDA" and e.time_range.elapsed_us() > 0 and "Memcpy" not in e.name)
# the last step: from the last stem conv (the step's first critical-path kernel)
starts = [i for i, (_, _, n) in enumerate(evs) if "conv_stem" in n]
step = evs[starts[-1]:]
t0 = step[0][0]
fam_k = collections.defaultdict(float)
fam_g = collections.defaultdict(float)
cnt = collections.Counter()
prev_end = t0
for s, e, n in step:
    short = n.split("(")[0].replace("void ", "").split("<")[0][:40]
    gap = max(0.0, s - prev_end)
    print(f"{s - t0:9.1f} {e - s:7.2f} us  gap {gap:6.2f}  {short}")
    fam_k[short] += e - s
    fam_g[short] += gap
    cnt[short] += 1
    prev_end = max(prev_end, e)
span = step[-1][1] - t0
print(f"\nstep span {span:.1f} us, kernels {len(step)}, kernel time {sum(fam_k.values()):.1f} us, "
      f"gaps {sum(fam_g.values()):.1f} us")
for k in sorted(fam_k, key=lambda k: -(fam_k[k] + fam_g[k])):
    print(f"  {k:40s} {cnt[k]:4d}x  kernel {fam_k[k]:8.1f} us  gaps-before {fam_g[k]:7.1f} us")
