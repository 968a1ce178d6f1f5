"""GPU: per-128-row-tile active-offset counts of every tensor-core conv of the
C3 step (forward and dgrad tables as the trainer stages them), saved to
gpurun_out/tile_costs.npz for the offline schedule simulation
(tools/sched_sim.py).  Usage: python tools/tile_costs.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import voxpipe_oracle as O  # noqa: E402
from paper_2012_13846_b200 import model  # noqa: E402

tr = model.SparseResNetTrainer(batch=64, points=2048, resolution=64)
pts, offs = O.synthetic_batch(64, 2048, 64, seed=1000, dtype=np.float32)
tr.train_step_from_host(pts, offs, np.arange(64) % 40)
out = {}
for L in tr.layers:
    if L["cin"] < 32:
        continue
    n_out = int(L["dst"].n.item())
    t = tr.fwd_table(L)[:n_out].cpu().numpy()
    out[f"{L['name']}.fwd"] = np.array([(t[i:i + 128] >= 0).any(0).sum() for i in range(0, n_out, 128)])
    out[f"{L['name']}.fwd.kd"] = np.array([L["cin"], L["cout"]])
    if L["name"] == "s0.down":
        continue
    table, flip, perm = tr.dgrad_table(L)
    n_in = int(L["src"].n.item())
    t = table[:n_in].cpu().numpy()
    out[f"{L['name']}.dgrad"] = np.array([(t[i:i + 128] >= 0).any(0).sum() for i in range(0, n_in, 128)])
    out[f"{L['name']}.dgrad.kd"] = np.array([L["cout"], L["cin"]])
os.makedirs("gpurun_out", exist_ok=True)
np.savez("gpurun_out/tile_costs.npz", **out)
for k, v in out.items():
    if not k.endswith(".kd"):
        q = len(v) // 8 or 1
        print(k, len(v), "tiles; mean active", round(float(v.mean()), 1), "by eighths:",
              [round(float(v[i:i + q].mean()), 1) for i in range(0, len(v), q)])
