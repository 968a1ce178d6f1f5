"""Per-layer GPU profile of the SparseResNet (C3 workload by default): prints
one JSON record per conv layer (fwd / BN-bwd / dgrad / wgrad device µs) and
writes the reference-format LayerProfile JSON the partitioner consumes."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import numpy as np
import torch

import voxpipe_oracle as O
from paper_2012_13846_b200 import model

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--points", type=int, default=2048)
ap.add_argument("--res", type=int, default=64)
ap.add_argument("--blocks", type=int, default=1)
ap.add_argument("--out", default="gpurun_out/layer_profile.json")
a = ap.parse_args()
tr = model.SparseResNetTrainer(batch=a.batch, points=a.points, resolution=a.res, blocks=a.blocks)
pts, _ = O.synthetic_batch(a.batch, a.points, a.res, seed=0, dtype=np.float32)
tr.set_batch(torch.from_numpy(pts).cuda(), torch.arange(a.batch, dtype=torch.int32).cuda() % 40)
recs = tr.profile_layers()
tot_f = tot_b = 0.0
for r in recs:
    tot_f += r["fwd_us"]
    tot_b += r["bwd_us"]
    print(json.dumps({k: (round(v, 2) if isinstance(v, float) else v) for k, v in r.items()}))
print(f"total fwd {tot_f:.1f} us  bwd {tot_b:.1f} us")
os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
with open(a.out, "w") as f:
    json.dump({"format_version": 1, "model_name": f"sparse_resnet_b{a.blocks}_{a.res}", "batch_size": a.batch,
               "processor_type": "B200", "records": recs}, f, indent=1)
