"""GPU: cost of the last (partial) round of work items in the tensor-core
conv.  A real C3 layer's forward (its own table, activations and weights) is
launched with the output row count capped at whole multiples of the grid's
128-row tiles and at the layer's real count; warm L2, CUDA events, median of
50 launches.  Usage: python tools/tail_probe.py [C]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import voxpipe_oracle as O  # noqa: E402
from paper_2012_13846_b200 import _lib, model  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 32
dev = torch.device("cuda")
tr = model.SparseResNetTrainer(batch=64, points=2048, resolution=64)
pts, offs = O.synthetic_batch(64, 2048, 64, seed=1000, dtype=np.float32)
tr.train_step_from_host(pts, offs, np.arange(64) % 40)
st = torch.cuda.current_stream().cuda_stream
for L in tr.layers:
    if L["cin"] != c or L["cout"] != c:
        continue
    x, w, nbr = L["x"], L["wb"], tr.fwd_table(L)
    perm = tr.fwd_perm(L)
    n = int(L["dst"].n.item())
    y = torch.empty_like(L["y"])
    ws = _lib.workspace(_lib.query("vp_conv_fwd_ws_bytes", c, c, tr.K), dev)
    print(f"layer {L['name']} rows {n} tiles {(n + 127) // 128}")
    for cap in sorted({n, 296 * 128, 2 * 296 * 128, 3 * 296 * 128, 4 * 296 * 128}):
        if cap > n:
            continue
        cnt = torch.tensor([cap], dtype=torch.int32, device=dev)

        def launch():
            _lib.call("vp_conv_fwd", x.data_ptr(), _lib.VP_BF16, x.shape[0], c, w.data_ptr(), _lib.VP_BF16, c, tr.K,
                      nbr.data_ptr(), 0, _lib.ptr(perm), cnt.data_ptr(), nbr.shape[0], y.data_ptr(), _lib.VP_BF16,
                      ws.data_ptr(), ws.numel(), st)

        for _ in range(5):
            launch()
        ts = []
        for _ in range(50):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            launch()
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        print(f"  rows {cap:7d} tiles {(cap + 127) // 128:5d} rounds {(cap + 127) // 128 / 296:5.2f}  "
              f"{np.median(ts):7.2f} us")
