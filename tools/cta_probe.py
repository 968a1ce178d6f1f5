"""GPU: per-CTA start / end (globaltimer) of the tensor-core conv on a real C3
layer (its own table, activations and weights): where a launch's time goes
(CTA start spread, per-CTA work, the slowest CTA).  The kernel records
(start, end, items, stages) per CTA when a debug trace buffer is set.
Usage: python tools/cta_probe.py [C]"""
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
L = [L for L in tr.layers if L["cin"] == c and L["cout"] == c and L["kind"] == "c1"][0]
x, w, nbr, perm = L["x"], L["wb"], tr.fwd_table(L), tr.fwd_perm(L)
n = int(L["dst"].n.item())
y = torch.empty_like(L["y"])
ws = _lib.workspace(_lib.query("vp_conv_fwd_ws_bytes", c, c, tr.K), dev)
buf = torch.zeros(2048 + 4 * 1024, dtype=torch.int64, device=dev)


def launch(cnt):
    _lib.call("vp_conv_fwd", x.data_ptr(), _lib.VP_BF16, x.shape[0], c, w.data_ptr(), _lib.VP_BF16, c, tr.K,
              nbr.data_ptr(), 0, _lib.ptr(perm), cnt.data_ptr(), nbr.shape[0], y.data_ptr(), _lib.VP_BF16,
              ws.data_ptr(), ws.numel(), st)


hits = (nbr[:n] >= 0).cpu().numpy()
print(f"layer {L['name']} rows {n} tiles {(n + 127) // 128} hits/row {hits.sum() / n:.2f}")
# active offsets per 128-row tile (what the kernel's scan finds)
act = np.array([hits[i:i + 128].any(0).sum() for i in range(0, n, 128)])
print(f"active offsets per tile: mean {act.mean():.1f} min {act.min()} max {act.max()} "
      f"quartiles {np.percentile(act, [25, 50, 75])}")
for cap in (296 * 128, n):
    cnt = torch.tensor([min(cap, n)], dtype=torch.int32, device=dev)
    for _ in range(3):
        launch(cnt)
    torch.cuda.synchronize()
    buf.zero_()
    _lib.call("vp_debug_conv_trace", buf.data_ptr())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    launch(cnt)
    e1.record()
    torch.cuda.synchronize()
    _lib.call("vp_debug_conv_trace", None)
    r = buf[2048:].view(-1, 4).cpu().numpy()
    r = r[r[:, 0] > 0]
    t0 = r[:, 0].min()
    s, e = (r[:, 0] - t0) / 1e3, (r[:, 1] - t0) / 1e3
    d = e - s
    print(f"\nrows {int(cnt.item())}: kernel (events) {e0.elapsed_time(e1) * 1e3:.1f} us, CTAs {len(r)}")
    print(f"  start spread: median {np.median(s):.2f} max {s.max():.2f} us")
    print(f"  end:          median {np.median(e):.2f} p90 {np.percentile(e, 90):.2f} max {e.max():.2f} us")
    print(f"  duration:     median {np.median(d):.2f} max {d.max():.2f} us")
    print(f"  stages/CTA:   mean {r[:, 3].mean():.1f} max {r[:, 3].max()}  items/CTA max {r[:, 2].max()}")
    if r[:, 3].std() > 0:
        print(f"  corr(duration, stages) {np.corrcoef(d, r[:, 3])[0, 1]:.2f}; us per stage (fit) "
              f"{np.polyfit(r[:, 3], d, 1)}")
    idx = np.argsort(-e)[:8]
    for i in idx:
        print(f"   slow CTA: start {s[i]:6.2f} end {e[i]:6.2f} items {r[i, 2]} stages {r[i, 3]}")
