"""GPU: clock64 timeline of CTA 0 of vp_conv_fwd on a synthetic table
(density d, random rows).  Usage: python tools/conv_trace.py [C] [density]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2012_13846_b200 import _lib  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 32
d = float(sys.argv[2]) if len(sys.argv) > 2 else 0.25
n = int(sys.argv[3]) if len(sys.argv) > 3 else 82000
K = 27
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
x = torch.randn(n, c, device=dev).to(torch.bfloat16)
w = (torch.randn(K, c, c, device=dev) / 16).to(torch.bfloat16)
rows = torch.randint(0, n, (n, K), device=dev, generator=g)
keep = torch.rand(n, K, device=dev, generator=g) < d
nbr = torch.where(keep, rows, torch.full_like(rows, -1)).to(torch.int32).contiguous()
ncount = torch.tensor([n], dtype=torch.int32, device=dev)
y = torch.empty(n, c, dtype=torch.bfloat16, device=dev)
ws = _lib.workspace(_lib.query("vp_conv_fwd_ws_bytes", c, c, K), dev)
st = torch.cuda.current_stream().cuda_stream


if len(sys.argv) > 4 and sys.argv[4] == "real":
    # a real C3 layer: the trainer's level tables and activations
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import voxpipe_oracle as O
    from paper_2012_13846_b200 import model
    tr = model.SparseResNetTrainer(batch=64, points=2048, resolution=64)
    pts, offs = O.synthetic_batch(64, 2048, 64, seed=1000, dtype=np.float32)
    tr.train_step_from_host(pts, offs, np.arange(64) % 40)
    L = [L for L in tr.layers if L["cin"] == c and L["cout"] == c and L["kind"] == "c1"][0]
    x = L["x"]
    w = L["wb"]
    nbr = tr.fwd_table(L)
    n = int(L["dst"].n.item())
    ncount = L["dst"].n
    y = L["y"]
    print("layer", L["name"], "rows", n, "hits/row", float((nbr[:n] >= 0).sum()) / n)


def launch():
    _lib.call("vp_conv_fwd", x.data_ptr(), _lib.VP_BF16, x.shape[0], c, w.data_ptr(), _lib.VP_BF16, c, K, nbr.data_ptr(),
              0, None, ncount.data_ptr(), nbr.shape[0], y.data_ptr(), _lib.VP_BF16, ws.data_ptr(), ws.numel(), st)


launch()
torch.cuda.synchronize()
buf = torch.zeros(1280, dtype=torch.int64, device=dev)
_lib.call("vp_debug_conv_trace", buf.data_ptr())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
launch()
e1.record()
torch.cuda.synchronize()
_lib.call("vp_debug_conv_trace", None)
t = buf.cpu().numpy().astype(np.float64)
st_ev = t[:1024].reshape(256, 4)
tl_ev = t[1024:].reshape(64, 4)
valid = tl_ev[:, 0] > 0
t0 = tl_ev[0, 0]
ghz = 1.965
print(f"C={c} density={d} kernel {e0.elapsed_time(e1) * 1e3:.1f} us")
for i in range(int(valid.sum())):
    a = (tl_ev[i] - t0) / ghz / 1e3
    b = (st_ev[i] - t0) / ghz / 1e3
    print(f" tile {i}: prologue {a[0]:7.2f} -> all in {b[0]:7.2f} scan {b[1]:7.2f} mask {b[2]:7.2f} -> published {a[1]:7.2f}  mma saw {b[3]:7.2f}  epi got acc {a[2]:7.2f} done {a[3]:7.2f} us")
ns = int((st_ev[:, 0] > 0).sum())
for gg in range(min(ns, 60)):
    a = (st_ev[gg] - t0) / ghz / 1e3
    print(f"  g={gg:3d} slot {a[0]:7.2f} issued {a[1]:7.2f} mma_full {a[2]:7.2f} committed {a[3]:7.2f}")
