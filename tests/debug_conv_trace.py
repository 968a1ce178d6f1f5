"""Debug helper (GPU): per-stage producer/MMA timeline of CTA 0 for a few
conv layers of the C3 step. Not collected by pytest."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np, torch
import voxpipe_oracle as O
from paper_2012_13846_b200 import _lib, model

tr = model.SparseResNetTrainer(batch=64, points=2048, resolution=64)
pts, offs = O.synthetic_batch(64, 2048, 64, seed=0, dtype=np.float32)
tr.train_step_from_host(pts, offs, np.arange(64) % 40)
torch.cuda.synchronize()
lib = _lib.load()
lib.vp_debug_set_trace.argtypes = [ctypes.c_void_p]
buf = torch.zeros(512 * 4, dtype=torch.int64, device="cuda")
for name in ["s0.b0.c1", "s1.b0.c1", "s2.b0.c1", "s3.b0.c1"]:
    L = [l for l in tr.layers if l["name"] == name][0]
    dst = L["dst"]
    st = torch.cuda.current_stream().cuda_stream
    def launch():
        _lib.call("vp_conv_fwd", L["x"].data_ptr(), _lib.VP_BF16, L["x"].shape[0], L["cin"], L["wb"].data_ptr(), _lib.VP_BF16,
                  L["cout"], tr.K, L["map"].nbr.data_ptr(), 0, dst.n.data_ptr(), dst.cap, L["y"].data_ptr(),
                  _lib.VP_BF16, L["fwd_ws"].data_ptr(), L["fwd_ws"].numel(), st)
    launch(); torch.cuda.synchronize()
    buf.zero_(); lib.vp_debug_set_trace(buf.data_ptr())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); launch(); e1.record(); torch.cuda.synchronize()
    lib.vp_debug_set_trace(None)
    t = buf.view(512, 4).cpu().numpy().astype(np.float64)
    n = int((t[:, 0] > 0).sum())
    t0 = t[0, 0]
    print(f"== {name} cin={L['cin']} cout={L['cout']} rows={int(dst.n.item())} kernel {e0.elapsed_time(e1)*1e3:.1f} us, CTA0 stages={n}")
    for g in range(min(n, 40)):
        a, b, c, d = (t[g] - t0) / 1e3
        print(f"  g={g:3d} prod_start {a:8.2f} prod_gotslot {b:8.2f} mma_full {c:8.2f} mma_done {d:8.2f}  (us)")
    if n > 1:
        print(f"  last stage mma at {(t[n-1,3]-t0)/1e3:.2f} us")
