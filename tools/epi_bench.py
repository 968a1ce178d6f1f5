"""Per-layer cost of the fused BN epilogue: each C3 layer's forward conv
plain vs with mode-1 statistics, and its dgrad plain vs with the mode-2
(masked gradient + statistics) epilogue for the previous layer, on the
trainer's own buffers after a step (warm L2, CUDA events, 30 reps)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import voxpipe_oracle as O  # noqa: E402
from paper_2012_13846_b200 import _lib, model  # noqa: E402


def timed(fn, reps=30):
    """reps back-to-back launches captured in one CUDA graph (no host
    overhead between them), replayed and timed with events."""
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s_ = torch.cuda.Stream()
    with torch.cuda.stream(s_):
        with torch.cuda.graph(g, stream=s_):
            for _ in range(reps):
                fn()
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) * 1000 / reps


tr = model.SparseResNetTrainer(batch=64, points=2048, resolution=64)
pts, offs = O.synthetic_batch(64, 2048, 64, seed=1000, dtype=np.float32)
tr.train_step_from_host(pts, offs, np.arange(64) % 40)
torch.cuda.synchronize()
fc = tr.fcode
print(f"{'layer':12s} {'fwd':>7s} {'fwd+m1':>7s} {'dgrad':>7s} {'dg+m2':>7s} {'apply':>7s} {'bwdapp':>7s} {'bnfwd0':>7s} {'bnbwd0':>7s}")
for i, L in enumerate(tr.layers):
    dst, src = L["dst"], L["src"]
    x = L["x"]
    conv = (x.data_ptr(), fc, x.shape[0], L["cin"], L["wb"].data_ptr(), L["wcode"], L["cout"], tr.K,
            tr.fwd_table(L).data_ptr(), 0, _lib.ptr(tr.fwd_perm(L)), dst.n.data_ptr(), dst.cap,
            L["y"].data_ptr(), fc, L["fwd_ws"].data_ptr(), L["fwd_ws"].numel())
    f0 = timed(lambda: _lib.call("vp_conv_fwd", *conv, _lib.stream()))
    f1 = timed(lambda: _lib.call("vp_conv_fwd_bn", *conv, 1, L["fpart"].data_ptr(), None, None, None, None, 1e-5, L["mean"].data_ptr(), L["rstd"].data_ptr(), None, _lib.stream()))
    ap = timed(lambda: _lib.call("vp_bn_apply_part", L["y"].data_ptr(), fc, dst.n.data_ptr(), dst.cap, L["cout"], 1e-5,
                                 L["fpart"].data_ptr(), L["mean"].data_ptr(), L["rstd"].data_ptr(),
                                 L["gamma"].data_ptr(), L["beta"].data_ptr(), None, fc, 1, L["a"].data_ptr(), fc, _lib.stream()))
    of = timed(lambda: _lib.call("vp_bn_forward", L["y"].data_ptr(), fc, dst.n.data_ptr(), dst.cap, L["cout"], 1e-5,
                                 L["mean"].data_ptr(), L["rstd"].data_ptr(), L["gamma"].data_ptr(), L["beta"].data_ptr(),
                                 None, fc, 1, L["a"].data_ptr(), fc, L["bn_ws"].data_ptr(), L["bn_ws"].numel(),
                                 _lib.stream()))
    ob = timed(lambda: _lib.call("vp_bn_backward", L["a"].data_ptr(), None, fc, L["a"].data_ptr(), fc,
                                 L["y"].data_ptr(), fc, dst.n.data_ptr(), dst.cap, L["cout"], L["mean"].data_ptr(),
                                 L["rstd"].data_ptr(), L["gamma"].data_ptr(), 1, L["gy"].data_ptr(), fc, None,
                                 L["ggamma"].data_ptr(), L["gbeta"].data_ptr(), L["bn_ws"].data_ptr(),
                                 L["bn_ws"].numel(), _lib.stream()))
    d0 = d2 = bp = float("nan")
    if i > 0:
        P = tr.layers[i - 1]
        table, flip, perm = tr.dgrad_table(L)
        gin = torch.empty((src.cap, L["cin"]), dtype=tr.fdt, device="cuda")
        dg = (L["gy"].data_ptr(), fc, L["gy"].shape[0], L["cout"], L["wb"].data_ptr(), L["wcode"], L["cin"], tr.K,
              table.data_ptr(), flip, _lib.ptr(perm), src.n.data_ptr(), src.cap, gin.data_ptr(), fc,
              L["dg_ws"].data_ptr(), L["dg_ws"].numel())
        d0 = timed(lambda: _lib.call("vp_conv_dgrad", *dg, _lib.stream()))
        d2 = timed(lambda: _lib.call("vp_conv_dgrad_bn", *dg, 2, P["bpart"].data_ptr(), None, P["a"].data_ptr(),
                                     P["y"].data_ptr(), P["mean"].data_ptr(), 0.0, P["ggamma"].data_ptr(), P["gbeta"].data_ptr(), P["rstd"].data_ptr(), _lib.stream()))
        bp = timed(lambda: _lib.call("vp_bn_backward_part", gin.data_ptr(), fc, P["y"].data_ptr(), fc,
                                     P["dst"].n.data_ptr(), P["dst"].cap, P["cout"], P["mean"].data_ptr(),
                                     P["rstd"].data_ptr(), P["gamma"].data_ptr(), P["bpart"].data_ptr(),
                                     P["gy"].data_ptr(), fc, P["ggamma"].data_ptr(), P["gbeta"].data_ptr(), _lib.stream()))
    print(f"{L['name']:12s} {f0:7.2f} {f1:7.2f} {d0:7.2f} {d2:7.2f} {ap:7.2f} {bp:7.2f} {of:7.2f} {ob:7.2f}")
