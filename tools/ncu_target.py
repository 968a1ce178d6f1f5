"""Launch ONE kernel of the C3 training step in isolation for ncu
(`ncu --profile-from-start off ...`): builds the C3 trainer, trains one step
on the bench's first synthetic batch, then brackets exactly one launch of the
requested layer/mode with cudaProfilerStart/Stop.  The launches are the ones
bench.py's `roofline` times (plain C-ABI entry points on the step's own
tables and activations), plus the fused-epilogue variants the step runs.

  python tools/ncu_target.py --layer s1.b0.c2 --mode wgrad
  modes: fwd dgrad wgrad fwd_bn dgrad_bn map
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import voxpipe_oracle as O  # noqa: E402
from paper_2012_13846_b200 import _lib, model  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layer", default="s1.b0.c2")
    ap.add_argument("--mode", default="wgrad")
    a = ap.parse_args()
    tr = model.SparseResNetTrainer(batch=64, points=2048, resolution=64)
    pts, offs = O.synthetic_batch(64, 2048, 64, seed=0, dtype=np.float32)  # bench.py's batch 0 (rank 0)
    tr.train_step_from_host(pts, offs, (np.arange(64) % 40).astype(np.int32))
    torch.cuda.synchronize()
    st = torch.cuda.current_stream().cuda_stream
    fc = _lib.VP_BF16
    idx = {L["name"]: i for i, L in enumerate(tr.layers)}
    if a.mode == "map":
        m = tr.map_s1[0]

        def launch():
            if tr.use_grid:
                tr._grid_set(0, st, clear=False)
            tr._build_map(m, st)
            if tr.use_grid:
                tr._grid_set(0, st, clear=True)
    else:
        L = tr.layers[idx[a.layer]]
        src, dst, m, x = L["src"], L["dst"], L["map"], L["x"]
        conv = (x.data_ptr(), fc, x.shape[0], L["cin"], L["wb"].data_ptr(), fc, L["cout"], tr.K,
                tr.fwd_table(L).data_ptr(), 0, _lib.ptr(tr.fwd_perm(L)), dst.n.data_ptr(), dst.cap,
                L["y"].data_ptr(), fc, L["fwd_ws"].data_ptr(), L["fwd_ws"].numel())
        table, flip, perm = tr.dgrad_table(L)
        gin = torch.empty((src.cap, L["cin"]), dtype=torch.bfloat16, device="cuda")
        dg = (L["gy"].data_ptr(), fc, L["gy"].shape[0], L["cout"], L["wb"].data_ptr(), fc, L["cin"], tr.K,
              table.data_ptr(), flip, _lib.ptr(perm), src.n.data_ptr(), src.cap, gin.data_ptr(), fc,
              L["dg_ws"].data_ptr(), L["dg_ws"].numel())
        P = tr.layers[idx[a.layer] - 1] if idx[a.layer] > 0 else None
        launches = {
            "fwd": lambda: _lib.call("vp_conv_fwd", *conv, st),
            "fwd_bn": lambda: _lib.call("vp_conv_fwd_bn", *conv, 1, L["fpart"].data_ptr(), None, None, None, None, 1e-5, L["mean"].data_ptr(), L["rstd"].data_ptr(), None, st),
            "dgrad": lambda: _lib.call("vp_conv_dgrad", *dg, st),
            "dgrad_bn": lambda: _lib.call("vp_conv_dgrad_bn", *dg, 2, P["bpart"].data_ptr(), None, P["a"].data_ptr(),
                                          P["y"].data_ptr(), P["mean"].data_ptr(), 0.0, P["ggamma"].data_ptr(), P["gbeta"].data_ptr(), P["rstd"].data_ptr(), st),
            "wgrad": lambda: _lib.call("vp_conv_wgrad", x.data_ptr(), fc, L["cin"], L["gy"].data_ptr(), fc, L["cout"],
                                       tr.K, m.pin.data_ptr(), m.pout.data_ptr(), m.ptr.data_ptr(), m.pin.numel(),
                                       L["gw"].data_ptr(), L["wg_ws"].data_ptr(), L["wg_ws"].numel(), st),
        }
        launch = launches[a.mode]
    for _ in range(2):
        launch()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    launch()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print(f"ncu target done: {a.layer} {a.mode}")


if __name__ == "__main__":
    main()
