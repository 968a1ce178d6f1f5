import os, sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/oracle")
import numpy as np, torch
import voxpipe_oracle as O
from paper_2012_13846_b200 import model, _lib
tr = model.SparseResNetTrainer(batch=64, points=2048, resolution=64)
pts, offs = O.synthetic_batch(64, 2048, 64, seed=0, dtype=np.float32)
tr.train_step_from_host(pts, offs, (np.arange(64) % 40).astype(np.int32))
torch.cuda.synchronize()
pb = tr.params; Ll = tr.layers[-1]; last = tr.levels[-1]; C = 256
def head(bn=True):
    _lib.call("vp_sparse_head", Ll["a"].data_ptr(), tr.fcode, last.seg.data_ptr(), tr.B, C,
              pb.view(pb.p, "fc.w").data_ptr(), pb.view(pb.p, "fc.b").data_ptr(), tr.classes,
              tr.labels.data_ptr(), tr.pooled.data_ptr(), tr.logits.data_ptr(), tr.loss.data_ptr(),
              pb.view(pb.g, "fc.w").data_ptr(), pb.view(pb.g, "fc.b").data_ptr(), Ll["a"].data_ptr(),
              Ll["y"].data_ptr() if bn else None, Ll["mean"].data_ptr(), Ll["rstd"].data_ptr(), tr._gm_buf(Ll).data_ptr(),
              Ll["bpart"].data_ptr(), Ll["ggamma"].data_ptr(), Ll["gbeta"].data_ptr(), tr.head_ws.data_ptr(),
              tr.head_ws.numel(), _lib.stream())
from torch.profiler import profile, ProfilerActivity
for bn in (True, False):
    for _ in range(3): head(bn)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(5): head(bn)
        torch.cuda.synchronize()
    for e in prof.key_averages():
        if "head" in e.key: print(bn, e.key[:40], round(e.device_time_total / e.count, 2) if e.count else 0, e.count)
print("B", tr.B, "seg", last.seg[:4].tolist(), last.seg[64:68].tolist(), "n", int(last.n.item()))
