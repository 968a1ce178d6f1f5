"""Critical-path breakdown of the captured C3 training step: CUDA-graph
replays of growing prefixes of the step (integer stage; + forward; + backward;
+ optimizer), device-timed, L2 flushed between replays."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import voxpipe_oracle as O  # noqa: E402
from paper_2012_13846_b200 import _lib, model  # noqa: E402

tr = model.SparseResNetTrainer(batch=64, points=2048, resolution=64)
pts, _ = O.synthetic_batch(64, 2048, 64, seed=0, dtype=np.float32)
tr.set_batch(torch.from_numpy(pts).cuda(), torch.arange(64, dtype=torch.int32).cuda() % 40)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def body(upto):
    st = _lib.stream()
    tr.launch_count = 0
    tr._integer_stage(st)
    if upto >= 1:
        tr._forward(st)
    if upto >= 2:
        tr._backward(st)
    if upto >= 3:
        tr._optimizer(st)
    tr.join_side_streams()


for upto, name in enumerate(["integer stage", "+ forward", "+ backward", "+ optimizer (full step)"]):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        body(upto)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        body(upto)
    ts = []
    for i in range(30):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        if i >= 5:
            ts.append(a.elapsed_time(b) * 1e3)
    print(f"{name:28s} {np.median(ts):8.1f} us  (kernels {tr.launch_count})")
