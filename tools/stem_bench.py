"""Device time of the stem conv (C_in = 1 -> 32, 27 offsets) at the C3 level-0
shape through vp_conv_fwd: 20 launches captured in a CUDA graph."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import voxpipe_oracle as O  # noqa: E402
from paper_2012_13846_b200 import _lib, conv, tensor  # noqa: E402

dev = torch.device("cuda")
pts, offs = O.synthetic_batch(64, 2048, 64, seed=7, dtype=np.float32)
t = tensor.voxelize_batch(torch.from_numpy(pts).to(dev), torch.from_numpy(offs), 1.0, (64, 64, 64),
                          feature_dtype=torch.bfloat16)
n = len(t)
km = conv._kernel_map4(t.coords4, t.coords4, conv.KernelShape.hypercubic(3, 3), (1, 1, 1), 3)
w = (torch.randn(27, 32, 1, device=dev) / 5).to(torch.bfloat16)
y = torch.empty(n, 32, dtype=torch.bfloat16, device=dev)
nd = torch.tensor([n], dtype=torch.int32, device=dev)
ws = _lib.workspace(_lib.query("vp_conv_fwd_ws_bytes", 1, 32, 27), dev)


def fwd():
    _lib.call("vp_conv_fwd", t.features.data_ptr(), 1, n, 1, w.data_ptr(), 1, 32, 27, km.nbr.data_ptr(), 0, None,
              nd.data_ptr(), n, y.data_ptr(), 1, ws.data_ptr(), ws.numel(), torch.cuda.current_stream().cuda_stream)


fwd()
torch.cuda.synchronize()
s = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    for _ in range(20):
        fwd()
g.replay()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5):
    g.replay()
b.record()
torch.cuda.synchronize()
print(f"stem fwd N={n}: {a.elapsed_time(b) * 1e3 / 100:.2f} us")
