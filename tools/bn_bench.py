"""Microbenchmark of the BN glue kernels at the C3 layer shapes: device time
per launch (20 back-to-back launches captured in a CUDA graph)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2012_13846_b200 import _lib  # noqa: E402

dev = torch.device("cuda")
st = torch.cuda.current_stream()
SHAPES = [(115000, 131072, 32), (83000, 131072, 32), (37500, 131072, 64), (10700, 32768, 128),
          (2600, 4096, 256)]
if len(sys.argv) > 1 and sys.argv[1] == "floor":  # fixed cost: almost no rows at the same capacities
    SHAPES = [(64, cap, C) for _, cap, C in SHAPES]
for n, cap, C in SHAPES:
    x = torch.randn(cap, C, device=dev).to(torch.bfloat16)
    nd = torch.tensor([n], dtype=torch.int32, device=dev)
    mean = torch.zeros(C, device=dev)
    rstd = torch.zeros(C, device=dev)
    g = torch.ones(C, device=dev)
    b = torch.zeros(C, device=dev)
    y = torch.empty_like(x)
    ws = torch.zeros(int(_lib.query("vp_bn_stats_ws_bytes", cap, C)), dtype=torch.uint8, device=dev)

    def stats():
        _lib.call("vp_bn_stats", x.data_ptr(), 1, nd.data_ptr(), cap, C, 1e-5, mean.data_ptr(), rstd.data_ptr(),
                  ws.data_ptr(), ws.numel(), torch.cuda.current_stream().cuda_stream)

    def apply():
        _lib.call("vp_bn_apply", x.data_ptr(), 1, nd.data_ptr(), cap, C, mean.data_ptr(), rstd.data_ptr(),
                  g.data_ptr(), b.data_ptr(), None, 1, 1, y.data_ptr(), 1, torch.cuda.current_stream().cuda_stream)

    gy = torch.randn(cap, C, device=dev).to(torch.bfloat16)
    gx = torch.empty_like(x)
    gg = torch.zeros(C, device=dev)
    gb = torch.zeros(C, device=dev)
    wsb = torch.zeros(int(_lib.query("vp_bn_backward_ws_bytes", cap, C)), dtype=torch.uint8, device=dev)

    def backward():
        _lib.call("vp_bn_backward", gy.data_ptr(), None, 1, y.data_ptr(), 1, x.data_ptr(), 1, nd.data_ptr(), cap, C,
                  mean.data_ptr(), rstd.data_ptr(), g.data_ptr(), 1, gx.data_ptr(), 1, None, gg.data_ptr(),
                  gb.data_ptr(), wsb.data_ptr(), wsb.numel(), torch.cuda.current_stream().cuda_stream)

    def forward():
        _lib.call("vp_bn_forward", x.data_ptr(), 1, nd.data_ptr(), cap, C, 1e-5, mean.data_ptr(), rstd.data_ptr(),
                  g.data_ptr(), b.data_ptr(), None, 1, 1, y.data_ptr(), 1, ws.data_ptr(), ws.numel(),
                  torch.cuda.current_stream().cuda_stream)

    def tiny():
        nd.add_(0)

    res = []
    for fn in (stats, apply, forward, backward, tiny):
        fn()
        torch.cuda.synchronize()
        s = torch.cuda.Stream()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=s):
            for _ in range(20):
                fn()
        gr.replay()
        torch.cuda.synchronize()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            gr.replay()
        e.record()
        torch.cuda.synchronize()
        res.append(a.elapsed_time(e) * 1e3 / 100)
    mb = n * C * 2 / 1e6
    print(f"N={n:6d} C={C:3d} ({mb:5.1f} MB): stats {res[0]:6.2f} us  apply {res[1]:6.2f} us  forward {res[2]:6.2f} us  backward {res[3]:6.2f} us  (1-elem op {res[4]:5.2f} us)")
