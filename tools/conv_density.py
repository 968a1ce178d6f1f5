"""GPU microbenchmark: vp_conv_fwd time vs neighbour-table density on
synthetic tables (random rows), to separate per-stage overheads from gather
bandwidth.  Usage: python tools/conv_density.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2012_13846_b200 import _lib  # noqa: E402


def run(n, c, density, K=27, iters=20, local=False):
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(0)
    x = torch.randn(n, c, device=dev).to(torch.bfloat16)
    w = (torch.randn(K, c, c, device=dev) / 16).to(torch.bfloat16)
    if local:  # neighbours near the row itself (spatially coherent gathers)
        rows = (torch.arange(n, device=dev)[:, None] + torch.randint(-64, 64, (n, K), device=dev, generator=g)).clamp(0, n - 1)
    else:
        rows = torch.randint(0, n, (n, K), device=dev, generator=g)
    keep = torch.rand(n, K, device=dev, generator=g) < density
    nbr = torch.where(keep, rows, torch.full_like(rows, -1)).to(torch.int32).contiguous()
    ncount = torch.tensor([n], dtype=torch.int32, device=dev)
    y = torch.empty(n, c, dtype=torch.bfloat16, device=dev)
    ws = _lib.workspace(_lib.query("vp_conv_fwd_ws_bytes", c, c, K), dev)
    st = torch.cuda.current_stream().cuda_stream

    def launch():
        _lib.call("vp_conv_fwd", x.data_ptr(), _lib.VP_BF16, n, c, w.data_ptr(), _lib.VP_BF16, c, K, nbr.data_ptr(), 0, None,
                  ncount.data_ptr(), n, y.data_ptr(), _lib.VP_BF16, ws.data_ptr(), ws.numel(), st)

    for _ in range(3):
        launch()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        launch()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / iters
    tiles = (n + 127) // 128
    act = (keep.view(-1)[: tiles * 0] if False else None)
    # active offsets per tile
    kp = torch.nn.functional.pad(keep, (0, 0, 0, tiles * 128 - n)).view(tiles, 128, K).any(1).sum(1).float()
    units = (kp / 2).ceil() if c == 32 else kp * (c // 64)
    stages = float(units.sum())
    print(f"n={n} C={c} density={density:.2f} local={local}: {us:7.1f} us  stages={stages:.0f} "
          f"-> {us / (max(stages, 1) / 148):.3f} us/stage/SM  pairs={int(keep.sum())}")


if __name__ == "__main__":
    for c in (32, 64, 128):
        for d in (0.0, 0.05, 0.25, 1.0):
            run(82000, c, d)
        run(82000, c, 0.25, local=True)
