"""Per-kernel breakdown of the kernel-map builders under CUPTI, each build
after an L2 flush (as bench.py's roofline.map times it):
  * the trainer's dense-grid path at C3 level 0 (grid set + probe + scan +
    emit + clear), on the bench's first batch;
  * the operator API's hash path (vp_kernel_map) at 1M rows (552 C2 clouds).
Prints mean us per kernel and the mean span (first start -> last end)."""
import collections
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import voxpipe_oracle as O  # noqa: E402
from paper_2012_13846_b200 import conv, model, tensor  # noqa: E402
from paper_2012_13846_b200 import roofline as RL  # noqa: E402

flush = RL.Flusher(torch.device("cuda"))


def breakdown(tag, launch, iters=10):
    for _ in range(3):
        flush()
        launch()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(iters):
            flush()
            launch()
        torch.cuda.synchronize()
    evs = sorted((e.time_range.start, e.time_range.end, e.name) for e in prof.events()
                 if e.device_type.name == "CUDA" and e.time_range.elapsed_us() > 0)
    per = collections.defaultdict(list)
    spans, cur = [], None
    for s, e, n in evs:
        if "elementwise" in n or "fill" in n.lower() and "Memset" not in n:  # the L2 flush
            if cur:
                spans.append(cur[1] - cur[0])
            cur = None
            continue
        short = n.split("(")[0].replace("void ", "").split("<")[0][:40]
        per[short].append(e - s)
        cur = [s, e] if cur is None else [cur[0], max(cur[1], e)]
    if cur:
        spans.append(cur[1] - cur[0])
    print(f"== {tag}: span {np.mean(spans):.1f} us (first start -> last end), {len(spans)} builds")
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        print(f"   {k:40s} {len(v) / len(spans):4.1f}x  {np.mean(v):8.2f} us")


if "--hash-only" not in sys.argv:
    tr = model.SparseResNetTrainer(batch=64, points=2048, resolution=64)
    pts, offs = O.synthetic_batch(64, 2048, 64, seed=0, dtype=np.float32)
    tr.train_step_from_host(pts, offs, (np.arange(64) % 40).astype(np.int32))
    torch.cuda.synchronize()
    st = torch.cuda.current_stream().cuda_stream
    m = tr.map_s1[0]

    def grid_map():
        tr._grid_set(0, st, clear=False)
        tr._build_map(m, st)
        tr._grid_set(0, st, clear=True)

    breakdown(f"C3 level 0 grid map (N={int(m.src.n.item())}, pairs={int(m.ptr[-1].item())})", grid_map)
    del tr
    torch.cuda.empty_cache()
dev = torch.device("cuda")
shape = conv.KernelShape.hypercubic(3, 3)
pts, offs = O.synthetic_batch(552, 2048, 64, seed=7, dtype=np.float32)
t = tensor.voxelize_batch(torch.from_numpy(pts).to(dev), torch.from_numpy(offs), 1.0, (64, 64, 64),
                          feature_dtype=torch.bfloat16)
c4 = t.coords4
breakdown(f"hash map, 1M rows (N={len(t)})", lambda: conv._kernel_map4(c4, c4, shape, (1, 1, 1), 3))

# the dense-grid index on the same 1M rows (B = 552 clouds at 64^3)
from paper_2012_13846_b200 import _lib  # noqa: E402

B, R, K = 552, 64, 27
n = len(t)
grid = torch.zeros(int(_lib.query("vp_grid_words", B, R)), dtype=torch.int32, device=dev)
nbr = torch.empty((n, K), dtype=torch.int32, device=dev)
pin = torch.empty(n * K, dtype=torch.int32, device=dev)
pout = torch.empty(n * K, dtype=torch.int32, device=dev)
ptr = torch.empty(K + 1, dtype=torch.int32, device=dev)
ws = _lib.workspace(_lib.query("vp_kernel_map_grid_ws_bytes", n, K), dev)
offs3 = _lib.i32_array(shape.offsets3().ravel())
one = _lib.i32_array((1, 1, 1))
st = _lib.stream()


def grid_map_1m():
    _lib.call("vp_grid_set", c4.data_ptr(), None, n, grid.data_ptr(), B, R, 1, 0, st)
    _lib.call("vp_kernel_map_grid", grid.data_ptr(), B, R, 1, c4.data_ptr(), None, n, offs3, K, one, nbr.data_ptr(),
              pin.data_ptr(), pout.data_ptr(), ptr.data_ptr(), ws.data_ptr(), ws.numel(), st)
    _lib.call("vp_grid_set", c4.data_ptr(), None, n, grid.data_ptr(), B, R, 1, 1, st)


breakdown(f"grid map, 1M rows (N={n})", grid_map_1m)
km = conv._kernel_map4(c4, c4, shape, (1, 1, 1), 3)
assert int(ptr[-1].item()) == km.total_pairs()
assert torch.equal(nbr, km.nbr), "grid and hash maps differ"
print("grid == hash map at 1M rows")
