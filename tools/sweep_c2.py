"""BASELINE config C2: single sparse-conv layer sweep on 1xB200 — N = 10k-1M
active voxels (6 / 55 / 552 synthetic ModelNet40-shaped clouds x 2048 pts at
64^3), C_in = C_out in {32, 64, 128, 256}, kernel 3^3, stride 1 / 2 and the
transposed (stride-2 adjoint) conv, forward + dgrad + wgrad.

Every kernel is timed alone with CUDA events on its launch stream, the L2
flushed before every launch (paper_2012_13846_b200/roofline.py), and reported
against SURVEY §8(d)'s algorithmic work:
  map  : B = 16 N_in + 16 N_out + 8 P                      (HBM bound)
  conv : F = 2 P C_in C_out ; B = 2 N_in C_in + 2 N_out C_out + 2*27*C_in*C_out
         + 8 P (wgrad: + 4*27*C_in*C_out fp32 instead of the bf16 weights)
         -> bound = tensor if F/B*HBM > TC
Prints one JSON line per (N, C, mode) and writes them to --out."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import voxpipe_oracle as O  # noqa: E402
from paper_2012_13846_b200 import _lib, conv, tensor  # noqa: E402
from paper_2012_13846_b200 import roofline as RL  # noqa: E402

HBM, TC, _ = RL.peaks()
_FLUSH = []


def timeit(fn, iters):
    if not _FLUSH:
        _FLUSH.append(RL.Flusher(torch.device("cuda")))
    return RL.time_cold(fn, _FLUSH[0], iters)


def conv_roof(P, n_in, n_out, cin, cout, t, mode="fwd"):
    F, B = RL.conv_work(P, n_in, n_out, cin, cout, 27, mode)
    r = RL.classify(F, B, t, HBM, TC)
    return {"us": r["us_per_launch"], "tflops": r["tflops"], "gbs": r["gbs"], "bound": r["bound"],
            "frac": r["frac"], "F": F, "B": B}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--clouds", default="6,55,552")
    ap.add_argument("--channels", default="32,64,128,256")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--out", default="gpurun_out/c2_sweep.jsonl")
    ap.add_argument("--no-sort", dest="sort", action="store_false", help="voxelization row order (no mask sort)")
    a = ap.parse_args()
    dev = torch.device("cuda")
    shape = conv.KernelShape.hypercubic(3, 3)
    K = 27
    st = torch.cuda.current_stream().cuda_stream
    out = open(a.out, "w")
    for nc in [int(v) for v in a.clouds.split(",")]:
        pts, offs = O.synthetic_batch(nc, 2048, 64, seed=7, dtype=np.float32)
        t = tensor.voxelize_batch(torch.from_numpy(pts).to(dev), torch.from_numpy(offs), 1.0, (64, 64, 64),
                                  feature_dtype=torch.bfloat16)
        n = len(t)
        c4 = t.coords4
        for stride in (1, 2):
            oc4, _ = conv._output_coords4(c4, (1, 1, 1), (stride,) * 3, 3)
            n_out = oc4.shape[0]
            km = conv._kernel_map4(c4, oc4, shape, (1, 1, 1), 3)
            P = km.total_pairs()
            # kernel map (hash index, the operator API's path) and output coords
            tm = timeit(lambda: conv._kernel_map4(c4, oc4, shape, (1, 1, 1), 3), a.iters)
            bm = 16 * n + 16 * n_out + 8 * P
            rec = {"mode": f"map_s{stride}", "N_in": n, "N_out": n_out, "pairs": P, "us": round(tm * 1e6, 2),
                   "gbs": round(bm / tm / 1e9, 1), "bound": "hbm", "frac": round(bm / tm / 1e9 / HBM, 4)}
            if stride == 2:
                to = timeit(lambda: conv._output_coords4(c4, (1, 1, 1), (2, 2, 2), 3), a.iters)
                rec["out_coords_us"] = round(to * 1e6, 2)
                rec["out_coords_gbs"] = round((16 * n + 16 * n_out) / to / 1e9, 1)
            print(json.dumps(rec), flush=True)
            out.write(json.dumps(rec) + "\n")
            inv = km.inverse() if stride > 1 else None
            # neighbour-pattern row grouping (vp_kernel_map_group), as the training engine uses it
            fwd_perm, fwd_tbl = conv.sort_table(km.nbr, n_out) if a.sort else (None, km.nbr)
            if inv is None:
                dg_perm, dg_tbl = fwd_perm, fwd_tbl
            else:
                dg_perm, dg_tbl = conv.sort_table(inv, n, 1) if a.sort else (None, inv)
            if a.sort:
                ts = timeit(lambda: conv.sort_table(km.nbr, n_out), a.iters)
                rec_sort = {"mode": f"map_sort_s{stride}", "N": n_out, "us": round(ts * 1e6, 2)}
                print(json.dumps(rec_sort), flush=True)
                out.write(json.dumps(rec_sort) + "\n")
            for c in [int(v) for v in a.channels.split(",")]:
                g = torch.Generator(device=dev).manual_seed(1)
                x = torch.randn(n, c, device=dev, generator=g).to(torch.bfloat16)
                w = (torch.randn(K, c, c, device=dev, generator=g) / (27 * c) ** 0.5).to(torch.bfloat16)
                gy = torch.randn(n_out, c, device=dev, generator=g).to(torch.bfloat16)
                y = torch.empty(n_out, c, dtype=torch.bfloat16, device=dev)
                gi = torch.empty(n, c, dtype=torch.bfloat16, device=dev)
                gw = torch.empty(K, c, c, dtype=torch.float32, device=dev)
                wsf = _lib.workspace(_lib.query("vp_conv_fwd_ws_bytes", c, c, K), dev)
                wsd = _lib.workspace(_lib.query("vp_conv_dgrad_ws_bytes", c, c, K), dev)
                wsw = _lib.workspace(_lib.query("vp_conv_wgrad_ws_bytes", c, c, K, km.pair_in.numel()), dev)
                table, flip = (dg_tbl, 1) if inv is None else (dg_tbl, 0)

                def fwd():
                    _lib.call("vp_conv_fwd", x.data_ptr(), 1, n, c, w.data_ptr(), 1, c, K, fwd_tbl.data_ptr(), 0,
                              _lib.ptr(fwd_perm), None, n_out, y.data_ptr(), 1, wsf.data_ptr(), wsf.numel(), st)

                def dgrad():
                    _lib.call("vp_conv_dgrad", gy.data_ptr(), 1, n_out, c, w.data_ptr(), 1, c, K, table.data_ptr(),
                              flip, _lib.ptr(dg_perm), None, n, gi.data_ptr(), 1, wsd.data_ptr(), wsd.numel(), st)

                def wgrad():
                    _lib.call("vp_conv_wgrad", x.data_ptr(), 1, c, gy.data_ptr(), 1, c, K, km.pair_in.data_ptr(),
                              km.pair_out.data_ptr(), km.pair_ptr.data_ptr(), km.pair_in.numel(), gw.data_ptr(),
                              wsw.data_ptr(), wsw.numel(), st)

                for mode, fn, ni, no in (("fwd", fwd, n, n_out), ("dgrad", dgrad, n_out, n), ("wgrad", wgrad, n, n_out)):
                    r = conv_roof(P, ni, no, c, c, timeit(fn, a.iters), mode)
                    rec = {"mode": f"{mode}_s{stride}", "N_in": n, "N_out": n_out, "C": c, "pairs": P, **r}
                    if stride == 2 and mode == "dgrad":
                        rec["note"] = "= transposed conv (coarse->fine) over the inverse map"
                    print(json.dumps(rec), flush=True)
                    out.write(json.dumps(rec) + "\n")
                del x, w, gy, y, gi, gw
            torch.cuda.empty_cache()
    out.close()


if __name__ == "__main__":
    main()
