"""Roofline bookkeeping shared by bench.py and tools/ (measurement only).

Algorithmic work per call, exactly SURVEY §8(d) (int32 coords 16 B/row,
int32 pairs 8 B/pair, bf16 features):

  kernel map   : B = 16 N_in + 16 N_out + 8 P            (HBM)
  output coords: B = 16 N_in + 16 N_out                   (HBM)
  conv fwd     : F = 2 P C_in C_out ;
                 B = 2 N_in C_in + 2 N_out C_out + 2 K C_in C_out + 8 P
  conv dgrad   : the same with the roles of the row sets swapped
  conv wgrad   : F as above ; B = 2 N_in C_in + 2 N_out C_out + 8 P + 4 K C_in C_out
  bound        : tensor when (F / B) * HBM_peak > TC_peak, else HBM

Kernel timing: every launch is preceded by an L2 flush (a write larger than
the 126 MB L2) outside the CUDA events, so the kernel starts cold as it does
inside the training step; the events sit on the launching stream.
"""
from __future__ import annotations

import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def peaks():
    """(hbm GB/s, bf16 TFLOP/s burst, source): the driver-measured
    MEASURED_PEAKS.json, else the profiling guide's nominal B200 numbers."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), "measured (MEASURED_PEAKS.json, burst)"
    except (OSError, KeyError, ValueError):
        return 7700.0, 2250.0, "nominal fallback (B200_PROFILING.md)"


def conv_work(P, n_in, n_out, cin, cout, K=27, mode="fwd"):
    """(FLOPs, bytes) of one conv pass; n_in/n_out are the rows read/written
    by that pass (dgrad: n_in = rows of g, n_out = rows of grad_in, and
    cin/cout its read/written widths)."""
    F = 2.0 * P * cin * cout
    if mode == "wgrad":
        B = 2 * n_in * cin + 2 * n_out * cout + 8 * P + 4 * K * cin * cout
    else:
        B = 2 * n_in * cin + 2 * n_out * cout + 2 * K * cin * cout + 8 * P
    return F, float(B)


def map_bytes(n_in, n_out, P):
    return float(16 * n_in + 16 * n_out + 8 * P)


def classify(F, B, seconds, hbm=None, tc=None):
    """Roofline record of one kernel: bound, achieved vs peak, frac."""
    if hbm is None or tc is None:
        hbm, tc, _ = peaks()
    tflops, gbs = (F / seconds / 1e12 if F else 0.0), B / seconds / 1e9
    tensor = F > 0 and (F / B) * hbm / 1e3 > tc
    ach, peak, unit = (tflops, tc, "TFLOP/s") if tensor else (gbs, hbm, "GB/s")
    return {"bound": "tensor" if tensor else "hbm", "achieved": round(ach, 2), "peak": peak, "unit": unit,
            "frac": round(ach / peak, 4), "us_per_launch": round(seconds * 1e6, 2),
            "algorithmic_flops": F, "algorithmic_bytes": B, "tflops": round(tflops, 2), "gbs": round(gbs, 1)}


class Flusher:
    """Writes a buffer larger than L2 (126 MB) on the current stream."""

    def __init__(self, device, mib=256):
        import torch

        self.buf = torch.empty(mib * 1024 * 1024, dtype=torch.uint8, device=device)

    def __call__(self):
        self.buf.zero_()


def time_cold(launch, flush, iters=20, warmup=3):
    """Mean seconds per launch, each launch after an L2 flush, CUDA events on
    the current (launching) stream bracketing the launch only."""
    import torch

    st = torch.cuda.current_stream()
    for _ in range(warmup):
        flush()
        launch()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
    torch.cuda.synchronize()
    for a, b in evs:
        flush()
        a.record(st)
        launch()
        b.record(st)
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in evs) / iters / 1e3


def ncu_traffic(config_tag, kernel, layer):
    """DRAM read+write bytes per launch of `kernel` for `layer` at
    `config_tag` from the committed ncu --set full summaries
    (profiles/ncu_traffic.json, keyed '<config> <kernel> <layer>'), else None
    — never another config's or layer's capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            t = json.load(f)
    except (OSError, ValueError):
        return None
    v = t.get(f"{config_tag} {kernel} {layer}")
    return int(v) if isinstance(v, (int, float)) else None
