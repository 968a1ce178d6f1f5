"""Fold the round's `ncu --set full` captures (gpurun_out/<round>_<layer>_<mode>.raw.csv
from tools/gpu_prof_r2.sh) into profiles/:

  * profiles/ncu_traffic.json — DRAM read+write bytes per timed launch (the
    conv kernel plus its split-K / chunk reduction, i.e. exactly what
    bench.py's roofline times), keyed '<config> <kernel> <layer>' as
    paper_2012_13846_b200.roofline.ncu_traffic looks them up;
  * profiles/<round>_ncu_summary.txt — the key metrics of every captured kernel.

Usage: python tools/ncu_traffic_update.py [round] [config]   (default r2 C3)"""
import csv
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "profiles"))
from ncu_summary import WANT  # noqa: E402

PLANES = (32, 64, 128, 256)


def widths(layer):
    """(C_in, C_out) of a C3 SparseResNet layer name (blocks=1)."""
    if layer == "stem":
        return 1, PLANES[0]
    s = int(layer[1])
    cout = PLANES[s]
    cin = (PLANES[s - 1] if s > 0 else PLANES[0]) if layer.endswith("down") else cout
    return cin, cout


def bench_key(layer, mode):
    cin, cout = widths(layer)
    if mode.startswith("fwd"):
        return f"conv_fwd_tc<{cin},{cout}>"
    if mode.startswith("dgrad"):
        return f"conv_dgrad_tc<{cout},{cin}>"
    if mode == "wgrad":
        return f"conv_wgrad_tc<{cin},{cout}>"
    return "map"


def rows_of(path):
    rows = list(csv.reader(open(path)))
    if len(rows) < 3:
        return [], [], []
    return rows[0], rows[1], rows[2:]


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return float(v.replace(",", "")) * scale


def main(rnd="r2", config="C3"):
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    lines = []
    for path in sorted(glob.glob(os.path.join(ROOT, "gpurun_out", f"{rnd}_*.raw.csv"))):
        tag = os.path.basename(path)[len(rnd) + 1:-len(".raw.csv")]
        layer, mode = tag.rsplit("_", 1) if not tag.endswith(("_fwd_bn", "_dgrad_bn")) else tag.rsplit("_", 2)[0:1] + [
            "_".join(tag.rsplit("_", 2)[1:])]
        h, units, data = rows_of(path)
        if not data:
            continue
        ir, iw = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
        total = sum(to_bytes(r[ir], units[ir]) + to_bytes(r[iw], units[iw]) for r in data)
        key = f"{config} {bench_key(layer, mode)} {layer}"
        if mode in ("fwd", "dgrad", "wgrad"):
            traffic[key] = int(total)
        lines.append(f"=== {config} {layer} {mode}  (DRAM read+write of the timed launch: {total / 1e6:.3f} MB)")
        idx = [(w, h.index(w)) for w in WANT if w in h]
        for r in data:
            lines.append("---")
            for w, i in idx:
                lines.append(f"  {w}: {r[i]} {units[i]}")
    traffic["_source"] = (f"ncu --set full --clock-control none, one launch of tools/ncu_target.py per key ({config}, "
                          "the step's own tables after one training step): dram__bytes_read.sum + "
                          "dram__bytes_write.sum summed over the kernels of the timed launch (conv + its reduction); "
                          f"keys '<config> <kernel> <layer>'; summaries in profiles/{rnd}_ncu_summary.txt")
    json.dump(traffic, open(tpath, "w"), indent=1, sort_keys=True)
    open(os.path.join(ROOT, "profiles", f"{rnd}_ncu_summary.txt"), "w").write("\n".join(lines) + "\n")
    print(f"{len(lines)} summary lines; traffic keys: {sorted(k for k in traffic if not k.startswith('_'))}")


if __name__ == "__main__":
    main(*sys.argv[1:])
