"""BASELINE.md §2 CPU baseline report, on the GPU box's host cores: the
reference's own CPU path (oracle/_ref voxpipe, compiled hash; numpy glue)
  * C1 (8 x 1024 pts @ 32^3) and a bounded C3 sample (16 of the 64 clouds of
    2048 pts @ 64^3), each with all host threads and with 1 BLAS thread;
  * the per-layer split of the C3 step into output coords + kernel map vs
    gather-GEMM-scatter (oracle/ref_runner.layer_split).
Writes one JSON object to stdout.  Bench/test infrastructure only."""
import json
import os
import platform
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def run(threads, B, npts, res, steps, warmup):
    env = dict(os.environ, OPENBLAS_NUM_THREADS=str(threads), OMP_NUM_THREADS=str(threads),
               MKL_NUM_THREADS=str(threads))
    code = (f"import sys, json; sys.path.insert(0, {os.path.join(ROOT, 'oracle')!r}); import ref_runner; "
            f"print(json.dumps(ref_runner.time_steps({B}, {npts}, {res}, {steps}, {warmup})))")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, check=True).stdout
    r = json.loads(out.strip().splitlines()[-1])
    return {"clouds": B, "threads": threads, "steps": steps, "clouds_per_s": round(r["clouds_per_s"], 3),
            "s_per_step": round(r["s_per_step"], 3), "kind": r["kind"]}


def main():
    import numpy as np

    import ref_runner
    nproc = os.cpu_count() or 1
    cpu = "unknown"
    try:
        cpu = next(l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name"))
    except (OSError, StopIteration):
        pass
    rep = {"host": {"cpu": cpu, "nproc": nproc, "python": platform.python_version(), "numpy": np.__version__},
           "C1": [run(nproc, 8, 1024, 32, 3, 1), run(1, 8, 1024, 32, 3, 1)],
           "C3_sample": [run(nproc, 16, 2048, 64, 2, 1), run(1, 16, 2048, 64, 2, 1)]}
    rep["C3_layer_split"] = ref_runner.layer_split(64, 2048, 64)
    L = rep["C3_layer_split"]["layers"]
    rep["C3_layer_split"]["totals_s"] = {k: round(sum(r[k] for r in L), 3)
                                         for k in ("coords_s", "map_s", "gemm_fwd_s", "gemm_bwd_s", "fwd_s", "bwd_s")}
    print(json.dumps(rep))


if __name__ == "__main__":
    main()
