#!/usr/bin/env bash
# Round-2 evidence: kernel launch list of the C3 step, and ncu --set full of
# the bench line's roofline candidates, each launched alone by
# tools/ncu_target.py (cudaProfilerStart/Stop around one launch); raw csv
# exports + DRAM traffic per launch into gpurun_out/.
set -u
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches.csv \
  python bench.py --profile-only --no-graph > gpurun_out/ncu_launch.log 2>&1; echo "ncu list rc=$?"
for t in "s1.b0.c2 wgrad" "s2.b0.c1 wgrad" "s3.b0.c1 wgrad" "s0.b0.c1 fwd" "s0.b0.c1 dgrad" "s0.b0.c1 fwd_bn" "s0.b0.c2 dgrad_bn" "s2.b0.c1 fwd" "s3.b0.c1 fwd" "s0.b0.c1 map"; do
  set -- $t
  tag="${1}_${2}"
  timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -o gpurun_out/r2_$tag -f python tools/ncu_target.py --layer $1 --mode $2 > gpurun_out/ncu_$tag.log 2>&1
  echo "ncu $tag rc=$?"
  ncu -i gpurun_out/r2_$tag.ncu-rep --page raw --csv > gpurun_out/r2_$tag.raw.csv 2>/dev/null
  [ -n "${KEEP_REPS:-}" ] || rm -f gpurun_out/r2_$tag.ncu-rep
done
