#!/usr/bin/env bash
# layer profile + ncu --set full captures of named kernels (one per regex)
set -u
mkdir -p gpurun_out
timeout 300 python tools/layer_profile.py > gpurun_out/layer_profile.txt 2>&1; echo "layer_profile rc=$?"
i=0
for k in "$@"; do
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$k" -s ${NCU_S:-2} -c 1 \
    -o gpurun_out/prof_$i -f python bench.py --profile-only --no-graph > gpurun_out/ncu_$i.log 2>&1; echo "ncu $k rc=$?"
  i=$((i+1))
done
