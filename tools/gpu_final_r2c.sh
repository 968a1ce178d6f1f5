#!/usr/bin/env bash
# Round-2 final lines after the integer-stage kernel work (coalesced grouping
# histogram + permute): bench (CPU baseline, e2e, roofline), reference arm,
# C5, critical path, launch list.
set -u
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 900 python bench.py --batch 256 --points 16384 --res 128 --blocks 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "c5 rc=$?"
timeout 600 python bench.py --dp-allreduce --steps 100 --no-cpu-baseline --no-roofline > gpurun_out/bench_dp1.json 2> gpurun_out/bench_dp1.err; echo "dp1 rc=$?"
rm -f gpurun_out/decomposition.txt
for v in "X=1" "VP_DBG_SKIP_WGRAD=1" "VP_DBG_SKIP_PREFETCH=1" "VP_DBG_SKIP_PREFETCH=1 VP_DBG_SKIP_WGRAD=1"; do
  env $v timeout 600 python bench.py --steps 200 --no-cpu-baseline --no-roofline > gpurun_out/b.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/b.json'));print('$v',d['value'],d['ms_per_step'],d['gpu_launches_per_step'])" >> gpurun_out/decomposition.txt
done
VP_DBG_SKIP_WGRAD=1 VP_DBG_SKIP_PREFETCH=1 timeout 600 python tools/critical_path.py > gpurun_out/critical_path.txt 2>&1; echo "critical rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG:-r2c}_launches.csv \
  python bench.py --profile-only --no-graph > gpurun_out/ncu_launch.log 2>&1; echo "ncu list rc=$?"
cat gpurun_out/decomposition.txt
