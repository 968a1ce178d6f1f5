#!/usr/bin/env bash
# Round-2 evidence: bench line (CPU baseline + e2e), reference arm, C5 on one
# GPU, DP all-reduce path at N=1, per-layer ncu --set full of every
# tensor-core conv launch the bench's roofline can name, launch list,
# critical-path timeline and the side-stream decomposition.
set -u
mkdir -p gpurun_out
lscpu | grep -E 'Model name|^CPU\(s\)' > gpurun_out/host.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 900 python bench.py --batch 256 --points 16384 --res 128 --blocks 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "c5 rc=$?"
timeout 600 python bench.py --dp-allreduce --steps 100 --no-cpu-baseline > gpurun_out/bench_dp1.json 2> gpurun_out/bench_dp1.err; echo "dp1 rc=$?"
for v in "X=1" "VP_DBG_SKIP_WGRAD=1" "VP_DBG_SKIP_PREFETCH=1" "VP_DBG_SKIP_PREFETCH=1 VP_DBG_SKIP_WGRAD=1"; do
  env $v timeout 600 python bench.py --steps 200 --no-cpu-baseline --no-roofline > gpurun_out/b.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/b.json'));print('$v',d['value'],d['ms_per_step'],d['gpu_launches_per_step'])" >> gpurun_out/decomposition.txt
done
VP_DBG_SKIP_WGRAD=1 VP_DBG_SKIP_PREFETCH=1 timeout 600 python tools/critical_path.py > gpurun_out/critical_path.txt 2>&1; echo "critical rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches.csv \
  python bench.py --profile-only --no-graph > gpurun_out/ncu_launch.log 2>&1; echo "ncu list rc=$?"
for L in s0.down s0.b0.c1 s0.b0.c2 s1.down s1.b0.c1 s1.b0.c2 s2.down s2.b0.c1 s2.b0.c2 s3.down s3.b0.c1 s3.b0.c2; do
  for M in fwd dgrad wgrad; do
    tag="${L}_${M}"
    timeout 300 ncu --set full --clock-control none --import-source on --profile-from-start off \
      -o gpurun_out/r2_$tag -f python tools/ncu_target.py --layer $L --mode $M > gpurun_out/ncu_$tag.log 2>&1
    echo "ncu $tag rc=$?"
    ncu -i gpurun_out/r2_$tag.ncu-rep --page raw --csv > gpurun_out/r2_$tag.raw.csv 2>/dev/null
    rm -f gpurun_out/r2_$tag.ncu-rep
  done
done
for t in "s0.b0.c1 fwd_bn" "s0.b0.c2 dgrad_bn" "s1.b0.c2 dgrad_bn" "s0.b0.c1 map"; do
  set -- $t
  tag="${1}_${2}"
  timeout 300 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -o gpurun_out/r2_$tag -f python tools/ncu_target.py --layer $1 --mode $2 > gpurun_out/ncu_$tag.log 2>&1
  echo "ncu $tag rc=$?"
  ncu -i gpurun_out/r2_$tag.ncu-rep --page raw --csv > gpurun_out/r2_$tag.raw.csv 2>/dev/null
  rm -f gpurun_out/r2_$tag.ncu-rep
done
