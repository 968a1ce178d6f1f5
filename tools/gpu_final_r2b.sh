#!/usr/bin/env bash
# Round-2 closing evidence after the level-1 tile schedule: bench line (CPU
# baseline + e2e + roofline), reference arm, C5 on one GPU, launch list,
# critical path, per-CTA probes of the level-1/2 convs, and ncu --set full of
# the convs whose tables changed (level 1) plus the bench's dominant launch.
set -u
mkdir -p gpurun_out
lscpu | grep -E 'Model name|^CPU\(s\)' > gpurun_out/host.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 900 python bench.py --batch 256 --points 16384 --res 128 --blocks 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "c5 rc=$?"
VP_DBG_SKIP_WGRAD=1 VP_DBG_SKIP_PREFETCH=1 timeout 600 python tools/critical_path.py > gpurun_out/critical_path.txt 2>&1; echo "critical rc=$?"
timeout 300 python tools/cta_probe.py 32 > gpurun_out/cta32.txt 2>&1; echo "cta32 rc=$?"
timeout 300 python tools/cta_probe.py 64 > gpurun_out/cta64.txt 2>&1; echo "cta64 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2b_launches.csv \
  python bench.py --profile-only --no-graph > gpurun_out/ncu_launch.log 2>&1; echo "ncu list rc=$?"
for t in "s0.b0.c1 fwd" "s0.b0.c1 dgrad" "s0.b0.c2 fwd" "s0.b0.c2 dgrad" "s2.b0.c2 wgrad" "s2.b0.c1 wgrad"; do
  set -- $t
  tag="${1}_${2}"
  timeout 300 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -o gpurun_out/r2b_$tag -f python tools/ncu_target.py --layer $1 --mode $2 > gpurun_out/ncu_$tag.log 2>&1
  echo "ncu $tag rc=$?"
  ncu -i gpurun_out/r2b_$tag.ncu-rep --page raw --csv > gpurun_out/r2b_$tag.raw.csv 2>/dev/null
  rm -f gpurun_out/r2b_$tag.ncu-rep
done
