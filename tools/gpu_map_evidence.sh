#!/usr/bin/env bash
# Round-2 kernel-map evidence after the bitmap / column probe / slab emit:
# bench line, C5 line, C2 sweep, per-kernel map breakdown, ncu --set full of
# the C3 level-0 map launches.
set -u
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --batch 256 --points 16384 --res 128 --blocks 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "c5 rc=$?"
timeout 900 python tools/sweep_c2.py --out gpurun_out/c2_sweep.jsonl > gpurun_out/c2_sweep.log 2>&1; echo "sweep rc=$?"
timeout 600 python tools/map_breakdown.py 2>&1 | grep -v -i warn > gpurun_out/map_breakdown.txt; echo "breakdown rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -o gpurun_out/r2_map -f python tools/ncu_target.py --layer s0.b0.c1 --mode map > gpurun_out/ncu_map.log 2>&1; echo "ncu map rc=$?"
ncu -i gpurun_out/r2_map.ncu-rep --page raw --csv > gpurun_out/r2_s0.b0.c1_map.raw.csv 2>/dev/null
rm -f gpurun_out/r2_map.ncu-rep
