#!/usr/bin/env bash
# Round-end evidence: full bench (with CPU baseline), reference arm, C5 one-GPU
# bench, launch list, ncu --set full of the dominant conv (traffic), timeline.
set -u
mkdir -p gpurun_out
lscpu | grep -E 'Model name|^CPU\(s\)' > gpurun_out/host.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 900 python bench.py --batch 256 --points 16384 --res 128 --blocks 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "c5 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --profile-only --no-graph > gpurun_out/ncu_launch.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_tc_kernel -s 7 -c 1 \
  -o gpurun_out/prof_fwd -f python bench.py --profile-only --no-graph > gpurun_out/ncu_f.log 2>&1; echo "ncu fwd rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_tc_kernel -s 1 -c 1 \
  -o gpurun_out/prof_fwd32 -f python bench.py --profile-only --no-graph > gpurun_out/ncu_f32.log 2>&1; echo "ncu fwd32 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_tc_kernel -s 0 -c 1 \
  -o gpurun_out/prof_fwd32d -f python bench.py --profile-only --no-graph > gpurun_out/ncu_f32d.log 2>&1; echo "ncu fwd32d rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"map_probe_grid|map_emit|grid_set" -s 0 -c 3 \
  -o gpurun_out/prof_map -f python bench.py --profile-only --no-graph > gpurun_out/ncu_m.log 2>&1; echo "ncu map rc=$?"
timeout 300 python tools/timeline.py > gpurun_out/timeline.txt 2>&1; echo "timeline rc=$?"
timeout 300 python tools/step_breakdown.py > gpurun_out/step_breakdown.txt 2>&1; echo "breakdown rc=$?"
# keep what comes back under gpurun's 64 MiB: raw csv exports of the captures
for r in gpurun_out/prof_*.ncu-rep; do
  [ -f "$r" ] || continue
  ncu -i "$r" --page raw --csv > "${r%.ncu-rep}.raw.csv" 2>/dev/null
  [ -n "${KEEP_REPS:-}" ] || rm -f "$r"
done
