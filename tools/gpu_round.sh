#!/usr/bin/env bash
# One gpurun call: GPU tests, smoke, bench (with clocks), launch list and one
# ncu --set full capture of the dominant conv kernel.  Outputs -> gpurun_out/.
set -u
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/gpu.txt 2>&1; lscpu | grep -E 'Model name|^CPU\(s\)' >> gpurun_out/gpu.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a gpurun_out/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" | tee -a gpurun_out/status.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" | tee -a gpurun_out/status.txt
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?" | tee -a gpurun_out/status.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --profile-only --no-graph > gpurun_out/ncu_launch.log 2>&1; echo "ncu list rc=$?" | tee -a gpurun_out/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:${NCU_K:-conv_tc_kernel}" -s ${NCU_S:-20} -c ${NCU_C:-3} \
  -o gpurun_out/prof -f python bench.py --profile-only --no-graph > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?" | tee -a gpurun_out/status.txt
