#!/usr/bin/env bash
# GPU tests + smoke + a short bench + ncu --set full of the dominant kernels
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -n 30 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -n 3 gpurun_out/smoke.log
timeout 600 python bench.py --steps ${BENCH_STEPS:-50} --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json; tail -n 5 gpurun_out/bench.err
if [ -n "${NCU:-}" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_wgrad -s 0 -c 1 -o gpurun_out/prof_wgrad -f python bench.py --profile-only --no-graph > gpurun_out/ncu_w.log 2>&1; echo "ncu wgrad rc=$?"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_tc_kernel -s 7 -c 1 -o gpurun_out/prof_fwd -f python bench.py --profile-only --no-graph > gpurun_out/ncu_f.log 2>&1; echo "ncu fwd rc=$?"
fi
