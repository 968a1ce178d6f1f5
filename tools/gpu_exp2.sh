set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tile_sched.py tests/test_gpu_model.py tests/test_gpu_bench_parity.py -x -q > gpurun_out/pytest_sched.log 2>&1; echo "pytest rc=$?"; tail -n 15 gpurun_out/pytest_sched.log
timeout 300 python tools/cta_probe.py 32 > gpurun_out/cta32_sched.txt 2>&1; echo "cta rc=$?"
rm -f gpurun_out/exp2.txt
for i in 1 2; do
for v in "VP_TILE_SCHED=0" "VP_TILE_SCHED=1"; do
  env $v timeout 600 python bench.py --steps 200 --no-cpu-baseline --no-roofline > gpurun_out/b.json 2>gpurun_out/b.err
  python -c "import json;d=json.load(open('gpurun_out/b.json'));print('$v',d['value'],d['ms_per_step'])" >> gpurun_out/exp2.txt
done; done
cat gpurun_out/exp2.txt; head -20 gpurun_out/cta32_sched.txt
