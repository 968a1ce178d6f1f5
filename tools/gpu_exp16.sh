set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bn_epi.py tests/test_gpu_model.py tests/test_gpu_bench_parity.py -x -q > gpurun_out/pytest16.log 2>&1; echo "pytest rc=$?"; tail -n 3 gpurun_out/pytest16.log
rm -f gpurun_out/exp16.txt
for i in 1 2; do
  timeout 600 python bench.py --steps 300 --no-cpu-baseline --no-roofline > gpurun_out/b.json 2>gpurun_out/b.err
  python -c "import json;d=json.load(open('gpurun_out/b.json'));print('headred',d['value'],d['ms_per_step'])" >> gpurun_out/exp16.txt
done
VP_DBG_SKIP_WGRAD=1 VP_DBG_SKIP_PREFETCH=1 timeout 600 python tools/critical_path.py 2>/dev/null | grep -E "head|step span" >> gpurun_out/exp16.txt
cat gpurun_out/exp16.txt
