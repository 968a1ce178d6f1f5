set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_pipeline.py tests/test_gpu_conv.py -x -q > gpurun_out/pytest20.log 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/pytest20.log
rm -f gpurun_out/exp20.txt
for i in 1 2; do
for v in "VP_WGRAD_SMS=148" "X=1"; do
  env $v timeout 600 python bench.py --dp-allreduce --steps 300 --no-cpu-baseline --no-roofline > gpurun_out/b.json 2>gpurun_out/b.err
  python -c "import json;d=json.load(open('gpurun_out/b.json'));print('dp $v',d['value'],d['ms_per_step'])" >> gpurun_out/exp20.txt
done; done
timeout 600 python bench.py --steps 300 --no-cpu-baseline --no-roofline > gpurun_out/b.json 2>gpurun_out/b.err
python -c "import json;d=json.load(open('gpurun_out/b.json'));print('c3',d['value'],d['ms_per_step'])" >> gpurun_out/exp20.txt
cat gpurun_out/exp20.txt
