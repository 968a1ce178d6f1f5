set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_conv.py tests/test_gpu_model.py -x -q > gpurun_out/pytest9.log 2>&1; echo "pytest rc=$?"; tail -n 3 gpurun_out/pytest9.log
rm -f gpurun_out/exp9.txt
for i in 1 2; do
  timeout 600 python bench.py --steps 200 --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err
  python -c "
import json;d=json.load(open('gpurun_out/b.json'));r=d['roofline']
w={k:round(v[0],1) for k,v in r['kernels'].items() if 'wgrad' in k}
print('pptr-par',d['value'],d['ms_per_step'],r['kernel'][:40],r['us_per_launch'],r['frac'],w)" >> gpurun_out/exp9.txt
done
cat gpurun_out/exp9.txt
