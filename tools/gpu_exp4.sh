set -u
mkdir -p gpurun_out
rm -f gpurun_out/exp4.txt
for v in "X=1" "VP_WGRAD_DEVICE_CHUNK=1 VP_WGRAD_MIN_F=8" "VP_WGRAD_DEVICE_CHUNK=1 VP_WGRAD_MIN_F=16" "VP_WGRAD_DEVICE_CHUNK=1 VP_WGRAD_MIN_F=4"; do
  env $v timeout 600 python bench.py --steps 200 --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err
  python -c "
import json;d=json.load(open('gpurun_out/b.json'));r=d['roofline']
w={k:v[0] for k,v in r['kernels'].items() if 'wgrad' in k}
print('$v',d['value'],d['ms_per_step'],r['kernel'][:40],r['us_per_launch'],r['frac'],'wgrad max',max(w.values()),'sum',round(sum(w.values()),1))" >> gpurun_out/exp4.txt
done
cat gpurun_out/exp4.txt
