set -u
mkdir -p gpurun_out
rm -f gpurun_out/exp7.txt
for v in "X=1" "VP_WGRAD_MAX_CHUNK=1024" "VP_WGRAD_MAX_CHUNK=512" "X=1" "VP_WGRAD_MAX_CHUNK=1024"; do
  env $v timeout 600 python bench.py --steps 200 --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err
  python -c "
import json;d=json.load(open('gpurun_out/b.json'));r=d['roofline']
w={k:v[0] for k,v in r['kernels'].items() if 'wgrad' in k}
print('$v',d['value'],d['ms_per_step'],r['kernel'][:40],r['us_per_launch'],r['frac'],'wgrad',{k:round(v,1) for k,v in w.items()})" >> gpurun_out/exp7.txt
done
cat gpurun_out/exp7.txt
