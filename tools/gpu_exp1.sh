set -u
mkdir -p gpurun_out
timeout 300 python tools/tail_probe.py 32 > gpurun_out/tail32.txt 2>&1; echo "tail32 rc=$?"
timeout 300 python tools/tail_probe.py 64 > gpurun_out/tail64.txt 2>&1; echo "tail64 rc=$?"
for i in 1 2; do
for v in "X=1" "VP_WGRAD_DEVICE_CHUNK=1"; do
  env $v timeout 600 python bench.py --steps 200 --no-cpu-baseline --no-roofline > gpurun_out/b.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/b.json'));print('$v',d['value'],d['ms_per_step'])" >> gpurun_out/exp1.txt
done; done
cat gpurun_out/tail32.txt gpurun_out/tail64.txt gpurun_out/exp1.txt
