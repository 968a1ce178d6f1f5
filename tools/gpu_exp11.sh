set -u
mkdir -p gpurun_out
rm -f gpurun_out/exp11.txt
for i in 1 2 3; do
for v in "VP_TILE_SCHED=0" "VP_TILE_SCHED=1"; do
  env $v timeout 600 python bench.py --steps 300 --no-cpu-baseline --no-roofline > gpurun_out/b.json 2>gpurun_out/b.err
  python -c "import json;d=json.load(open('gpurun_out/b.json'));print('$v',d['value'],d['ms_per_step'])" >> gpurun_out/exp11.txt
done; done
cat gpurun_out/exp11.txt
