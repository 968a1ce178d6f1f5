set -u
mkdir -p gpurun_out
rm -f gpurun_out/exp15.txt
for i in 1 2; do
  timeout 600 python bench.py --steps 300 --no-cpu-baseline --no-roofline > gpurun_out/b.json 2>gpurun_out/b.err
  python -c "import json;d=json.load(open('gpurun_out/b.json'));print('C3',d['value'],d['ms_per_step'])" >> gpurun_out/exp15.txt
  timeout 900 python bench.py --batch 256 --points 16384 --res 128 --blocks 2 --steps 10 --warmup 3 --no-cpu-baseline --no-roofline > gpurun_out/b5.json 2>gpurun_out/b5.err
  python -c "import json;d=json.load(open('gpurun_out/b5.json'));print('C5',d['value'],d['ms_per_step'])" >> gpurun_out/exp15.txt
done
cat gpurun_out/exp15.txt
