set -u
mkdir -p gpurun_out
rm -f gpurun_out/exp17.txt
for i in 1 2; do
for v in "X=1" "VP_ROWS_PASS_BLOCKS=148" "VP_ROWS_PASS_BLOCKS=296"; do
  env $v timeout 600 python bench.py --steps 300 --no-cpu-baseline --no-roofline > gpurun_out/b.json 2>gpurun_out/b.err
  python -c "import json;d=json.load(open('gpurun_out/b.json'));print('$v',d['value'],d['ms_per_step'])" >> gpurun_out/exp17.txt
done; done
cat gpurun_out/exp17.txt
