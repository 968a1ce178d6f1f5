set -u
mkdir -p gpurun_out
rm -f gpurun_out/exp18.txt
for i in 1 2; do
for v in "X=1" "VP_BN_APPLY_PER_SM=2" "VP_CONV_MAX_SPLIT=8" "VP_CONV_CFG_128=3" "VP_WGRAD_SMS=80" "VP_WGRAD_SMS=110" "VP_EPI_ROWS_MIN_ND=128" "VP_SORT_LEVELS=1,2" "VP_WGRAD_CPS=1"; do
  env $v timeout 600 python bench.py --steps 300 --no-cpu-baseline --no-roofline > gpurun_out/b.json 2>gpurun_out/b.err
  python -c "import json;d=json.load(open('gpurun_out/b.json'));print('$v',d['value'],d['ms_per_step'])" >> gpurun_out/exp18.txt
done; done
cat gpurun_out/exp18.txt
