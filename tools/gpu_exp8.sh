set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tile_sched.py tests/test_gpu_model.py tests/test_gpu_conv.py -x -q -k "sched or mask_sorted or kernel_maps or grid or tc_grid or prefetch" > gpurun_out/pytest8.log 2>&1; echo "pytest rc=$?"; tail -n 4 gpurun_out/pytest8.log
timeout 300 python tools/intstage_time.py 2>/dev/null | grep -E "group_hist|tile_|permute"
rm -f gpurun_out/exp8.txt
for i in 1 2; do
  timeout 600 python bench.py --steps 200 --no-cpu-baseline --no-roofline > gpurun_out/b.json 2>gpurun_out/b.err
  python -c "import json;d=json.load(open('gpurun_out/b.json'));print('hist-coalesced',d['value'],d['ms_per_step'])" >> gpurun_out/exp8.txt
done
cat gpurun_out/exp8.txt
