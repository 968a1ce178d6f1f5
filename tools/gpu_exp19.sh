set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bn_epi.py tests/test_gpu_model.py tests/test_gpu_bench_parity.py tests/test_gpu_conv.py -x -q > gpurun_out/pytest19.log 2>&1; echo "pytest rc=$?"; tail -n 3 gpurun_out/pytest19.log
rm -f gpurun_out/exp19.txt
for i in 1 2; do
for v in "VP_STEM_MMA=0" "VP_STEM_MMA=1"; do
  env $v timeout 600 python bench.py --steps 300 --no-cpu-baseline --no-roofline > gpurun_out/b.json 2>gpurun_out/b.err
  python -c "import json;d=json.load(open('gpurun_out/b.json'));print('$v',d['value'],d['ms_per_step'],d['final_loss'])" >> gpurun_out/exp19.txt
done; done
VP_DBG_SKIP_WGRAD=1 VP_DBG_SKIP_PREFETCH=1 timeout 600 python tools/critical_path.py 2>/dev/null | grep -E "stem|step span" >> gpurun_out/exp19.txt
cat gpurun_out/exp19.txt
