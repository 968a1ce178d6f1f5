mkdir -p gpurun_out; rm -f gpurun_out/decomposition.txt
for v in "X=1" "VP_DBG_SKIP_WGRAD=1" "VP_DBG_SKIP_PREFETCH=1" "VP_DBG_SKIP_PREFETCH=1 VP_DBG_SKIP_WGRAD=1"; do
  env $v timeout 600 python bench.py --steps 200 --no-cpu-baseline --no-roofline > gpurun_out/b.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/b.json'));print('$v',d['value'],d['ms_per_step'],d['gpu_launches_per_step'])" >> gpurun_out/decomposition.txt
done
VP_DBG_SKIP_WGRAD=1 VP_DBG_SKIP_PREFETCH=1 timeout 600 python tools/critical_path.py > gpurun_out/critical_path.txt 2>&1; echo "critical rc=$?"
cat gpurun_out/decomposition.txt; tail -25 gpurun_out/critical_path.txt
