mkdir -p gpurun_out
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_grid_map.py tests/test_gpu_intstage.py tests/test_gpu_vs_reference.py tests/test_gpu_model.py tests/test_gpu_conv.py 2>&1 | tail -2
timeout 300 python tools/map_breakdown.py 2>&1 | grep -v -i warn
timeout 300 python bench.py --steps 30 --warmup 5 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'],d['ms_per_step'],d['roofline']['map'])"
timeout 300 python tools/sweep_c2.py --clouds 6,55,552 --channels 32 --iters 10 --out gpurun_out/m_sweep.jsonl 2>&1 | grep map
