mkdir -p gpurun_out
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_grid_map.py tests/test_gpu_model.py tests/test_gpu_bench_parity.py 2>&1 | tail -3
timeout 300 python tools/map_breakdown.py 2>&1 | grep -v -i warn | head -8
VP_MAP_CUBE=0 timeout 300 python tools/map_breakdown.py 2>&1 | grep -v -i warn | head -7
timeout 300 python bench.py --steps 30 --warmup 5 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'],d['ms_per_step'],d['roofline']['map'])"
