mkdir -p gpurun_out
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_grid_map.py tests/test_gpu_intstage.py 2>&1 | tail -2
timeout 300 python tools/map_breakdown.py 2>&1 | grep -v -i warn | head -12
