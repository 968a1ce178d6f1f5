python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in 1 2 3 4; do VP_CONV_CPS=$c python bench.py --steps 50 --warmup 5 --no-cpu-baseline 2>&1 | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('CPS', $c, d['value'], d['ms_per_step'], d['roofline']['per_layer_fwd_us'])"; done
