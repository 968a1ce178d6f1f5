python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in 0 1 3; do echo CFG $c; VP_CONV_CFG=$c python tools/conv_density.py 2>&1 | grep "density=0.25 local=False"; done
for c in 0 1 3; do VP_CONV_CFG=$c python bench.py --steps 50 --warmup 5 --no-cpu-baseline 2>&1 | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('CFG', $c, d['value'], d['ms_per_step'], d['roofline']['per_layer_fwd_us'])"; done
