#!/usr/bin/env bash
# C3 bench under environment-knob variants (one line each): value, ms/step
run() { echo -n "$*: "; env "$@" timeout 200 python bench.py --steps 100 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"; }
run X=0
for v in "$@"; do run $v; done
run X=0
