run() { echo -n "$1: "; env $1 timeout 200 python bench.py --steps 100 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"; }
run "X=0"
for nd in 32 64 128 256; do for c in 0 1 2 4; do run "VP_CONV_CFG_$nd=$c"; done; done
run "X=0"
