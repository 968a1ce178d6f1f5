# A/B of the step-level knobs after the bitmap map (200 steps each, alternating)
for i in 1 2; do
for v in "X=1" "VP_WGRAD_DEVICE_CHUNK=1" "VP_FULL_MASK_ROWS=65536" "VP_FULL_MASK_ROWS=8192" "VP_WGRAD_CPS=1"; do
  env $v timeout 600 python bench.py --steps 200 --no-cpu-baseline --no-roofline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v',d['value'],d['ms_per_step'])"
done; done
