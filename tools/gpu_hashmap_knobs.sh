# hash kernel-map experiments: table load factor, z-grouped homes, streaming nbr stores
for cfg in "4 0 0" "2 0 0" "4 2 0" "4 3 0" "2 2 0" "2 3 0" "2 3 1" "4 3 1"; do
  set -- $cfg
  echo "### LOADF=$1 ZG=$2 STREAM=$3"
  VP_MAP_LOADF=$1 VP_MAP_ZG=$2 VP_MAP_STREAM_NBR=$3 timeout 300 python tools/map_breakdown.py --hash-only 2>&1 | grep -v Warn | grep -v warn_once | tail -6
done
VP_MAP_LOADF=2 VP_MAP_ZG=3 timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_intstage.py tests/test_gpu_vs_reference.py tests/test_gpu_model.py -k "map or pairs or kmap or hash or golden or reference" 2>&1 | tail -3
