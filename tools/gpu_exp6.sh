set -u
mkdir -p gpurun_out
rm -f gpurun_out/exp6.txt
for c in 32 64; do
for v in 0 1 8 9 7 15; do
  echo "C=$c VP_CONV_DBG=$v" >> gpurun_out/exp6.txt
  VP_CONV_DBG=$v timeout 300 python tools/cta_probe.py $c 2>/dev/null | grep -E "^rows|end:|fit" >> gpurun_out/exp6.txt
done; done
cat gpurun_out/exp6.txt
