set -u
mkdir -p gpurun_out
rm -f gpurun_out/exp5.txt
for c in 32 64 128; do
for v in 0 2 4 6; do
  echo "C=$c VP_CONV_DBG=$v" >> gpurun_out/exp5.txt
  VP_CONV_DBG=$v timeout 300 python tools/cta_probe.py $c 2>/dev/null | grep -E "^rows|end:" >> gpurun_out/exp5.txt
done; done
cat gpurun_out/exp5.txt
