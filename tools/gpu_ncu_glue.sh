set -u
mkdir -p gpurun_out
for k in conv_stem_kernel bn_apply_kernel split_reduce_epi_kernel head_kernel; do
  timeout 300 ncu --set full --clock-control none -k regex:$k -s 20 -c 1 -o gpurun_out/glue_$k -f python bench.py --profile-only --no-graph > gpurun_out/ncu_glue_$k.log 2>&1
  echo "ncu $k rc=$?"
  ncu -i gpurun_out/glue_$k.ncu-rep --page raw --csv > gpurun_out/glue_$k.raw.csv 2>/dev/null
  ncu -i gpurun_out/glue_$k.ncu-rep --page details > gpurun_out/glue_$k.details.txt 2>/dev/null
  rm -f gpurun_out/glue_$k.ncu-rep
done
