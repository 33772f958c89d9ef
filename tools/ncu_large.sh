#!/bin/bash
# ncu --set full of the discretisation kernels on the large config (k = 50).
export CFG=large REPS=1
python tools/prof_run.py > gpurun_out/plain_large_run.log 2>&1 || { echo plain-failed; tail -5 gpurun_out/plain_large_run.log; exit 1; }
for spec in "onmf_rtu:2:1" "aw_stream:3:1" "assign_small:5:1" "ups_update:2:1" "cluster_sums:5:1" "dgemm_kernel<1:0:1"; do
  IFS=: read name skip cnt <<< "$spec"
  tag=$(echo $name | tr -cd 'a-z_')
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$name" -s $skip -c $cnt -o gpurun_out/L_$tag python tools/prof_run.py > gpurun_out/ncuL_$tag.log 2>&1
  echo "$name=$?"
done
