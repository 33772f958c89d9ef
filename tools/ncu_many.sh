#!/bin/bash
# ncu --set full of several kernels of one tpo_run (second run), one capture per kernel family.
python tools/prof_run.py > gpurun_out/plain_run.log 2>&1 || { echo plain-failed; exit 1; }
for spec in "aw_stream:6:1" "onmf_rtu:5:1" "gram_tc:1:1" "features_tc:1:1" "spmm_kernel:10:2" "chol_inv_blk:45:1" "nci_fused:19:1"; do
  IFS=: read name skip cnt <<< "$spec"
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:$name -s $skip -c $cnt -o gpurun_out/k_$name python tools/prof_run.py > gpurun_out/ncu_$name.log 2>&1
  echo "$name=$?"
done
