#!/bin/bash
# Round-2 session-g ncu --set full captures on the large config (one B200, under gpurun): the SpMM pair of
# hop 1, the tcgen05 features / Gram kernels, the integer-tensor-core ONMF products and the Alg. 2 / 3
# row kernels, each from one tpo_run (tools/prof_run.py CFG=large REPS=1); summaries by tools/ncu_summary.py.
set -u
export CFG=large REPS=1
python tools/prof_run.py > gpurun_out/r2g_plain_run.log 2>&1 || { echo plain-failed; tail -5 gpurun_out/r2g_plain_run.log; exit 1; }
for spec in "spmm:spmm_kernel:0:2" "tc:features_tc_kernel|gram_tc_kernel:0:2" "oz:oz_rtu_kernel|oz_aw_kernel:1:2" \
            "rows:oa_assign_kernel|dm_rowk_kernel|dm_atb_bulk_kernel|cluster_sums_kernel:4:6"; do
  IFS=: read tag name skip cnt <<< "$spec"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$name" -s $skip -c $cnt \
      -f -o gpurun_out/r2g_${tag}_large python tools/prof_run.py > gpurun_out/r2g_ncu_$tag.log 2>&1
  echo "$tag=$?"
  python tools/ncu_summary.py gpurun_out/r2g_${tag}_large.ncu-rep > gpurun_out/r2g_${tag}_large_summary.txt 2>&1
  cat gpurun_out/r2g_${tag}_large_summary.txt
  [ "$tag" = rows ] && rm -f gpurun_out/r2g_rows_large.ncu-rep
done
echo done
