#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "propagate or run_" > gpurun_out/pt_par.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pt_par.log
CFG=large REPS=1 timeout 600 ncu --set full --clock-control none --import-source on \
    -k regex:"features_tc_kernel|gram_tc_kernel|split_tf32_kernel|degree_scale" -c 4 \
    -o gpurun_out/feat_large python tools/prof_run.py > gpurun_out/ncu_feat.log 2>&1
