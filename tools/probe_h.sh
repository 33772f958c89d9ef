#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "features or run_ or rfree" > gpurun_out/pt_par.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pt_par.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -m gpu -k "features" > gpurun_out/pt_full.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pt_full.log
CFG=large REPS=3 timeout 600 python tools/kprof.py > gpurun_out/kprof_large.txt 2>&1
