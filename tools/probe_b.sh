#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_oz.py -x -q -m gpu > gpurun_out/pt_oz.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pt_oz.log
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q -m gpu > gpurun_out/pt_full.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pt_full.log
CFG=large REPS=3 timeout 600 python tools/kprof.py > gpurun_out/kprof_large.txt 2>&1
CFG=large timeout 600 python tools/prof_topk.py > gpurun_out/prof_topk_large.txt 2>&1
