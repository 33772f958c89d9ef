#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_oz.py -x -q -m gpu > gpurun_out/pt_par.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pt_par.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -m gpu -k "large or xl" > gpurun_out/pt_c.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pt_c.log
CFG=large TPO_TRACE_EIG=1 timeout 600 python tools/prof_topk.py > gpurun_out/prof_topk_large.txt 2>&1
CFG=large REPS=3 timeout 600 python tools/kprof.py > gpurun_out/kprof_large.txt 2>&1
