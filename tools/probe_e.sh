#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_oz.py tests/test_gpu_eval.py tests/test_gpu_reduce.py -x -q -m gpu > gpurun_out/pt_par.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pt_par.log
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q -m gpu > gpurun_out/pt_full.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pt_full.log
CFG=large REPS=3 timeout 600 python tools/kprof.py > gpurun_out/kprof_large.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/be_large.log 2>&1
