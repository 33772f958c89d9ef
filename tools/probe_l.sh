#!/bin/bash
# R-free a7-a9 GPU tests, the fused Ups-update column maxima (cluster parity), per-kernel profile
set -u
python -m paper_2405_11922_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_rfree.py -q -x > gpurun_out/l_rfree.log 2>&1; tail -2 gpurun_out/l_rfree.log
REPS=2 timeout 300 python tools/kprof.py 2>&1 | grep -v Warn | head -16 > gpurun_out/l_kprof.txt
timeout 1500 python -m pytest tests -q -m gpu -k "cluster or run_ or ups" -x > gpurun_out/l_pytest.log 2>&1; tail -2 gpurun_out/l_pytest.log
