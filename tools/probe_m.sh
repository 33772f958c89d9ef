#!/bin/bash
# R-free a7-a9 GPU tests (full file) + per-kernel profile of a large step
set -u
python -m paper_2405_11922_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_rfree.py -q > gpurun_out/m_rfree.log 2>&1; tail -2 gpurun_out/m_rfree.log
REPS=2 timeout 300 python tools/kprof.py 2>&1 | grep -v Warn > gpurun_out/m_kprof.txt
