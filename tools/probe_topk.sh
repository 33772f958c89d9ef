#!/bin/bash
# top-k stage probe: parity subset, eigen-round trace and warm kernel profile on large
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "topk or cluster or run_" > gpurun_out/pt_topk.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pt_topk.log
CFG=large TPO_TRACE_EIG=1 python tools/topk_probe.py > gpurun_out/topk_large.log 2>&1
CFG=large REPS=3 python tools/kprof.py > gpurun_out/kprof_large.txt 2>&1
