#!/bin/bash
# Gram A^T A single-copy + two row splits per SM, UPS 3 CTAs/SM: per-kernel profile + affected parity tests
set -u
python -m paper_2405_11922_b200.build > /dev/null 2>&1
REPS=2 timeout 300 python tools/kprof.py 2>&1 | grep -v Warn | head -14 > gpurun_out/k_kprof.txt
timeout 1500 python -m pytest tests -q -m gpu -k "cluster or run_ or atb or topk or ups or sharded" -x > gpurun_out/k_pytest.log 2>&1; tail -2 gpurun_out/k_pytest.log
