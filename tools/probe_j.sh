#!/bin/bash
# A/B of the UPS kernel launch (one CTA with a 2-slot ring vs several 1-slot CTAs per SM) + cluster parity
set -u
python -m paper_2405_11922_b200.build > /dev/null 2>&1
TPO_UPS_OLD=1 REPS=2 timeout 300 python tools/kprof.py 2>&1 | grep -v Warn | head -12 > gpurun_out/j_kprof_old.txt
REPS=2 timeout 300 python tools/kprof.py 2>&1 | grep -v Warn | head -12 > gpurun_out/j_kprof_new.txt
timeout 1200 python -m pytest tests -q -m gpu -k "cluster or run_matches or ups" -x > gpurun_out/j_pytest.log 2>&1; tail -2 gpurun_out/j_pytest.log
