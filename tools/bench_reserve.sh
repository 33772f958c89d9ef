#!/bin/bash
# tpo_run step time under Haar-reserve schedules (sms,launches)
for r in ${RESERVES:-"8,1000" "16,4" "24,2" "24,4" "32,2" "0,0"}; do
  TPO_HAAR_RESERVE=$r timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/br_$r.log 2>&1
  echo "$r $(grep -o '"ms_per_step": [0-9.]*\|"stages_ms": {[^}]*}' gpurun_out/br_$r.log | tr '\n' ' ')"
done
