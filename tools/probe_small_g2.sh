#!/bin/bash
# Session g: run-to-run spread of the small config's propagation stage inside tpo_run under Haar-reserve
# schedules TPO_HAAR_RESERVE = "sms,launches" (default 16 SMs for every launch); three runs each.
for r in "16,1073741824" "32,1073741824" "0,0" "16,4"; do
  for i in 1 2 3; do
    TPO_HAAR_RESERVE=$r timeout 300 python bench.py --config small --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2g_bs_${r}_$i.log 2>&1
    echo "$r run $i $(grep -o '"ms_per_step": [0-9.]*\|"stages_ms": {[^}]*}' gpurun_out/r2g_bs_${r}_$i.log | head -2 | tr '\n' ' ')"
  done
done
