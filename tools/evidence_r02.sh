#!/bin/bash
# Round-2 evidence on one B200: bench line (large), launch list of one large step, ncu --set full
# of the dominant kernels.  Run from the repo root under gpurun; outputs in gpurun_out/.
set -u
python -m paper_2405_11922_b200.build > /dev/null 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2e_bench.log 2>&1
CFG=large REPS=2 python tools/prof_run.py > gpurun_out/r2e_plain.log 2>&1 && \
CFG=large REPS=2 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv \
    --log-file gpurun_out/r2e_launches_large.csv python tools/prof_run.py > /dev/null 2>&1
CFG=large REPS=1 ncu --set full --clock-control none --import-source on \
    -k regex:"dm_rowgemm|dm_rtu|dm_rowk|dm_atb_bulk|features_tc|gram_tc" -c 8 \
    -o gpurun_out/r2e_tensor_large python tools/prof_run.py > gpurun_out/r2e_ncu.log 2>&1
echo done
