#!/bin/bash
# Round-2 evidence (session g) on one B200 (run from the repo root under gpurun; outputs in gpurun_out/):
# full GPU suite, smoke, bench lines for every config + the reference arm, the ncu launch list of the
set -u
python -m paper_2405_11922_b200.build > /dev/null 2>&1
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r2g_pytest.log 2>&1; tail -2 gpurun_out/r2g_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/r2g_smoke.log 2>&1; tail -1 gpurun_out/r2g_smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2g_bench_large.log 2>&1
timeout 600 python bench.py --config small --steps 10 --warmup 3 > gpurun_out/r2g_bench_small.log 2>&1
timeout 600 python bench.py --config medium --steps 10 --warmup 3 > gpurun_out/r2g_bench_medium.log 2>&1
timeout 900 python bench.py --config xl --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2g_bench_xl.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2g_bench_ref.log 2>&1
timeout 300 python tools/kprof.py > gpurun_out/r2g_kprof_large.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv \
    --log-file gpurun_out/r2g_launches_large.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
    > gpurun_out/r2g_ncu_bench.log 2>&1
echo done
