#!/bin/bash
# host-input path: B's column ids copied on a side stream during hop 1's V-side SpMM (parity + e2e)
set -u
python -m paper_2405_11922_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests -q -m gpu -k "run_host or run_tiny or smoke" > gpurun_out/n_pytest.log 2>&1; tail -2 gpurun_out/n_pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/n_bench_large.log 2>&1; grep '^{' gpurun_out/n_bench_large.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e'])"
