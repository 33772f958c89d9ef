#!/bin/bash
# One gpurun pass: build, GPU parity suite, default bench, launch list of one bench step.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build-failed; tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo bench=$?; tail -c 1500 gpurun_out/bench.log
if [ -n "$LAUNCHES" ]; then
  timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/ncu.log 2>&1; echo ncu=$?
fi
