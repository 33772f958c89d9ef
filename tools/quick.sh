#!/bin/bash
# quick GPU iteration: build, a subset of the GPU tests (PYK), small + large bench stages, launch list of KREGEX
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build-failed; tail -20 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests -m gpu -x -q --ignore=tests/test_gpu_fullsize.py ${PYK:+-k "$PYK"} > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
for c in ${CFGS:-small large}; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 5 --warmup 3 > gpurun_out/b_$c.log 2>&1
  echo $c; grep -o "\"ms_per_step\": [0-9.]*\|\"stages_ms\": {[^}]*}" gpurun_out/b_$c.log
done
if [ -n "$KREGEX" ]; then
  timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$KREGEX" -c 200 --csv --log-file gpurun_out/klaunch.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu=$?
  python tools/launches.py gpurun_out/klaunch.csv
fi
