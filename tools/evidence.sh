#!/bin/bash
# Round-end evidence in one gpurun call: full GPU suite, bench lines (default, reference arm,
# medium, large), the launch list of one bench step, ncu --set full of the propagation SpMMs.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build-failed; tail -20 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/ev_pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/ev_pytest_gpu.log
timeout 400 python bench.py > gpurun_out/ev_bench_small.log 2>&1; echo bench=$?; tail -1 gpurun_out/ev_bench_small.log | cut -c1-300
timeout 400 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/ev_bench_reference.log 2>&1; echo ref=$?
for c in medium large; do
  timeout 400 python bench.py --config $c --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/ev_bench_$c.log 2>&1; echo $c=$?
done
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/ev_launches_small.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ev_ncu_launch.log 2>&1; echo launches=$?
timeout 400 ncu --set full --clock-control none --import-source on -k regex:spmm_kernel -s 10 -c 2 -o gpurun_out/ev_spmm_small python tools/prof_prop.py > gpurun_out/ev_ncu_spmm.log 2>&1; echo ncu_spmm=$?
