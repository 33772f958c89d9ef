#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_oz.py -x -q -m gpu -k rtu > gpurun_out/pt_rtu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pt_rtu.log
timeout 300 python tools/bench_rtu.py > gpurun_out/bench_rtu.log 2>&1
K=64 timeout 300 python tools/bench_rtu.py >> gpurun_out/bench_rtu.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"oz_|dm_rtu" --csv python tools/bench_rtu.py > gpurun_out/rtu_launches.csv 2>&1
