#!/bin/bash
mkdir -p gpurun_out
CFG=large timeout 600 python tools/prof_run_gaps.py > gpurun_out/gaps_large.txt 2>&1
