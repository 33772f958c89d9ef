#!/bin/bash
# Session g: the small config's device-resident propagation measured 7.4 ms in the evidence run against
# 4.3-4.8 ms in every earlier session with the same SpMM code: re-measure (two bench runs, warm per-kernel profile).
set -u
timeout 600 python bench.py --config small --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2g_small_a.log 2>&1; tail -1 gpurun_out/r2g_small_a.log | cut -c1-100
timeout 600 python bench.py --config small --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2g_small_b.log 2>&1; tail -1 gpurun_out/r2g_small_b.log | cut -c1-100
CFG=small timeout 300 python tools/kprof.py > gpurun_out/r2g_kprof_small.log 2>&1; grep -v Warn gpurun_out/r2g_kprof_small.log | head -14
CFG=small REPS=3 timeout 300 python tools/prof_prop.py > gpurun_out/r2g_prop_small.log 2>&1
python - <<'PY' > gpurun_out/r2g_prop_small_times.log 2>&1
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2405_11922_b200 as T
from synth import make_config
g = make_config("small")
dg = T.to_device_graph(g.n, g.m, g.B_rowptr, g.B_col, g.Bt_rowptr, g.Bt_col, device="cuda:0")
X = torch.from_numpy(g.X).cuda()
for _ in range(3): T.propagate(dg, X, g.alpha, g.T)
torch.cuda.synchronize()
ts = []
for _ in range(10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); T.propagate(dg, X, g.alpha, g.T); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
print("tpo_propagate alone, small, ms:", [round(t, 3) for t in ts])
PY
cat gpurun_out/r2g_prop_small_times.log
echo done
