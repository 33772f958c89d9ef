"""GPU idle gaps inside one warm tpo_run step (torch.profiler / CUPTI): the kernels in launch order
with the idle time before each, summed per stage window; CFG (default large)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
import paper_2405_11922_b200 as T
from synth import make_config

g = make_config(os.environ.get("CFG", "large"))
dg = T.to_device_graph(g.n, g.m, g.B_rowptr, g.B_col, g.Bt_rowptr, g.Bt_col, device="cuda:0")
X = torch.from_numpy(g.X).cuda()
runner = T.Runner(dg, g.d, g.k, device="cuda:0")
for _ in range(3):
    runner(X, g.alpha, g.T, g.G, 5, 20)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    runner(X, g.alpha, g.T, g.G, 5, 20)
    runner(X, g.alpha, g.T, g.G, 5, 20)
    torch.cuda.synchronize()
ev = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA],
            key=lambda e: e.time_range.start)
half = len(ev) // 2
ev = ev[half:]                                   # the second step (the first absorbs CUPTI buffer setup)
t0 = ev[0].time_range.start
prev = ev[0].time_range.start
gaps = []
for e in ev:
    gap = (e.time_range.start - prev) / 1000.0
    gaps.append((gap, (e.time_range.start - t0) / 1000.0, e.name[:70]))
    prev = max(prev, e.time_range.end)
print(f"kernels {len(ev)} span {(prev - t0) / 1000.0:.3f} ms, total idle {sum(g for g, _, _ in gaps):.3f} ms")
for gap, t, name in sorted(gaps, reverse=True)[:25]:
    print(f"  idle {gap:7.3f} ms before t={t:8.3f} ms  {name}")
