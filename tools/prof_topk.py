"""Kernel-by-kernel device times of ONE warm topk_eig call (torch.profiler / CUPTI), in launch order,
with the host gaps: where the exact top-k's time goes (CFG, default large)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
import paper_2405_11922_b200 as T
from synth import make_config

g = make_config(os.environ.get("CFG", "large"))
dg = T.to_device_graph(g.n, g.m, g.B_rowptr, g.B_col, g.Bt_rowptr, g.Bt_col)
X = torch.from_numpy(g.X).cuda()
Z, Zh = T.propagate(dg, X, g.alpha, g.T)
del Z
Q = T.haar_q_dev(g.G)
Rp, dinv, r = T.features(Zh, Q, want_r=True)
for _ in range(2):
    T.topk_eig(Rp, dinv, g.k)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    T.topk_eig(Rp, dinv, g.k)
    torch.cuda.synchronize()
ev = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA],
            key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
prev_end = t0
tot = 0.0
for e in ev:
    gap = (e.time_range.start - prev_end) / 1000.0
    d = (e.time_range.end - e.time_range.start) / 1000.0
    tot += d
    print(f"{(e.time_range.start - t0) / 1000.0:9.3f} ms  +gap {gap:7.3f}  {d * 1000:8.1f} us  {e.name[:90]}")
    prev_end = e.time_range.end
print(f"kernels {len(ev)}  busy {tot:.3f} ms  span {(ev[-1].time_range.end - t0) / 1000.0:.3f} ms")
api = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CPU],
             key=lambda e: e.time_range.start)
print("host-side runtime calls longer than 20 us:")
for e in api:
    d = (e.time_range.end - e.time_range.start) / 1000.0
    if d > 0.02:
        print(f"  {(e.time_range.start - t0) / 1000.0:9.3f} ms  {d:8.3f} ms  {e.name[:80]}")
