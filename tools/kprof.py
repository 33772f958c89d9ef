"""Per-kernel device time of warm tpo_run steps (CUPTI via torch.profiler; real stream overlap,
warm caches -- the complement of ncu's serialised cold-cache launch list).  CFG (default large),
REPS timed steps after 2 warm-ups; prints kernels sorted by total time per step."""
import os
import sys
from collections import defaultdict
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
import paper_2405_11922_b200 as T
from synth import make_config

g = make_config(os.environ.get("CFG", "large"))
reps = int(os.environ.get("REPS", 3))
dg = T.to_device_graph(g.n, g.m, g.B_rowptr, g.B_col, g.Bt_rowptr, g.Bt_col, device="cuda:0")
X = torch.from_numpy(g.X).cuda()
runner = T.Runner(dg, g.d, g.k, device="cuda:0")
for _ in range(2):
    runner(X, g.alpha, g.T, g.G, 5, 20)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(reps):
        runner(X, g.alpha, g.T, g.G, 5, 20)
    torch.cuda.synchronize()
tot, cnt = defaultdict(float), defaultdict(int)
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        tot[e.name] += e.device_time_total / 1000.0
        cnt[e.name] += 1
print(f"{os.environ.get('CFG', 'large')}: stage ms of the last step {list(runner.timings)}")
s = sum(tot.values()) / reps
for name, t in sorted(tot.items(), key=lambda x: -x[1])[:40]:
    short = name if len(name) < 70 else name[:67] + "..."
    print(f"{short:72s} {cnt[name] / reps:7.1f} {t / reps:9.3f} ms/step {100 * t / reps / s:5.1f}%  "
          f"{t / cnt[name] * 1000:9.1f} us/launch")
print(f"total kernel time {s:.3f} ms/step")
