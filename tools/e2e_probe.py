"""Time the host->device input copies alone, the device-input run and the host-input run."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2405_11922_b200 as T
from synth import make_config

g = make_config(os.environ.get("CFG", "small"))
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
hX, hBr, hBc, hTr, hTc, hG = pin(g.X), pin(g.B_rowptr), pin(g.B_col), pin(g.Bt_rowptr), pin(g.Bt_col), pin(np.asarray(g.G, np.float64))
dX = torch.empty_like(hX, device="cuda")
dB = [torch.empty_like(t, device="cuda") for t in (hBr, hBc, hTr, hTc, hG)]
st = torch.cuda.current_stream()


def timed(fn, reps=5):
    ts = []
    for _ in range(reps + 1):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fn()
        e1.record(st)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts[1:]))


def copies():
    for d, h in zip(dB, (hBr, hBc, hTr, hTc, hG)):
        d.copy_(h, non_blocking=True)
    dX.copy_(hX, non_blocking=True)


print("copies only      %.3f ms (%.1f GB/s)" % (timed(copies), 0))
dg = T.to_device_graph(g.n, g.m, g.B_rowptr, g.B_col, g.Bt_rowptr, g.Bt_col)
X = torch.from_numpy(g.X).cuda()
Gd = torch.from_numpy(np.asarray(g.G, np.float64)).cuda()
r = T.Runner(dg, g.d, g.k)
print("device run       %.3f ms" % timed(lambda: r(X, g.alpha, g.T, Gd)), r.timings)
hr = T.HostRunner(g.n, g.m, g.nnz, g.d, g.k)
hl = torch.empty(g.n, dtype=torch.int32).pin_memory()
print("host run         %.3f ms" % timed(lambda: hr(hBr, hBc, hTr, hTc, hX, hG, g.alpha, g.T, labels=hl)), hr.timings)
Gh = np.asarray(g.G, np.float64)
print("haar alone (host G, incl. ws alloc)  %.3f ms" % timed(lambda: T.haar_q_dev(Gh)))
