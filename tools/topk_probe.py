"""Warm timings of the top-k stage pieces on a config: gram alone, topk_eig (incl. gram, ws alloc)."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2405_11922_b200 as T
from synth import make_config

g = make_config(os.environ.get("CFG", "small"))
dg = T.to_device_graph(g.n, g.m, g.B_rowptr, g.B_col, g.Bt_rowptr, g.Bt_col)
X = torch.from_numpy(g.X).cuda()
Z, Zh = T.propagate(dg, X, g.alpha, g.T)
Q = T.haar_q_dev(g.G)
Rp, dinv, r = T.features(Zh, Q, want_r=True)


def timed(fn, reps=5):
    ts = []
    for _ in range(reps + 1):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append((e0.elapsed_time(e1), 1e3 * (time.perf_counter() - t0)))
    ts = ts[1:]
    return np.median([a for a, b in ts]), np.median([b for a, b in ts])


print("gram      device %.3f ms  wall %.3f ms" % timed(lambda: T.gram(Rp, dinv)))
print("topk_eig  device %.3f ms  wall %.3f ms" % timed(lambda: T.topk_eig(Rp, dinv, g.k)))
