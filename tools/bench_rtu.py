"""Warm timing of Alg. 2's R^T Ups (tpo_shard_onmf_rtu over all rows) on the large shape:
integer tensor cores (default) vs the fp64 DMMA path (TPO_OZ=0)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2405_11922_b200 as T

n, D, k = int(os.environ.get("N", 2_000_000)), int(os.environ.get("D", 256)), int(os.environ.get("K", 50))
g = torch.Generator(device="cuda").manual_seed(0)
A = (np.sqrt(np.e / (D // 2)) * torch.sin(torch.rand(n, D, device="cuda", generator=g) * 12 - 6)).float()
U = (torch.rand(n, k, device="cuda", generator=g, dtype=torch.float64) / np.sqrt(n) + 1e-12)
dinv = (torch.rand(n, device="cuda", generator=g) * 2 + 0.5).float()


def timed(reps=10):
    out = T.onmf_rtu(A, dinv, U)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        T.onmf_rtu(A, dinv, U, out=out)
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps, out


t_oz, o1 = timed()
os.environ["TPO_OZ"] = "0"
t_dm, o2 = timed()
rel = ((o1 - o2).abs().max() / o2.abs().max()).item()
print(f"R^T Ups n={n} D={D} k={k}: oz {t_oz:.3f} ms, DMMA {t_dm:.3f} ms, max|oz-dm|/max|dm| = {rel:.2e}")
