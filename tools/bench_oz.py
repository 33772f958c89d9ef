"""Time tpo_rowgemm_f64 (RH = dinv . (R' H)) on the integer tensor cores vs the fp64 DMMA path
(TPO_OZ=0) at a config's shape (n, D = 2d, k): median of REPS calls, L2 flushed between calls."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2405_11922_b200 as T

shapes = {"large": (2_000_000, 256, 50), "medium": (500_000, 512, 20), "xl": (10_000_000, 256, 100),
          "small": (50_000, 2000, 10)}
reps = int(os.environ.get("REPS", 7))
for cfg in os.environ.get("CFGS", "large,medium").split(","):
    n, D, k = shapes[cfg]
    g = torch.Generator(device="cuda").manual_seed(0)
    A = (torch.rand(n, D, device="cuda", generator=g) - 0.5) * 0.2
    W = torch.rand(D, k, device="cuda", generator=g, dtype=torch.float64) * 0.1
    rs = torch.rand(n, device="cuda", generator=g) + 0.5
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    res = {}
    for mode in ("1", "0"):
        os.environ["TPO_OZ"] = mode
        out = T.rowgemm_f64(A, W, rs)
        ts = []
        for _ in range(reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            T.rowgemm_f64(A, W, rs, out=out)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        res[mode] = (sorted(ts)[reps // 2], out.clone())
    d = (res["1"][1] - res["0"][1]).abs().max().item() / res["0"][1].abs().max().item()
    print(f"{cfg} n={n} D={D} k={k}: integer-TC {res['1'][0]:.3f} ms  fp64 DMMA {res['0'][0]:.3f} ms  "
          f"max|diff|/max|out| {d:.2e}", flush=True)
