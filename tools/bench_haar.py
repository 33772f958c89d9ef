"""Time the device Haar rotation (tpo_haar_q_dev) alone for d in DS under TPO_HAAR_PANEL values."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2405_11922_b200 as T

for d in [int(x) for x in os.environ.get("DS", "1000,512,256").split(",")]:
    G = np.random.default_rng(d).standard_normal((d, d))
    for pw in os.environ.get("PANELS", "32,64,96,112").split(","):
        os.environ["TPO_HAAR_PANEL"] = pw
        for _ in range(2):
            T.haar_q_dev(G)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            Q = T.haar_q_dev(G)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        err = float(np.abs(Q.cpu().numpy().astype(np.float64).T @ Q.cpu().numpy() - np.eye(d)).max())
        print(f"d={d} panel={pw}: {1e3 * sorted(ts)[2]:.3f} ms  |QtQ-I|={err:.1e}", flush=True)
