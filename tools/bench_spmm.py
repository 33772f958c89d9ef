"""Time tpo_propagate under the SpMM layouts on BASELINE configs:
  LAYOUTS -- TPO_SPMM_L = "Lp,Lq" (column-group widths in float4 of P and Q; "0,0" = row-major).
  (RANGES -- TPO_SPMM_RANGES, the column-range passes measured in round 2, were removed: slower
  everywhere and a register-pressure cost to the default kernel.)
Variants sum in different (fixed) orders: results agree to fp32 rounding (relF printed vs the
first variant).  The L2 is flushed before every timed call."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2405_11922_b200 as T
from synth import make_config

cfgs = os.environ.get("CFGS", "large").split(",")
ranges = ["1,1"]
layouts = os.environ.get("LAYOUTS", "0,0").split(";")
reps = int(os.environ.get("REPS", "5"))
for cfg in cfgs:
    g = make_config(cfg)
    dg = T.to_device_graph(g.n, g.m, g.B_rowptr, g.B_col, g.Bt_rowptr, g.Bt_col, device="cuda:0")
    X = torch.from_numpy(g.X).cuda()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda:0")
    ref = None
    for lay in layouts:
        for rg in ranges:
            if lay != "0,0" and rg != ranges[0]:
                continue
            os.environ["TPO_SPMM_L"] = lay
            if rg == "auto":
                os.environ.pop("TPO_SPMM_RANGES", None)
            else:
                os.environ["TPO_SPMM_RANGES"] = rg
            Z, Zh = T.propagate(dg, X, g.alpha, g.T)
            torch.cuda.synchronize()
            ts = []
            for _ in range(reps):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                Z, Zh = T.propagate(dg, X, g.alpha, g.T, Z=Z, Zhat=Zh)
                e1.record()
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            if ref is None:
                ref = Z.clone()
                rel = 0.0
            else:
                rel = float(torch.linalg.norm((Z - ref).double()) / torch.linalg.norm(ref.double()))
            ts.sort()
            print(f"{cfg} d={g.d} nnz={g.nnz} T={g.T} layout={lay} ranges={rg}: median {ts[reps // 2]:.3f} ms "
                  f"min {ts[0]:.3f} ms per hop {ts[reps // 2] / g.T:.3f} ms  relF vs first {rel:.2e}", flush=True)
    del dg, X, Z, Zh, flush, ref
    torch.cuda.empty_cache()
