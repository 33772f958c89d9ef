#!/usr/bin/env python
"""bench.py -- the TPO hot path (arXiv 2405.11922) on B200: one step = one whole pass of
propagate -> Haar Q -> features -> exact top-k -> ONMF + NCI over BASELINE.json's
configs[3] ("large", the largest configuration that fits one GPU; xl is the 8-GPU config) by
default, through libtpo's C-ABI (tpo_run).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config large]

Prints ONE JSON line (rank 0).  BASELINE.json's metric is the pair "MSA propagation GB/s &
nnz*d/s; end-to-end TPO seconds": `value` is the MSA-propagation work of a step
(2 * nnz * d * T multiply-adds, i.e. nnz*d per SpMM) per END-TO-END TPO second with inputs
resident in HBM (so it moves with the whole step, not only with the propagation);
`tpo_seconds` is the end-to-end step time, and `propagation_nnz_d_per_s` /
`propagation_gb_per_s` the propagation alone.  `e2e` is the same metric with host inputs
copied in and labels copied out inside the timed region.  --impl reference times the fp64
CPU oracle (oracle/) on a bounded, stage-by-stage sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import threading
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return PEAKS_FALLBACK, "fallback"


def propagation_bytes(n, m, nnz, d):
    """SURVEY.md §8(d) compulsory bytes per hop (unit weights): Z read (SpMM-1), X read and
    Z write (SpMM-2), the V-side block written and read, int32 indices of both CSRs, int64
    row pointers, and the two degree-scale vectors."""
    return 4 * (3 * n * d + 2 * m * d) + 2 * 4 * nnz + 8 * (n + m + 2) + 4 * (n + m)


class ClockSampler:
    """SM clocks and clock-event reasons sampled DURING the timed region: NVML every 10 ms from a
    background thread (a 50 ms region is shorter than nvidia-smi's start-up), with `nvidia-smi
    -lms 100` as the fallback when NVML is unavailable."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # NVML clocks-event reason bits (nvmlClocksEventReason*)
    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40}

    def __init__(self, index=0):
        self.index = index
        self.p = None
        self.nv = None
        self.samples = []
        self.lines = []

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.nv = (pynvml, h)
            self.mx = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            self.stop = threading.Event()

            def loop():
                while True:
                    try:
                        sm = float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                        rs = int(pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)) \
                            if hasattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons") \
                            else int(pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h))
                        self.samples.append((sm, rs))
                    except Exception:
                        pass
                    if self.stop.wait(0.010):
                        break
            self.th = threading.Thread(target=loop, daemon=True)
            self.th.start()
            return self
        except Exception:
            self.nv = None
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.nv is not None:
            self.stop.set()
            self.th.join(timeout=1)
            return
        if self.p is not None:
            self.p.terminate()
            try:
                out, _ = self.p.communicate(timeout=5)
                self.lines = [l for l in out.splitlines() if l.strip()]
            except Exception:
                self.p.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        if self.nv is not None:
            mx = self.mx
            for f, rs in self.samples:
                sm.append(f)
                for nm, bit in self.BITS.items():
                    if rs & bit:
                        reasons.add(nm)
            return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                    "samples": len(sm), "source": "nvml"}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
                for nm, v in zip(names, f[2:6]):
                    if v.lower().startswith("active"):
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvidia-smi"}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


ORACLE_ROW_FRACTION = 32      # a5-a9 of the oracle sample run on n / 32 rows (their cost is linear in n)


def oracle_stage_sample(g, args):
    """One bounded, stage-by-stage sample of the whole oracle pipeline (a1-a9) on this workload,
    extrapolated to one full step.  a1-a3: ONE of the T hops over the full graph (each hop costs
    the same).  a4: the Haar QR of G (d x d, once per step).  a5-a9 on the first n/16 U rows
    of that hop's Zhat (the ids are shuffled, so this is a random row sample; features, Gram,
    Gamma, ONMF and NCI costs are linear in n): features, the exact top-k, ONE ONMF iteration and
    ONE Alg. 3 iteration, scaled by 32 and by Tf / Tg -- except the top-k's D x D Jacobi
    eigensolve, which does not depend on n and is timed on its own and counted once.  Returns (seconds per full step, stage
    dict, sample text)."""
    from oracle import core as O
    O.lib()
    t = {}
    t0 = time.perf_counter()
    _, Zh = O.propagate(g.n, g.m, g.B_rowptr, g.B_col, g.X, g.alpha, 1, g.B_val)
    t["propagate_hop"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    Q = O.haar_q(g.G)
    t["haar"] = time.perf_counter() - t0
    ns = max(min(g.n, 4096), g.n // ORACLE_ROW_FRACTION)
    scale = g.n / ns
    Zs = np.ascontiguousarray(Zh[:ns], np.float32)
    del Zh
    t0 = time.perf_counter()
    Rp, dinv, _ = O.features(Zs, Q.astype(np.float32))
    t["features"] = time.perf_counter() - t0
    Rp32, dv32 = Rp.astype(np.float32), dinv.astype(np.float32)
    del Rp
    # the D x D eigensolve: the oracle's Jacobi, or LAPACK eigh for D > 600 (as the parity tests;
    # cyclic Jacobi at D = 2000 alone takes minutes)
    eig = "lapack" if Rp32.shape[1] > 600 else "jacobi"
    t0 = time.perf_counter()
    Gm, s, Ps, _ = O.topk(Rp32, dv32, g.k, eig=eig)
    t["topk"] = time.perf_counter() - t0
    Gs = O.gram(Rp32, dv32)
    t0 = time.perf_counter()
    if eig == "lapack":
        np.linalg.eigh(Gs)
    else:
        O.sym_eig(Gs)
    t_jac = min(time.perf_counter() - t0, t["topk"])
    t0 = time.perf_counter()
    U, _ = O.onmf(Rp32, dv32, Gm.astype(np.float32), s, Ps.astype(np.float32), 1)
    t["onmf_iter"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    O.nci(U, 1)
    t["nci_iter"] = time.perf_counter() - t0
    stages = {"propagate": g.T * t["propagate_hop"] + t["haar"], "features": scale * t["features"],
              "topk_eig": scale * (t["topk"] - t_jac) + t_jac, "cluster": scale * (args.tf * t["onmf_iter"] + args.tg * t["nci_iter"])}
    step_s = sum(stages.values())
    sample = (f"oracle (fp64 C, OpenMP) stage by stage on {g.name}: 1 of T={g.T} propagation hops over the full graph "
              f"+ Haar QR; features, exact top-k, 1 of Tf={args.tf} ONMF and 1 of Tg={args.tg} NCI iterations on "
              f"{ns:,} of {g.n:,} U rows; extrapolated to the full step (x T, x n/{ns} except the D x D "
              f"Jacobi, x Tf, x Tg); "
              f"measured {sum(t.values()):.1f} s")
    return step_s, {k: round(v * 1e3, 1) for k, v in stages.items()}, sample


def run_reference(args, g, ws, rank):
    """The fp64 oracle as it stands (the reference arm of this tier), each step one bounded
    stage-by-stage sample of the whole pipeline (oracle_stage_sample) on this workload; the
    step's time is the extrapolated full-step time, so `value` is our arm's metric."""
    if rank != 0:
        return
    cores = omp_cores()
    units = 2.0 * g.nnz * g.d * g.T
    times, stages, sample = [], None, ""
    for it in range(args.warmup + args.steps):
        step_s, stages, sample = oracle_stage_sample(g, args)
        if it >= args.warmup:
            times.append(step_s)
    tot = sum(times)
    value = units * len(times) / tot
    unit = "nnz*d/s"
    line = {"impl": "reference", "metric": metric_name(), "value": value, "unit": unit, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(g, args, ws), "stages_ms": stages, "tpo_seconds": tot / len(times),
            "cpu_baseline": {"value": value, "unit": unit, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def omp_cores():
    """Threads the oracle's OpenMP loops use (OMP_NUM_THREADS, else every core of the affinity mask)."""
    n = len(os.sched_getaffinity(0))
    try:
        return min(n, int(os.environ["OMP_NUM_THREADS"]))
    except (KeyError, ValueError):
        return n


def metric_name():
    return ("MSA-propagation nnz*d per end-to-end TPO second (pair: propagation_nnz_d_per_s / "
            "propagation_gb_per_s and tpo_seconds)")


def config_dict(g, args, ws):
    return {"workload": f"{g.name} planted ABG (BASELINE.json configs[{['tiny','small','medium','large','xl'].index(g.name)}])",
            "n_u": g.n, "n_v": g.m, "nnz": g.nnz, "d": g.d, "k": g.k, "alpha": g.alpha, "T": g.T, "Tf": args.tf,
            "Tg": args.tg, "eig": "exact", "seed": 0, "parallelism": f"replicas{ws}" if ws > 1 else "single",
            "units_per_step": "2*nnz*d*T (MSA-propagation multiply-adds)",
            "l2": "256 MiB L2 flush between timed steps; inputs also exceed L2"}


def cpu_baseline_sample(g, args):
    step_s, stages, sample = oracle_stage_sample(g, args)
    return {"value": 2.0 * g.nnz * g.d * g.T / step_s, "unit": "nnz*d/s", "cores": omp_cores(), "kind": "oracle",
            "sample": sample, "tpo_seconds": step_s, "stages_ms": stages}


def shard_inputs(args, ws, rank):
    """Every rank's share of the workload without every rank materialising the whole graph: rank 0
    generates it, writes each rank's U slice (CSR(B_p), CSR(B_p^T), X_p) to /dev/shm, and each rank
    loads only its own (host memory per rank ~ 1/ws of the graph; xl is ~22 GB whole)."""
    import shutil
    import types
    import torch.distributed as dist
    from paper_2405_11922_b200.sharded import HostShard, shard_graph
    from synth import make_config
    base = f"/dev/shm/tpo_bench_{os.environ.get('MASTER_PORT', '0')}"
    if rank == 0:
        g = make_config(args.config)
        os.makedirs(base, exist_ok=True)
        for r in range(ws):
            sh = shard_graph(g.n, g.m, g.B_rowptr, g.B_col, r, ws, g.B_val)
            np.savez(f"{base}/shard{r}.npz", Bp_rowptr=sh.Bp_rowptr, Bp_col=sh.Bp_col, Btp_rowptr=sh.Btp_rowptr,
                     Btp_col=sh.Btp_col, X=g.X[sh.u0:sh.u1], u0=sh.u0, u1=sh.u1)
        np.savez(f"{base}/meta.npz", G=g.G, n=g.n, m=g.m, nnz=g.nnz, d=g.d, k=g.k, alpha=g.alpha, T=g.T)
        del g
    dist.barrier()
    z = np.load(f"{base}/shard{rank}.npz")
    mt = np.load(f"{base}/meta.npz")
    meta = types.SimpleNamespace(name=args.config, G=mt["G"], n=int(mt["n"]), m=int(mt["m"]), nnz=int(mt["nnz"]),
                                 d=int(mt["d"]), k=int(mt["k"]), alpha=float(mt["alpha"]), T=int(mt["T"]))
    sh = HostShard(rank, ws, meta.n, meta.m, int(z["u0"]), int(z["u1"]), z["Bp_rowptr"], z["Bp_col"], z["Btp_rowptr"],
                   z["Btp_col"])
    Xp = np.ascontiguousarray(z["X"])
    dist.barrier()
    if rank == 0:
        shutil.rmtree(base, ignore_errors=True)
    return meta, sh, Xp


def run_sharded(args, g, ws, rank, local, dev, pre=None):
    """One graph, U rows split over the ranks: sharded propagation (NCCL
    reduce-scatter / all-gather of the V-side block per hop) and the sharded solver (fp64
    partials all-reduced); every rank computes the Haar rotation from G (replicated)."""
    import torch
    import torch.distributed as dist
    import paper_2405_11922_b200 as T
    from paper_2405_11922_b200._lib import lib
    from paper_2405_11922_b200.sharded import (GpuShardOps, GpuSolverOps, LibRunner, NcclComm, TorchCollectives,
                                               propagate_sharded, shard_graph, solve_sharded)
    if ws == 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    coll = TorchCollectives()
    if pre is not None:                       # (meta, shard, X_p) from shard_inputs
        g, sh, Xp_host = pre
    else:
        sh = shard_graph(g.n, g.m, g.B_rowptr, g.B_col, rank, ws, g.B_val)
        Xp_host = g.X[sh.u0:sh.u1]
    ops = GpuShardOps(sh, dev, g.d)
    sops = GpuSolverOps(sh.n_p, g.d, g.k, dev)
    Xp = torch.from_numpy(np.ascontiguousarray(Xp_host)).to(dev)
    L = lib()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    lib_run, comm = None, None
    if args.comm == "lib" and args.exchange == "full":
        # collectives inside libtpo (tpo_run_sharded on a library-owned NCCL communicator)
        uid = [NcclComm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = NcclComm(rank, ws, dev, uid[0])
        lib_run = LibRunner(comm, ops, g.d, g.k)
        Gd = torch.from_numpy(np.ascontiguousarray(g.G, np.float64)).to(dev)

    def step():
        if lib_run is not None:
            return lib_run(Xp, g.alpha, g.T, Gd, args.tf, args.tg)
        Q = T.haar_q_dev(g.G, device=dev)
        _, Zh = propagate_sharded(ops, coll, Xp, g.alpha, g.T, exchange=args.exchange)
        lab, _ = solve_sharded(sops, coll, Zh, Q, sh.u0, args.tf, args.tg)
        return lab

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    launches0 = L.tpo_launch_count()
    times = []
    stream = torch.cuda.current_stream()
    with ClockSampler(local) as cs:
        for _ in range(args.steps):
            flush.zero_()
            dist.barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    launches = L.tpo_launch_count() - launches0
    t = torch.tensor([float(sum(times))], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.barrier()
    tot_ms = float(t.item())
    units = 2.0 * g.nnz * g.d * g.T
    cfg = config_dict(g, args, ws)
    cfg["parallelism"] = (f"U-rows sharded over {ws} rank(s) ("
                          + ("NCCL RS/AG of the V block" if args.exchange == "full" else "NCCL all-to-all of touched V rows")
                          + " per hop, all-reduced solver partials; collectives "
                          + ("inside libtpo: tpo_run_sharded" if lib_run is not None else "through torch.distributed") + ")")
    # end to end: this rank's shard (X_p, CSR(B_p), CSR(B_p^T), G) copied in from pinned host memory
    # and its labels copied out inside the timed region, every step
    e2e = None
    if not args.no_e2e:
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
        hX = pin(Xp_host)
        hB = [pin(sh.Bp_rowptr), pin(sh.Bp_col), pin(sh.Btp_rowptr), pin(sh.Btp_col)]
        hG = pin(np.ascontiguousarray(g.G, np.float64))
        dB = [ops.Bp[0], ops.Bp[1], ops.Btp[0], ops.Btp[1]]
        Gd_e = torch.empty_like(hG, device=dev)
        hlab = torch.empty(max(sh.n_p, 1), dtype=torch.int32).pin_memory()
        h2d = sum(t.numel() * t.element_size() for t in [hX, hG] + hB)
        et = []
        for it in range(max(2, args.steps // 2) + 1):
            flush.zero_()
            dist.barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            Xp.copy_(hX, non_blocking=True)
            for dsrc, ddst in zip(hB, dB):
                ddst.copy_(dsrc, non_blocking=True)
            Gd_e.copy_(hG, non_blocking=True)
            if lib_run is not None:
                lab = lib_run(Xp, g.alpha, g.T, Gd_e, args.tf, args.tg)
            else:
                lab = step()
            hlab[: sh.n_p].copy_(lab[: sh.n_p], non_blocking=True)
            e1.record(stream)
            e1.synchronize()
            if it > 0:
                et.append(e0.elapsed_time(e1))
        t2 = torch.tensor([float(np.mean(et))], device=dev, dtype=torch.float64)
        dist.all_reduce(t2, op=dist.ReduceOp.MAX)
        e2e_ms = float(t2.item())
        e2e = {"value": units / (e2e_ms / 1e3), "unit": "nnz*d/s", "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(sh.n_p * 4)}
    line = {"metric": metric_name(), "value": units * args.steps / (tot_ms / 1e3), "unit": "nnz*d/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32+f64", "data": "synthetic", "config": cfg,
            "e2e": e2e, "gpu_launches": int(launches), "clocks": cs.summary(), "mode": "sharded",
            "tpo_seconds": tot_ms / args.steps / 1e3}
    if lib_run is not None:
        line["stages_ms"] = dict(zip(["propagate", "features", "topk_eig", "cluster"],
                                     [float(x) for x in lib_run.timings]))
    if rank == 0:
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="large")
    ap.add_argument("--tf", type=int, default=5)
    ap.add_argument("--tg", type=int, default=20)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--comm", default="lib", choices=["lib", "torch"],
                    help="sharded mode: collectives inside libtpo (tpo_run_sharded on its own NCCL communicator) or "
                         "issued from Python through torch.distributed")
    ap.add_argument("--exchange", default="full", choices=["full", "touched"],
                    help="sharded mode: per-hop exchange of the whole V block (reduce-scatter + all-gather) or of "
                         "the touched V rows only (all-to-all, SURVEY.md §8f #2)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--mode", default=None, choices=["replicas", "sharded"],
                    help="N > 1: one graph with its U rows sharded across the ranks (default: strong scaling, "
                         "NCCL reduce-scatter / all-gather per hop, all-reduced solver partials) or N independent "
                         "replicas (weak scaling, no data-path collective)")
    args = ap.parse_args()
    ws, rank, local = dist_env()
    if args.mode is None:
        args.mode = "sharded" if ws > 1 else "replicas"

    from synth import make_config
    if args.impl != "reference" and args.mode == "sharded" and ws > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dev = torch.device("cuda", local)
        dist.init_process_group("nccl", device_id=dev)
        run_sharded(args, None, ws, rank, local, dev, pre=shard_inputs(args, ws, rank))
        return
    if args.impl == "reference" and rank != 0:
        return      # rank 0 alone runs and prints the oracle arm; the other ranks exit 0 without work
    g = make_config(args.config)

    if args.impl == "reference":
        run_reference(args, g, ws, rank)
        return

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    import paper_2405_11922_b200 as T
    from paper_2405_11922_b200._lib import lib

    if args.mode == "sharded":
        run_sharded(args, g, ws, rank, local, dev)
        return

    L = lib()
    dg = T.to_device_graph(g.n, g.m, g.B_rowptr, g.B_col, g.Bt_rowptr, g.Bt_col, device=dev)
    X = torch.from_numpy(g.X).to(dev)
    Gd = torch.from_numpy(np.ascontiguousarray(g.G, np.float64)).to(dev)   # Alg. 1 L6 input, resident like X
    runner = T.Runner(dg, g.d, g.k, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    def step():
        return runner(X, g.alpha, g.T, Gd, args.tf, args.tg)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # --- timed region: device-resident inputs ------------------------------------------
    stage = np.zeros(4)
    times = []
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = L.tpo_launch_count()
    with ClockSampler(local) as cs:
        for _ in range(args.steps):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
            stage += runner.timings
    torch.cuda.synchronize()
    launches = L.tpo_launch_count() - launches0
    tot_ms = float(sum(times))
    if ws > 1:
        t = torch.tensor([tot_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
        tot_ms = float(t.item())
    units = 2.0 * g.nnz * g.d * g.T
    value = ws * units * args.steps / (tot_ms / 1e3)
    ms_step = tot_ms / args.steps
    stage_ms = stage / args.steps

    # --- end to end through the public API with host buffers ----------------------------
    e2e = None
    if not args.no_e2e:
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
        hX, hBr, hBc, hTr, hTc = pin(g.X), pin(g.B_rowptr), pin(g.B_col), pin(g.Bt_rowptr), pin(g.Bt_col)
        hG = pin(np.ascontiguousarray(g.G, np.float64))
        h2d = sum(t.numel() * t.element_size() for t in (hX, hBr, hBc, hTr, hTc, hG))
        d2h = g.n * 4
        hlab = torch.empty(g.n, dtype=torch.int32).pin_memory()
        # the public host-input entry point (tpo_run_host): copies inside the call, the Haar QR
        # of G beside the input copies, labels copied back
        hrun = T.HostRunner(g.n, g.m, g.nnz, g.d, g.k, device=dev)
        et = []
        for it in range(max(2, args.steps // 2) + 1):
            flush.zero_()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            hrun(hBr, hBc, hTr, hTc, hX, hG, g.alpha, g.T, args.tf, args.tg, labels=hlab, stream=stream)
            e1.record(stream)
            e1.synchronize()
            if it > 0:
                et.append(e0.elapsed_time(e1))
        e2e_ms = float(np.mean(et))
        if ws > 1:
            t = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        e2e = {"value": ws * units / (e2e_ms / 1e3), "unit": "nnz*d/s", "ms_per_step": e2e_ms,
               "stages_ms": dict(zip(["copies+propagate", "features", "topk_eig", "cluster"],
                                     [float(x) for x in hrun.timings])),
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)}

    # --- roofline of the propagation (the paper's dominant cost) --
    pk, src = peaks()
    bytes_hop = propagation_bytes(g.n, g.m, g.nnz, g.d)
    prop_ms = stage_ms[0]
    achieved = bytes_hop * g.T / (prop_ms / 1e3) / 1e9
    traffic = None
    tf = os.path.join(ROOT, "profiles", f"traffic_{args.config}.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get("bytes_per_hop") * g.T      # per launch of the T-hop loop
        except Exception:
            traffic = None
    # the gather view: every edge reads a d-wide fp32 row in both SpMMs (2 nnz d 4 bytes per hop),
    # against the measured gather ceilings of tools/probes/gather_bw.cu (context: a table that fits
    # L2 vs one that lives in DRAM; the large config's two tables are 1 GB and 512 MB)
    gather = None
    gc = os.path.join(ROOT, "profiles", "gather_ceilings.json")
    if os.path.exists(gc):
        try:
            ceil = json.load(open(gc))
            gbytes = 2.0 * g.nnz * g.d * 4
            gather = {"achieved": gbytes * g.T / (prop_ms / 1e3) / 1e9, "unit": "GB/s", "gathered_bytes_per_hop": gbytes,
                      "ceiling_l2_resident_gbs": ceil.get("l2_resident_gbs"), "ceiling_dram_resident_gbs": ceil.get("dram_gbs"),
                      "ceiling_source": "profiles/gather_ceilings.json (measured gather probe)"}
        except Exception:
            gather = None
    roof = {"kernel": "spmm_kernel pair (one hop: SpMM-1 V side + SpMM-2 U side, fix-ups, per-call schedule)",
            "bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
            "frac": achieved / pk["hbm_gbs"], "traffic": traffic, "peak_source": src,
            "algorithmic_bytes_per_hop": bytes_hop, "hops": g.T, "propagate_ms": prop_ms, "gather": gather}

    line = {"metric": metric_name(), "value": value, "unit": "nnz*d/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32+f64", "data": "synthetic",
            "config": config_dict(g, args, ws),
            "stages_ms": {"propagate": stage_ms[0], "features": stage_ms[1], "topk_eig": stage_ms[2],
                          "cluster": stage_ms[3]},
            "tpo_seconds": ms_step / 1e3,
            "propagation_nnz_d_per_s": 2.0 * g.nnz * g.d * g.T / (prop_ms / 1e3),
            "propagation_gb_per_s": bytes_hop * g.T / (prop_ms / 1e3) / 1e9,
            "roofline": roof, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": cs.summary()}
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_sample(g, args)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
