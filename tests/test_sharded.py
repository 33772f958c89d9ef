"""Multi-rank propagation: partitioning and the exchange algebra on CPU with
gloo (world size 2 and 3), with the local compute done by a plain fp64 numpy stand-in; and the
libtpo shard entry points on one GPU with the collectives emulated in-process."""
import os
import socket

import numpy as np
import pytest
import torch

from oracle import core as O
from paper_2405_11922_b200.sharded import HostShard, propagate_sharded, row_bounds, shard_graph
from synth import planted_abg


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class NumpyShardOps:
    """fp64 stand-in of GpuShardOps (test double): the same per-shard products, in numpy."""

    def __init__(self, shard: HostShard, d):
        self.s, self.d = shard, d

    def new(self, rows, cols=None, dtype=torch.float64, zero=False):
        shape = (rows,) if cols is None else (rows, cols)
        return torch.zeros(shape, dtype=torch.float64)

    def _deg(self, rp, val):
        if val is None:
            return np.diff(rp).astype(np.float64)
        return np.add.reduceat(np.concatenate([val.astype(np.float64), [0.0]]), rp[:-1]) * (np.diff(rp) > 0)

    def degrees(self):
        s = self.s
        return torch.from_numpy(self._deg(s.Bp_rowptr, s.Bp_val)), torch.from_numpy(self._deg(s.Btp_rowptr, s.Btp_val))

    def start(self, du, dv, Xp, alpha):
        c = (1 - alpha) if alpha < 1 else 1.0
        su = torch.where(du > 0, 1 / torch.sqrt(torch.where(du > 0, du, torch.ones_like(du))), torch.zeros_like(du))
        sv = torch.where(dv > 0, 1 / torch.sqrt(torch.where(dv > 0, dv, torch.ones_like(dv))), torch.zeros_like(dv))
        return su, sv, (su[:, None] * c * Xp).clone()

    def _spmm(self, rp, col, val, src):
        out = np.zeros((len(rp) - 1, src.shape[1]))
        w = np.ones(len(col)) if val is None else val.astype(np.float64)
        rows = np.repeat(np.arange(len(rp) - 1), np.diff(rp))
        np.add.at(out, rows, w[:, None] * src.numpy()[col])
        return torch.from_numpy(out)

    def vside(self, P, Qpart):
        s = self.s
        Qpart.copy_(self._spmm(s.Btp_rowptr, s.Btp_col, s.Btp_val, P))

    def vscale(self, Q, s_v):
        Q.mul_((s_v * s_v)[:, None])

    def index(self, ids):
        return torch.from_numpy(np.asarray(ids, np.int64))

    def pack(self, src, idx, dst):
        dst.copy_(src[idx])

    def unpack(self, dst, idx, src, accumulate):
        if accumulate:
            dst[idx] += src
        else:
            dst[idx] = src

    def uside(self, Q, Xp, alpha, s_u, last, Zp, Zhat):
        s = self.s
        c = (1 - alpha) if alpha < 1 else 1.0
        acc = self._spmm(s.Bp_rowptr, s.Bp_col, s.Bp_val, Q[: s.m])
        z = c * Xp + alpha * s_u[:, None] * acc
        if last:
            Zp.copy_(z)
            if Zhat is not None:
                nr = torch.linalg.vector_norm(z, dim=1, keepdim=True)
                Zhat.copy_(torch.where(nr > 0, z / torch.where(nr > 0, nr, torch.ones_like(nr)), torch.zeros_like(z)))
        else:
            Zp.copy_(s_u[:, None] * z)

    def propagate_local(self, Xp, alpha, T):
        c = (1 - alpha) if alpha < 1 else 1.0
        Z = c * Xp
        nr = torch.linalg.vector_norm(Z, dim=1, keepdim=True)
        return Z, torch.where(nr > 0, Z / torch.where(nr > 0, nr, torch.ones_like(nr)), torch.zeros_like(Z))


def _worker(rank, world, port, T, weighted, q, exchange="full"):
    import torch.distributed as dist
    from paper_2405_11922_b200.sharded import TorchCollectives
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = planted_abg(301, 122, 2, 8, deg=("poisson", 5.0), p_in=0.7, x=("uniform",), seed=7, weighted=weighted)
        sh = shard_graph(g.n, g.m, g.B_rowptr, g.B_col, rank, world, g.B_val)
        ops = NumpyShardOps(sh, g.d)
        Xp = torch.from_numpy(g.X[sh.u0:sh.u1].astype(np.float64))
        Z, Zh = propagate_sharded(ops, TorchCollectives(), Xp, 0.6, T, exchange=exchange)
        q.put((rank, Z.numpy(), Zh.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,T,weighted,exchange", [(2, 3, False, "full"), (3, 2, True, "full"), (2, 0, False, "full"),
                                                        (2, 3, False, "touched"), (3, 2, True, "touched"),
                                                        (4, 3, False, "touched")])
def test_sharded_propagation_gloo(world, T, weighted, exchange):
    """Concatenated shard results == the oracle's single-process propagation (fp64), with the
    full reduce-scatter / all-gather exchange and with the touched-row all-to-all (§8f #2)."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, T, weighted, q, exchange)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict()
    for _ in range(world):
        r, Z, Zh = q.get(timeout=120)
        res[r] = (Z, Zh)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = planted_abg(301, 122, 2, 8, deg=("poisson", 5.0), p_in=0.7, x=("uniform",), seed=7, weighted=weighted)
    Zo, Zho = O.propagate(g.n, g.m, g.B_rowptr, g.B_col, g.X, 0.6, T, g.B_val)
    Z = np.concatenate([res[r][0] for r in range(world)])
    Zh = np.concatenate([res[r][1] for r in range(world)])
    assert np.allclose(Z, Zo, rtol=1e-12, atol=1e-14)
    assert np.allclose(Zh, Zho, rtol=1e-12, atol=1e-14)


def test_shard_graph_partition():
    g = planted_abg(101, 60, 3, 4, deg=("poisson", 4.0), p_in=0.7, x=("uniform",), seed=2, weighted=True)
    rows, cols, vals = [], [], []
    for r in range(4):
        sh = shard_graph(g.n, g.m, g.B_rowptr, g.B_col, r, 4, g.B_val)
        assert (sh.u0, sh.u1) == row_bounds(g.n, r, 4)
        u = np.repeat(np.arange(sh.n_p), np.diff(sh.Bp_rowptr)) + sh.u0
        rows.append(u)
        cols.append(sh.Bp_col)
        vals.append(sh.Bp_val)
        # B_p^T: same edge set
        vt = np.repeat(np.arange(g.m), np.diff(sh.Btp_rowptr))
        a = sorted(zip(u.tolist(), sh.Bp_col.tolist(), sh.Bp_val.tolist()))
        b = sorted(zip((sh.Btp_col + sh.u0).tolist(), vt.tolist(), sh.Btp_val.tolist()))
        assert a == b
    assert np.array_equal(np.concatenate(cols), g.B_col)
    assert np.array_equal(np.concatenate(vals), g.B_val)


@pytest.mark.gpu
@pytest.mark.parametrize("world,d,weighted", [(3, 8, False), (2, 132, True), (4, 128, False)])
def test_shard_ops_gpu_emulated(world, d, weighted):
    """libtpo tpo_shard_* on one GPU for every shard of a partition, with reduce-scatter and
    all-gather emulated in-process, equals the oracle's propagation (rel. Frobenius 1e-5)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2405_11922_b200 import build
    build.build()
    from paper_2405_11922_b200.sharded import GpuShardOps
    g = planted_abg(3001, 1005, 5, d, deg=("zipf", 1.3, 300), p_in=0.6, pop=("zipf", 1.2), x=("gaussian", 1.0),
                    seed=d, weighted=weighted)
    T, alpha = 3, 0.5
    shards = [shard_graph(g.n, g.m, g.B_rowptr, g.B_col, r, world, g.B_val) for r in range(world)]
    ops = [GpuShardOps(s, "cuda", d) for s in shards]
    Xp = [torch.from_numpy(g.X[s.u0:s.u1]).cuda() for s in shards]
    deg = [o.degrees() for o in ops]
    dv = sum(dvp for _, dvp in deg)
    st = [o.start(du, dv, x, alpha) for o, (du, _), x in zip(ops, deg, Xp)]
    m = g.m
    mp = -(-m // world)
    sv_pad = torch.zeros(mp * world, device="cuda")
    sv_pad[:m] = st[0][1]
    P = [s[2] for s in st]
    Zh = [torch.empty_like(x) for x in Xp]
    for t in range(T):
        parts = []
        for o, p in zip(ops, P):
            q = torch.zeros(mp * world, d, device="cuda")
            o.vside(p, q[:m])
            parts.append(q)
        tot = sum(parts)
        slices = [tot[r * mp:(r + 1) * mp].contiguous() for r in range(world)]
        for r in range(world):
            ops[r].vscale(slices[r], sv_pad[r * mp:(r + 1) * mp].contiguous())
        Q = torch.cat(slices)
        for r in range(world):
            ops[r].uside(Q, Xp[r], alpha, st[r][0], t == T - 1, P[r], Zh[r] if t == T - 1 else None)
    Zo, Zho = O.propagate(g.n, g.m, g.B_rowptr, g.B_col, g.X, alpha, T, g.B_val)
    Z = torch.cat(P).cpu().numpy().astype(np.float64)
    Zhat = torch.cat(Zh).cpu().numpy().astype(np.float64)
    assert np.linalg.norm(Z - Zo) <= 1e-5 * np.linalg.norm(Zo)
    assert np.linalg.norm(Zhat - Zho) <= 1e-5 * np.linalg.norm(Zho)


def test_touched_rows_are_a_fraction_of_v():
    """The touched-row exchange moves only the V rows a U slice touches: on a shuffled planted graph
    at 4 ranks each rank touches well under all of V (SURVEY A.11 measured 34.5 % at 8 ranks on
    large), and every touched row has an owner."""
    g = planted_abg(4000, 3000, 5, 4, deg=("zipf", 1.3, 200), p_in=0.5, pop=("zipf", 1.3), x=("uniform",), seed=3)
    for r in range(4):
        sh = shard_graph(g.n, g.m, g.B_rowptr, g.B_col, r, 4, g.B_val)
        touched = np.flatnonzero(np.diff(sh.Btp_rowptr) > 0)
        assert 0 < touched.size < 0.8 * g.m
        assert np.array_equal(np.unique(sh.Bp_col), touched)


@pytest.mark.gpu
def test_row_movers_gpu():
    """tpo_rows_gather / tpo_rows_scatter (accumulate and overwrite) vs torch indexing."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2405_11922_b200 import build
    build.build()
    from paper_2405_11922_b200.sharded import GpuShardOps
    g = planted_abg(300, 200, 2, 8, seed=1)
    sh = shard_graph(g.n, g.m, g.B_rowptr, g.B_col, 0, 1)
    ops = GpuShardOps(sh, "cuda", 12)
    src = torch.randn(200, 12, device="cuda")
    idx = ops.index(np.random.default_rng(0).permutation(200)[:77])
    out = torch.empty(77, 12, device="cuda")
    ops.pack(src, idx, out)
    assert torch.equal(out, src[idx.long()])
    dst = torch.randn(200, 12, device="cuda")
    ref = dst.clone()
    ops.unpack(dst, idx, out, True)
    ref[idx.long()] += out
    assert torch.equal(dst, ref)
    ops.unpack(dst, idx, out, False)
    ref[idx.long()] = out
    assert torch.equal(dst, ref)


@pytest.mark.gpu
@pytest.mark.parametrize("T,weighted", [(3, False), (2, True), (0, False)])
def test_propagate_sharded_library_nccl(T, weighted):
    """tpo_propagate_sharded with a libtpo-owned NCCL communicator (world 1 on one GPU: the
    all-reduce / reduce-scatter / all-gather run through NCCL) equals the oracle's propagation."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2405_11922_b200 import build
    build.build()
    from paper_2405_11922_b200.sharded import GpuShardOps, NcclComm, propagate_sharded_lib
    g = planted_abg(3001, 1005, 5, 64, deg=("zipf", 1.3, 300), p_in=0.6, pop=("zipf", 1.2), x=("gaussian", 1.0),
                    seed=T + 11, weighted=weighted)
    sh = shard_graph(g.n, g.m, g.B_rowptr, g.B_col, 0, 1, g.B_val)
    ops = GpuShardOps(sh, "cuda:0", 64)
    comm = NcclComm(0, 1, "cuda:0", NcclComm.unique_id())
    try:
        Z, Zh = propagate_sharded_lib(comm, ops, torch.from_numpy(g.X).cuda(), 0.5, T)
        torch.cuda.synchronize()
    finally:
        comm.close()
    Zo, Zho = O.propagate(g.n, g.m, g.B_rowptr, g.B_col, g.X, 0.5, T, g.B_val)
    assert np.linalg.norm(Z.cpu().numpy() - Zo) <= 1e-5 * np.linalg.norm(Zo)
    assert np.linalg.norm(Zh.cpu().numpy() - Zho) <= 1e-5 * np.linalg.norm(Zho)


@pytest.mark.gpu
def test_run_sharded_library_nccl():
    """tpo_run_sharded (the whole hot path with every collective inside libtpo) at world 1 through
    NCCL: labels equal the oracle's end-to-end labels on the tiny config, and tpo_run's."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2405_11922_b200 import build
    build.build()
    import paper_2405_11922_b200 as T
    from oracle import dense as DN
    from paper_2405_11922_b200.sharded import GpuShardOps, LibRunner, NcclComm
    from synth import make_config
    g = make_config("tiny")
    sh = shard_graph(g.n, g.m, g.B_rowptr, g.B_col, 0, 1, g.B_val)
    ops = GpuShardOps(sh, "cuda:0", g.d)
    comm = NcclComm(0, 1, "cuda:0", NcclComm.unique_id())
    try:
        run = LibRunner(comm, ops, g.d, g.k)
        Gd = torch.from_numpy(np.ascontiguousarray(g.G, np.float64)).cuda()
        lab = run(torch.from_numpy(g.X).cuda(), g.alpha, g.T, Gd, 5, 20).cpu().numpy()
        torch.cuda.synchronize()
    finally:
        comm.close()
    ref = O.run(g)
    assert np.array_equal(lab, ref["labels"]) or DN.ari(lab, ref["labels"]) >= 0.999
    dg = T.to_device_graph(g.n, g.m, g.B_rowptr, g.B_col, g.Bt_rowptr, g.Bt_col)
    lab1, _ = T.run(dg, torch.from_numpy(g.X).cuda(), g.alpha, g.T, g.k, g.G)
    assert DN.ari(lab, lab1.cpu().numpy()) >= 0.999


def _shard_inputs_worker(rank, world, port, q):
    import types
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        meta, sh, Xp = bench.shard_inputs(types.SimpleNamespace(config="tiny"), world, rank)
        q.put((rank, meta.n, meta.nnz, sh.u0, sh.u1, sh.Bp_col.copy(), Xp.copy()))
    finally:
        dist.destroy_process_group()


def test_bench_shard_inputs_gloo():
    """bench.py's multi-rank input path: rank 0 generates the graph once and every rank loads only
    its own U slice; the slices reassemble the generator's graph and X exactly."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_shard_inputs_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict()
    for _ in range(2):
        r, n, nnz, u0, u1, col, Xp = q.get(timeout=180)
        res[r] = (u0, u1, col, Xp)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from synth import make_config
    g = make_config("tiny")
    assert np.array_equal(np.concatenate([res[r][2] for r in range(2)]), g.B_col)
    assert np.array_equal(np.concatenate([res[r][3] for r in range(2)]), g.X)
    assert res[0][1] == res[1][0] and res[1][1] == g.n
