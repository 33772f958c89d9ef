"""Row-sharded a5-a9 (the solver's fp64 partials all-reduced across ranks).

CPU: the orchestration `solve_sharded` with a plain fp64 numpy stand-in of the per-shard
compute, world size 2 and 3 over gloo, gives the single-rank labels, which match the fp64
oracle's discretisation.  GPU: libtpo's tpo_shard_* solver entry points for every shard of a
partition, the ranks emulated by threads with in-process collectives (host barriers only; no
kernel waits on another), give the labels of the single-GPU path and of the oracle."""
import os
import socket
import threading

import numpy as np
import pytest
import torch

from oracle import core as O
from oracle import dense as DN
from paper_2405_11922_b200.sharded import _sign_rule, row_bounds, solve_sharded
from synth import planted_abg

EPS = 1e-12


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class NumpySolverOps:
    """fp64 stand-in of GpuSolverOps (test double), written from the paper's definitions."""

    def __init__(self, n_p, d, k):
        self.n_p, self.d, self.k, self.D = n_p, d, k, 2 * d

    def features(self, Zhat_p, Q):
        Zh, Qd = Zhat_p.double().numpy(), Q.double().numpy()
        Zo = np.sqrt(self.d) * Zh @ Qd.T                                    # Eq. R-prime
        Rp = np.sqrt(np.e / self.d) * np.concatenate([np.sin(Zo), np.cos(Zo)], axis=1)
        return torch.from_numpy(Rp), torch.from_numpy(Rp.sum(0))

    def dinv(self, Rp, r):
        return torch.from_numpy(1.0 / np.sqrt(np.maximum(Rp.numpy() @ r.numpy(), 1e-12)))   # Eq. Ri, R6

    def gram(self, Rp, dinv):
        R = dinv.numpy()[:, None] * Rp.numpy()
        return torch.from_numpy(R.T @ R)

    def eig(self, G, r):
        w, V = np.linalg.eigh(G.numpy())
        order = np.argsort(-w)[: self.k]
        return torch.from_numpy(V[:, order].copy()), np.sqrt(np.maximum(w[order], 0.0))

    def gamma(self, Rp, dinv, Psi64, sigma):
        R = dinv.numpy()[:, None] * Rp.numpy()
        return torch.from_numpy(R @ (Psi64.numpy() / sigma[None, :]))

    def atb(self, A, B):
        return torch.from_numpy(A.numpy().T @ B.numpy())

    def apply_chol(self, X, g):
        gn = g.numpy()
        s = 1.0 / np.sqrt(np.diag(gn))
        C = np.linalg.cholesky(s[:, None] * gn * s[None, :]).T             # upper: S g S = C^T C
        X.copy_(torch.from_numpy(X.numpy() @ (s[:, None] * np.linalg.inv(C))))

    def colstats(self, G64, row0):
        A = G64.numpy()
        if A.shape[0] == 0:
            z = np.zeros(self.k)
            return torch.from_numpy(z), torch.from_numpy(z), torch.from_numpy(z - 1), torch.zeros(self.k, dtype=torch.int64)
        am = np.argmax(np.abs(A), axis=0)                                   # first index among ties
        return (torch.from_numpy(A.sum(0)), torch.from_numpy(np.abs(A).sum(0)),
                torch.from_numpy(A[am, np.arange(self.k)]), torch.from_numpy((am + row0).astype(np.int64)))

    def gamma_final(self, G64, signs, Psi64):
        sg = signs.astype(np.float64)
        return (torch.from_numpy((Psi64.numpy() * sg).astype(np.float32)),
                torch.from_numpy((G64.numpy() * sg).astype(np.float32)))

    def onmf_init(self, Gamma_p, Psi, sigma):
        U = np.maximum(Gamma_p.double().numpy(), 0.0) + EPS                 # R9
        H = np.maximum(Psi.double().numpy() * sigma[None, :], 0.0) + EPS
        return torch.from_numpy(U), torch.from_numpy(H)

    def rtu(self, Rp, dinv, U):
        return torch.from_numpy(Rp.numpy().T @ (dinv.numpy()[:, None] * U.numpy()))

    def h_update(self, H, RtU, UtU):                                        # Eq. update-Q
        Hn = H.numpy() * np.maximum(RtU.numpy(), 0.0) / (H.numpy() @ UtU.numpy() + EPS)
        H.copy_(torch.from_numpy(Hn))

    def rh(self, Rp, dinv, H):
        return torch.from_numpy(dinv.numpy()[:, None] * (Rp.numpy() @ H.numpy()))

    def u_update(self, U, RH, M):                                          # Eq. update-Y, R9
        Un = U.numpy() * np.sqrt(np.maximum(RH.numpy(), 0.0) / (np.maximum(U.numpy() @ M.numpy(), 0.0) + EPS))
        U.copy_(torch.from_numpy(Un))

    def nci_assign(self, U, Phi, labels):                                  # Eq. ell-ast
        lab = np.argmax(U.numpy() @ Phi.numpy(), axis=1).astype(np.int32) if self.n_p else np.zeros(0, np.int32)
        changed = int(np.any(lab != labels.numpy()))
        labels.copy_(torch.from_numpy(lab))
        sums = np.zeros((self.k, self.k))
        np.add.at(sums, lab, U.numpy())
        counts = np.bincount(lab, minlength=self.k).astype(np.float64)
        return torch.tensor([changed], dtype=torch.int32), torch.from_numpy(sums), torch.from_numpy(counts)

    def phi(self, sums, counts):
        c = counts.numpy()
        Phi = np.where(c[None, :] > 0, sums.numpy().T / np.sqrt(np.where(c > 0, c, 1.0))[None, :], 0.0)
        return torch.from_numpy(Phi)

    def eye(self):
        return torch.eye(self.k, dtype=torch.float64)

    def labels(self):
        return torch.full((self.n_p,), -1, dtype=torch.int32)


def _inputs():
    g = planted_abg(900, 600, 4, 12, deg=("poisson", 8.0), p_in=0.85, x=("gaussian", 1.0), alpha=0.5, T=2, seed=11)
    _, Zh = O.propagate(g.n, g.m, g.B_rowptr, g.B_col, g.X, g.alpha, g.T)
    Q = O.haar_q(np.random.default_rng(3).standard_normal((g.d, g.d)))
    return g, Zh.astype(np.float32), Q.astype(np.float32)


def _solver_worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2405_11922_b200.sharded import TorchCollectives
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g, Zh, Q = _inputs()
        u0, u1 = row_bounds(g.n, rank, world)
        ops = NumpySolverOps(u1 - u0, g.d, g.k)
        lab, it = solve_sharded(ops, TorchCollectives(), torch.from_numpy(Zh[u0:u1]), torch.from_numpy(Q), u0, 5, 20)
        q.put((rank, lab.numpy(), it))
    finally:
        dist.destroy_process_group()


def _run_gloo(world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_solver_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, lab, it = q.get(timeout=300)
        res[r] = (lab, it)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return np.concatenate([res[r][0] for r in range(world)]), {res[r][1] for r in range(world)}


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_solver_gloo(world):
    """world ranks over gloo == one rank (the exchange algebra), == the oracle's labels."""
    lab_w, its = _run_gloo(world)
    assert len(its) == 1                                 # every rank stops at the same iteration
    g, Zh, Q = _inputs()

    class One:
        world, rank = 1, 0

        def allreduce_sum(self, t):
            pass

        def all_gather_rows(self, t):
            return t[None]

    lab_1, it_1 = solve_sharded(NumpySolverOps(g.n, g.d, g.k), One(), torch.from_numpy(Zh), torch.from_numpy(Q), 0)
    assert its == {it_1}
    assert np.array_equal(lab_w, lab_1.numpy())
    Rp, dinv, _ = O.features(Zh, Q)
    Rp32, dinv32 = Rp.astype(np.float32), dinv.astype(np.float32)
    Gm, s, Ps, _ = O.topk(Rp32, dinv32, g.k)
    lab_o, _, _ = O.cluster(Rp32, dinv32, Gm.astype(np.float32), s, Ps.astype(np.float32), 5, 20)
    assert DN.ari(lab_w, lab_o) >= 0.999


def test_sign_rule_tie_break():
    """R8 across ranks: near-zero column sum -> sign of the largest |entry|, smallest index on ties."""
    s = np.array([1e-20, -3.0, 1e-20])
    a = np.array([1.0, 3.0, 1.0])
    vals = np.array([[-0.5, 1.0, 0.4], [0.5, 1.0, -0.4]])
    idxs = np.array([[7, 0, 9], [3, 5, 2]])
    assert list(_sign_rule(s, a, vals, idxs)) == [1, -1, -1]


class ThreadCollectives:
    """In-process collectives for ranks emulated by threads (host barriers; sums in rank order)."""

    def __init__(self, world):
        self.world = world
        self.slots = [None] * world
        self.bar = threading.Barrier(world)

    def view(self, rank):
        outer = self

        class V:
            world = outer.world

            def __init__(self):
                self.rank = rank

            def allreduce_sum(self, t):
                torch.cuda.synchronize()
                outer.slots[rank] = t.clone()
                outer.bar.wait()
                tot = outer.slots[0].clone()
                for r in range(1, outer.world):
                    tot += outer.slots[r]
                outer.bar.wait()
                t.copy_(tot)

            def all_gather_rows(self, t):
                torch.cuda.synchronize()
                outer.slots[rank] = t.clone()
                outer.bar.wait()
                out = torch.stack([outer.slots[r] for r in range(outer.world)])
                outer.bar.wait()
                return out
        return V()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 2, 3])
def test_sharded_solver_gpu_emulated(world):
    """libtpo's tpo_shard_* solver pieces, ranks emulated by threads on one GPU: the labels
    equal the single-GPU path's (tpo_features -> tpo_topk_eig -> tpo_cluster) and the oracle's."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2405_11922_b200 import build
    build.build()
    import paper_2405_11922_b200 as T
    from paper_2405_11922_b200.sharded import GpuSolverOps
    g, Zh, Q = _inputs()
    coll = ThreadCollectives(world)
    res, errs = {}, []

    def run(r):
        try:
            u0, u1 = row_bounds(g.n, r, world)
            ops = GpuSolverOps(u1 - u0, g.d, g.k, "cuda")
            lab, it = solve_sharded(ops, coll.view(r), torch.from_numpy(Zh[u0:u1]).cuda(), torch.from_numpy(Q).cuda(),
                                    u0, 5, 20)
            res[r] = (lab.cpu().numpy(), it)
        except Exception as e:              # pragma: no cover - surfaced below
            errs.append(e)
            coll.bar.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    lab = np.concatenate([res[r][0] for r in range(world)])
    Rp, dv, _ = T.features(torch.from_numpy(Zh).cuda(), torch.from_numpy(Q).cuda(), want_r=True)
    Gm, s, Ps = T.topk_eig(Rp, dv, g.k)
    lab_1, _ = T.cluster(Rp, dv, Gm, s, Ps, 5, 20)
    assert DN.ari(lab, lab_1.cpu().numpy()) >= 0.999
    Rpo, dinvo, _ = O.features(Zh, Q)
    Rp32, dinv32 = Rpo.astype(np.float32), dinvo.astype(np.float32)
    Gmo, so, Pso, _ = O.topk(Rp32, dinv32, g.k)
    lab_o, _, _ = O.cluster(Rp32, dinv32, Gmo.astype(np.float32), so, Pso.astype(np.float32), 5, 20)
    assert DN.ari(lab, lab_o) >= 0.999


@pytest.mark.gpu
@pytest.mark.parametrize("k", [40, 50, 100])
def test_shard_nci_assign_tensor_path_gpu(k):
    """Alg. 3 through the sharded solver's per-rank step tpo_shard_nci_assign at
    32 < k <= 104, where the assignment runs the certified fp64-tensor-path argmax (R13): labels equal
    the oracle's bit for bit on a ragged row count (equal rows and exact ties included)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2405_11922_b200 import build
    build.build()
    from paper_2405_11922_b200.sharded import GpuSolverOps
    n, Tg = 20011, 20
    rng = np.random.default_rng(100 + k)
    Ups = np.abs(rng.standard_normal((n, k))) * 0.3
    Ups[np.arange(n), rng.integers(0, k, n)] += 1.0          # a dominant cluster per row, noisy
    Ups[:64] = Ups[0]                                         # equal rows
    Ups[64:96] = 0.25                                         # exact ties -> smallest l
    ref, it_ref = O.nci(Ups, Tg)
    ops = GpuSolverOps(n, 8, k, "cuda")
    U = torch.from_numpy(Ups).cuda()
    Phi, labels, iters = ops.eye(), ops.labels(), 0
    for t in range(Tg):
        changed, sums, counts = ops.nci_assign(U, Phi, labels)
        iters += 1
        if int(changed.item()) == 0 or t == Tg - 1:
            break
        Phi = ops.phi(sums, counts)
    assert np.array_equal(labels.cpu().numpy(), ref)
    assert abs(iters - it_ref) <= 1      # the oracle counts the iterations it used; the fix-point check is one more pass here
