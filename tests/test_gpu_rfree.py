"""f3 "R-free" a7-a9: the exact top-k and the discretisation with R' rows
recomputed from Zhat and Q in row chunks (tpo_topk_eig_rfree, tpo_cluster_rfree) -- against the
oracle's materialised-R' path and against the GPU's own materialised path on the same inputs."""
import os
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import core as O  # noqa: E402
from oracle import dense as DN  # noqa: E402
from synth import make_config, planted_abg  # noqa: E402

pytestmark = pytest.mark.gpu


def relF(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


@pytest.fixture(scope="module")
def tpo():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2405_11922_b200 import build
    build.build()
    import paper_2405_11922_b200 as T
    return T


def oracle_chain(g):
    """Oracle Zhat, Q and the materialised R', dinv, exact top-k on them (fp64, Algs. 1-2 inputs)."""
    _, Zh = O.propagate(g.n, g.m, g.B_rowptr, g.B_col, g.X, g.alpha, g.T, g.B_val)
    Zh32 = Zh.astype(np.float32)
    Q32 = O.haar_q(g.G).astype(np.float32)
    Rp, dinv, _ = O.features(Zh32, Q32)
    Rp32, dv32 = Rp.astype(np.float32), dinv.astype(np.float32)
    return Zh32, Q32, Rp32, dv32, O.topk(Rp32, dv32, g.k)


@pytest.fixture(scope="module")
def tiny():
    g = make_config("tiny")
    return g, oracle_chain(g)


@pytest.fixture(scope="module")
def k40():
    g = planted_abg(6000, 4000, 40, 48, deg=("poisson", 10.0), p_in=0.8, x=("gaussian", 1.0), alpha=0.5, T=2, seed=41)
    return g, oracle_chain(g)


def check_topk(g, Gm, s, Ps, dv, ref):
    Zh32, Q32, Rp32, dv32, (Gmo, so, Pso, _) = ref
    Gm, Ps, dv = Gm.cpu().numpy(), Ps.cpu().numpy(), dv.cpu().numpy()
    assert relF(dv, dv32) <= 1e-5                                                   # Eq. dinv
    assert DN.sin_theta(Gm, Gmo) <= 1e-4
    assert DN.sin_theta(Ps, Pso) <= 1e-4
    assert np.allclose(s, so, rtol=1e-5)
    assert abs(s[0] - 1.0) < 1e-5                                                   # F5 / E5
    assert np.max(np.abs(Gm.astype(np.float64).T @ Gm - np.eye(g.k))) <= 1e-6      # E2
    assert np.all(Gm.astype(np.float64).sum(0) >= 0)                                # R8


@pytest.mark.parametrize("chunk", [0, 700, 64])
def test_topk_rfree_vs_oracle_tiny(tpo, tiny, chunk):
    """Three sweeps over ragged chunks (2000 rows: 700 -> 3 chunks with a 600-row tail; 64 -> 32)."""
    g, ref = tiny
    Gm, s, Ps, dv = tpo.topk_eig_rfree(torch.from_numpy(ref[0]).cuda(), torch.from_numpy(ref[1]).cuda(), g.k,
                                       chunk_rows=chunk)
    check_topk(g, Gm, s, Ps, dv, ref)


def test_topk_rfree_vs_oracle_k40(tpo, k40):
    g, ref = k40
    Gm, s, Ps, dv = tpo.topk_eig_rfree(torch.from_numpy(ref[0]).cuda(), torch.from_numpy(ref[1]).cuda(), g.k,
                                       chunk_rows=2500)
    check_topk(g, Gm, s, Ps, dv, ref)


def test_topk_rfree_matches_materialised_gpu(tpo, k40):
    """Same subspace as tpo_features -> tpo_topk_eig on the GPU's own R' (the recomputed rows equal the
    materialised ones; dinv differs at most by the fp32 rounding of r's chunk-order sum)."""
    g, ref = k40
    Zh, Q = torch.from_numpy(ref[0]).cuda(), torch.from_numpy(ref[1]).cuda()
    Rg, dg, _ = tpo.features(Zh, Q)
    Gm_m, s_m, Ps_m = tpo.topk_eig(Rg, dg, g.k)
    Gm, s, Ps, dv = tpo.topk_eig_rfree(Zh, Q, g.k, chunk_rows=1000)
    assert float(((dv - dg).abs() / dg.abs()).max()) <= 1e-6
    assert DN.sin_theta(Gm.cpu().numpy(), Gm_m.cpu().numpy()) <= 1e-5
    assert np.allclose(s, s_m, rtol=1e-6)       # the Gram's fp32 tile sums flush at other row boundaries


@pytest.mark.parametrize("chunk", [0, 700])
def test_cluster_rfree_tiny(tpo, tiny, chunk):
    """k = 5 (DMMA products on both paths): labels and Alg. 3 iterations identical to tpo_cluster on the
    GPU's materialised R' (same Gamma, sigma, Psi, dinv); ARI >= 0.999 against the oracle's labels
    on its own staged inputs (north_star's end-to-end bar)."""
    g, ref = tiny
    Zh32, Q32, Rp32, dv32, (Gmo, so, Pso, _) = ref
    Zh, Q = torch.from_numpy(Zh32).cuda(), torch.from_numpy(Q32).cuda()
    Rg, dg, _ = tpo.features(Zh, Q)
    Gm, s, Ps = tpo.topk_eig(Rg, dg, g.k)
    lab_m, it_m = tpo.cluster(Rg, dg, Gm, s, Ps, 5, 20)
    lab, it = tpo.cluster_rfree(Zh, Q, dg, Gm, s, Ps, 5, 20, chunk_rows=chunk)
    assert it == it_m and torch.equal(lab, lab_m)
    lab_o, _, _ = O.cluster(Rp32, dv32, Gmo.astype(np.float32), so, Pso.astype(np.float32), 5, 20)
    assert DN.ari(lab.cpu().numpy(), lab_o) >= 0.999


def test_cluster_rfree_k40(tpo, k40):
    """k = 40: the R-free passes run on the fp64 tensor path while the materialised path uses the
    integer-tensor-core products (R16, ~1e-14 relative): the same labels, and ARI >= 0.999 vs the
    oracle's labels on its own staged inputs."""
    g, ref = k40
    Zh32, Q32, Rp32, dv32, (Gmo, so, Pso, _) = ref
    Zh, Q = torch.from_numpy(Zh32).cuda(), torch.from_numpy(Q32).cuda()
    Rg, dg, _ = tpo.features(Zh, Q)
    Gm, s, Ps = tpo.topk_eig(Rg, dg, g.k)
    lab_m, it_m = tpo.cluster(Rg, dg, Gm, s, Ps, 3, 20)
    lab, it = tpo.cluster_rfree(Zh, Q, dg, Gm, s, Ps, 3, 20, chunk_rows=2500)
    lab, lab_m = lab.cpu().numpy(), lab_m.cpu().numpy()
    assert np.mean(lab != lab_m) <= 1e-3
    lab_o, _, _ = O.cluster(Rp32, dv32, Gmo.astype(np.float32), so, Pso.astype(np.float32), 3, 20)
    assert DN.ari(lab, lab_o) >= 0.999
