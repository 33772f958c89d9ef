"""GPU parity: the CUDA path (through the C-ABI) vs the fp64 oracle on the same seeded inputs.

Tolerances (north_star): propagated Z within 1e-5 relative Frobenius;
features / affinity products within 1e-5 relative Frobenius (fp32 storage); top-k subspace
sin(max principal angle) <= 1e-4 against the oracle's exact top-k; cluster labels bit-exact
given identical eigen inputs; end-to-end ARI(GPU, oracle) >= 0.999.
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import core as O  # noqa: E402
from oracle import dense as DN  # noqa: E402
from synth import csr_from_edges, make_config, planted_abg, random_unit_rows  # noqa: E402


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


def dev_graph(T, g):
    return T.to_device_graph(g.n, g.m, g.B_rowptr, g.B_col, g.Bt_rowptr, g.Bt_col, g.B_val, g.Bt_val)


def hub_graph(seed=0, weighted=False, n=1500, m=900, d=8):
    """Random edges plus a V hub of degree 1400 and a U hub of degree 700 (> the 512-edge chunk),
    isolated U rows 3 and 4, isolated V 7."""
    rng = np.random.default_rng(seed)
    u = rng.integers(0, n, 9000)
    v = rng.integers(0, m, 9000)
    u = np.concatenate([u, np.arange(1400) + 5, np.full(700, 11)])
    v = np.concatenate([v, np.full(1400, 13), rng.permutation(m)[:700]])
    keep = (u != 3) & (u != 4) & (v != 7)
    key = np.unique(u[keep].astype(np.int64) * m + v[keep])
    u, v = key // m, key % m
    w = (rng.random(u.shape[0]).astype(np.float32) + 0.5) if weighted else None
    B_rowptr, B_col, Bt_rowptr, Bt_col, B_val, Bt_val = csr_from_edges(u, v, n, m, w)
    X = random_unit_rows(n, d, seed=seed + 1)
    return dict(n=n, m=m, B_rowptr=B_rowptr, B_col=B_col, Bt_rowptr=Bt_rowptr, Bt_col=Bt_col, B_val=B_val,
                Bt_val=Bt_val, X=X)


class G:
    def __init__(self, **kw):
        self.__dict__.update(kw)


# ------------------------------------------------------------------------------------------
# a1-a3 propagation
# ------------------------------------------------------------------------------------------

@pytest.mark.parametrize("d,T,alpha,weighted", [(4, 3, 0.5, False), (132, 3, 0.5, False), (128, 5, 0.9, True),
                                                (300, 2, 0.6, False), (8, 0, 0.5, False), (12, 4, 0.0, False),
                                                (16, 3, 1.0, True)])
def test_propagate_planted(tpo, d, T, alpha, weighted):
    g = planted_abg(3001, 2005, 5, d, deg=("zipf", 1.3, 120), p_in=0.6, pop=("zipf", 1.2), x=("gaussian", 1.0),
                    seed=d + T, weighted=weighted)
    Zo, Zho = O.propagate(g.n, g.m, g.B_rowptr, g.B_col, g.X, alpha, T, g.B_val)
    Z, Zh = tpo.propagate(dev_graph(tpo, g), torch.from_numpy(g.X).cuda(), alpha, T)
    assert relF(Z.cpu().numpy(), Zo) <= 1e-5
    assert relF(Zh.cpu().numpy(), Zho) <= 1e-5


@pytest.mark.parametrize("weighted", [False, True])
@pytest.mark.parametrize("d", [8, 128, 136])
def test_propagate_hubs_isolated(tpo, weighted, d):
    """Rows longer than one 512-edge chunk (fix-up path), isolated U and V nodes (R3)."""
    h = hub_graph(seed=d, weighted=weighted, d=d)
    g = G(**h)
    Zo, Zho = O.propagate(g.n, g.m, g.B_rowptr, g.B_col, g.X, 0.5, 3, g.B_val)
    dg = tpo.to_device_graph(g.n, g.m, g.B_rowptr, g.B_col, g.Bt_rowptr, g.Bt_col, g.B_val, g.Bt_val)
    Z, Zh = tpo.propagate(dg, torch.from_numpy(g.X).cuda(), 0.5, 3)
    Z, Zh = Z.cpu().numpy(), Zh.cpu().numpy()
    assert relF(Z, Zo) <= 1e-5 and relF(Zh, Zho) <= 1e-5
    for u in (3, 4):   # isolated U keeps X-hat
        assert np.allclose(Zh[u], g.X[u] / np.linalg.norm(g.X[u]), atol=1e-6)
    # run twice: bitwise identical (no float atomics)
    Z2, Zh2 = tpo.propagate(dg, torch.from_numpy(g.X).cuda(), 0.5, 3)
    assert np.array_equal(Z, Z2.cpu().numpy()) and np.array_equal(Zh, Zh2.cpu().numpy())


@pytest.mark.parametrize("layout", ["0,0", "4,4", "4,8", "8,16", "16,8", "32,32", "32,4"])
@pytest.mark.parametrize("weighted", [False, True])
def test_propagate_column_group_layouts(tpo, monkeypatch, layout, weighted):
    """Every column-group layout of the propagation (TPO_SPMM_L = "Lp,Lq": the iterate P and the
    V-side block Q stored in Lp / Lq-float4 column groups, gathered E = 32 / L edges per load;
    "0,0" = the row-major slice kernel) on a graph with rows longer than one chunk (the
    last-arriving-chunk path) and isolated U / V nodes, at d = 128 (4 .. 32-float4 groups) and
    d = 64: parity with the oracle and bitwise-deterministic re-runs."""
    monkeypatch.setenv("TPO_SPMM_L", layout)
    for d in (128, 64):
        if d == 64 and "32" in layout:
            continue                              # 32-float4 groups need d4 % 32 == 0
        h = hub_graph(seed=d + 7, weighted=weighted, d=d)
        g = G(**h)
        Zo, Zho = O.propagate(g.n, g.m, g.B_rowptr, g.B_col, g.X, 0.6, 4, g.B_val)
        dg = tpo.to_device_graph(g.n, g.m, g.B_rowptr, g.B_col, g.Bt_rowptr, g.Bt_col, g.B_val, g.Bt_val)
        Z, Zh = tpo.propagate(dg, torch.from_numpy(g.X).cuda(), 0.6, 4)
        Z2, Zh2 = tpo.propagate(dg, torch.from_numpy(g.X).cuda(), 0.6, 4)
        assert torch.equal(Z, Z2) and torch.equal(Zh, Zh2)
        Z, Zh = Z.cpu().numpy(), Zh.cpu().numpy()
        assert relF(Z, Zo) <= 1e-5 and relF(Zh, Zho) <= 1e-5
        for u in (3, 4):   # isolated U keeps X-hat
            assert np.allclose(Zh[u], g.X[u] / np.linalg.norm(g.X[u]), atol=1e-6)
        gp = planted_abg(3001, 2005, 5, d, deg=("zipf", 1.3, 120), p_in=0.6, pop=("zipf", 1.2),
                         x=("gaussian", 1.0), seed=d + 1, weighted=weighted)
        Zo, _ = O.propagate(gp.n, gp.m, gp.B_rowptr, gp.B_col, gp.X, 0.5, 3, gp.B_val)
        Z, _ = tpo.propagate(dev_graph(tpo, gp), torch.from_numpy(gp.X).cuda(), 0.5, 3)
        assert relF(Z.cpu().numpy(), Zo) <= 1e-5


def test_propagate_empty_graph(tpo):
    """nnz = 0: every node is isolated, Z = (1 - alpha) X."""
    n, m, d = 37, 5, 8
    rp = np.zeros(n + 1, np.int64)
    rpt = np.zeros(m + 1, np.int64)
    X = random_unit_rows(n, d, seed=3)
    dg = tpo.to_device_graph(n, m, rp, np.zeros(0, np.int32), rpt, np.zeros(0, np.int32))
    Z, Zh = tpo.propagate(dg, torch.from_numpy(X).cuda(), 0.25, 4)
    assert np.allclose(Z.cpu().numpy(), 0.75 * X, atol=1e-7)


def test_propagate_sqrt_degree_closed_form_full_size(tpo):
    """P2 at the bench configuration's graph (BASELINE configs[1], 'small'): x = sqrt(D_U) is a
    fixed point of L L^T, so Z_T = (1 - alpha^{T+1}) x."""
    g = make_config("small")
    du = np.diff(g.B_rowptr).astype(np.float64)
    X = np.repeat(np.sqrt(du)[:, None], 8, axis=1).astype(np.float32)
    Z, _ = tpo.propagate(dev_graph(tpo, g), torch.from_numpy(X).cuda(), g.alpha, g.T)
    exp = (1 - g.alpha ** (g.T + 1)) * X.astype(np.float64)
    assert relF(Z.cpu().numpy(), exp) <= 1e-5


@pytest.mark.slow
def test_propagate_full_small_vs_oracle(tpo):
    """Full-size parity on BASELINE configs[1] ('small': 50k x 80k, ~1M edges, d = 1000, T = 5)."""
    g = make_config("small")
    Zo, Zho = O.propagate(g.n, g.m, g.B_rowptr, g.B_col, g.X, g.alpha, g.T)
    Z, Zh = tpo.propagate(dev_graph(tpo, g), torch.from_numpy(g.X).cuda(), g.alpha, g.T)
    assert relF(Z.cpu().numpy(), Zo) <= 1e-5
    assert relF(Zh.cpu().numpy(), Zho) <= 1e-5


# ------------------------------------------------------------------------------------------
# a4-a5 Haar rotation and features
# ------------------------------------------------------------------------------------------

@pytest.mark.parametrize("d", [1, 12, 64, 65, 300, 1000])
def test_haar_q_device(tpo, d):
    """Device BCGS2 + CholeskyQR2 panels vs the oracle's Householder QR (unique positive QR)."""
    G = np.random.default_rng(d).standard_normal((d, d))
    Q = tpo.haar_q_dev(G).cpu().numpy()
    Qo = O.haar_q(G)
    assert np.max(np.abs(Q - Qo)) <= 1e-5
    assert np.linalg.norm(Q.astype(np.float64).T @ Q - np.eye(d), 2) <= 1e-5


# ------------------------------------------------------------------------------------------
# features
# ------------------------------------------------------------------------------------------

@pytest.mark.parametrize("n,d", [(3001, 12), (1000, 132), (777, 300), (130, 4)])
def test_features(tpo, n, d):
    Zh = random_unit_rows(n, d, seed=d, zero_rows=(5,))
    Q = O.haar_q(np.random.default_rng(d).standard_normal((d, d))).astype(np.float32)
    Rpo, dvo, ro = O.features(Zh, Q)
    Rp, dv, r = tpo.features(torch.from_numpy(Zh).cuda(), torch.from_numpy(Q).cuda(), want_r=True)
    assert relF(Rp.cpu().numpy(), Rpo) <= 1e-5
    assert relF(dv.cpu().numpy(), dvo) <= 1e-5
    assert relF(r.cpu().numpy(), ro) <= 1e-5
    Rp2, dv2, _ = tpo.features(torch.from_numpy(Zh).cuda(), torch.from_numpy(Q).cuda())
    assert torch.equal(Rp, Rp2) and torch.equal(dv, dv2)


def test_features_wide_d(tpo):
    """d = 4096 (D = 8192): dinv's r staging needs 64 KB of dynamic shared memory, above the default
    48 KB opt-in limit.  Q is any orthogonal matrix (numpy QR of a Gaussian; features take Q as input)."""
    n, d = 300, 4096
    Zh = random_unit_rows(n, d, seed=41)
    Q = np.linalg.qr(np.random.default_rng(42).standard_normal((d, d)))[0].astype(np.float32)
    Rpo, dvo, ro = O.features(Zh, Q)
    Rp, dv, r = tpo.features(torch.from_numpy(Zh).cuda(), torch.from_numpy(Q).cuda(), want_r=True)
    # the sin / cos arguments sqrt(d) Zhat Q^T grow as sqrt(d) (up to 64 here) and their fp32 rounding
    # with them: the fp32-vs-fp64 tolerance is scaled from the 1e-5 of d <= 256 by sqrt(d / 256)
    tol = 1e-5 * np.sqrt(d / 256)
    assert relF(Rp.cpu().numpy(), Rpo) <= tol
    assert relF(dv.cpu().numpy(), dvo) <= tol
    assert relF(r.cpu().numpy(), ro) <= tol
    assert np.allclose(np.sum(Rp.double().cpu().numpy() ** 2, axis=1), np.e, rtol=1e-5)   # F1


# ------------------------------------------------------------------------------------------
# a6-a7 implicit affinity and top-k
# ------------------------------------------------------------------------------------------

def oracle_features_of(g):
    Z, Zh = O.propagate(g.n, g.m, g.B_rowptr, g.B_col, g.X, g.alpha, g.T, g.B_val)
    Q = O.haar_q(g.G)
    Rp, dinv, _ = O.features(Zh.astype(np.float32), Q.astype(np.float32))
    return Rp.astype(np.float32), dinv.astype(np.float32)


@pytest.fixture(scope="module")
def tiny_feats():
    g = make_config("tiny")
    Rp, dinv = oracle_features_of(g)
    return g, Rp, dinv


@pytest.mark.parametrize("n,D", [(2000, 600), (777, 136), (5003, 256), (40, 8)])
def test_gram_tcgen05(tpo, n, D):
    """tcgen05 3xTF32 Gram vs the oracle's fp64 Gram (ragged row / column tails, diagonal and
    off-diagonal 128 x 128 tiles, several row splits)."""
    Zh = random_unit_rows(n, D // 2, seed=n)
    Q = O.haar_q(np.random.default_rng(D).standard_normal((D // 2, D // 2))).astype(np.float32)
    Rp, dinv, _ = O.features(Zh, Q)
    Rp, dinv = Rp.astype(np.float32), dinv.astype(np.float32)
    Go = O.gram(Rp, dinv)
    G = tpo.gram(torch.from_numpy(Rp).cuda(), torch.from_numpy(dinv).cuda()).cpu().numpy()
    assert np.array_equal(G, G.T)
    # 3xTF32 products are fp32-accurate; the tensor-core fp32 accumulation over a 128-row
    # segment truncates, which shows up as a small one-sided bias
    assert np.max(np.abs(G - Go)) <= 3e-6 * np.max(np.abs(Go))
    G2 = tpo.gram(torch.from_numpy(Rp).cuda(), torch.from_numpy(dinv).cuda()).cpu().numpy()
    assert np.array_equal(G, G2)


def test_affinity_matvec(tpo, tiny_feats):
    g, Rp, dinv = tiny_feats
    Y = np.random.default_rng(1).standard_normal((g.n, 15)).astype(np.float32)
    out_o = O.affinity_matvec(Rp, dinv, Y)
    out = tpo.affinity_matvec(torch.from_numpy(Rp).cuda(), torch.from_numpy(dinv).cuda(), torch.from_numpy(Y).cuda())
    assert relF(out.cpu().numpy(), out_o) <= 1e-5
    # F5: S~ (1/dinv) = 1/dinv
    v = (1.0 / dinv)[:, None].astype(np.float32)
    o2 = tpo.affinity_matvec(torch.from_numpy(Rp).cuda(), torch.from_numpy(dinv).cuda(), torch.from_numpy(v).cuda())
    assert relF(o2.cpu().numpy(), v) <= 1e-5


@pytest.mark.parametrize("chunk", [0, 700, 2000, 64])
def test_affinity_matvec_rfree(tpo, chunk):
    """f3: S~Y from Zhat and Q with R' recomputed in row chunks (ragged last chunk)
    vs the oracle's features -> affinity chain, and vs the materialised GPU product."""
    g = make_config("tiny")
    _, Zh = O.propagate(g.n, g.m, g.B_rowptr, g.B_col, g.X, g.alpha, g.T)
    Zh32 = Zh.astype(np.float32)
    Q = O.haar_q(g.G).astype(np.float32)
    Rp, dinv, _ = O.features(Zh32, Q)
    Rp32, dv32 = Rp.astype(np.float32), dinv.astype(np.float32)
    Y = np.random.default_rng(5).standard_normal((g.n, 15)).astype(np.float32)
    ref = O.affinity_matvec(Rp32, dv32, Y)
    out = tpo.affinity_matvec_rfree(torch.from_numpy(Zh32).cuda(), torch.from_numpy(Q).cuda(), torch.from_numpy(Y).cuda(),
                                    chunk_rows=chunk)
    assert relF(out.cpu().numpy(), ref) <= 1e-5
    Rg, dg_, _ = tpo.features(torch.from_numpy(Zh32).cuda(), torch.from_numpy(Q).cuda())
    mat = tpo.affinity_matvec(Rg, dg_, torch.from_numpy(Y).cuda())
    assert relF(out.cpu().numpy(), mat.cpu().numpy()) <= 1e-6


@pytest.fixture(scope="module")
def tiny_topk(tiny_feats):
    g, Rp, dinv = tiny_feats
    return O.topk(Rp, dinv, g.k)


def test_topk_exact_tiny(tpo, tiny_feats, tiny_topk):
    g, Rp, dinv = tiny_feats
    Gmo, so, Pso, lam = tiny_topk
    Gm, s, Ps = tpo.topk_eig(torch.from_numpy(Rp).cuda(), torch.from_numpy(dinv).cuda(), g.k)
    Gm, Ps = Gm.cpu().numpy(), Ps.cpu().numpy()
    assert DN.sin_theta(Gm, Gmo) <= 1e-4
    assert DN.sin_theta(Ps, Pso) <= 1e-4
    assert np.allclose(s, so, rtol=1e-5)
    assert abs(s[0] - 1.0) < 1e-5                                   # F5 / E5
    assert np.max(np.abs(Gm.astype(np.float64).T @ Gm - np.eye(g.k))) <= 1e-6   # E2
    assert np.all(Gm.astype(np.float64).sum(0) >= 0)                 # R8


def test_topk_not_converged_is_an_error(tpo, tiny_feats, monkeypatch):
    """A subspace iteration that runs out of rounds before its Ritz residuals reach 1e-9 lambda_1
    returns TPO_ENUMERIC instead of unconverged vectors (TPO_EIG_MAX_ROUNDS lowers the cap)."""
    from paper_2405_11922_b200._lib import TPO_ENUMERIC, TpoError
    g, Rp, dinv = tiny_feats
    monkeypatch.setenv("TPO_EIG_MAX_ROUNDS", "0")
    with pytest.raises(TpoError) as ei:
        tpo.topk_eig(torch.from_numpy(Rp).cuda(), torch.from_numpy(dinv).cuda(), g.k)
    assert ei.value.code == TPO_ENUMERIC and "did not converge" in str(ei.value)
    monkeypatch.delenv("TPO_EIG_MAX_ROUNDS")
    Gm, s, Ps = tpo.topk_eig(torch.from_numpy(Rp).cuda(), torch.from_numpy(dinv).cuda(), g.k)
    assert abs(s[0] - 1.0) < 1e-5


def test_topk_planted_svd(tpo):
    """E8: R' = U diag(s) V^T with dinv = 1 -> Gamma = U[:, :k], sigma = s[:k]."""
    rng = np.random.default_rng(3)
    n, D, k = 2500, 48, 6
    U, _ = np.linalg.qr(rng.standard_normal((n, D)))
    V, _ = np.linalg.qr(rng.standard_normal((D, D)))
    sig = np.geomspace(3.0, 0.05, D)
    Rp = ((U * sig) @ V.T).astype(np.float32)
    Gm, s, Ps = tpo.topk_eig(torch.from_numpy(Rp).cuda(), torch.ones(n, device="cuda"), k)
    assert np.allclose(s, sig[:k], rtol=1e-5)
    assert DN.sin_theta(Gm.cpu().numpy(), U[:, :k]) <= 1e-4
    assert DN.sin_theta(Ps.cpu().numpy(), V[:, :k]) <= 1e-4


def test_topk_halko_mode_vs_oracle(tpo, tiny_feats):
    """TPO_EIG_HALKO (the paper-cited rSVD, p = 10, q = 2) vs the same algorithm in the oracle with
    the same Omega (same-algorithm parity; orth by CholeskyQR2 on the GPU,
    Householder in the oracle -- the same subspaces)."""
    g, Rp, dinv = tiny_feats
    k, p, q = g.k, 10, 2
    Om = np.random.default_rng(7).standard_normal((Rp.shape[1], k + p)).astype(np.float32)
    Gmo, so, Pso = DN.halko_topk(Rp, dinv, k, p, q, Om)
    Gm, s, Ps = tpo.topk_eig(torch.from_numpy(Rp).cuda(), torch.from_numpy(dinv).cuda(), k, mode=tpo.TPO_EIG_HALKO,
                             p=p, q=q, Omega=torch.from_numpy(Om).cuda())
    Gm, Ps = Gm.cpu().numpy(), Ps.cpu().numpy()
    assert np.allclose(s, so, rtol=1e-5)
    assert DN.sin_theta(Gm, Gmo) <= 1e-4
    assert DN.sin_theta(Ps, Pso) <= 1e-4
    assert np.max(np.abs(Gm.astype(np.float64).T @ Gm - np.eye(k))) <= 1e-6
    assert np.all(Gm.astype(np.float64).sum(0) >= 0)


# ------------------------------------------------------------------------------------------
# a8-a9 discretisation
# ------------------------------------------------------------------------------------------

def test_cluster_bit_exact_given_eigen_inputs(tpo, tiny_feats, tiny_topk):
    """D4: identical fp32 (R', dinv, Gamma, Psi) and fp64 sigma -> identical labels."""
    g, Rp, dinv = tiny_feats
    Gmo, so, Pso, _ = tiny_topk
    Gm32, Ps32 = Gmo.astype(np.float32), Pso.astype(np.float32)
    lab_o, it_o, U_o = O.cluster(Rp, dinv, Gm32, so, Ps32, 5, 20)
    lab, it = tpo.cluster(torch.from_numpy(Rp).cuda(), torch.from_numpy(dinv).cuda(), torch.from_numpy(Gm32).cuda(), so,
                          torch.from_numpy(Ps32).cuda(), 5, 20)
    lab = lab.cpu().numpy()
    assert it == it_o
    assert np.array_equal(lab, lab_o)


@pytest.mark.parametrize("Tf,Tg", [(0, 1), (1, 3), (7, 30)])
def test_cluster_iterations(tpo, Tf, Tg):
    g = planted_abg(1200, 1200, 4, 16, deg=("poisson", 8.0), p_in=0.85, x=("gaussian", 1.0), alpha=0.5, T=3, seed=5)
    Rp, dinv = oracle_features_of(g)
    Gmo, so, Pso, _ = O.topk(Rp, dinv, g.k)
    Gm32, Ps32 = Gmo.astype(np.float32), Pso.astype(np.float32)
    lab_o, it_o, _ = O.cluster(Rp, dinv, Gm32, so, Ps32, Tf, Tg)
    lab, it = tpo.cluster(torch.from_numpy(Rp).cuda(), torch.from_numpy(dinv).cuda(), torch.from_numpy(Gm32).cuda(), so,
                          torch.from_numpy(Ps32).cuda(), Tf, Tg)
    assert it == it_o and np.array_equal(lab.cpu().numpy(), lab_o)


@pytest.mark.parametrize("k,Tf,Tg", [(40, 3, 20), (50, 2, 10)])
def test_cluster_bit_exact_k_over_32(tpo, k, Tf, Tg):
    """The k > 32 discretisation path (warp-per-row assign with 4 rows per warp, column-chunked
    cluster sums, smem-staged M in the Upsilon update): labels bit-exact vs the oracle."""
    g = planted_abg(6000, 4000, k, 48, deg=("poisson", 10.0), p_in=0.8, x=("gaussian", 1.0), alpha=0.5, T=2,
                    seed=k)
    Rp, dinv = oracle_features_of(g)
    Gmo, so, Pso, _ = O.topk(Rp, dinv, k)
    Gm32, Ps32 = Gmo.astype(np.float32), Pso.astype(np.float32)
    lab_o, it_o, _ = O.cluster(Rp, dinv, Gm32, so, Ps32, Tf, Tg)
    lab, it = tpo.cluster(torch.from_numpy(Rp).cuda(), torch.from_numpy(dinv).cuda(), torch.from_numpy(Gm32).cuda(), so,
                          torch.from_numpy(Ps32).cuda(), Tf, Tg)
    assert it == it_o and np.array_equal(lab.cpu().numpy(), lab_o)


@pytest.mark.parametrize("k", [40, 50])
def test_cluster_exact_ties_k_over_32(tpo, k):
    """Exact ties in Alg. 3 on the k > 32 path (integer-tensor-core scores, certified argmax):
    columns j and j+1 of Gamma and Psi are made identical with sigma_{j+1} = sigma_j, so the ONMF
    keeps Upsilon's columns j and j+1 identical and every row whose best cluster is j ties.  Those
    rows fail certification and are rescored with R13's sequential fma: ties -> smallest index,
    labels bit-exact vs the oracle."""
    g = planted_abg(6000, 4000, k, 48, deg=("poisson", 10.0), p_in=0.8, x=("gaussian", 1.0), alpha=0.5, T=2,
                    seed=k + 3)
    Rp, dinv = oracle_features_of(g)
    Gmo, so, Pso, _ = O.topk(Rp, dinv, k)
    for j in range(2, k - 1):                      # the first non-trivial pair whose tie is exercised
        Gm32, Ps32 = Gmo.astype(np.float32).copy(), Pso.astype(np.float32).copy()
        sj = np.array(so, np.float64).copy()
        Gm32[:, j + 1] = Gm32[:, j]
        Ps32[:, j + 1] = Ps32[:, j]
        sj[j + 1] = sj[j]
        lab_o, it_o, _ = O.cluster(Rp, dinv, Gm32, sj, Ps32, 3, 1)       # first assignment: Phi = I
        if np.any(lab_o == j):
            break
    so = sj
    assert np.any(lab_o == j)                      # the tie is exercised
    assert not np.any(lab_o == j + 1)              # ... and resolved to the smaller index
    args = (torch.from_numpy(Rp).cuda(), torch.from_numpy(dinv).cuda(), torch.from_numpy(Gm32).cuda(), so,
            torch.from_numpy(Ps32).cuda(), 3)
    lab, it = tpo.cluster(*args, 1)
    assert it == it_o and np.array_equal(lab.cpu().numpy(), lab_o)
    lab_o, it_o, _ = O.cluster(Rp, dinv, Gm32, so, Ps32, 3, 10)        # and through the later iterations
    lab, it = tpo.cluster(*args, 10)
    assert it == it_o and np.array_equal(lab.cpu().numpy(), lab_o)


# ------------------------------------------------------------------------------------------
# end to end
# ------------------------------------------------------------------------------------------

def test_run_tiny_end_to_end(tpo, tiny_topk):
    g = make_config("tiny")
    res = O.run(g)
    labels, tm = tpo.run(dev_graph(tpo, g), torch.from_numpy(g.X).cuda(), g.alpha, g.T, g.k, g.G)
    labels = labels.cpu().numpy()
    assert DN.ari(labels, res["labels"]) >= 0.999
    assert labels.min() >= 0 and labels.max() < g.k
    assert np.all(tm > 0)


@pytest.mark.parametrize("k", [40, 50])
def test_run_matches_stage_calls_k_over_32(tpo, k):
    """tpo_run shares R''s row exponents / feature maxima between a7 and a8 (formed in the dinv pass
    of a5, dinv bit-identical) and runs the integer-tensor-core Gamma, RH and R^T Ups: the same
    labels, bit for bit, as the stage-by-stage ABI calls (tpo_propagate, tpo_haar_q_dev,
    tpo_features, tpo_topk_eig, tpo_cluster), which compute those statistics themselves."""
    g = planted_abg(9000, 5000, k, 64, deg=("poisson", 10.0), p_in=0.8, x=("gaussian", 1.0), alpha=0.5, T=2,
                    seed=k + 11)
    dg = dev_graph(tpo, g)
    X = torch.from_numpy(g.X).cuda()
    lab_run, _ = tpo.run(dg, X, g.alpha, g.T, k, g.G)
    _, Zh = tpo.propagate(dg, X, g.alpha, g.T)
    Rp, dinv, _ = tpo.features(Zh, tpo.haar_q_dev(g.G))
    Gm, sig, Ps = tpo.topk_eig(Rp, dinv, k)
    lab, _ = tpo.cluster(Rp, dinv, Gm, sig, Ps, 5, 20)
    assert np.array_equal(lab_run.cpu().numpy(), lab.cpu().numpy())


@pytest.mark.parametrize("weighted", [False, True])
def test_run_host_matches_device_inputs(tpo, weighted):
    """tpo_run_host (host inputs copied inside the call, Haar beside the copies, no SMs held
    back) runs the same kernels on the same data as tpo_run: identical labels."""
    g = make_config("tiny")
    rng = np.random.default_rng(5)
    bval = tval = None
    if weighted:   # weights of B and the matching entries of B^T
        bval = rng.uniform(0.5, 2.0, g.nnz).astype(np.float32)
        rows = np.repeat(np.arange(g.n, dtype=np.int64), np.diff(g.B_rowptr))
        key_b = rows * g.m + g.B_col
        trows = np.repeat(np.arange(g.m, dtype=np.int64), np.diff(g.Bt_rowptr))
        key_t = g.Bt_col.astype(np.int64) * g.m + trows
        tval = bval[np.searchsorted(key_b, key_t)] if np.all(np.diff(key_b) > 0) else None
        assert tval is not None
    dg = tpo.to_device_graph(g.n, g.m, g.B_rowptr, g.B_col, g.Bt_rowptr, g.Bt_col, bval, tval)
    X = torch.from_numpy(g.X).cuda()
    lab_d = tpo.Runner(dg, g.d, g.k)(X, g.alpha, g.T, g.G).cpu().numpy()
    hr = tpo.HostRunner(g.n, g.m, g.nnz, g.d, g.k, weighted=weighted)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    lab_h = hr(pin(g.B_rowptr), pin(g.B_col), pin(g.Bt_rowptr), pin(g.Bt_col), pin(g.X),
               pin(np.asarray(g.G, np.float64)), g.alpha, g.T,
               B_val=None if bval is None else pin(bval), Bt_val=None if tval is None else pin(tval)).numpy()
    assert np.array_equal(lab_h, lab_d)
    assert np.all(hr.timings > 0)
    # pageable numpy inputs work too (synchronous copies)
    lab_h2 = hr(g.B_rowptr, g.B_col, g.Bt_rowptr, g.Bt_col, g.X, np.asarray(g.G, np.float64), g.alpha, g.T,
                B_val=bval, Bt_val=tval).numpy()
    assert np.array_equal(lab_h2, lab_d)


@pytest.mark.parametrize("n_p,k", [(20000, 7), (20000, 16), (12345, 20), (9000, 32), (20000, 40), (100, 20)])
def test_skinny_atb64(tpo, n_p, k):
    """A^T B of two n_p x k fp64 blocks (the k x k products of Alg. 2 and the Gamma polish):
    the whole-output skinny kernel (k <= 32, n_p >= 8192) and the dgemm path both match
    numpy's fp64 product to rounding."""
    from paper_2405_11922_b200.sharded import GpuSolverOps
    rng = np.random.default_rng(n_p + k)
    A = rng.standard_normal((n_p, k))
    B = rng.standard_normal((n_p, k))
    ops = GpuSolverOps(n_p, 64, k, "cuda")
    out = ops.atb(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()).cpu().numpy()
    ref = A.T @ B
    scale = np.abs(A).T @ np.abs(B)
    assert np.max(np.abs(out - ref) / scale) <= 1e-13
