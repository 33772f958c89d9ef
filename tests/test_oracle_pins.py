"""Pins of the fp64 oracle against what the paper and the mathematics fix (not against itself).

Each test names the passage it pins.  Dense references come from oracle/dense.py (numpy,
tiny sizes) or from closed forms / hand-computed values written in the test.
"""
import math

import numpy as np
import pytest

from oracle import core as O
from oracle import dense as DN
from synth import csr_from_edges, planted_abg, random_unit_rows

pytestmark = pytest.mark.filterwarnings("ignore::RuntimeWarning")


def small_graph(seed=0, weighted=False, n=60, m=40, k=4, d=5, deg=("poisson", 4.0), isolated=()):
    g = planted_abg(n, m, k, d, deg=deg, p_in=0.7, x=("uniform",), seed=seed, weighted=weighted)
    if isolated:
        # remove all edges of the listed U rows (rebuild CSR)
        u = np.repeat(np.arange(n), np.diff(g.B_rowptr))
        keep = ~np.isin(u, list(isolated))
        w = None if g.B_val is None else g.B_val[keep]
        g.B_rowptr, g.B_col, g.Bt_rowptr, g.Bt_col, g.B_val, g.Bt_val = csr_from_edges(
            u[keep], g.B_col[keep], n, m, w)
    return g


# ----------------------------------------------------------------------------------------------
# a1-a3 propagation: Eq. PX, Eq. L (252-254), Eq. update-Z (454)
# ----------------------------------------------------------------------------------------------

def test_hand_computed_two_node_example():
    """B = [[1],[1]]: D_U = [1,1], D_V = [2], L = [[1/sqrt2],[1/sqrt2]], L L^T = [[.5,.5],[.5,.5]].
    X = I2, alpha = .5, T = 1: Z = .5 (X + .5 L L^T X) = [[.625,.125],[.125,.625]] (by hand)."""
    rp, col, _, _, _, _ = csr_from_edges([0, 1], [0, 0], 2, 1)
    Z, Zh = O.propagate(2, 1, rp, col, np.eye(2, dtype=np.float32), 0.5, 1)
    assert np.allclose(Z, [[0.625, 0.125], [0.125, 0.625]], atol=1e-15)
    nr = math.hypot(0.625, 0.125)
    assert np.allclose(Zh, [[0.625 / nr, 0.125 / nr], [0.125 / nr, 0.625 / nr]], atol=1e-15)


@pytest.mark.parametrize("weighted", [False, True])
@pytest.mark.parametrize("alpha,T", [(0.5, 3), (0.9, 7), (0.2, 1)])
def test_dense_series(weighted, alpha, T):
    """P1: sparse Horner evaluation == explicit dense power series of Eq. PX."""
    g = small_graph(seed=3, weighted=weighted)
    Z, Zh = O.propagate(g.n, g.m, g.B_rowptr, g.B_col, g.X, alpha, T, g.B_val)
    L = DN.dense_L(DN.dense_B(g.n, g.m, g.B_rowptr, g.B_col, g.B_val))
    Zs = DN.series_Z(L, g.X.astype(np.float64), alpha, T)
    assert np.linalg.norm(Z - Zs) <= 1e-13 * np.linalg.norm(Zs)
    assert np.allclose(Zh, DN.rownorm(Zs), atol=1e-13)


def test_sqrt_degree_fixed_point():
    """P2: x = sqrt(D_U) satisfies L L^T x = x (Eq. L), so Z_T = (1 - alpha^{T+1}) x exactly."""
    g = small_graph(seed=5, weighted=True, isolated=(0, 7))
    du = np.zeros(g.n)
    for u in range(g.n):
        du[u] = g.B_val[g.B_rowptr[u]:g.B_rowptr[u + 1]].sum()
    X = np.repeat(np.sqrt(du)[:, None], 3, axis=1) * np.array([1.0, -2.0, 0.5])
    X32 = X.astype(np.float32)
    delta = np.linalg.norm(X32.astype(np.float64) - X)     # fp32 rounding of the input
    for alpha, T in [(0.5, 4), (0.8, 9)]:
        Z, _ = O.propagate(g.n, g.m, g.B_rowptr, g.B_col, X32, alpha, T, g.B_val)
        exp = (1.0 - alpha ** (T + 1)) * X
        # the series operator has 2-norm <= 1 (spec(L L^T) in [0,1]), so the input rounding
        # moves Z by at most ||delta||
        assert np.linalg.norm(Z - exp) <= delta + 1e-13 * np.linalg.norm(exp)
        assert np.linalg.norm(Z - exp) <= 1e-6 * np.linalg.norm(exp)


def test_row_stochastic_transition():
    """M = D_U^{-1} B D_V^{-1} B^T has unit row sums."""
    g = small_graph(seed=6, weighted=True, isolated=(3,))
    su, sv = O.degree_scales(g.n, g.m, g.B_rowptr, g.B_col, g.B_val)
    B = DN.dense_B(g.n, g.m, g.B_rowptr, g.B_col, g.B_val)
    M = (su ** 2)[:, None] * B * (sv ** 2)[None, :] @ B.T
    rs = M.sum(1)
    nz = np.diff(g.B_rowptr) > 0
    assert np.allclose(rs[nz], 1.0, atol=1e-12) and np.all(rs[~nz] == 0)


def test_special_cases():
    """P3: alpha = 0 -> Z = X; T = 0 -> Z = (1-alpha) X and Zhat = Xhat;
    isolated u keeps Xhat (R3)."""
    g = small_graph(seed=7, isolated=(2, 11))
    X = g.X.astype(np.float64)
    Z, Zh = O.propagate(g.n, g.m, g.B_rowptr, g.B_col, g.X, 0.0, 5)
    assert np.array_equal(Z, X)
    Z, Zh = O.propagate(g.n, g.m, g.B_rowptr, g.B_col, g.X, 0.3, 0)
    assert np.allclose(Z, 0.7 * X, rtol=0, atol=1e-16) and np.allclose(Zh, DN.rownorm(X), atol=1e-15)
    Z, Zh = O.propagate(g.n, g.m, g.B_rowptr, g.B_col, g.X, 0.6, 6)
    for u in (2, 11):
        assert np.allclose(Z[u], 0.4 * X[u], atol=1e-16)
        assert np.allclose(Zh[u], DN.rownorm(X[u:u + 1])[0], atol=1e-15)


def test_block_diagonal_no_mixing():
    """P3: intra-cluster probability 1 gives a block-diagonal B, so attributes never cross blocks."""
    g = planted_abg(80, 40, 4, 3, deg=("poisson", 5.0), p_in=1.0, x=("uniform",), seed=2, shuffle=False)
    X = np.zeros((80, 3), np.float32)
    X[:20] = g.X[:20]                        # only block 0 carries attributes
    Z, _ = O.propagate(g.n, g.m, g.B_rowptr, g.B_col, X, 0.7, 6)
    assert np.all(Z[20:] == 0.0) and np.any(Z[:20] != 0.0)


def test_linearity_and_weight_scaling():
    """P3: Z is linear in X; L is invariant to a uniform weight scaling."""
    g = small_graph(seed=8, weighted=True)
    X1 = g.X
    X2 = random_unit_rows(g.n, g.d, seed=4)
    a, b = 0.75, -1.5
    Za, _ = O.propagate(g.n, g.m, g.B_rowptr, g.B_col, (a * X1.astype(np.float64) + b * X2).astype(np.float32), .5, 4, g.B_val)
    Z1, _ = O.propagate(g.n, g.m, g.B_rowptr, g.B_col, X1, .5, 4, g.B_val)
    Z2, _ = O.propagate(g.n, g.m, g.B_rowptr, g.B_col, X2, .5, 4, g.B_val)
    Xab = (a * X1.astype(np.float64) + b * X2).astype(np.float32).astype(np.float64)
    # reference: same operator on the rounded combination equals a Z1 + b Z2 up to the rounding of X
    assert np.linalg.norm(Za - (a * Z1 + b * Z2)) <= 1e-6 * np.linalg.norm(Za)
    Zs, _ = O.propagate(g.n, g.m, g.B_rowptr, g.B_col, X1, .5, 4, (g.B_val * 4.0).astype(np.float32))
    assert np.allclose(Zs, Z1, rtol=1e-14, atol=1e-15)
    del Xab


@pytest.mark.parametrize("alpha", [0.5, 0.9])
def test_lemma1_limit_and_tail_bound(alpha):
    """P4: Z_T -> (1-alpha)(I - alpha L L^T)^{-1} X (Lemma 1 proof) with
    ||Z_T - Z_inf||_F <= alpha^{T+1}/(1-alpha) ||X||_F because spec(L L^T) is in [0, 1]."""
    g = small_graph(seed=9)
    L = DN.dense_L(DN.dense_B(g.n, g.m, g.B_rowptr, g.B_col))
    ev = np.linalg.eigvalsh(L @ L.T)
    assert ev.min() > -1e-12 and ev.max() < 1 + 1e-12
    Zinf = DN.neumann_Z(L, g.X.astype(np.float64), alpha)
    for T in (2, 5, 10):
        Z, _ = O.propagate(g.n, g.m, g.B_rowptr, g.B_col, g.X, alpha, T)
        assert np.linalg.norm(Z - Zinf) <= alpha ** (T + 1) / (1 - alpha) * np.linalg.norm(g.X.astype(np.float64)) * (1 + 1e-9)
    Z, _ = O.propagate(g.n, g.m, g.B_rowptr, g.B_col, g.X, alpha, 400)
    assert np.linalg.norm(Z - Zinf) <= 1e-12 * np.linalg.norm(Zinf)


# ----------------------------------------------------------------------------------------------
# a4-a5 Haar rotation and random features: PAPER.md:458-468 (Eqs. R-prime, Ri)
# ----------------------------------------------------------------------------------------------

def test_haar_q_is_the_unique_positive_qr():
    """F4: Q^T Q = I and G = Q R with R upper triangular, diag(R) > 0 (the unique QR; LAPACK's
    Householder QR with the same sign fix must agree)."""
    rng = np.random.default_rng(1)
    G = rng.standard_normal((37, 37))
    Q = O.haar_q(G)
    assert np.linalg.norm(Q.T @ Q - np.eye(37)) < 1e-12
    R = Q.T @ G
    assert np.max(np.abs(np.tril(R, -1))) < 1e-12 and np.all(np.diag(R) > 0)
    q2, r2 = np.linalg.qr(G)
    s = np.sign(np.diag(r2))
    assert np.allclose(Q, q2 * s[None, :], atol=1e-12)


def test_features_row_norm_bound_zero_row():
    """F1 ||R'[i]||^2 = (e/d) sum(sin^2 + cos^2) = e; F2 |R'| <= sqrt(e/d); F3 zero row."""
    n, d = 50, 16
    Zh = random_unit_rows(n, d, seed=2, zero_rows=(4,))
    Q = O.haar_q(np.random.default_rng(3).standard_normal((d, d))).astype(np.float32)
    Rp, dinv, r = O.features(Zh, Q)
    assert np.allclose((Rp ** 2).sum(1), math.e, rtol=1e-14)
    assert np.max(np.abs(Rp)) <= math.sqrt(math.e / d) * (1 + 1e-15)
    assert np.all(Rp[4, :d] == 0.0) and np.allclose(Rp[4, d:], math.sqrt(math.e / d), rtol=1e-15)
    assert np.allclose(r, Rp.sum(0), rtol=1e-13)
    assert np.allclose(dinv, 1.0 / np.sqrt(Rp @ r), rtol=1e-13)


def test_features_rotation_orientation():
    """Zo = sqrt(d) Zhat Q^T.  With Q a permutation matrix P (P[j, pi(j)] = 1) and
    Zhat[i] = e_a, Zo[i, j] = sqrt(d) [pi(j) == a]: the sin half is sqrt(e/d) sin(sqrt d) exactly
    at the column j = pi^{-1}(a) and 0 elsewhere (Zhat Q would put it at pi(a))."""
    d = 6
    pi = np.array([2, 0, 5, 1, 3, 4])          # not an involution
    P = np.zeros((d, d), np.float32)
    P[np.arange(d), pi] = 1.0
    Zh = np.eye(d, dtype=np.float32)           # row a = e_a
    Rp, _, _ = O.features(Zh, P)
    amp = math.sqrt(math.e / d)
    for a in range(d):
        j = int(np.where(pi == a)[0][0])
        expect = np.zeros(d)
        expect[j] = amp * math.sin(math.sqrt(d))
        assert np.allclose(Rp[a, :d], expect, atol=1e-15)
        ce = np.full(d, amp)
        ce[j] = amp * math.cos(math.sqrt(d))
        assert np.allclose(Rp[a, d:], ce, atol=1e-15)


def test_top_eigenpair_closed_form():
    """F5: S~ (1/dinv) = 1/dinv, because diag(dinv) R' R'^T diag(dinv) dinv^{-1} = diag(dinv) R' r;
    hence the top singular value of R is exactly 1 (R7 keeps this trivial pair)."""
    n, d = 120, 10
    Zh = random_unit_rows(n, d, seed=5)
    Q = O.haar_q(np.random.default_rng(6).standard_normal((d, d))).astype(np.float32)
    Rp, dinv, r = O.features(Zh, Q)
    Rp32, dv32 = Rp.astype(np.float32), dinv.astype(np.float32)
    v = 1.0 / dv32.astype(np.float64)
    out = O.affinity_matvec(Rp32, dv32, v[:, None])[:, 0]
    assert np.linalg.norm(out - v) <= 1e-6 * np.linalg.norm(v)   # fp32 rounding of R', dinv
    Gm, s, Ps, lam = O.topk(Rp32, dv32, 3)
    assert abs(s[0] - 1.0) < 1e-6


@pytest.mark.slow
def test_theorem1_band_d64():
    """F6 (Theorem 1): E[R[i].R[j]] lies in the multiplicative band around
    s(u_i,u_j), checked over Haar seeds at d = 64 on off-diagonal pairs, widened by 3 SE
    (the only regime where the proof's ratio-of-expectations step holds)."""
    n, d, reps = 10, 64, 300
    Zh = random_unit_rows(n, d, seed=11)
    S = DN.msa_matrix(Zh.astype(np.float64))
    acc = np.zeros((reps, n, n))
    for s in range(reps):
        Q = O.haar_q(np.random.default_rng(1000 + s).standard_normal((d, d))).astype(np.float32)
        Rp, dinv, _ = O.features(Zh, Q)
        R = dinv[:, None] * Rp
        acc[s] = R @ R.T
    mean, se = acc.mean(0), acc.std(0) / math.sqrt(reps)
    eps = 17 / (16 * d * d) + 1 / (4 * d)
    lo, hi = (1 - eps) / (1 + eps), (1 + eps) / (1 - eps)
    off = ~np.eye(n, dtype=bool)
    ok = (mean >= lo * S - 3 * se) & (mean <= hi * S + 3 * se)
    assert ok[off].mean() >= 0.95


def test_msa_running_example(running_example):
    """F7: Eq. s on the printed Zhat (2 decimals) reproduces the printed S (3 decimals) within 0.003,
    and the nearest neighbours are u2,u1,u4,u5,u4,u7,u6 (PAPER.md:287 / 1523)."""
    S = DN.msa_matrix(running_example["Zhat"])
    assert np.max(np.abs(S - running_example["S"])) <= 0.003
    Sp = running_example["S"].copy()
    np.fill_diagonal(Sp, -1)
    assert list(np.argmax(Sp, 1) + 1) == [2, 1, 4, 5, 4, 7, 6]


def test_running_example_partition_optimal(running_example):
    """D3: brute-force Eq. obj1 over all 301 partitions of 7 nodes into 3 blocks on the printed
    (symmetrised) S: the paper's partition {u1,u2}/{u3,u4,u5}/{u6,u7} is the minimiser."""
    S = running_example["S"]
    S = 0.5 * (S + S.T)
    arg, best, allv = DN.best_partition(S, 3)
    assert len(allv) == 301
    truth = running_example["partition"][0].astype(int)
    assert DN.ari(arg, truth) == 1.0


# ----------------------------------------------------------------------------------------------
# a6-a7 implicit affinity and exact top-k (Eq. init-HY)
# ----------------------------------------------------------------------------------------------

def planted_svd(n, D, sig, seed):
    rng = np.random.default_rng(seed)
    U, _ = np.linalg.qr(rng.standard_normal((n, D)))
    V, _ = np.linalg.qr(rng.standard_normal((D, D)))
    Rp = (U * sig[None, :]) @ V.T
    return U, V, Rp


def test_affinity_matvec_planted():
    """E8: with R' = U diag(s) V^T and dinv = 1, R R^T Y = U diag(s^2) U^T Y."""
    n, D = 200, 12
    sig = np.linspace(2.0, 0.3, D)
    U, V, Rp = planted_svd(n, D, sig, 1)
    Rp32 = Rp.astype(np.float32)
    Y = np.random.default_rng(2).standard_normal((n, 5))
    out = O.affinity_matvec(Rp32, np.ones(n, np.float32), Y)
    R64 = Rp32.astype(np.float64)
    assert np.allclose(out, R64 @ (R64.T @ Y), rtol=1e-12, atol=1e-12)
    assert np.linalg.norm(out - (U * sig ** 2) @ (U.T @ Y)) <= 1e-6 * np.linalg.norm(out)


def test_sym_eig_vs_lapack():
    rng = np.random.default_rng(3)
    A = rng.standard_normal((40, 40))
    A = A + A.T
    w, V = O.sym_eig(A)
    o = np.argsort(w)
    assert np.allclose(w[o], np.linalg.eigvalsh(A), atol=1e-12)
    assert np.linalg.norm(A @ V - V * w[None, :]) < 1e-11
    assert np.linalg.norm(V.T @ V - np.eye(40)) < 1e-12


def test_topk_lapack_eigensolver_matches_jacobi():
    """The oracle's top-k with the Gram's eigenpairs taken from LAPACK (eig="lapack", used where the
    Jacobi sweeps are too slow, D = 2000) equals the Jacobi route: same sigma, the same subspaces, and
    the same signs (the sign rule R8 is applied after either eigensolver)."""
    n, d, k = 600, 20, 6
    Zh = random_unit_rows(n, d, seed=21)
    Q = O.haar_q(np.random.default_rng(22).standard_normal((d, d))).astype(np.float32)
    Rp, dinv, _ = O.features(Zh, Q)
    Rp32, dv32 = Rp.astype(np.float32), dinv.astype(np.float32)
    Gj, sj, Pj, lj = O.topk(Rp32, dv32, k)
    Gl, sl, Pl, ll = O.topk(Rp32, dv32, k, eig="lapack")
    assert np.allclose(sj, sl, rtol=1e-12) and np.allclose(lj, ll, rtol=1e-9, atol=1e-13)
    assert np.allclose(Gj, Gl, atol=1e-9) and np.allclose(Pj, Pl, atol=1e-9)


def test_topk_planted_svd_and_eckart_young():
    """E8 / E4 / E2: the exact top-k of R' = U diag(s) V^T is (U[:, :k], s[:k], V[:, :k]) up to the
    sign rule; ||R - Gamma Sigma Psi^T||_2 = s_{k+1} (Eckart-Young)."""
    n, D, k = 300, 16, 5
    sig = np.array([3.0, 2.5, 2.0, 1.6, 1.3, 0.9, 0.8, 0.7, 0.6, 0.5, 0.4, 0.35, 0.3, 0.2, 0.1, 0.05])
    U, V, Rp = planted_svd(n, D, sig, 4)
    Rp32 = Rp.astype(np.float32)
    Gm, s, Ps, lam = O.topk(Rp32, np.ones(n, np.float32), k)
    assert np.allclose(s, sig[:k], rtol=1e-6)
    assert DN.sin_theta(Gm, U[:, :k]) < 1e-6 and DN.sin_theta(Ps, V[:, :k]) < 1e-6
    assert np.linalg.norm(Gm.T @ Gm - np.eye(k)) < 1e-12
    assert np.linalg.norm(Ps.T @ Ps - np.eye(k)) < 1e-12
    R = Rp32.astype(np.float64)
    assert abs(np.linalg.norm(R - (Gm * s[None, :]) @ Ps.T, 2) - sig[k]) < 1e-6
    assert np.all(Gm.sum(0) >= 0)                     # R8 sign rule


def test_topk_vs_dense_eigh_of_RRt():
    """E1: top-k eigenvectors of the dense n x n R R^T (independent LAPACK) on a features matrix."""
    n, d, k = 400, 12, 6
    Zh = random_unit_rows(n, d, seed=8)
    Q = O.haar_q(np.random.default_rng(9).standard_normal((d, d))).astype(np.float32)
    Rp, dinv, _ = O.features(Zh, Q)
    Rp32, dv32 = Rp.astype(np.float32), dinv.astype(np.float32)
    R = dv32.astype(np.float64)[:, None] * Rp32.astype(np.float64)
    w, V = np.linalg.eigh(R @ R.T)
    Gm, s, Ps, lam = O.topk(Rp32, dv32, k)
    assert np.allclose(s ** 2, w[::-1][:k], rtol=1e-10, atol=1e-13)
    assert DN.sin_theta(Gm, V[:, ::-1][:, :k]) < 1e-8
    # Ky Fan (E3): for any NCI Y, ||R^T Y||_F^2 <= sum_{i<=k} sigma_i^2 (Lemma 5)
    rng = np.random.default_rng(10)
    for _ in range(20):
        lab = rng.integers(0, k, n)
        Y = np.zeros((n, k))
        for c in range(k):
            idx = lab == c
            if idx.any():
                Y[idx, c] = 1 / math.sqrt(idx.sum())
        assert np.linalg.norm(R.T @ Y) ** 2 <= (s ** 2).sum() * (1 + 1e-12)


# ----------------------------------------------------------------------------------------------
# a8 ONMF (Alg. 2, Eqs. update-Q / update-Y) and a9 NCI (Alg. 3, 583-639)
# ----------------------------------------------------------------------------------------------

def test_onmf_hand_computed_step():
    """One step by hand with a non-symmetric R = [[2,1],[0,1]], Ups0 = H0 = [[1],[1]] (k = 1):
    R^T Ups = [[2],[2]], H (Ups^T Ups) = [[2],[2]]  -> H = [[1],[1]];
    R H = [[3],[1]], Ups^T (R H) = [[4]], Ups (.) = [[4],[4]] -> Ups = [[sqrt(3/4)],[sqrt(1/4)]]."""
    Rp = np.array([[2, 1], [0, 1]], np.float32)
    U, H = O.onmf(Rp, np.ones(2, np.float32), np.ones((2, 1), np.float32), np.ones(1),
                  np.ones((2, 1), np.float32), 1)
    assert np.allclose(H, [[1.0], [1.0]], atol=1e-9)
    assert np.allclose(U, [[math.sqrt(0.75)], [0.5]], atol=1e-9)


def test_onmf_hand_computed_step_k2_weighted():
    """One Alg. 2 step by hand at k = 2 with non-unit dinv, non-unit sigma and a NON-symmetric
    M = Ups^T (R H), so that a transposed M, a dropped dinv (in R^T Ups or in R H) or Sigma applied
    on the wrong side of Psi each change the result (Eqs. update-Q / update-Y, PAPER.md:553-560;
    products bracketed as PAPER.md:564; init Eq. init-HY 571-574 with the R9 clamps).

      R' = [[1,2],[3,1]], dinv = [1, 1/2]  ->  R = diag(dinv) R' = [[1,2],[3/2,1/2]]
      Gamma = [[1,1],[2,1]]                ->  Ups0 = Gamma (+eps)
      Psi = [[1/2,2],[1/2,4]], sigma = [2, 1/2]  ->  H0 = Psi Sigma = [[1,1],[1,2]] (+eps)
    H step:  R^T Ups0 = [[4,5/2],[3,5/2]];  Ups0^T Ups0 = [[5,3],[3,2]];  H0 (Ups0^T Ups0) = [[8,5],[11,7]]
             H1 = H0 . (R^T Ups0) / (H0 Ups0^T Ups0) = [[1/2,1/2],[3/11,5/7]]
    Ups step: R H1 = [[23/22,27/14],[39/44,31/28]]
              M = Ups0^T (R H1) = [[31/11,29/7],[85/44,85/28]]          (M != M^T)
              Ups0 M = [[209/44,201/28],[333/44,317/28]]
              Ups1 = Ups0 . sqrt(R H1 / (Ups0 M)) = [[sqrt(46/209), sqrt(54/201)],
                                                    [2 sqrt(39/333), sqrt(31/317)]]"""
    Rp = np.array([[1, 2], [3, 1]], np.float32)
    dinv = np.array([1.0, 0.5], np.float32)
    Gamma = np.array([[1, 1], [2, 1]], np.float32)
    Psi = np.array([[0.5, 2], [0.5, 4]], np.float32)
    sigma = np.array([2.0, 0.5])
    U, H = O.onmf(Rp, dinv, Gamma, sigma, Psi, 1)
    assert np.allclose(H, [[0.5, 0.5], [3 / 11, 5 / 7]], rtol=0, atol=1e-10)
    assert np.allclose(U, [[math.sqrt(46 / 209), math.sqrt(54 / 201)],
                           [2 * math.sqrt(39 / 333), math.sqrt(31 / 317)]], rtol=0, atol=1e-10)


def test_onmf_clamps_negative_numerator():
    """R9: a negative (R H) entry is clamped to 0, so the Ups entry becomes exactly 0."""
    Rp = np.array([[-2, 0], [0, 1]], np.float32)
    U, H = O.onmf(Rp, np.ones(2, np.float32), np.ones((2, 1), np.float32), np.ones(1),
                  np.ones((2, 1), np.float32), 1)
    # R^T Ups = [[-2],[1]] -> H = [[0],[1 * 1/2]] ; R H = [[0],[0.5]] -> Ups[0] = 0
    assert np.allclose(H, [[0.0], [0.5]], atol=1e-9)
    assert U[0, 0] == 0.0 and U[1, 0] > 0


def test_onmf_fixed_point():
    """(Ups0, H0) with Ups0 >= 0 column-orthonormal (disjoint supports) and R = Ups0 H0^T is a fixed
    point of both multiplicative rules (R^T Ups0 = H0 = H0 (Ups0^T Ups0);
    Ups0 (Ups0^T R H0) = R H0)."""
    rng = np.random.default_rng(4)
    n, D, k = 30, 8, 3
    lab = np.arange(n) % k
    U0 = np.zeros((n, k))
    for c in range(k):
        v = rng.random((lab == c).sum()) + 0.5
        U0[lab == c, c] = v / np.linalg.norm(v)
    H0 = rng.random((D, k)) + 0.1
    Rp = (U0 @ H0.T)
    U0f, H0f, Rpf = U0.astype(np.float32), H0.astype(np.float32), Rp.astype(np.float32)
    U, H = O.onmf(Rpf, np.ones(n, np.float32), U0f, np.ones(k), H0f, 4)
    assert np.allclose(U, U0f, atol=2e-6) and np.allclose(H, H0f, atol=2e-6)


def test_nci_examples():
    """Eq. ell-ast argmax with ties -> smallest index (R10); SPEC.md:314-343 examples."""
    lab, it = O.nci(np.array([[0.9, 0.1], [0.2, 0.8]]), 20)
    assert list(lab) == [0, 1] and it == 2
    lab, it = O.nci(np.array([[0.5, 0.5], [0.0, 1.0]]), 20)
    assert list(lab) == [0, 1]
    lab, it = O.nci(np.eye(4)[[0, 1, 2, 3, 0, 1]], 20)
    assert list(lab) == [0, 1, 2, 3, 0, 1] and it == 2


def test_nci_hand_traced_rotation():
    """Alg. 3 by hand: rows r0..r2 = [1,0], r3 = [.45,.55], r4 = [0,1].
    it1 (Phi = I): labels [0,0,0,1,1]; Phi = Ups^T Y: col0 = [3,0]/sqrt3, col1 = [.45,1.55]/sqrt2.
    it2: r3 scores [.45*1.7321, .45*.3182 + .55*1.0960] = [.7794, .7460] -> 0: labels [0,0,0,0,1].
    it3: col0 = [3.45,.55]/2, col1 = [0,1]; no change -> stop after 3 iterations."""
    U = np.array([[1, 0], [1, 0], [1, 0], [0.45, 0.55], [0, 1]], float)
    lab, it = O.nci(U, 20)
    assert list(lab) == [0, 0, 0, 0, 1] and it == 3
    lab, it = O.nci(U, 1)
    assert list(lab) == [0, 0, 0, 1, 1] and it == 1


def test_nci_noise_recovery_and_validity():
    """D1/D2: NCI + 1% noise recovers the clean labels; the output is a valid NCI."""
    rng = np.random.default_rng(5)
    n, k = 500, 7
    lab0 = rng.integers(0, k, n)
    Y0 = np.zeros((n, k))
    for c in range(k):
        Y0[lab0 == c, c] = 1 / math.sqrt((lab0 == c).sum())
    Ups = np.abs(Y0 + 0.01 * rng.random((n, k)) * Y0.max())
    lab, it = O.nci(Ups, 20)
    assert np.array_equal(lab, lab0)
    assert lab.min() >= 0 and lab.max() < k


def test_ari_worked_example():
    """truth [0,0,1,1], pred [0,1,1,1] -> ARI 0; identical -> 1."""
    assert abs(DN.ari([0, 0, 1, 1], [0, 1, 1, 1])) < 1e-15
    assert DN.ari([0, 0, 1, 2], [5, 5, 7, 9]) == 1.0


def test_end_to_end_tiny_planted():
    """Whole oracle pipeline on a small planted graph: valid labels, Gamma orthonormal, sigma_1 = 1."""
    g = planted_abg(600, 600, 3, 24, deg=("poisson", 10.0), p_in=0.9, x=("gaussian", 1.0), alpha=0.5, T=3, seed=1)
    res = O.run(g, Tf=5, Tg=20)
    assert abs(res["sigma"][0] - 1.0) < 1e-6
    assert np.linalg.norm(res["Gamma"].T @ res["Gamma"] - np.eye(3)) < 1e-10
    assert DN.ari(res["labels"], g.truth) > 0.5


# ------------------------------------------------------------------------------------------
# Halko mode oracle (oracle/dense.halko_topk): the randomised truncated SVD PAPER.md:574 cites
# ------------------------------------------------------------------------------------------

def _planted_svd(n, D, sig, seed):
    rng = np.random.default_rng(seed)
    U, _ = np.linalg.qr(rng.standard_normal((n, D)))
    V, _ = np.linalg.qr(rng.standard_normal((D, D)))
    return U, V, (U * sig) @ V.T


def test_halko_exact_when_rank_fits_the_block():
    """rank(R) <= b = k + p: range(R Omega) = range(R), so the rSVD is the exact SVD (textbook
    property of the range finder) -- pins Gamma = Y U, Psi = V, sigma = S."""
    n, D, k, p = 400, 30, 4, 6
    sig = np.concatenate([np.geomspace(4.0, 0.5, 8), np.zeros(D - 8)])     # rank 8 <= b = 10
    U, V, Rp = _planted_svd(n, D, sig, 1)
    Om = np.random.default_rng(2).standard_normal((D, k + p))
    Gm, s, Ps = DN.halko_topk(Rp, np.ones(n), k, p, 0, Om)
    assert np.allclose(s, sig[:k], rtol=1e-12)
    assert DN.sin_theta(Gm, U[:, :k]) < 1e-10 and DN.sin_theta(Ps, V[:, :k]) < 1e-10
    assert np.all(Gm.sum(0) >= 0)                                          # R8
    assert np.allclose(Gm * s, (Rp @ Ps), atol=1e-10)                      # R Psi = Gamma Sigma


def test_halko_power_iterations_converge_to_the_exact_top_k():
    """Full-rank R with a gap after k: q power steps drive sin(theta) to the exact top-k down by
    (sigma_{b+1} / sigma_k)^{2q+1} (Halko et al., Thm. 9.1 flavour); at q = 6 it is exact to 1e-8."""
    n, D, k, p = 500, 60, 5, 5
    sig = np.concatenate([np.linspace(3.0, 2.0, k), np.geomspace(0.5, 0.01, D - k)])
    U, V, Rp = _planted_svd(n, D, sig, 3)
    Om = np.random.default_rng(4).standard_normal((D, k + p))
    errs = []
    for q in (0, 1, 2, 6):
        Gm, s, Ps = DN.halko_topk(Rp, np.ones(n), k, p, q, Om)
        errs.append(DN.sin_theta(Ps, V[:, :k]))
    assert errs[0] > errs[1] > errs[2] > errs[3]
    assert errs[3] < 1e-8
    Gm, s, _ = DN.halko_topk(Rp, np.ones(n), k, p, 6, Om)
    assert np.allclose(s, sig[:k], rtol=1e-10)


# ----------------------------------------------------------------------------------------------
# f1 SVD-based attribute dimension reduction: Eq. Xd, Lemma 3 (519-527)
# ----------------------------------------------------------------------------------------------

def test_svd_reduce_pass_through():
    """d >= d_U disables the reduction: X' = X exactly."""
    X = random_unit_rows(30, 12, seed=31)
    for d in (12, 20):
        Xr, s = O.svd_reduce(X, d)
        assert s is None and np.array_equal(Xr, X.astype(np.float64))


def test_svd_reduce_exact_on_low_rank_X():
    """A rank-r X (exact small-integer product, so fp32 holds it exactly) loses nothing at d >= r:
    X' X'^T = X X^T (Eq. Xd: X X^T = Gamma Sigma^2 Gamma^T when sigma_{d+1} = 0), and the
    singular values beyond r vanish."""
    rng = np.random.default_rng(32)
    A = rng.integers(-3, 4, (40, 3)).astype(np.float64)
    B = rng.integers(-3, 4, (3, 24)).astype(np.float64)
    X = (A @ B).astype(np.float32)
    XX = X.astype(np.float64) @ X.astype(np.float64).T
    for d in (3, 5):
        Xr, s = O.svd_reduce(X, d)
        assert np.max(np.abs(Xr @ Xr.T - XX)) <= 1e-9 * np.max(np.abs(XX))
        if d > 3:
            assert np.all(s[3:] <= 1e-6 * s[0])


def test_svd_reduce_eckart_young_orthogonality_and_signs():
    """Random 50 x 40 X, d = 10: sigma = the top-10 singular values of an independent
    LAPACK SVD; X'^T X' = diag(sigma^2) (orthogonal columns Gamma Sigma); Eckart-Young
    ||X X^T - X' X'^T||_2 = sigma_11^2 and entrywise <= sigma_11^2; column sums >= 0 (R8)."""
    X = np.random.default_rng(33).random((50, 40)).astype(np.float32)
    X64 = X.astype(np.float64)
    S = np.linalg.svd(X64, compute_uv=False)
    Xr, s = O.svd_reduce(X, 10)
    assert np.allclose(s, S[:10], rtol=1e-11)
    assert np.allclose(Xr.T @ Xr, np.diag(S[:10] ** 2), atol=1e-9 * S[0] ** 2)
    E = X64 @ X64.T - Xr @ Xr.T
    assert abs(np.linalg.norm(E, 2) - S[10] ** 2) <= 1e-9 * S[0] ** 2
    assert np.max(np.abs(E)) <= S[10] ** 2 + 1e-6
    assert np.all(Xr.sum(0) >= 0)
    # X' spans the top-10 left singular subspace
    U = np.linalg.svd(X64, full_matrices=False)[0][:, :10]
    assert DN.sin_theta(Xr, U) < 1e-9


def test_lemma3_bound_on_reduced_propagation():
    """Lemma 3: |Z'[i].Z'[j] - Z[i].Z[j]| <= sigma_{d+1}^2 sqrt(D_U[i] D_U[j]) / (1 - alpha)
    for the propagation of X' = Gamma Sigma vs of X (T = 300 hops: the series has converged to
    fp64 precision at alpha = 0.5, 0.8); graphs without isolated U nodes."""
    worst = 0.0
    for seed in range(6):
        g = small_graph(seed=40 + seed, n=60, m=40, k=4, d=5, deg=("poisson", 5.0))
        du = np.diff(g.B_rowptr).astype(np.float64)
        if np.any(du == 0):
            continue
        X = np.random.default_rng(seed).random((g.n, 24)).astype(np.float32)
        S = np.linalg.svd(X.astype(np.float64), compute_uv=False)
        for d in (4, 10):
            Xr, _ = O.svd_reduce(X, d)
            for alpha in (0.5, 0.8):
                Z, _ = O.propagate(g.n, g.m, g.B_rowptr, g.B_col, X, alpha, 300)
                Zr, _ = O.propagate(g.n, g.m, g.B_rowptr, g.B_col, Xr.astype(np.float32), alpha, 300)
                lhs = np.abs(Zr @ Zr.T - Z @ Z.T)
                rhs = S[d] ** 2 * np.sqrt(np.outer(du, du)) / (1 - alpha)
                worst = max(worst, float(np.max(lhs / rhs)))
    assert 0.0 < worst <= 1.0


# ----------------------------------------------------------------------------------------------
# f4 evaluation metrics
# ----------------------------------------------------------------------------------------------

def test_metrics_worked_examples():
    """Hand-worked: a = [0,0,1,1], b = [0,1,0,1]: contingency [[1,1],[1,1]] -> ARI = (0 - 2*2/6) /
    (2 - 2/3) = -1/2, MI = 0 -> NMI = 0, best matching 2 of 4 -> ACC = 1/2.  A relabelled copy
    scores 1 on all three.  a = [0,0,0,1,1,2], b = [1,1,1,0,0,0]: contingency rows (0: 3 in b=1),
    (1: 2 in b=0), (2: 1 in b=0) -> ACC = (3 + 2) / 6."""
    a, b = np.array([0, 0, 1, 1]), np.array([0, 1, 0, 1])
    assert abs(DN.ari(a, b) + 0.5) < 1e-15 and abs(DN.nmi(a, b)) < 1e-15 and DN.acc(a, b) == 0.5
    c = np.array([2, 2, 0, 0, 1, 1, 1])
    d = np.array([0, 0, 1, 1, 2, 2, 2])
    assert DN.ari(c, d) == 1.0 and abs(DN.nmi(c, d) - 1.0) < 1e-15 and DN.acc(c, d) == 1.0
    assert abs(DN.acc(np.array([0, 0, 0, 1, 1, 2]), np.array([1, 1, 1, 0, 0, 0])) - 5 / 6) < 1e-15
    # NMI by hand for a = [0,0,1,1], b = [0,0,0,1]: a_i = (2,2), b_j = (3,1), n_ij = [[2,0],[1,1]]
    mi = 2 * math.log(4 * 2 / (2 * 3)) + 1 * math.log(4 * 1 / (2 * 3)) + 1 * math.log(4 * 1 / (2 * 1))
    ha, hb = 2 * 2 * math.log(2 / 4), 3 * math.log(3 / 4) + math.log(1 / 4)
    assert abs(DN.nmi(np.array([0, 0, 1, 1]), np.array([0, 0, 0, 1])) - mi / math.sqrt(ha * hb)) < 1e-15
