"""GPU parity of the SVD-based attribute dimension reduction (Sec. 3.2.1, Eq. Xd, PAPER.md:501-517;
SURVEY.md §8f #1) through the C-ABI (tpo_svd_reduce) against the fp64 oracle (oracle_svd_reduce).

X' = Gamma Sigma of the exact top-d SVD (R14), sign-fixed by R8.  Where the top-d singular values
are separated, X' itself is unique and compared column by column (relative Frobenius <= 1e-5,
fp32 storage); where the cut falls inside a noise bulk only the singular values, the orthogonality
X'^T X' = diag(sigma^2) and the Eckart-Young bound are fixed, and those are checked.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import core as O  # noqa: E402
from oracle import dense as DN  # noqa: E402
from synth import make_config, planted_abg  # noqa: E402


def relF(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(scope="module")
def tpo():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2405_11922_b200 import build
    build.build()
    import paper_2405_11922_b200 as T
    return T


def planted_spectrum_X(n, du, seed, s_top=4.0, ratio=0.85):
    """X = U diag(s) V^T (fp32) with geometric, well-separated singular values."""
    rng = np.random.default_rng(seed)
    U, _ = np.linalg.qr(rng.standard_normal((n, du)))
    V, _ = np.linalg.qr(rng.standard_normal((du, du)))
    s = s_top * ratio ** np.arange(du)
    return ((U * s) @ V.T).astype(np.float32), s


@pytest.mark.parametrize("n,du,d", [(6000, 96, 16), (3001, 64, 8), (777, 40, 4)])
def test_svd_reduce_planted_spectrum(tpo, n, du, d):
    X, s = planted_spectrum_X(n, du, seed=n + d)
    Xo, so = O.svd_reduce(X, d)
    Xg, sg = tpo.svd_reduce(torch.from_numpy(X).cuda(), d)
    Xg = Xg.cpu().numpy()
    assert np.allclose(sg, so, rtol=1e-6)
    assert relF(Xg, Xo) <= 1e-5
    assert np.all(Xg.astype(np.float64).sum(0) >= 0)                                  # R8
    # Xg and Xo agree, and both are Gamma Sigma of the planted SVD
    assert np.allclose(so, s[:d], rtol=1e-5)


def test_svd_reduce_pass_through(tpo):
    X, _ = planted_spectrum_X(500, 24, seed=3)
    Xg, sg = tpo.svd_reduce(torch.from_numpy(X).cuda(), 24)
    assert sg is None and np.array_equal(Xg.cpu().numpy(), X)


@pytest.mark.slow
def test_svd_reduce_small_config_X(tpo):
    """BASELINE configs[1]'s attribute matrix (50,000 x 1,000, 1 % density + cluster signatures):
    d = 10 (the signature subspace, separated) column by column; d = 64 (cut inside the bulk):
    singular values, orthogonality and the Eckart-Young bound on sampled pairs."""
    X = make_config("small").X
    Xt = torch.from_numpy(X).cuda()
    Xo, so = O.svd_reduce(X, 10, eig="lapack")
    Xg, sg = tpo.svd_reduce(Xt, 10)
    Xg = Xg.cpu().numpy()
    assert np.allclose(sg, so, rtol=1e-5)
    assert DN.sin_theta(Xg, Xo) <= 1e-4
    assert relF(Xg, Xo) <= 1e-4
    Xo64, so64 = O.svd_reduce(X, 68, eig="lapack")
    Xg, sg = tpo.svd_reduce(Xt, 64)
    Xg = Xg.cpu().numpy().astype(np.float64)
    assert np.allclose(sg, so64[:64], rtol=1e-5)
    assert np.max(np.abs(Xg.T @ Xg - np.diag(sg ** 2))) <= 1e-5 * sg[0] ** 2
    rng = np.random.default_rng(0)
    i, j = rng.integers(0, X.shape[0], 20000), rng.integers(0, X.shape[0], 20000)
    X64 = X.astype(np.float64)
    err = np.abs(np.einsum("ij,ij->i", X64[i], X64[j]) - np.einsum("ij,ij->i", Xg[i], Xg[j]))
    assert np.all(err <= so64[64] ** 2 * (1 + 1e-3) + 1e-5 * sg[0] ** 2)        # Eckart-Young entrywise


def test_reduced_pipeline_end_to_end(tpo):
    """The paper's default 'TPO' variant: reduce X (d_U = 96 -> d = 16), then the whole hot path
    (tpo_run) on X'; the oracle runs the same two steps; ARI(GPU, oracle) >= 0.999."""
    g = planted_abg(3000, 2000, 5, 96, deg=("poisson", 8.0), p_in=0.8, x=("gaussian", 1.0), alpha=0.5, T=3, seed=9)
    X, _ = planted_spectrum_X(g.n, 96, seed=10, ratio=0.9)
    d = 16
    Gd = np.random.default_rng(11).standard_normal((d, d))
    Xo, _ = O.svd_reduce(X, d)
    g.X, g.G, g.d = Xo.astype(np.float32), Gd, d
    ref = O.run(g, Tf=5, Tg=20)
    Xg, _ = tpo.svd_reduce(torch.from_numpy(X).cuda(), d)
    dg = tpo.to_device_graph(g.n, g.m, g.B_rowptr, g.B_col, g.Bt_rowptr, g.Bt_col)
    labels, _ = tpo.run(dg, Xg, g.alpha, g.T, g.k, Gd)
    assert DN.ari(labels.cpu().numpy(), ref["labels"]) >= 0.999
