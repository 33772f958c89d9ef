"""GPU evaluation and monitors through the C-ABI: tpo_eval (ARI / NMI / ACC,
PAPER.md:2448-2462) and tpo_objective (the Lemma 4 monitor, Eq. obj5) against the
oracle's definitions (oracle/dense.py: contingency-table formulas, Hungarian matching by scipy,
explicit n x n R R^T), and clustering the V side by swapping B and B^T."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import core as O  # noqa: E402
from oracle import dense as DN  # noqa: E402
from synth import make_config, planted_abg, random_unit_rows  # noqa: E402


@pytest.fixture(scope="module")
def tpo():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2405_11922_b200 import build
    build.build()
    import paper_2405_11922_b200 as T
    return T


@pytest.mark.parametrize("n,kp,kt,noise", [(100_000, 7, 5, 0.3), (2_000_000, 50, 50, 0.1), (999, 3, 4, 0.9), (10, 2, 2, 0.0)])
def test_eval_metrics_vs_oracle(tpo, n, kp, kt, noise):
    rng = np.random.default_rng(n + kp)
    truth = rng.integers(0, kt, n).astype(np.int32)
    pred = (truth * 7 + 3) % kp
    flip = rng.random(n) < noise
    pred[flip] = rng.integers(0, kp, flip.sum())
    pred = pred.astype(np.int32)
    m = tpo.evaluate(torch.from_numpy(pred).cuda(), torch.from_numpy(truth).cuda(), kp, kt)
    assert abs(m["ari"] - DN.ari(pred, truth)) <= 1e-12
    assert abs(m["nmi"] - DN.nmi(pred, truth)) <= 1e-12
    assert abs(m["acc"] - DN.acc(pred, truth)) <= 1e-15


def test_eval_rejects_out_of_range_labels(tpo):
    from paper_2405_11922_b200._lib import TpoError
    p = torch.tensor([0, 1, 5], dtype=torch.int32, device="cuda")
    t = torch.tensor([0, 1, 1], dtype=torch.int32, device="cuda")
    with pytest.raises(TpoError):
        tpo.evaluate(p, t, 2, 2)


def test_objective_monitor_vs_explicit_affinity(tpo):
    """||R^T Y||^2 and ||R^T Ups||^2 against Tr(Y^T (R R^T) Y) and Tr(Ups^T (R R^T) Ups) with the n x n
    R R^T formed explicitly; Ky Fan (E3): ||R^T Y||^2 <= sum_{l<=k} sigma_l^2."""
    g = make_config("tiny")
    Z, Zh = O.propagate(g.n, g.m, g.B_rowptr, g.B_col, g.X, g.alpha, g.T)
    Rp, dinv, _ = O.features(Zh.astype(np.float32), O.haar_q(g.G).astype(np.float32))
    Rp, dinv = Rp.astype(np.float32), dinv.astype(np.float32)
    Gm, s, Ps, _ = O.topk(Rp, dinv, g.k)
    labels, _, U = O.cluster(Rp, dinv, Gm.astype(np.float32), s, Ps.astype(np.float32), 5, 20)
    t1, t2 = DN.nci_objective(Rp, dinv, labels, g.k, U)
    o1, o2 = tpo.objective(torch.from_numpy(Rp).cuda(), torch.from_numpy(dinv).cuda(),
                           torch.from_numpy(labels.astype(np.int32)).cuda(), g.k, torch.from_numpy(U).cuda())
    assert abs(o1 - t1) <= 1e-9 * abs(t1) and abs(o2 - t2) <= 1e-9 * abs(t2)
    assert o1 <= (s ** 2).sum() * (1 + 1e-9)


def test_target_side_v(tpo):
    """Clustering V: the same hot path on the swapped graph and X_V; parity of the
    propagation with the oracle run on B^T, end-to-end ARI with the oracle's V-side run."""
    g = planted_abg(1500, 2500, 5, 64, deg=("poisson", 8.0), p_in=0.8, x=("gaussian", 1.0), alpha=0.5, T=3, seed=21)
    Xv = random_unit_rows(g.m, 64, seed=22)
    dg = tpo.to_device_graph(g.n, g.m, g.B_rowptr, g.B_col, g.Bt_rowptr, g.Bt_col).target("V")
    Zo, Zho = O.propagate(g.m, g.n, g.Bt_rowptr, g.Bt_col, Xv, g.alpha, g.T)
    Z, Zh = tpo.propagate(dg, torch.from_numpy(Xv).cuda(), g.alpha, g.T)
    rel = np.linalg.norm(Z.cpu().numpy() - Zo) / np.linalg.norm(Zo)
    assert rel <= 1e-5
    from synth import ABG
    gv = ABG(n=g.m, m=g.n, d=64, k=5, alpha=g.alpha, T=g.T, B_rowptr=g.Bt_rowptr, B_col=g.Bt_col,
             Bt_rowptr=g.B_rowptr, Bt_col=g.B_col, X=Xv, G=np.random.default_rng(23).standard_normal((64, 64)),
             Omega=None, truth=np.zeros(g.m, np.int32))
    ref = O.run(gv)
    labels, _ = tpo.run(dg, torch.from_numpy(Xv).cuda(), g.alpha, g.T, 5, gv.G)
    assert DN.ari(labels.cpu().numpy(), ref["labels"]) >= 0.999
