"""NGD-CG baseline (optim.py:273-327) and the Gramian spectrum (harness.py:237-266) on the device
path, against fixtures from the live reference (tests/golden/make_golden.py:
baselines)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ngd = pytest.importorskip("paper_2505_11638_b200")


@pytest.fixture(scope="module")
def setup(gold):
    G = gold("baselines")
    top = ngd.MlpTopology((2, 8, 8, 1))
    prob = ngd.make_problem("poisson2d", topology=top)
    quad = prob.sample_quadrature(200, 40, 0)
    theta = ngd.init(top, 0).values
    assert np.array_equal(theta, G["theta0"])
    cfg = ngd.NystromNgdConfig(ell0=10, ell_max=40, cg_maxit=20, iterations=4, seed=0)
    return G, prob, quad, theta, cfg


@pytest.mark.parametrize("name", ["ngd_cg"])
def test_baseline_trajectory(setup, name):
    G, prob, quad, theta, cfg = setup
    theta_f, recs = ngd.run_optimizer(name, prob, theta, cfg, quad, quad_eval=quad)
    assert isinstance(theta_f, np.ndarray) and theta_f.shape == theta.shape
    np.testing.assert_allclose([r.loss for r in recs], G[f"{name}_loss"], rtol=1e-6)
    np.testing.assert_allclose([r.h1_rel_error for r in recs], G[f"{name}_h1"], rtol=1e-6)
    np.testing.assert_allclose([r.mu for r in recs], G[f"{name}_mu"], rtol=1e-12)
    assert [r.pcg_iters for r in recs] == list(G[f"{name}_pcg"].astype(int))
    assert [r.matvecs for r in recs] == list(G[f"{name}_matvecs"].astype(int))


def test_unknown_optimizer(setup):
    _, prob, quad, theta, cfg = setup
    for name in ("adam", "bfgs", "gd", "ngd_dense"):  # off the hot path: not provided
        with pytest.raises(KeyError):
            ngd.run_optimizer(name, prob, theta, cfg, quad)


def test_dense_gramian_spectrum(setup):
    """Device assembly of J^T diag(w) J (Jacobian-row chunks on the DMMA GEMM): symmetric, equal to
    matvecs of I, and the normalised spectrum matches the reference's."""
    G, prob, quad, theta, _ = setup
    gop = ngd.GramianOperator.from_problem(prob, theta, quad)
    dense = ngd.assemble_dense(gop)
    assert np.array_equal(dense, dense.T)
    eye = np.eye(gop.dim)
    cols = np.column_stack([gop.matvec(eye[:, i]) for i in range(0, gop.dim, 13)])
    np.testing.assert_allclose(dense[:, ::13], cols, rtol=1e-10, atol=1e-12 * np.abs(dense).max())
    spec = ngd.gramian_spectrum(prob, theta, quad, top=30)
    np.testing.assert_allclose(spec, G["spectrum"], rtol=1e-8, atol=1e-13)
