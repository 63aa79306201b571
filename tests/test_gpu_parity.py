"""Parity of the CUDA path (through the C-ABI) against the golden fixtures from
the live reference (tests/golden/make_golden.py).  Tolerances are the north
star's: Gramian matvec / sketch 1e-10, PCG direction 1e-8 at a fixed iteration
count, loss trajectory 1e-6 (see test_c1_trajectory for the horizon)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ngd = pytest.importorskip("paper_2505_11638_b200")


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.fixture(scope="module")
def c1(gold):
    G = gold("c1")
    top = ngd.MlpTopology((2, 32, 32, 1))
    prob = ngd.Poisson2D(top)
    quad = prob.sample_quadrature(900, 120, 0)
    theta = ngd.init(top, 0).values
    return G, prob, quad, theta


def test_c1_loss_metric_grad_matvec(c1):
    G, prob, quad, theta = c1
    assert prob.loss_value(theta, quad) == pytest.approx(float(G["loss"]), rel=1e-12)
    assert rel(prob.metric_stack(theta, None, quad), G["metric"]) <= 1e-12
    assert rel(prob.loss_grad(theta, quad), G["grad"]) <= 1e-10
    gop = ngd.GramianOperator.from_problem(prob, theta, quad)
    assert rel(gop.matvec(G["v"]), G["gv"]) <= 1e-10
    assert rel(gop.matmat(G["omega8"]), G["y8"]) <= 1e-10
    assert gop.matvec_count == 9


@pytest.mark.parametrize("svd", [3, 2, 1, 0])
def test_c1_nystrom_preconditioner_pcg(c1, svd):
    G, prob, quad, theta = c1
    from paper_2505_11638_b200 import _lib

    with _lib.option("svd", svd):
        _check_c1_pcg(G, prob, quad, theta)


def _check_c1_pcg(G, prob, quad, theta):
    gop = ngd.GramianOperator.from_problem(prob, theta, quad)
    fac = ngd.nystrom_approximate(gop, 100, seed=7, omega_source="host")
    assert gop.matvec_count == 100
    top = G["eig100"] > 1e-8 * G["eig100"][0]
    assert rel(fac.eig_host[top], G["eig100"][top]) <= 1e-10
    mu = float(G["mu"])
    pre = ngd.NystromPreconditioner(fac, mu)
    assert rel(pre.apply(G["v"]), G["pinv_v"]) <= 1e-8
    for k in (1, 5, 20):
        rep = ngd.pcg(ngd.ShiftedOperator(gop, mu), G["grad"], 1e-300, k, precond=pre)
        meta = G[f"pcg{k}_meta"]
        assert rel(rep.solution, G[f"pcg{k}_x"]) <= 1e-8, k
        assert (rep.iterations, rep.matvecs, rep.breakdown) == (int(meta[0]), int(meta[1]), bool(meta[4]))


def test_c1_device_omega_sketch_statistics(c1):
    """Throughput-mode (device Philox) sketches resolve the same top spectrum."""
    G, prob, quad, theta = c1
    gop = ngd.GramianOperator.from_problem(prob, theta, quad)
    fac = ngd.nystrom_approximate(gop, 100, seed=7, omega_source="device")
    top = G["eig100"] > 1e-6 * G["eig100"][0]
    assert rel(fac.eig_host[top], G["eig100"][top]) <= 1e-8


def test_c1_trajectory(c1):
    """20-step fixed-rank NGD trajectory vs the reference.  The first 12 steps must
    agree to 1e-6; beyond that the reference itself amplifies 1-ulp matvec noise
    past 1e-6 (profiles/r01_traj_sensitivity_oracle_1e-16.txt: 2.9e-6 at step 13,
    2.4e-4 at step 18), so later steps are held to that measured envelope (x10)."""
    G, prob, quad, theta = c1
    cfg = ngd.NystromNgdConfig(ell0=100, ell_max=100, cg_maxit=20, kappa=1e-300, mu_floor_mode="grad-power",
                               mu_floor_coeff=1e-6, mu_floor_exponent=1.0, iterations=20, seed=0, fixed_rank=True)
    _, recs = ngd.nystrom_ngd_run(prob, theta, cfg, quad)
    loss = np.array([r.loss for r in recs])
    dev = np.abs(loss - G["traj_loss"]) / np.abs(G["traj_loss"])
    assert np.all(dev[:12] <= 1e-6), dev
    envelope = np.array([1e-12] * 6 + [3e-9, 2e-8, 1e-8, 1e-7, 5e-7, 1.2e-6, 1.3e-6, 3e-5, 1.1e-4, 9.3e-5,
                                       4.7e-5, 8.6e-4, 2.4e-3, 1.2e-3])
    assert np.all(dev <= np.maximum(envelope, 1e-6)), dev
    assert [r.pcg_iters for r in recs] == list(G["traj_pcg"].astype(int))
    assert [r.matvecs for r in recs] == list(G["traj_matvecs"].astype(int))


def test_c1_adaptive_rank_trajectory(c1):
    G, prob, quad, theta = c1
    cfg = ngd.NystromNgdConfig(ell0=10, ell_max=100, cg_maxit=20, iterations=8, seed=3)
    _, recs = ngd.nystrom_ngd_run(prob, theta, cfg, quad)
    assert [r.ell for r in recs] == list(G["adapt_ell"].astype(int))
    assert [r.pcg_iters for r in recs] == list(G["adapt_pcg"].astype(int))
    np.testing.assert_allclose([r.loss for r in recs], G["adapt_loss"], rtol=1e-6)


@pytest.mark.parametrize("name,widths,kind,nint,nbnd", [
    ("c2", (2, 64, 64, 64, 1), "sin2d", 4096, 512),
    ("c3_sub", (5, 128, 128, 128, 1), "sinsum", 256, 64),
    ("c5_sub", (10, 256, 256, 256, 256, 1), "gauss", 24, 8),
])
def test_configs_loss_grad_matvec(gold, name, widths, kind, nint, nbnd):
    G = gold(name)
    top = ngd.MlpTopology(widths)
    prob = ngd.Poisson2D(top) if kind == "sin2d" else ngd.PoissonND(top, kind)
    quad = prob.sample_quadrature(nint, nbnd, 0)
    theta = ngd.init(top, 0).values
    assert prob.loss_value(theta, quad) == pytest.approx(float(G["loss"]), rel=1e-12)
    assert rel(prob.loss_grad(theta, quad), G["grad"]) <= 1e-10
    gop = ngd.GramianOperator.from_problem(prob, theta, quad)
    assert rel(gop.matvec(G["v"]), G["gv"]) <= 1e-10


def test_c4_interior_only(gold):
    G = gold("c4_sub")
    top = ngd.MlpTopology((2, 256, 256, 256, 1))
    prob = ngd.LaplacianStack(top)
    n = G["x"].shape[0]
    quad = ngd.QuadratureSet(G["x"], np.full(n, 1.0 / n), np.zeros((0, 2)), np.zeros(0))
    gop = ngd.GramianOperator.from_problem(prob, ngd.init(top, 0).values, quad)
    assert rel(gop.matvec(G["v"]), G["gv"]) <= 1e-10
