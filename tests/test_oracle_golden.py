"""Pin the CPU oracle against fixtures produced by the live reference
(tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from oracle import ngd_oracle as O


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b))


def c1_setup():
    prob = O.PoissonProblem((2, 32, 32, 1))
    quad = prob.sample_quadrature(900, 120, 0)
    theta = O.init_theta((2, 32, 32, 1), 0)
    return prob, quad, theta


def test_c1_inputs_and_stack(gold):
    g = gold("c1")
    prob, quad, theta = c1_setup()
    assert np.array_equal(theta, g["theta0"])
    assert prob.loss_value(theta, quad) == pytest.approx(float(g["loss"]), rel=1e-13)
    lin = O.Linearization(prob, theta, quad)
    assert rel(lin.value, g["metric"]) <= 1e-13
    assert rel(prob.loss_grad(theta, quad), g["grad"]) <= 1e-12
    gop = O.GramianOracle(prob, theta, quad)
    assert rel(gop.matvec(g["v"]), g["gv"]) <= 1e-12
    assert rel(gop.matmat(g["omega8"]), g["y8"]) <= 1e-12


def test_c1_nystrom_precond_pcg(gold):
    g = gold("c1")
    prob, quad, theta = c1_setup()
    gop = O.GramianOracle(prob, theta, quad)
    fac = O.nystrom_approximate(gop, 100, seed=7)
    top = fac.eigenvalues > 1e-8 * fac.eigenvalues[0]
    assert rel(fac.eigenvalues[top], g["eig100"][top]) <= 1e-10
    mu = float(g["mu"])
    pre = O.PreconditionerOracle(fac, mu)
    assert rel(pre.apply(g["v"]), g["pinv_v"]) <= 1e-10
    for k in (1, 5, 20):
        rep = O.pcg(O.ShiftedOracle(gop, mu), g["grad"], 1e-300, k, precond=pre)
        assert rel(rep.solution, g[f"pcg{k}_x"]) <= 1e-8
        meta = g[f"pcg{k}_meta"]
        assert rep.iterations == int(meta[0]) and rep.matvecs == int(meta[1])
        assert rep.breakdown == bool(meta[4])


def test_c1_trajectory_fixed_rank(gold):
    g = gold("c1")
    prob, quad, theta = c1_setup()
    cfg = O.NgdConfigOracle(ell0=100, ell_max=100, cg_maxit=20, kappa=1e-300,
                            mu_floor_mode="grad-power", mu_floor_coeff=1e-6,
                            mu_floor_exponent=1.0, iterations=6, seed=0, fixed_rank=True)
    _, recs = O.nystrom_ngd_run(prob, theta, cfg, quad)
    loss = np.array([r.loss for r in recs])
    np.testing.assert_allclose(loss, g["traj_loss"][:6], rtol=1e-6)
    assert [r.pcg_iters for r in recs] == list(g["traj_pcg"][:6].astype(int))
    assert [r.matvecs for r in recs] == list(g["traj_matvecs"][:6].astype(int))


@pytest.mark.parametrize("name,widths,kind,nint,nbnd", [
    ("c2", (2, 64, 64, 64, 1), "sin2d", 4096, 512),
    ("c3_sub", (5, 128, 128, 128, 1), "sinsum", 256, 64),
    ("c5_sub", (10, 256, 256, 256, 256, 1), "gauss", 24, 8),
])
def test_nd_stacks(gold, name, widths, kind, nint, nbnd):
    g = gold(name)
    prob = O.PoissonProblem(widths, kind=kind)
    quad = prob.sample_quadrature(nint, nbnd, 0)
    theta = O.init_theta(widths, 0)
    assert prob.loss_value(theta, quad) == pytest.approx(float(g["loss"]), rel=1e-12)
    assert rel(prob.loss_grad(theta, quad), g["grad"]) <= 1e-12
    gop = O.GramianOracle(prob, theta, quad)
    assert rel(gop.matvec(g["v"]), g["gv"]) <= 1e-12


def test_c4_interior_only(gold):
    g = gold("c4_sub")
    widths = (2, 256, 256, 256, 1)
    prob = O.PoissonProblem(widths, interior_only=True)
    n = g["x"].shape[0]
    quad = O.Quadrature(g["x"], np.full(n, 1.0 / n), np.zeros((0, 2)), np.zeros(0))
    gop = O.GramianOracle(prob, O.init_theta(widths, 0), quad)
    assert rel(gop.matvec(g["v"]), g["gv"]) <= 1e-12


def test_policy_kats():
    # reference KATs (test_optim.py:54-98)
    assert O.adapt_mu(1.0, 1217, 0.0, 0.0, "constant", 0.0, 0.0) == pytest.approx(2.702e-13, rel=1e-3)
    assert O.adapt_mu(1e-10, 100, 1e-2, 0.0, "loss-power", 1e-4, 2.0) == pytest.approx(1e-8, rel=1e-12)
    assert O.adapt_rank(np.array([1.0]), 0.05, 8, 100) == 16
    assert O.adapt_rank(np.array([1.0]), 0.05, 80, 100) == 100
    assert O.adapt_rank(np.array([1.0, 0.5, 1e-6]), 1e-3, 3, 50) == 4
    assert O.adapt_rank(np.full(10, 1.0), 1e-6, 10, 10) == 10
    assert O.Topology((3, 32, 32, 1)).param_count == 1217


def oracle_problem(name, widths):
    if name == "poisson1d":
        return O.PoissonProblem(widths, kind="sin1d")
    if name == "heat1p1d":
        return O.HeatProblem(widths)
    return O.NonlinearPoissonProblem(widths)


PROBLEM_CASES = [("poisson1d", (1, 16, 16, 1), 200, 2, 20),
                 ("heat1p1d", (2, 24, 24, 1), 600, 80, 40),
                 ("nlpoisson2d", (2, 24, 24, 1), 600, 80, 40)]


@pytest.mark.parametrize("name,widths,nint,nbnd,ell", PROBLEM_CASES)
def test_other_problems_stacks(gold, name, widths, nint, nbnd, ell):
    """poisson1d / heat1p1d / nlpoisson2d (problems.py:128-385): stacks, loss, gradient,
    Gramian, the frozen-coefficient metric and H1 error against the live reference."""
    g = gold(name)
    prob = oracle_problem(name, widths)
    quad = prob.sample_quadrature(nint, nbnd, 0)
    theta = O.init_theta(widths, 0)
    assert np.array_equal(theta, g["theta0"])
    assert rel(prob.residual_stack(theta, quad), g["residual"]) <= 1e-13
    assert prob.loss_value(theta, quad) == pytest.approx(float(g["loss"]), rel=1e-13)
    assert rel(prob.metric_stack(theta, quad), g["metric"]) <= 1e-13
    assert rel(prob.loss_grad(theta, quad), g["grad"]) <= 1e-12
    gop = O.GramianOracle(prob, theta, quad)
    assert rel(gop.matvec(g["v"]), g["gv"]) <= 1e-12
    assert rel(gop.matmat(g["omega8"]), g["y8"]) <= 1e-12
    assert prob.h1_relative_error(theta, quad) == pytest.approx(float(g["h1"]), rel=1e-13)
    lin = O.Linearization(prob, g["theta1"], quad, "metric", theta_bar=theta)
    assert rel(lin.value, g["metric_bar"]) <= 1e-13
    assert rel(lin.jvp(g["v"]), g["jvp_bar"]) <= 1e-12


@pytest.mark.parametrize("name,widths,nint,nbnd,ell", PROBLEM_CASES)
def test_other_problems_trajectory(gold, name, widths, nint, nbnd, ell):
    g = gold(name)
    prob = oracle_problem(name, widths)
    quad = prob.sample_quadrature(nint, nbnd, 0)
    theta = O.init_theta(widths, 0)
    cfg = O.NgdConfigOracle(ell0=ell, ell_max=ell, cg_maxit=20, kappa=1e-300, mu_floor_mode="grad-power",
                            mu_floor_coeff=1e-6, mu_floor_exponent=1.0, iterations=4, seed=0, fixed_rank=True)
    _, recs = O.nystrom_ngd_run(prob, theta, cfg, quad)
    np.testing.assert_allclose([r.loss for r in recs], g["traj_loss"][:4], rtol=1e-6)
    assert [r.pcg_iters for r in recs] == list(g["traj_pcg"][:4].astype(int))
