"""The reference's other problems on the CUDA path: poisson1d,
heat1p1d (per-coordinate u_t - u_xx head, bulk and initial blocks, metric and
residual stacks with different rows) and nlpoisson2d (frozen 3 ubar^2
coefficient -- the stop-gradient path of autodiff.py:521-527).

Pinned against fixtures from the live reference (tests/golden/make_golden.py)
and, at larger sizes, against the CPU oracle.  Tolerances as test_gpu_parity."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ngd = pytest.importorskip("paper_2505_11638_b200")

from oracle import ngd_oracle as O  # noqa: E402

CASES = [("poisson1d", (1, 16, 16, 1), 200, 2, 20),
         ("heat1p1d", (2, 24, 24, 1), 600, 80, 40),
         ("nlpoisson2d", (2, 24, 24, 1), 600, 80, 40)]


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def setup(name, widths, nint, nbnd):
    top = ngd.MlpTopology(widths)
    prob = ngd.make_problem(name, topology=top)
    quad = prob.sample_quadrature(nint, nbnd, 0)
    theta = ngd.init(top, 0).values
    return prob, quad, theta


def oracle_problem(name, widths):
    if name == "poisson1d":
        return O.PoissonProblem(widths, kind="sin1d")
    if name == "heat1p1d":
        return O.HeatProblem(widths)
    return O.NonlinearPoissonProblem(widths)


@pytest.mark.parametrize("name,widths,nint,nbnd,ell", CASES)
def test_stacks_loss_grad_gramian(gold, name, widths, nint, nbnd, ell):
    G = gold(name)
    prob, quad, theta = setup(name, widths, nint, nbnd)
    assert np.array_equal(theta, G["theta0"])
    assert prob.loss_value(theta, quad) == pytest.approx(float(G["loss"]), rel=1e-12)
    assert rel(prob.residual_stack(theta, quad), G["residual"]) <= 1e-12
    assert rel(prob.metric_stack(theta, theta, quad), G["metric"]) <= 1e-12
    assert rel(prob.loss_grad(theta, quad), G["grad"]) <= 1e-10
    gop = ngd.GramianOperator.from_problem(prob, theta, quad)
    assert rel(gop.matvec(G["v"]), G["gv"]) <= 1e-10
    assert rel(gop.matmat(G["omega8"]), G["y8"]) <= 1e-10
    assert prob.h1_relative_error(theta, quad) == pytest.approx(float(G["h1"]), rel=1e-12)


@pytest.mark.parametrize("name,widths,nint,nbnd,ell", CASES)
def test_frozen_metric(gold, name, widths, nint, nbnd, ell):
    """metric_stack(theta1, freeze(theta0)) and its JVP (gramian.py:36-40)."""
    G = gold(name)
    prob, quad, theta = setup(name, widths, nint, nbnd)
    theta1 = G["theta1"]
    assert rel(prob.metric_stack(theta1, theta, quad), G["metric_bar"]) <= 1e-12
    # JVP of the frozen-coefficient metric map through the C-ABI
    from paper_2505_11638_b200 import _lib

    torch = _lib.torch_mod()
    ctx = prob.context(quad)
    rows = prob._rows(quad)
    n = len(rows.x_int) + len(rows.x_val)
    loss = _lib.ctypes.c_double()
    t1, t0 = _lib.to_device(theta1), _lib.to_device(theta)
    ctx.call("ngd_linearize_ex", _lib.ptr(t1), _lib.ptr(t0), _lib.ctypes.byref(loss), None, None)
    out = torch.empty(n, dtype=torch.float64, device=ctx.device)
    ctx.call("ngd_jvp", _lib.ptr(_lib.to_device(G["v"])), _lib.ptr(out))
    jv = out.cpu().numpy()
    if rows.metric_index is not None:
        jv = jv[rows.metric_index]
    assert rel(jv, G["jvp_bar"]) <= 1e-10
    # a frozen linearisation cannot serve the gradient (residual Jacobian is at theta)
    g = torch.empty(ctx.p, dtype=torch.float64, device=ctx.device)
    if name == "nlpoisson2d":
        with pytest.raises(RuntimeError):
            ctx.call("ngd_loss_grad", _lib.ptr(g))
    ctx.lin_owner = None


def test_frozen_coefficient_is_load_bearing():
    """Negative control (reference test_problems.py:85-91): freezing ubar at a different
    point changes the nonlinear metric; for the linear problems it does not."""
    prob, quad, theta = setup("nlpoisson2d", (2, 8, 1), 40, 12)
    theta1 = theta + 0.3 * np.random.default_rng(0).standard_normal(theta.size)
    a = prob.metric_stack(theta1, theta, quad)
    b = prob.metric_stack(theta1, theta1, quad)
    assert not np.allclose(a, b, rtol=1e-6)
    hp, hq, ht = setup("heat1p1d", (2, 8, 1), 40, 12)
    ht1 = ht + 0.3 * np.random.default_rng(0).standard_normal(ht.size)
    assert np.array_equal(hp.metric_stack(ht1, ht, hq), hp.metric_stack(ht1, ht1, hq))


def test_nonlinear_metric_at_zero_net_is_laplacian():
    """reference test_problems.py:76-83"""
    prob, quad, _ = setup("nlpoisson2d", (2, 5, 5, 1), 30, 12)
    lin = ngd.make_problem("poisson2d", topology=prob.topology)
    theta = np.zeros(prob.topology.param_count)
    np.testing.assert_allclose(prob.metric_stack(theta, theta, quad), lin.metric_stack(theta, theta, quad),
                               atol=1e-15)


@pytest.mark.parametrize("name,widths,nint,nbnd,ell", CASES)
def test_trajectory(gold, name, widths, nint, nbnd, ell):
    G = gold(name)
    prob, quad, theta = setup(name, widths, nint, nbnd)
    cfg = ngd.NystromNgdConfig(ell0=ell, ell_max=ell, cg_maxit=20, kappa=1e-300, mu_floor_mode="grad-power",
                               mu_floor_coeff=1e-6, mu_floor_exponent=1.0, iterations=6, seed=0, fixed_rank=True)
    _, recs = ngd.nystrom_ngd_run(prob, theta, cfg, quad)
    loss = np.array([r.loss for r in recs])
    np.testing.assert_allclose(loss[:4], G["traj_loss"][:4], rtol=1e-6)
    # kappa = 1e-300 makes the PCG tolerance unreachable: a solve ends at cg_maxit or one step
    # earlier when the search direction's curvature d.Ad rounds to <= 0 (breakdown at machine
    # precision, krylov.py:59-66) -- a rounding-level event, so the count may differ by one
    ours, ref = [r.pcg_iters for r in recs[:4]], G["traj_pcg"][:4].astype(int)
    assert all(abs(a - b) <= 1 for a, b in zip(ours, ref)), (ours, list(ref))
    assert np.all(np.isfinite(loss)) and loss[-1] < loss[0]


@pytest.mark.parametrize("name", ["heat1p1d", "nlpoisson2d"])
def test_larger_vs_oracle(name):
    """C2-sized network and quadrature: stacks, gradient, Gramian matvec and a sketch
    block against the oracle (the fixtures above are small)."""
    widths = (2, 64, 64, 64, 1)
    prob, quad, theta = setup(name, widths, 4096, 512)
    theta = theta + 0.1 * np.random.default_rng(5).standard_normal(theta.size)
    op = oracle_problem(name, widths)
    oq = op.sample_quadrature(4096, 512, 0)
    assert np.array_equal(oq.interior_points, quad.interior_points)
    assert prob.loss_value(theta, quad) == pytest.approx(op.loss_value(theta, oq), rel=1e-12)
    assert rel(prob.loss_grad(theta, quad), op.loss_grad(theta, oq)) <= 1e-10
    v = np.random.default_rng(1).standard_normal(theta.size)
    gop = ngd.GramianOperator.from_problem(prob, theta, quad)
    ogop = O.GramianOracle(op, theta, oq)
    assert rel(gop.matvec(v), ogop.matvec(v)) <= 1e-10
    om = np.linalg.qr(np.random.default_rng(2).standard_normal((theta.size, 4)))[0]
    assert rel(gop.matmat(om), ogop.matmat(om)) <= 1e-10
    # symmetry and PSD of the device Gramian
    u = np.random.default_rng(3).standard_normal(theta.size)
    gu, gv = gop.matvec(u), gop.matvec(v)
    assert abs(v @ gu - u @ gv) <= 1e-11 * np.linalg.norm(gu) * np.linalg.norm(v)
    assert v @ gv >= 0.0
