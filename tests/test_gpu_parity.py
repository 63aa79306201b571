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


@pytest.mark.parametrize("svd", [3, 1])
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


def test_c1_trajectory(c1, gold):
    """20-step fixed-rank NGD trajectory vs the reference, judged against the reference's own
    rounding sensitivity: tests/golden/c1_ensemble.npz holds 24 runs of the unmodified reference
    whose Gramian matvec output carries an independent relative 1-ulp perturbation (delta * U(-1, 1),
    make_golden.py case_c1_ensemble).  Where every ensemble run stays within 1e-6 of the reference
    (steps 0-12) the GPU must too (north-star bar); beyond, the GPU must stay within the ensemble's
    largest deviation at that step (x1.5 for the finite ensemble: 24 draws)."""
    G, prob, quad, theta = c1
    E = gold("c1_ensemble")
    cfg = ngd.NystromNgdConfig(ell0=100, ell_max=100, cg_maxit=20, kappa=1e-300, mu_floor_mode="grad-power",
                               mu_floor_coeff=1e-6, mu_floor_exponent=1.0, iterations=20, seed=0, fixed_rank=True)
    _, recs = ngd.nystrom_ngd_run(prob, theta, cfg, quad)
    loss = np.array([r.loss for r in recs])
    ref = G["traj_loss"]
    dev = np.abs(loss - ref) / np.abs(ref)
    ens = np.max(np.abs(E["ens_loss"] - ref) / np.abs(ref), axis=0)
    print("gpu dev", dev, "ensemble max", ens)
    strict = ens <= 1e-6
    assert strict[:13].all(), ens  # the reference itself holds 1e-6 for 13 steps
    assert np.all(dev[strict] <= 1e-6), dev
    assert np.all(dev[~strict] <= 1.5 * ens[~strict]), (dev, ens)
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


# ---------------------------------------------------------------------------
# The benchmarked configurations: the C2 step's pieces on the reference's own
# seeded inputs, and point subsets of >= 1024 points at C3 / C4 / C5 with sketch columns.
# ---------------------------------------------------------------------------


@pytest.fixture(scope="module")
def c2(gold):
    G = gold("c2_step")
    top = ngd.MlpTopology((2, 64, 64, 64, 1))
    prob = ngd.Poisson2D(top)
    quad = prob.sample_quadrature(4096, 512, 0)
    theta = ngd.init(top, 0).values
    return G, prob, quad, theta


def test_c2_factor_preconditioner_pcg(c2):
    """C2 (p = 8577): rank-300 Nystrom factor on host Omega (sketch.py:58-90: the FP32 + FP64 block
    Jacobi path), the step's mu, P^-1 v, and PCG at k = 5 / 20 / 50 (krylov.py:24-88; the reference
    breaks down at 19 iterations) -- same iteration, matvec and breakdown accounting."""
    G, prob, quad, theta = c2
    gop = ngd.GramianOperator.from_problem(prob, theta, quad)
    fac = ngd.nystrom_approximate(gop, 300, seed=11, omega_source="host")
    top = G["eig300"] > 1e-8 * G["eig300"][0]
    assert rel(fac.eig_host[top], G["eig300"][top]) <= 1e-10
    g = prob.loss_grad(theta, quad)
    mu = ngd.adapt_mu(fac.eig_host[0], float(len(theta)), prob.loss_value(theta, quad), float(np.linalg.norm(g)),
                      "grad-power", 1e-6, 1.0)
    assert mu == pytest.approx(float(G["mu"]), rel=1e-10)
    pre = ngd.NystromPreconditioner(fac, float(G["mu"]))
    assert rel(pre.apply(G["v"]), G["pinv_v"]) <= 1e-8
    for k in (5, 20, 50):
        rep = ngd.pcg(ngd.ShiftedOperator(gop, float(G["mu"])), g, 1e-300, k, precond=pre)
        meta = G[f"pcg{k}_meta"]
        assert (rep.iterations, rep.matvecs, rep.breakdown) == (int(meta[0]), int(meta[1]), bool(meta[4])), k
        assert rel(rep.solution, G[f"pcg{k}_x"]) <= 1e-8, k


def test_c2_trajectory(c2):
    """5 fixed-rank NGD steps of the benchmarked C2 configuration (ell = 300, 50 PCG iterations)
    with host Omega: loss and mu within 1e-6.  Every C2 step ends in a PCG breakdown (d.Ad <= 0 once
    the residual reaches rounding level), and WHEN it triggers is itself a rounding event: the
    oracle with a relative 1-ulp perturbation of each matvec stops at 23 / 25 / 28 iterations in
    step 5 (profiles/r02_c2_pcg_breakdown_sensitivity.txt, tools/c2_pcg_sensitivity.py) while its
    loss moves by 2e-10.  So the iteration counts are held to that measured spread (+-5), and the
    matvec totals to the accounting identity of the exit each solve took."""
    G, prob, quad, theta = c2
    cfg = ngd.NystromNgdConfig(ell0=300, ell_max=300, cg_maxit=50, kappa=1e-300, mu_floor_mode="grad-power",
                               mu_floor_coeff=1e-6, mu_floor_exponent=1.0, iterations=5, seed=0, fixed_rank=True)
    reports = []
    theta_f, recs = ngd.nystrom_ngd_run(prob, theta, cfg, quad, step_hook=lambda k, info: reports.append(info["report"]))
    loss = np.array([r.loss for r in recs])
    dev = np.abs(loss - G["traj_loss"]) / np.abs(G["traj_loss"])
    print("c2 trajectory dev", dev)
    assert np.all(dev <= 1e-6), dev
    np.testing.assert_allclose([r.mu for r in recs], G["traj_mu"], rtol=1e-6)
    its = np.array([r.pcg_iters for r in recs])
    print("pcg iterations", its, "reference", G["traj_pcg"])
    assert np.all(np.abs(its - G["traj_pcg"]) <= 5)
    assert np.all(its[:2] == G["traj_pcg"][:2])  # the first steps agree exactly
    per_step = np.diff(np.concatenate([[0], [r.matvecs for r in recs]]))
    # krylov.py:59-88: one matvec per iteration + the final true residual, + the breakdown iteration's own
    # matvec when d.Ad <= 0 ends the loop.  At this point r.z is in the denormal range (measured 1e-310 ..
    # 1e-322), so either d.Ad underflows to 0 first (breakdown) or ||r||^2 does (recurrence residual
    # <= 1e-300, no extra matvec): both are exits of the reference's loop, neither "converged" on the
    # true residual (~2e-16).
    brk = np.array([int(rep.breakdown) for rep in reports])
    assert np.array_equal(per_step, 300 + its + 1 + brk)
    assert not any(rep.converged for rep in reports)


def _omega8(p):
    return np.linalg.qr(np.random.default_rng(123).standard_normal((p, 8)), mode="reduced")[0]


@pytest.mark.parametrize("name,widths,kind", [("c3_1k", (5, 128, 128, 128, 1), "sinsum"),
                                              ("c5_1k", (10, 256, 256, 256, 256, 1), "gauss")])
def test_nd_1k_subsets_with_sketch_columns(gold, name, widths, kind):
    """1024 + 256 points of C3 / C5 (the full configs' samplers, first points): loss, metric,
    gradient, Gv and 8 sketch columns Y = G Omega (the J-chunk DMMA GEMM path) vs the reference."""
    G = gold(name)
    top = ngd.MlpTopology(widths)
    prob = ngd.PoissonND(top, kind)
    quad = prob.sample_quadrature(1024, 256, 0)
    theta = ngd.init(top, 0).values
    p = len(theta)
    assert prob.loss_value(theta, quad) == pytest.approx(float(G["loss"]), rel=1e-12)
    assert rel(prob.metric_stack(theta, None, quad), G["metric"]) <= 1e-12
    assert rel(prob.loss_grad(theta, quad), G["grad"]) <= 1e-10
    gop = ngd.GramianOperator.from_problem(prob, theta, quad)
    assert rel(gop.matvec(np.random.default_rng(1).standard_normal(p)), G["gv"]) <= 1e-10
    assert rel(gop.matmat(_omega8(p)), G["y8"]) <= 1e-10


def test_c4_1k_with_sketch_columns(gold):
    G = gold("c4_1k")
    top = ngd.MlpTopology((2, 256, 256, 256, 1))
    prob = ngd.LaplacianStack(top)
    n = G["x"].shape[0]
    quad = ngd.QuadratureSet(G["x"], np.full(n, 1.0 / n), np.zeros((0, 2)), np.zeros(0))
    theta = ngd.init(top, 0).values
    p = len(theta)
    gop = ngd.GramianOperator.from_problem(prob, theta, quad)
    assert rel(gop.matvec(np.random.default_rng(1).standard_normal(p)), G["gv"]) <= 1e-10
    assert rel(gop.matmat(_omega8(p)), G["y8"]) <= 1e-10
