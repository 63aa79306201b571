"""Generate the golden fixtures in tests/golden/ by running the LIVE reference.

Run in the build container (the only place /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src:/root/repo python tests/golden/make_golden.py

Inputs (theta0, quadrature points, probe vectors, Omega seeds) are seeded and
reproducible by ``oracle.ngd_oracle``; the *outputs* stored here come from the
unmodified reference package (``nystromngd``), so the fixtures pin both the
oracle and the CUDA path.  The N-D Poisson problems of BASELINE C3/C5 do not
exist in the reference; they are defined here by subclassing the
reference's ``Poisson1D`` exactly as SURVEY 7.1 step 0 prescribes, and the
interior-only microbench (C4) uses the reference's ``GramianOperator.from_stack``.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from nystromngd import gramian, krylov, model, optim, problems, sketch  # noqa: E402
from nystromngd import autodiff as ad  # noqa: E402

from oracle import ngd_oracle as O  # noqa: E402  (inputs only: points, boundary sampler)


class PoissonND(problems.Poisson1D):
    """Reference-side N-D Poisson (subclass of problems.Poisson1D)."""

    def __init__(self, topology, kind):
        self.input_dim = topology.input_dim
        self.kind = kind
        self._o = O.PoissonProblem(topology.widths, kind=kind)
        super().__init__(topology)

    def exact(self, x):
        return self._o.exact(x)

    def exact_grad(self, x):
        return self._o.exact_grad(x)

    def exact_laplacian(self, x):
        return -self._o.source(x)

    def source(self, x):
        return self._o.source(x)

    def dirichlet(self, x):
        return self._o.exact(x)

    def sample_quadrature(self, n_interior, n_boundary, seed):
        q = self._o.sample_quadrature(n_interior, n_boundary, seed)
        return problems.QuadratureSet(q.interior_points, q.interior_weights, q.boundary_points, q.boundary_weights)


def _basic(prob, theta, quad, v):
    gop = gramian.GramianOperator.from_problem(prob, theta, quad)
    frozen = ad.freeze(theta)
    return {
        "loss": np.array(prob.loss_value(theta, quad)),
        "grad": prob.loss_grad(theta, quad),
        "metric": np.asarray(ad.primal_value(prob.metric_stack(theta, frozen, quad))),
        "v": v,
        "gv": gop.matvec(v),
    }


def case_c1():
    widths = (2, 32, 32, 1)
    prob = problems.make_problem("poisson2d", topology=model.MlpTopology(widths))
    quad = prob.sample_quadrature(900, 120, 0)
    theta = model.init(prob.topology, 0).values
    p = theta.shape[0]
    out = _basic(prob, theta, quad, np.random.default_rng(1).standard_normal(p))
    out["theta0"] = theta
    gop = gramian.GramianOperator.from_problem(prob, theta, quad)
    # sketch block on a fixed post-QR Omega (compare Y on the same Omega)
    omega, _ = np.linalg.qr(np.random.default_rng(123).standard_normal((p, 8)), mode="reduced")
    out["omega8"] = omega
    out["y8"] = gop.matmat(omega)
    # full Nystrom factor at rank 100, preconditioner, PCG at a fixed iteration count
    factor = sketch.nystrom_approximate(gop, 100, seed=7)
    mu = 1e-4
    pre = sketch.NystromPreconditioner(factor, mu)
    out["eig100"] = factor.eigenvalues
    out["mu"] = np.array(mu)
    out["pinv_v"] = pre.apply(out["v"])
    g = out["grad"]
    for k in (1, 5, 20):
        rep = krylov.pcg(gramian.ShiftedOperator(gop, mu), g, 1e-300, k, precond=pre)
        out[f"pcg{k}_x"] = rep.solution
        out[f"pcg{k}_meta"] = np.array([rep.iterations, rep.matvecs, rep.relative_residual, rep.converged, rep.breakdown], dtype=float)
    # 20-step NGD loss trajectory, fixed rank 100
    cfg = optim.NystromNgdConfig(ell0=100, ell_max=100, cg_maxit=20, kappa=1e-300,
                                 mu_floor_mode="grad-power", mu_floor_coeff=1e-6,
                                 mu_floor_exponent=1.0, iterations=20, seed=0)
    saved = optim.adapt_rank
    optim.adapt_rank = lambda eigenvalues, mu, ell, ell_max, ratio=10.0: ell
    try:
        t0 = time.time()
        theta_f, recs = optim.nystrom_ngd_run(prob, theta, cfg, quad)
        print(f"  c1 20 NGD steps in {time.time() - t0:.1f}s")
    finally:
        optim.adapt_rank = saved
    out["traj_loss"] = np.array([r.loss for r in recs])
    out["traj_mu"] = np.array([r.mu for r in recs])
    out["traj_pcg"] = np.array([r.pcg_iters for r in recs])
    out["traj_matvecs"] = np.array([r.matvecs for r in recs])
    out["traj_theta"] = theta_f
    # adaptive-rank trajectory (default policy), 8 steps, small ell0
    cfg2 = optim.NystromNgdConfig(ell0=10, ell_max=100, cg_maxit=20, iterations=8, seed=3)
    _, recs2 = optim.nystrom_ngd_run(prob, theta, cfg2, quad)
    out["adapt_loss"] = np.array([r.loss for r in recs2])
    out["adapt_ell"] = np.array([r.ell for r in recs2])
    out["adapt_mu"] = np.array([r.mu for r in recs2])
    out["adapt_pcg"] = np.array([r.pcg_iters for r in recs2])
    out["adapt_matvecs"] = np.array([r.matvecs for r in recs2])
    return out


def case_c2():
    widths = (2, 64, 64, 64, 1)
    prob = problems.make_problem("poisson2d", topology=model.MlpTopology(widths))
    quad = prob.sample_quadrature(4096, 512, 0)
    theta = model.init(prob.topology, 0).values
    out = _basic(prob, theta, quad, np.random.default_rng(1).standard_normal(theta.shape[0]))
    return out


def case_nd(widths, kind, n_int, n_bnd):
    top = model.MlpTopology(widths)
    prob = PoissonND(top, kind)
    quad = prob.sample_quadrature(n_int, n_bnd, 0)
    theta = model.init(top, 0).values
    return _basic(prob, theta, quad, np.random.default_rng(1).standard_normal(theta.shape[0]))


def case_c4(n):
    widths = (2, 256, 256, 256, 1)
    top = model.MlpTopology(widths)
    x = np.random.default_rng(0).random((n, 2))
    w = np.full(n, 1.0 / n)
    theta = model.init(top, 0).values
    stack = lambda th: model.input_derivatives(top, th, x)[2]
    gop = gramian.GramianOperator.from_stack(stack, theta, w)
    v = np.random.default_rng(1).standard_normal(theta.shape[0])
    return {"x": x, "v": v, "gv": gop.matvec(v)}


def _traj(prob, theta, quad, iterations, ell, seed):
    """Fixed-rank NGD trajectory (adapt_rank patched out, as in case_c1)."""
    cfg = optim.NystromNgdConfig(ell0=ell, ell_max=ell, cg_maxit=20, kappa=1e-300,
                                 mu_floor_mode="grad-power", mu_floor_coeff=1e-6,
                                 mu_floor_exponent=1.0, iterations=iterations, seed=seed)
    saved = optim.adapt_rank
    optim.adapt_rank = lambda eigenvalues, mu, ell, ell_max, ratio=10.0: ell
    try:
        theta_f, recs = optim.nystrom_ngd_run(prob, theta, cfg, quad)
    finally:
        optim.adapt_rank = saved
    return {"traj_loss": np.array([r.loss for r in recs]), "traj_pcg": np.array([r.pcg_iters for r in recs]),
            "traj_matvecs": np.array([r.matvecs for r in recs]), "traj_mu": np.array([r.mu for r in recs])}


def case_problem(name, widths, n_int, n_bnd, ell):
    """The reference's other problems (problems.py:128-385) at a small size."""
    prob = problems.make_problem(name, topology=model.MlpTopology(widths))
    quad = prob.sample_quadrature(n_int, n_bnd, 0)
    theta = model.init(prob.topology, 0).values
    p = theta.shape[0]
    out = _basic(prob, theta, quad, np.random.default_rng(1).standard_normal(p))
    out["theta0"] = theta
    out["residual"] = np.asarray(ad.primal_value(prob.residual_stack(theta, quad)))
    out["h1"] = np.array(prob.h1_relative_error(theta, quad))
    # metric frozen at theta_bar != theta (the stop-gradient path, autodiff.py:521-527)
    theta1 = theta + 0.05 * np.random.default_rng(2).standard_normal(p)
    out["theta1"] = theta1
    out["metric_bar"] = np.asarray(ad.primal_value(prob.metric_stack(theta1, ad.freeze(theta), quad)))
    lin = ad.linearize(lambda th: prob.metric_stack(th, ad.freeze(theta), quad), theta1)
    out["jvp_bar"] = lin.jvp(out["v"])
    omega, _ = np.linalg.qr(np.random.default_rng(123).standard_normal((p, 8)), mode="reduced")
    gop = gramian.GramianOperator.from_problem(prob, theta, quad)
    out["omega8"] = omega
    out["y8"] = gop.matmat(omega)
    t0 = time.time()
    out.update(_traj(prob, theta, quad, 6, ell, 0))
    print(f"  {name} 6 NGD steps in {time.time() - t0:.1f}s")
    return out


def case_baselines():
    """The reference's baseline optimizers (optim.py:273-455) and spectrum (harness.py:237-266)."""
    from nystromngd import harness
    widths = (2, 8, 8, 1)
    prob = problems.make_problem("poisson2d", topology=model.MlpTopology(widths))
    quad = prob.sample_quadrature(200, 40, 0)
    theta = model.init(prob.topology, 0).values
    cfg = optim.NystromNgdConfig(ell0=10, ell_max=40, cg_maxit=20, iterations=4, seed=0)
    out = {"theta0": theta}
    for name in ("ngd_cg", "ngd_dense", "gd", "bfgs"):
        _, recs = optim.run_optimizer(name, prob, theta, cfg, quad, quad_eval=quad)
        out[f"{name}_loss"] = np.array([r.loss for r in recs])
        out[f"{name}_h1"] = np.array([r.h1_rel_error for r in recs])
        out[f"{name}_mu"] = np.array([r.mu for r in recs])
        out[f"{name}_pcg"] = np.array([r.pcg_iters for r in recs])
        out[f"{name}_matvecs"] = np.array([r.matvecs for r in recs])
    out["spectrum"] = harness.gramian_spectrum(prob, theta, quad, top=30)
    return out


def case_c2_step():
    """C2 full step pieces on the benchmarked shapes: the rank-300 Nystrom factor
    on host Omega (sketch.py:58-90), the step's mu (optim.py:86-103), P^-1 v (sketch.py:101-112),
    PCG iterates at k = 5/20/50 (krylov.py:24-88) and a 5-step fixed-rank trajectory
    (optim.py:188-270) with the bench config (ell = 300, 50 PCG iterations)."""
    widths = (2, 64, 64, 64, 1)
    prob = problems.make_problem("poisson2d", topology=model.MlpTopology(widths))
    quad = prob.sample_quadrature(4096, 512, 0)
    theta = model.init(prob.topology, 0).values
    p = theta.shape[0]
    out = {"v": np.random.default_rng(1).standard_normal(p)}
    loss = prob.loss_value(theta, quad)
    g = prob.loss_grad(theta, quad)
    gop = gramian.GramianOperator.from_problem(prob, theta, quad)
    t0 = time.time()
    factor = sketch.nystrom_approximate(gop, 300, seed=11)
    print(f"  c2 rank-300 sketch in {time.time() - t0:.1f}s")
    mu = optim.adapt_mu(factor.eigenvalues[0], float(p), loss, float(np.linalg.norm(g)), "grad-power", 1e-6, 1.0)
    pre = sketch.NystromPreconditioner(factor, mu)
    out["eig300"] = factor.eigenvalues
    out["mu"] = np.array(mu)
    out["pinv_v"] = pre.apply(out["v"])
    for k in (5, 20, 50):
        rep = krylov.pcg(gramian.ShiftedOperator(gop, mu), g, 1e-300, k, precond=pre)
        out[f"pcg{k}_x"] = rep.solution
        out[f"pcg{k}_meta"] = np.array([rep.iterations, rep.matvecs, rep.relative_residual, rep.converged,
                                        rep.breakdown], dtype=float)
    cfg = optim.NystromNgdConfig(ell0=300, ell_max=300, cg_maxit=50, kappa=1e-300,
                                 mu_floor_mode="grad-power", mu_floor_coeff=1e-6,
                                 mu_floor_exponent=1.0, iterations=5, seed=0)
    saved = optim.adapt_rank
    optim.adapt_rank = lambda eigenvalues, mu, ell, ell_max, ratio=10.0: ell
    try:
        t0 = time.time()
        theta_f, recs = optim.nystrom_ngd_run(prob, theta, cfg, quad)
        print(f"  c2 5 NGD steps in {time.time() - t0:.1f}s")
    finally:
        optim.adapt_rank = saved
    out["traj_loss"] = np.array([r.loss for r in recs])
    out["traj_mu"] = np.array([r.mu for r in recs])
    out["traj_pcg"] = np.array([r.pcg_iters for r in recs])
    out["traj_matvecs"] = np.array([r.matvecs for r in recs])
    out["traj_theta"] = theta_f
    return out


def case_c1_ensemble(k_runs=24, delta=2.220446049250313e-16):
    """Rounding sensitivity of the reference's own 20-step C1 trajectory:
    k_runs runs of the unmodified nystrom_ngd_run whose Gramian matvec output is perturbed
    elementwise by a relative delta * U(-1, 1) (about one ulp, independent draws per run).
    The spread of these runs is the parity envelope of any correct reimplementation."""
    widths = (2, 32, 32, 1)
    prob = problems.make_problem("poisson2d", topology=model.MlpTopology(widths))
    quad = prob.sample_quadrature(900, 120, 0)
    theta = model.init(prob.topology, 0).values
    cfg = optim.NystromNgdConfig(ell0=100, ell_max=100, cg_maxit=20, kappa=1e-300,
                                 mu_floor_mode="grad-power", mu_floor_coeff=1e-6,
                                 mu_floor_exponent=1.0, iterations=20, seed=0)
    orig_mv = gramian.GramianOperator.matvec
    saved = optim.adapt_rank
    optim.adapt_rank = lambda eigenvalues, mu, ell, ell_max, ratio=10.0: ell
    losses, pcgs = [], []
    try:
        for run in range(k_runs):
            prng = np.random.default_rng(1000 + run)

            def mv(self, v, _prng=prng):
                y = orig_mv(self, v)
                return y * (1.0 + delta * _prng.uniform(-1.0, 1.0, y.shape))

            gramian.GramianOperator.matvec = mv
            t0 = time.time()
            _, recs = optim.nystrom_ngd_run(prob, theta, cfg, quad)
            print(f"  ensemble run {run}: {time.time() - t0:.1f}s")
            losses.append([r.loss for r in recs])
            pcgs.append([r.pcg_iters for r in recs])
    finally:
        gramian.GramianOperator.matvec = orig_mv
        optim.adapt_rank = saved
    return {"ens_loss": np.array(losses), "ens_pcg": np.array(pcgs), "delta": np.array(delta)}


def case_nd_sketch(widths, kind, n_int, n_bnd):
    """Point subsets of C3 / C5 with >= 1024 points: loss, grad, matvec and 8 sketch columns on a
    fixed post-QR Omega (gramian.py:48-61)."""
    top = model.MlpTopology(widths)
    prob = PoissonND(top, kind)
    quad = prob.sample_quadrature(n_int, n_bnd, 0)
    theta = model.init(top, 0).values
    p = theta.shape[0]
    out = _basic(prob, theta, quad, np.random.default_rng(1).standard_normal(p))
    gop = gramian.GramianOperator.from_problem(prob, theta, quad)
    omega, _ = np.linalg.qr(np.random.default_rng(123).standard_normal((p, 8)), mode="reduced")
    out["y8"] = gop.matmat(omega)
    del out["v"]  # regenerated by the tests from the seeds (default_rng(1), default_rng(123) + QR)
    return out


def case_c4_sketch(n):
    """C4 microbench on n points: matvec + 8 sketch columns on a fixed post-QR Omega."""
    widths = (2, 256, 256, 256, 1)
    top = model.MlpTopology(widths)
    x = np.random.default_rng(0).random((n, 2))
    w = np.full(n, 1.0 / n)
    theta = model.init(top, 0).values
    p = theta.shape[0]
    stack = lambda th: model.input_derivatives(top, th, x)[2]
    gop = gramian.GramianOperator.from_stack(stack, theta, w)
    v = np.random.default_rng(1).standard_normal(p)
    omega, _ = np.linalg.qr(np.random.default_rng(123).standard_normal((p, 8)), mode="reduced")
    return {"x": x, "gv": gop.matvec(v), "y8": gop.matmat(omega)}  # v, omega: regenerated from the seeds


def main():
    cases = {
        "c1": case_c1,
        "c2": case_c2,
        "c3_sub": lambda: case_nd((5, 128, 128, 128, 1), "sinsum", 256, 64),
        "c5_sub": lambda: case_nd((10, 256, 256, 256, 256, 1), "gauss", 24, 8),
        "c4_sub": lambda: case_c4(96),
        "poisson1d": lambda: case_problem("poisson1d", (1, 16, 16, 1), 200, 2, 20),
        "heat1p1d": lambda: case_problem("heat1p1d", (2, 24, 24, 1), 600, 80, 40),
        "nlpoisson2d": lambda: case_problem("nlpoisson2d", (2, 24, 24, 1), 600, 80, 40),
        "baselines": case_baselines,
        "c2_step": case_c2_step,
        "c1_ensemble": case_c1_ensemble,
        "c3_1k": lambda: case_nd_sketch((5, 128, 128, 128, 1), "sinsum", 1024, 256),
        "c5_1k": lambda: case_nd_sketch((10, 256, 256, 256, 256, 1), "gauss", 1024, 256),
        "c4_1k": lambda: case_c4_sketch(1024),
    }
    default_skip = {"baselines"}  # out-of-scope baselines (removed in round 2); run explicitly if needed
    only = sys.argv[1:]
    for name, fn in cases.items():
        if only and name not in only:
            continue
        if not only and name in default_skip:
            continue
        t0 = time.time()
        data = fn()
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **data)
        print(f"{name}: {time.time() - t0:.1f}s -> {path} ({os.path.getsize(path) / 1e6:.2f} MB)")


if __name__ == "__main__":
    main()
