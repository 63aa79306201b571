"""Size-independent properties at the BASELINE configs' FULL sizes (GPU), plus
the reference's own operator / sketch / PCG known-answer tests run against the
CUDA path (test_gramian.py, test_sketch.py, test_krylov.py)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ngd = pytest.importorskip("paper_2505_11638_b200")
torch = pytest.importorskip("torch")

from oracle import ngd_oracle as O  # noqa: E402

CONFIGS = {
    "c1": ((2, 32, 32, 1), "sin2d", 900, 120),
    "c2": ((2, 64, 64, 64, 1), "sin2d", 4096, 512),
    "c3": ((5, 128, 128, 128, 1), "sinsum", 16384, 4096),
    "c4": ((2, 256, 256, 256, 1), "lap", 65536, 0),
    "c5": ((10, 256, 256, 256, 256, 1), "gauss", 131072, 16384),
}


def make(name):
    widths, kind, nint, nbnd = CONFIGS[name]
    top = ngd.MlpTopology(widths)
    if kind == "sin2d":
        prob = ngd.Poisson2D(top)
    elif kind == "lap":
        prob = ngd.LaplacianStack(top)
    else:
        prob = ngd.PoissonND(top, kind)
    quad = prob.sample_quadrature(nint, nbnd, 0)
    return prob, quad, ngd.init(top, 0).values


def dev(x):
    return torch.as_tensor(x, dtype=torch.float64, device="cuda")


@pytest.mark.parametrize("name", ["c2", "c3", "c4", "c5"])
def test_full_size_operator_properties(name):
    prob, quad, theta = make(name)
    gop = ngd.GramianOperator.from_problem(prob, theta, quad)
    p = gop.dim
    rng = np.random.default_rng(5)
    u, v = dev(rng.standard_normal(p)), dev(rng.standard_normal(p))
    gu, gv = gop.matvec(u), gop.matvec(v)
    # symmetry and positive semidefiniteness
    assert abs(float(u @ gv) - float(v @ gu)) <= 1e-12 * float(torch.linalg.norm(gu) * torch.linalg.norm(v))
    assert float(v @ gv) >= 0.0
    # linearity
    g2 = gop.matvec(2.5 * u - 0.5 * v)
    assert float(torch.linalg.norm(g2 - (2.5 * gu - 0.5 * gv))) <= 1e-12 * float(torch.linalg.norm(g2))
    # matmat columns == matvecs (two formulations: factored jets vs explicit J chunks)
    Y = gop.matmat(torch.stack([u, v], dim=1))
    assert float(torch.linalg.norm(Y[:, 0] - gu)) <= 1e-10 * float(torch.linalg.norm(gu))
    assert float(torch.linalg.norm(Y[:, 1] - gv)) <= 1e-10 * float(torch.linalg.norm(gv))
    # bitwise determinism
    assert torch.equal(gop.matvec(v), gv)
    # zero vector
    assert float(torch.linalg.norm(gop.matvec(torch.zeros_like(v)))) == 0.0


@pytest.mark.parametrize("name", ["c4", "c5"])
def test_back_to_back_matvecs_are_bitwise_reproducible(name):
    """Matvecs enqueued back to back (no host synchronisation in between) against results made in isolation.
    The warp-specialised phase kernels refill a ring slot the moment its last consumer warp has released
    it; without the consumers' fence.proxy.async ahead of the release one 16-column box of the C5 phase A
    was stale in ~10% of the launches (tools/ws_stress.py; csrc/ngd_phag.cu)."""
    prob, quad, theta = make(name)
    gop = ngd.GramianOperator.from_problem(prob, theta, quad)
    p = gop.dim
    rng = np.random.default_rng(7)
    u, v = dev(rng.standard_normal(p)), dev(rng.standard_normal(p))
    torch.cuda.synchronize()
    gu = gop.matvec(u).clone()
    torch.cuda.synchronize()
    gv = gop.matvec(v).clone()
    torch.cuda.synchronize()
    reps = 20 if name == "c5" else 40
    outs = []
    for _ in range(reps):
        outs.append((gop.matvec(u), gop.matvec(v)))
    torch.cuda.synchronize()
    for k, (a, b) in enumerate(outs):
        assert torch.equal(a, gu), f"repeat {k}: matvec(u) differs"
        assert torch.equal(b, gv), f"repeat {k}: matvec(v) differs"


@pytest.mark.parametrize("name", ["c3", "c5"])
def test_point_subset_against_oracle(name):
    """Gv is a sum of per-point terms: a point subset is an exact oracle."""
    widths, kind, nint, nbnd = CONFIGS[name]
    prob, quad, theta = make(name)
    sub = ngd.QuadratureSet(quad.interior_points[:40], quad.interior_weights[:40], quad.boundary_points[:16],
                            quad.boundary_weights[:16])
    oprob = O.PoissonProblem(widths, kind=kind)
    oq = O.Quadrature(sub.interior_points, sub.interior_weights, sub.boundary_points, sub.boundary_weights)
    v = np.random.default_rng(9).standard_normal(len(theta))
    want = O.GramianOracle(oprob, theta, oq).matvec(v)
    got = ngd.GramianOperator.from_problem(prob, theta, sub).matvec(v)
    assert np.linalg.norm(got - want) <= 1e-10 * np.linalg.norm(want)
    assert prob.loss_value(theta, sub) == pytest.approx(oprob.loss_value(theta, oq), rel=1e-12)


@pytest.mark.parametrize("name,ncols", [("c3", 8), ("c4", 4), ("c5", 2)])
def test_full_size_against_oracle(name, ncols):
    """FULL-size C3 / C4 / C5 (20480 / 65536 / 147456 points): Gv and sketch columns Y = G Omega
    against the CPU oracle on the GPU box's host cores -- the large-N phase-B split plans, the
    reductions and the J-chunk DMMA GEMMs (several chunks at C5) at the benchmarked sizes."""
    import os

    import psutil

    widths, kind, nint, nbnd = CONFIGS[name]
    need_gb = {"c3": 4, "c4": 24, "c5": 64}[name]  # oracle linearisation (jets + adjoints) + temporaries
    if psutil.virtual_memory().available < need_gb * (1 << 30):
        pytest.skip(f"oracle at full {name} needs ~{need_gb} GB of host memory")
    prob, quad, theta = make(name)
    p = len(theta)
    okind = "sin2d" if kind == "lap" else kind
    oprob = O.PoissonProblem(widths, kind=okind, interior_only=(kind == "lap"))
    oq = O.Quadrature(quad.interior_points, quad.interior_weights, quad.boundary_points, quad.boundary_weights)
    v = np.random.default_rng(9).standard_normal(p)
    om = np.linalg.qr(np.random.default_rng(10).standard_normal((p, ncols)), mode="reduced")[0]
    gop = ngd.GramianOperator.from_problem(prob, theta, quad)
    got_v, got_y = gop.matvec(v), gop.matmat(om)
    ogop = O.GramianOracle(oprob, theta, oq)
    want_v = ogop.matvec(v)
    want_y = ogop.matmat(om)
    print(f"{name}: host cores {os.cpu_count()}")
    assert np.linalg.norm(got_v - want_v) <= 1e-10 * np.linalg.norm(want_v)
    for j in range(ncols):
        assert np.linalg.norm(got_y[:, j] - want_y[:, j]) <= 1e-10 * np.linalg.norm(want_y[:, j]), j


def test_shard_additivity():
    """Sum of per-shard Gramians == full Gramian (the multi-GPU reduction identity)."""
    prob, quad, theta = make("c2")
    v = np.random.default_rng(2).standard_normal(len(theta))
    full = ngd.GramianOperator.from_problem(prob, theta, quad).matvec(v)
    from paper_2505_11638_b200.distributed import shard_slices

    acc = np.zeros_like(full)
    for r in range(4):
        si, sb = shard_slices(len(quad.interior_points), len(quad.boundary_points), r, 4)
        q = ngd.QuadratureSet(quad.interior_points[si], quad.interior_weights[si], quad.boundary_points[sb],
                              quad.boundary_weights[sb])
        p2 = ngd.Poisson2D(prob.topology)
        acc += ngd.GramianOperator.from_problem(p2, theta, q).matvec(v)
    assert np.linalg.norm(acc - full) <= 1e-13 * np.linalg.norm(full)


def test_ragged_and_tiny_point_sets():
    top = ngd.MlpTopology((2, 8, 8, 1))
    prob = ngd.Poisson2D(top)
    theta = ngd.init(top, 1).values
    oprob = O.PoissonProblem((2, 8, 8, 1))
    rng = np.random.default_rng(4)
    for nint, nbnd in ((1, 0), (0, 1), (17, 3), (33, 31)):
        bnd = rng.random((nbnd, 2))
        bnd[:, 0] = np.round(bnd[:, 0])
        quad = ngd.QuadratureSet(rng.random((nint, 2)), np.full(nint, 1.0 / max(nint, 1)), bnd,
                                 np.full(nbnd, 4.0 / max(nbnd, 1)))
        oq = O.Quadrature(quad.interior_points, quad.interior_weights, quad.boundary_points, quad.boundary_weights)
        v = np.random.default_rng(0).standard_normal(len(theta))
        want = O.GramianOracle(oprob, theta, oq).matvec(v)
        got = ngd.GramianOperator.from_problem(prob, theta, quad).matvec(v)
        assert np.linalg.norm(got - want) <= 1e-10 * max(np.linalg.norm(want), 1e-300)


# ---- the reference's KATs (test_gramian.py / test_sketch.py / test_krylov.py) on the CUDA path ----

def test_matvec_count_and_shape_errors():
    prob, quad, theta = make("c1")
    gop = ngd.GramianOperator.from_problem(prob, theta, quad)
    gop.matvec(np.ones(gop.dim))
    gop.matmat(np.ones((gop.dim, 3)))
    assert gop.matvec_count == 4
    with pytest.raises(ValueError):
        gop.matvec(np.ones(gop.dim + 1))


def test_sketch_kats():
    p = 12
    f = ngd.nystrom_approximate(np.eye(p), rank=p, seed=0)
    np.testing.assert_allclose(f.dense(), np.eye(p), atol=1e-12)
    rng = np.random.default_rng(1)
    z = rng.standard_normal(15)
    g = np.outer(z, z)
    f = ngd.nystrom_approximate(g, rank=3, seed=2)
    assert f.eig_host[0] == pytest.approx(z @ z, rel=1e-10)
    assert f.eig_host[1] <= 1e-10 * (z @ z)
    a = rng.standard_normal((20, 20))
    spsd = a @ a.T
    f1 = ngd.nystrom_approximate(spsd, rank=5, seed=9)
    f2 = ngd.nystrom_approximate(spsd, rank=5, seed=9)
    assert torch.equal(f1.basis, f2.basis) and torch.equal(f1.eigenvalues, f2.eigenvalues)
    op = ngd.DenseOperator(spsd)
    ngd.nystrom_approximate(op, rank=8, seed=0)
    assert op.matvec_count == 8
    with pytest.raises(ValueError):
        ngd.nystrom_approximate(np.eye(4), rank=5, seed=0)


def test_preconditioner_kats():
    rng = np.random.default_rng(0)
    p = 25
    q, _ = np.linalg.qr(rng.standard_normal((p, p)))
    g = (q * 2.0 ** -np.arange(p)) @ q.T
    f = ngd.nystrom_approximate(g, rank=8, seed=0)
    pre = ngd.NystromPreconditioner(f, 1e-3)
    u = np.asarray(f.basis.cpu())
    v = np.random.default_rng(5).standard_normal(p)
    v -= u @ (u.T @ v)
    np.testing.assert_allclose(pre.apply(v), v, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(pre.apply(u[:, -1]), u[:, -1], rtol=1e-12, atol=1e-14)
    w = np.random.default_rng(6).standard_normal(p)
    np.testing.assert_allclose(pre.apply(w), pre.dense_inverse() @ w, rtol=1e-12)
    with pytest.raises(ValueError):
        ngd.NystromPreconditioner(f, -1.0)
    with pytest.raises(ngd.SketchFailure):  # Omega^T Y_nu == 0 is never PD (sketch.py:83-85)
        ngd.nystrom_approximate(np.zeros((4, 4)), 2, 0)


def test_pcg_kats():
    b = np.array([3.0, -1.0, 2.0])
    rep = ngd.pcg(ngd.DenseOperator(np.eye(3)), b, rel_tol=1e-12, maxit=10)
    assert rep.iterations == 1 and rep.converged
    np.testing.assert_allclose(rep.solution, b, rtol=1e-14)
    rng = np.random.default_rng(0)
    a = rng.standard_normal((10, 10))
    spd = a @ a.T + 10.0 * np.eye(10)
    bb = rng.standard_normal(10)
    rep = ngd.pcg(ngd.DenseOperator(spd), bb, rel_tol=1e-12, maxit=100)
    np.testing.assert_allclose(rep.solution, np.linalg.solve(spd, bb), rtol=1e-10)
    rep = ngd.pcg(ngd.DenseOperator(np.eye(4)), np.zeros(4), rel_tol=1e-8, maxit=5)
    assert rep.converged and rep.iterations == 0 and rep.matvecs == 0
    rng = np.random.default_rng(1)
    a = rng.standard_normal((20, 20))
    op = ngd.DenseOperator(a @ a.T + np.eye(20))
    rep = ngd.pcg(op, rng.standard_normal(20), rel_tol=1e-10, maxit=100)
    assert rep.matvecs == rep.iterations + 1 and op.matvec_count == rep.matvecs
    rep = ngd.pcg(ngd.DenseOperator(np.diag([1.0, -1.0])), np.array([0.0, 1.0]), 1e-10, 10)
    assert rep.breakdown and not rep.converged
    with pytest.raises(ValueError):
        ngd.pcg(ngd.DenseOperator(np.eye(2)), np.ones(2), rel_tol=0.0, maxit=5)
    with pytest.raises(ValueError):
        ngd.pcg(ngd.DenseOperator(np.eye(2)), np.ones(2), rel_tol=1.0, maxit=5)
    # exact preconditioner: <= 2 iterations (test_krylov.py:42-53)
    rng = np.random.default_rng(2)
    f = rng.standard_normal((30, 4))
    g = f @ f.T
    fac = ngd.nystrom_approximate(g, rank=7, seed=0)
    pre = ngd.NystromPreconditioner(fac, 1e-3)
    rep = ngd.pcg(ngd.ShiftedOperator(ngd.DenseOperator(g), 1e-3), rng.standard_normal(30), 1e-10, 50, precond=pre)
    assert rep.converged and rep.iterations <= 2
    # callable operator and preconditioner (generic path)
    spd3 = np.diag([1.0, 4.0, 9.0])
    rep = ngd.pcg(lambda v: spd3 @ v, np.ones(3), 1e-12, 20, precond=lambda v: v / spd3.diagonal())
    np.testing.assert_allclose(rep.solution, np.ones(3) / spd3.diagonal(), rtol=1e-10)


def test_pcg_recompute_every_accounting():
    rng = np.random.default_rng(3)
    a = rng.standard_normal((60, 60))
    op = ngd.DenseOperator(a @ a.T + 1e-3 * np.eye(60))
    b = rng.standard_normal(60)
    rep = ngd.pcg(op, b, 1e-300, 7, recompute_every=3)
    want = O.pcg(O.DenseOracle(a @ a.T + 1e-3 * np.eye(60)), b, 1e-300, 7, recompute_every=3)
    assert (rep.iterations, rep.matvecs) == (want.iterations, want.matvecs)
    np.testing.assert_allclose(rep.solution, want.solution, rtol=1e-8)


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_pcg_bitwise_across_launch_modes(name):
    """Programmatic dependent launch and CUDA-graph replay only change how the PCG kernel chain is
    scheduled, never what it computes: a preconditioned 50-iteration solve is bitwise identical with
    pdl on/off and graphs on/off (each kernel waits for its predecessor before touching memory)."""
    from paper_2505_11638_b200 import _lib

    prob, quad, theta = make(name)
    gop = ngd.GramianOperator.from_problem(prob, theta, quad)
    g = prob.loss_grad(theta, quad)
    fac = ngd.nystrom_approximate(gop, 100, seed=1, omega_source="device")
    out = {}
    for pdl, graphs in ((1, 1), (0, 1), (1, 0), (0, 0)):
        with _lib.option("pdl", pdl), _lib.option("graphs", graphs):
            pre = ngd.NystromPreconditioner(fac, 1e-9)
            rep = ngd.pcg(ngd.ShiftedOperator(gop, 1e-9), g, 1e-300, 50, precond=pre)
            out[(pdl, graphs)] = (np.asarray(rep.solution).copy(), rep.iterations)
    ref = out[(1, 1)]
    for k, (x, its) in out.items():
        assert its == ref[1], k
        assert np.array_equal(x, ref[0]), k
