"""Phase A (J v, ngd_jet.cu and ngd_phag.cu) and phase B (J^T c, ngd_phb2.cu and ngd_phbg.cu) on
topologies that exercise their tile plans: partial 64x64 tiles,
several m/n tiles per layer, 'heavy' layers just above the thin threshold (17 x 33), thin
input layers with N = d up to 10 (two 8-column blocks) and the M = 1 output layer.  Each
Gramian matvec and gradient is checked against the CPU oracle."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ngd = pytest.importorskip("paper_2505_11638_b200")

from oracle import ngd_oracle as O  # noqa: E402

CASES = [
    ("sin2d", (2, 50, 100, 1), 256, 64),
    ("sin2d", (2, 17, 33, 1), 200, 40),
    ("sin2d", (2, 64, 130, 1), 256, 64),
    ("sin2d", (2, 8, 16, 8, 1), 160, 32),
    ("sinsum", (10, 40, 24, 1), 192, 48),
    ("gauss", (5, 70, 1), 192, 48),
    # wide layers (both sides >= 256) on the DMMA GEMM core (ngd_phbg.cu): full / partial 128 tiles,
    # several tiles per layer, mixed with phb2 layers in the same matvec
    ("sin2d", (2, 256, 256, 1), 256, 64),
    ("gauss", (10, 256, 300, 260, 1), 192, 48),
    ("sinsum", (3, 130, 257, 300, 64, 1), 160, 32),
    # phase A of uniform wide layers on the GEMM core (ngd_phag.cu): 128-column tiles spanning
    # several point blocks (C = 4, 7), partial m-tiles (300 rows), ragged boundary tiles
    ("sin2d", (2, 300, 300, 1), 200, 40),
    ("sinsum", (5, 256, 256, 256, 1), 150, 37),
    ("gauss", (10, 256, 256, 1), 64, 16),
]


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b))


def build(kind, widths, nint, nbnd):
    top = ngd.MlpTopology(widths)
    prob = ngd.Poisson2D(top) if kind == "sin2d" else ngd.PoissonND(top, kind)
    quad = prob.sample_quadrature(nint, nbnd, 0)
    theta = ngd.init(top, 0).values + 0.05 * np.random.default_rng(1).standard_normal(top.param_count)
    return prob, quad, theta


@pytest.mark.parametrize("kind,widths,nint,nbnd", CASES)
def test_phase_b_tile_plans(kind, widths, nint, nbnd):
    prob, quad, theta = build(kind, widths, nint, nbnd)
    v = np.random.default_rng(2).standard_normal(prob.topology.param_count)
    oprob = O.PoissonProblem(widths, kind=kind)
    oq = oprob.sample_quadrature(nint, nbnd, 0)
    ref = O.GramianOracle(oprob, theta, oq).matvec(v)
    gop = ngd.GramianOperator.from_problem(prob, theta, quad)
    assert rel(gop.matvec(v), ref) <= 1e-10
    # the gradient runs phase B with the residual cotangent
    assert rel(prob.loss_grad(theta, quad), oprob.loss_grad(theta, oq)) <= 1e-10


# every phase-A / phase-B route on the same problems: the wide layers' phase A on the GEMM core
# (pha_gemm, ngd_phag.cu) or on pha_all_kernel, and the output layer from its precontracted Jacobian
# rows (out_pre: out_contract / out_phase_b / reduce_pha_cols) or from its jets (pha_all / phb2)
ROUTE_CASES = [
    ("gauss", (10, 256, 256, 1), 64, 16),
    ("sin2d", (2, 300, 300, 1), 200, 40),
    ("sin2d", (2, 50, 100, 1), 256, 64),
    ("sinsum", (3, 17, 1), 97, 21),
]


@pytest.mark.parametrize("kind,widths,nint,nbnd", ROUTE_CASES)
def test_phase_routes_agree(kind, widths, nint, nbnd):
    from paper_2505_11638_b200 import _lib

    prob, quad, theta = build(kind, widths, nint, nbnd)
    v = np.random.default_rng(2).standard_normal(prob.topology.param_count)
    oprob = O.PoissonProblem(widths, kind=kind)
    oq = oprob.sample_quadrature(nint, nbnd, 0)
    ref_mv = O.GramianOracle(oprob, theta, oq).matvec(v)
    ref_g = oprob.loss_grad(theta, oq)
    outs = {}
    for pg in (0, 1):
        for op in (0, 1):
            with _lib.option("pha_gemm", pg), _lib.option("out_pre", op):
                gop = ngd.GramianOperator.from_problem(prob, theta, quad)
                mv = gop.matvec(v)
                g = prob.loss_grad(theta, quad)
            assert rel(mv, ref_mv) <= 1e-10, (pg, op)
            assert rel(g, ref_g) <= 1e-10, (pg, op)
            outs[pg, op] = mv
    for key, mv in outs.items():
        assert rel(mv, outs[0, 0]) <= 1e-13, key


def test_route_options_validate():
    from paper_2505_11638_b200 import _lib

    prob, quad, theta = build("sin2d", (2, 8, 1), 32, 16)
    prob.loss_value(theta, quad)  # a live context validates the values
    with pytest.raises(ValueError):
        _lib.set_option("out_pre", 3)
    with pytest.raises(ValueError):
        _lib.set_option("pha_gemm", -1)
