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
