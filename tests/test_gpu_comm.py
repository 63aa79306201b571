"""The multi-rank code path (NCCL all-reduce inside the C-ABI, split reductions) exercised on ONE
GPU: a single-rank communicator built through torch.distributed (nccl backend) with the
"force_comm" option, so every collective and every multi-rank branch runs (an all-reduce over
one rank is a copy).  Results must match the communicator-free path."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ngd = pytest.importorskip("paper_2505_11638_b200")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_single_rank_nccl_path_matches():
    import torch
    import torch.distributed as dist
    from paper_2505_11638_b200 import _lib, distributed

    top = ngd.MlpTopology((2, 32, 32, 1))
    cfg = ngd.NystromNgdConfig(ell0=40, ell_max=40, cg_maxit=15, kappa=1e-300, mu_floor_mode="grad-power",
                               mu_floor_coeff=1e-6, mu_floor_exponent=1.0, iterations=3, seed=0, fixed_rank=True)
    theta0 = ngd.init(top, 0).values

    def run(comm):
        prob = ngd.make_problem("poisson2d", topology=top)
        if comm is not None:
            distributed.attach(prob, comm)
        quad = prob.sample_quadrature(900, 120, 0)
        g = prob.loss_grad(theta0, quad)
        gop = ngd.GramianOperator.from_problem(prob, theta0, quad)
        v = np.random.default_rng(1).standard_normal(gop.dim)
        mv = gop.matvec(v)
        om = np.linalg.qr(np.random.default_rng(2).standard_normal((gop.dim, 8)))[0]
        y = gop.matmat(om)
        theta, recs = ngd.nystrom_ngd_run(prob, theta0, cfg, quad, quad_eval=quad)
        # a solve that converges long before maxit: with a communicator the host enqueues all maxit
        # iterations (no timing-dependent early exit), the device-side stop is unchanged.
        # mu = 1 (lambda_max ~ 73) keeps CG insensitive to rounding: a 1-ulp matvec perturbation
        # moves the 12-iteration iterate by ~4e-13 in the oracle (at mu = 1e-3, tol 1e-3: 1.3e-4)
        gop = ngd.GramianOperator.from_problem(prob, theta0, quad)
        rep = ngd.pcg(ngd.ShiftedOperator(gop, 1.0), g, 1e-8, 40)
        return g, mv, y, theta, recs, rep

    base = run(None)
    if not dist.is_initialized():
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(_port())
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        _lib.set_option("force_comm", 1)
        comm = distributed.NcclComm()
        assert (comm.rank, comm.nranks) == (0, 1)
        forced = run(comm)
    finally:
        _lib.set_option("force_comm", 0)
        dist.destroy_process_group()
    for a, b in zip(base[:3], forced[:3]):
        np.testing.assert_allclose(b, a, rtol=1e-12, atol=1e-14 * np.abs(a).max())
    np.testing.assert_allclose([r.loss for r in forced[4]], [r.loss for r in base[4]], rtol=1e-9)
    np.testing.assert_allclose([r.h1_rel_error for r in forced[4]], [r.h1_rel_error for r in base[4]], rtol=1e-9)
    assert [r.pcg_iters for r in forced[4]] == [r.pcg_iters for r in base[4]]
    a, b = base[5], forced[5]
    assert a.converged and a.iterations < 40
    assert (b.iterations, b.matvecs, b.converged, b.breakdown) == (a.iterations, a.matvecs, a.converged, a.breakdown)
    # split partials summed in a different order before the all-reduce: rounding-level differences
    np.testing.assert_allclose(b.solution, a.solution, rtol=1e-8, atol=1e-10 * np.abs(a.solution).max())
