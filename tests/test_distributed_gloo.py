"""Multi-rank host logic of the point-sharded path, world_size 2 over gloo on CPU.

Each rank takes its contiguous point shard (distributed.shard_slices), computes
its partial loss / gradient / Gramian matvec / sketch block with the CPU oracle
(standing in for the per-GPU kernels), and the partials are summed with the
same all-reduce the GPU path issues through NCCL.  The result must
equal the single-process full-quadrature oracle -- the identity the sharded
CUDA path relies on -- and every rank must hold bitwise-identical replicated
results (so replicated PCG / factorisation work stays in lock step).
"""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys

        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from oracle import ngd_oracle as O
        from paper_2505_11638_b200.distributed import shard_slices

        widths = (2, 16, 16, 1)
        prob = O.PoissonProblem(widths)
        quad = prob.sample_quadrature(300, 60, 0)
        theta = O.init_theta(widths, 0)
        si, sb = shard_slices(len(quad.interior_points), len(quad.boundary_points), rank, world)
        shard = O.Quadrature(quad.interior_points[si], quad.interior_weights[si], quad.boundary_points[sb],
                             quad.boundary_weights[sb])
        lin = O.Linearization(prob, theta, shard)
        w = prob.metric_weights(shard)
        r = lin.value + prob.data_offsets(shard)
        loss2 = torch.tensor([float(np.sum(w * r * r))], dtype=torch.float64)  # un-halved, as ngd_loss sums
        grad = torch.from_numpy(lin.vjp(w * r))
        v = np.random.default_rng(7).standard_normal(len(theta))
        gv = torch.from_numpy(lin.vjp(w * lin.jvp(v)))
        omega = np.linalg.qr(np.random.default_rng(8).standard_normal((len(theta), 6)))[0]
        y = torch.from_numpy(np.stack([lin.vjp(w * lin.jvp(omega[:, j])) for j in range(6)], axis=1))
        for t in (loss2, grad, gv, y):
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
        np.savez(out_path.format(rank=rank), loss=0.5 * loss2.numpy(), grad=grad.numpy(), gv=gv.numpy(),
                 y=y.numpy(), n_int=si.stop - si.start, n_bnd=sb.stop - sb.start)
    finally:
        dist.destroy_process_group()


def test_two_rank_shard_allreduce_equals_full(tmp_path):
    from oracle import ngd_oracle as O

    world = 2
    out = str(tmp_path / "rank{rank}.npz")
    mp.start_processes(_worker, args=(world, _free_port(), out), nprocs=world, start_method="spawn")
    res = [dict(np.load(out.format(rank=r))) for r in range(world)]
    # shards partition the points
    assert sum(int(r["n_int"]) for r in res) == 300 and sum(int(r["n_bnd"]) for r in res) == 60
    # replicated results are identical on every rank
    for k in ("loss", "grad", "gv", "y"):
        assert np.array_equal(res[0][k], res[1][k])
    # and equal the single-process full-quadrature oracle
    widths = (2, 16, 16, 1)
    prob = O.PoissonProblem(widths)
    quad = prob.sample_quadrature(300, 60, 0)
    theta = O.init_theta(widths, 0)
    full = O.GramianOracle(prob, theta, quad)
    v = np.random.default_rng(7).standard_normal(len(theta))
    omega = np.linalg.qr(np.random.default_rng(8).standard_normal((len(theta), 6)))[0]
    np.testing.assert_allclose(res[0]["loss"], prob.loss_value(theta, quad), rtol=1e-13)
    np.testing.assert_allclose(res[0]["grad"], prob.loss_grad(theta, quad), rtol=1e-11, atol=1e-13)
    np.testing.assert_allclose(res[0]["gv"], full.matvec(v), rtol=1e-11, atol=1e-13)
    np.testing.assert_allclose(res[0]["y"], full.matmat(omega), rtol=1e-11, atol=1e-13)


def test_nccl_unique_id_roundtrip():
    """The 128-byte NCCL id the ranks exchange is produced by the C-ABI (no GPU needed)."""
    import ctypes

    from paper_2505_11638_b200 import _lib

    lib = _lib.load()
    buf = (ctypes.c_char * 128)()
    rc = lib.ngd_nccl_unique_id(buf)
    if rc != 0:
        pytest.skip("NCCL unique id unavailable in this container: " + lib.ngd_last_error().decode())
    assert len(bytes(buf.raw)) == 128 and any(bytes(buf.raw))
