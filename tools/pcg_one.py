"""A few preconditioned CG iterations at a BASELINE config with the iteration launched directly (graphs off),
for ncu captures of the PCG vector / preconditioner / thin-layer kernels."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import bench
import paper_2505_11638_b200 as ngd
from paper_2505_11638_b200 import _lib

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 4
prob, quad, theta0, _ = bench.make_problem(ngd, cfg)
ell = bench.CONFIGS[cfg][4]
gop = ngd.GramianOperator.from_problem(prob, theta0, quad)
g = _lib.to_device(prob.loss_grad(theta0, quad))
fac = ngd.nystrom_approximate(gop, ell, seed=1, omega_source="device")
mu = 1e-6 * float(torch.linalg.norm(g))
pre = ngd.NystromPreconditioner(fac, mu)
with _lib.option("graphs", 0):
    rep = ngd.pcg(ngd.ShiftedOperator(gop, mu), g, 1e-300, iters, precond=pre)
torch.cuda.synchronize()
print(f"{cfg}: {rep.iterations} PCG iterations, {rep.matvecs} matvecs, relative residual {rep.relative_residual:.3e}")
