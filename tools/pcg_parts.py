"""In-graph cost split of one PCG solve at a BASELINE config: full preconditioned PCG vs the
unpreconditioned solve (same iteration count) vs bare matvecs."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import bench
import paper_2505_11638_b200 as ngd

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
prob, quad, theta0, c = bench.make_problem(ngd, cfg)
gop = ngd.GramianOperator.from_problem(prob, theta0, quad)
g = prob.loss_grad(theta0, quad)
gop = ngd.GramianOperator.from_problem(prob, theta0, quad)
ell, maxit = bench.CONFIGS[cfg][4], bench.CONFIGS[cfg][5]
fac = ngd.nystrom_approximate(gop, ell, seed=1, omega_source="device")
mu = 1e-4
pre = ngd.NystromPreconditioner(fac, mu)
gt = torch.as_tensor(g, device="cuda")
def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); e.synchronize()
    return s.elapsed_time(e) / reps
t_pre = timed(lambda: ngd.pcg(ngd.ShiftedOperator(gop, mu), gt, 1e-300, maxit, precond=pre))
t_nop = timed(lambda: ngd.pcg(ngd.ShiftedOperator(gop, mu), gt, 1e-300, maxit))
v = torch.randn(gop.dim, dtype=torch.float64, device="cuda"); out = torch.empty_like(v)
t_mv = timed(lambda: [gop.matvec_device(v, mu, out) for _ in range(maxit)])
print(f"{cfg}: PCG {maxit} its with precond {t_pre:.3f} ms, without {t_nop:.3f} ms, {maxit} bare matvecs {t_mv:.3f} ms"
      f" -> per it: precond {1e3*(t_pre-t_nop)/maxit:.1f} us, vector/scalar {1e3*(t_nop-t_mv)/maxit:.1f} us, matvec {1e3*t_mv/maxit:.1f} us")
