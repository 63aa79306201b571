"""Per-iteration cost of a preconditioned PCG solve at a BASELINE config (fixed 50 iterations, no
convergence: tiny mu, rel_tol 1e-300), optionally A/B over a library option."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch, bench
import paper_2505_11638_b200 as ngd
from paper_2505_11638_b200 import _lib
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
opts = sys.argv[2:]
prob, quad, theta0, c = bench.make_problem(ngd, cfg)
gop = ngd.GramianOperator.from_problem(prob, theta0, quad)
g = torch.as_tensor(prob.loss_grad(theta0, quad), device="cuda")
fac = ngd.nystrom_approximate(gop, bench.CONFIGS[cfg][4], seed=1, omega_source="device")
for kv in [None] + opts:
    if kv:
        k, v = kv.split("=")
        _lib.set_option(k, int(v))
    pre = ngd.NystromPreconditioner(fac, 1e-9)
    run = lambda: ngd.pcg(ngd.ShiftedOperator(gop, 1e-9), g, 1e-300, 50, precond=pre)
    rep = run(); torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        rep = run()
    e.record(); e.synchronize()
    print(f"{cfg} {kv or 'default'}: {rep.iterations} its, {1e3 * s.elapsed_time(e) / 5 / max(rep.iterations, 1):.1f} us/it")
