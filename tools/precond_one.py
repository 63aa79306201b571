"""Nystrom preconditioner applies at C2 (for ncu): one factorisation, then reps applies."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch, bench
import paper_2505_11638_b200 as ngd
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
prob, quad, theta0, c = bench.make_problem(ngd, cfg)
gop = ngd.GramianOperator.from_problem(prob, theta0, quad)
fac = ngd.nystrom_approximate(gop, bench.CONFIGS[cfg][4], seed=1, omega_source="device")
pre = ngd.NystromPreconditioner(fac, 1e-4)
v = torch.randn(gop.dim, dtype=torch.float64, device="cuda")
for _ in range(3):
    pre.apply_device(v)
torch.cuda.synchronize()
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(reps):
    pre.apply_device(v)
e.record(); e.synchronize()
print(f"{cfg}: precond apply {1e3 * s.elapsed_time(e) / reps:.1f} us (incl. host call overhead)")
