"""One linearisation + one ell-column sketch block Y = G Omega at a BASELINE config (for ncu)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2505_11638_b200 as ngd  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
prob, quad, theta0, _ = bench.make_problem(ngd, cfg)
ell = bench.CONFIGS[cfg][4]
gop = ngd.GramianOperator.from_problem(prob, theta0, quad)
V = torch.randn((ell, gop.dim), dtype=torch.float64, device="cuda")
Y = torch.empty_like(V)
gop.matmat_colmajor(V, Y)
torch.cuda.synchronize()
s = torch.cuda.Event(enable_timing=True)
e = torch.cuda.Event(enable_timing=True)
s.record()
gop.matmat_colmajor(V, Y)
e.record()
e.synchronize()
n = len(quad.interior_points) + len(quad.boundary_points)
ms = s.elapsed_time(e)
print(f"{cfg}: sketch block ({ell} columns) {ms:.1f} ms = {4.0 * n * gop.dim * ell / ms / 1e9:.2f} TFLOP/s")
