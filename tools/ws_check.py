"""Gramian matvec at a config: GEMM-core routes (default) vs the 64 x 64-tile kernels, repeated (race hunting)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import bench
import paper_2505_11638_b200 as ngd
from paper_2505_11638_b200 import _lib

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
prob, quad, theta0, _ = bench.make_problem(ngd, cfg)
gop = ngd.GramianOperator.from_problem(prob, theta0, quad)
torch.manual_seed(0)
u = torch.randn(gop.dim, dtype=torch.float64, device="cuda")
v = torch.randn(gop.dim, dtype=torch.float64, device="cuda")


def mv(x):
    out = torch.empty_like(x)
    gop.matvec_device(x, 0.0, out)
    torch.cuda.synchronize()
    return out


outs = [mv(v) for _ in range(reps)]
gu = mv(u)
sym = abs(float(u @ outs[0]) - float(v @ gu)) / float(torch.linalg.norm(gu) * torch.linalg.norm(v))
print(f"{cfg} default routes: symmetry {sym:.2e}; repeats differ from the first by",
      [f"{float(torch.linalg.norm(o - outs[0]) / torch.linalg.norm(outs[0])):.1e}" for o in outs[1:]])
for opts in ({"pha_gemm": 0},):
    for k, val in opts.items():
        _lib.set_option(k, val)
    gop2 = ngd.GramianOperator.from_problem(prob, theta0, quad)
    o = torch.empty_like(v)
    gop2.matvec_device(v, 0.0, o)
    torch.cuda.synchronize()
    print(f"   vs {opts}: rel diff {float(torch.linalg.norm(o - outs[0]) / torch.linalg.norm(o)):.2e}",
          " max abs", float((o - outs[0]).abs().max()), " at", int((o - outs[0]).abs().argmax()))
    for k in opts:
        _lib.set_option(k, 2)
