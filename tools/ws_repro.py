"""Reproduce tests/test_gpu_properties.py::test_full_size_operator_properties[c5]'s symmetry check and locate the error."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import bench
import paper_2505_11638_b200 as ngd
from paper_2505_11638_b200 import _lib

mode = sys.argv[1] if len(sys.argv) > 1 else "plain"
prob, quad, theta0, _ = bench.make_problem(ngd, "c5")
if mode == "nopdl":
    _lib.set_option("pdl", 0)
gop = ngd.GramianOperator.from_problem(prob, theta0, quad)
p = gop.dim
rng = np.random.default_rng(5)
u = torch.as_tensor(rng.standard_normal(p), dtype=torch.float64, device="cuda")
v = torch.as_tensor(rng.standard_normal(p), dtype=torch.float64, device="cuda")
gu = gop.matvec(u)
if mode == "sync":
    torch.cuda.synchronize()
gv = gop.matvec(v)
torch.cuda.synchronize()
sym = abs(float(u @ gv) - float(v @ gu)) / float(torch.linalg.norm(gu) * torch.linalg.norm(v))
gu2, gv2 = gop.matvec(u), gop.matvec(v)
torch.cuda.synchronize()
print(f"[{mode}] symmetry {sym:.2e}; first-call vs repeat: gu {float(torch.linalg.norm(gu - gu2) / torch.linalg.norm(gu2)):.2e}"
      f" gv {float(torch.linalg.norm(gv - gv2) / torch.linalg.norm(gv2)):.2e}")
for name, a, b in (("gu", gu, gu2), ("gv", gv, gv2)):
    d = (a - b).abs()
    nz = torch.nonzero(d > 0).flatten()
    if nz.numel():
        print(f"   {name}: {nz.numel()} entries differ, index range {int(nz.min())}..{int(nz.max())}, max abs {float(d.max()):.3e}"
              f" (|entry| ~ {float(b.abs().mean()):.3e})")
        # layer offsets of the flat layout (W then b per layer)
        off, lay = 0, []
        w = [10, 256, 256, 256, 256, 1]
        for l in range(5):
            lay.append((off, off + w[l] * w[l + 1], off + w[l] * w[l + 1] + w[l + 1]))
            off += w[l] * w[l + 1] + w[l + 1]
        for l, (o0, o1, o2) in enumerate(lay):
            k = int(((nz >= o0) & (nz < o1)).sum()); kb = int(((nz >= o1) & (nz < o2)).sum())
            if k or kb:
                sel = nz[(nz >= o0) & (nz < o1)] - o0
                rows = torch.unique(sel // w[l]) if k else sel
                print(f"      layer {l}: {k} weight entries (rows {rows[:6].tolist()}.. {rows.numel()} rows), {kb} bias entries")
