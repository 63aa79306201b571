"""One linearisation + a few Gramian matvecs at a BASELINE config (for ncu)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import bench
import paper_2505_11638_b200 as ngd

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
from paper_2505_11638_b200 import _lib
for kv in sys.argv[3:]:  # key=value library options, e.g. phb_cs=1
    k, v = kv.split("=") if "=" in kv else ("l2window", kv)
    _lib.set_option(k, int(v))
side = torch.cuda.Stream()
torch.cuda.set_stream(side)  # a non-default stream can carry the L2 access-policy window
prob, quad, theta0, _ = bench.make_problem(ngd, cfg)
gop = ngd.GramianOperator.from_problem(prob, theta0, quad)
v = torch.randn(gop.dim, dtype=torch.float64, device="cuda")
out = torch.empty_like(v)
for _ in range(reps):
    gop.matvec_device(v, 0.0, out)
torch.cuda.synchronize()
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20):
    gop.matvec_device(v, 0.0, out)
e.record(); e.synchronize()
print(f"{cfg}: matvec {1e3 * s.elapsed_time(e) / 20:.1f} us  (args {sys.argv[1:]})")
