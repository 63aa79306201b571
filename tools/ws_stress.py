"""Back-to-back Gramian matvec / JVP stress at C5: every repeat against a reference made in isolation."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import bench
import paper_2505_11638_b200 as ngd
from paper_2505_11638_b200 import _lib

mode = sys.argv[1] if len(sys.argv) > 1 else "plain"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 12
prob, quad, theta0, _ = bench.make_problem(ngd, "c5")
if mode == "nopdl":
    _lib.set_option("pdl", 0)
gop = ngd.GramianOperator.from_problem(prob, theta0, quad)
ctx = gop.ctx
p = gop.dim
n = 131072 + 16384
rng = np.random.default_rng(5)
u = torch.as_tensor(rng.standard_normal(p), dtype=torch.float64, device="cuda")
v = torch.as_tensor(rng.standard_normal(p), dtype=torch.float64, device="cuda")
gop.matvec_device(u); torch.cuda.synchronize()


def jvp(x):
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    ctx.call("ngd_jvp", _lib.ptr(x), _lib.ptr(out))
    return out


torch.cuda.synchronize()
c_ref = jvp(v); torch.cuda.synchronize()
g_ref = gop.matvec_device(v).clone(); torch.cuda.synchronize()
bad_j, bad_m = [], []
for k in range(reps):
    gop.matvec_device(u)          # a matvec in flight ...
    c = jvp(v)                    # ... then phase A alone, back to back
    torch.cuda.synchronize()
    d = torch.nonzero(c != c_ref).flatten()
    if d.numel():
        bad_j.append((k, d.numel(), int(d.min()), int(d.max()), float((c - c_ref).abs().max() / c_ref.abs().max())))
    gop.matvec_device(u)
    g = gop.matvec_device(v)
    torch.cuda.synchronize()
    d = torch.nonzero(g != g_ref).flatten()
    if d.numel():
        bad_m.append((k, d.numel(), float(torch.linalg.norm(g - g_ref) / torch.linalg.norm(g_ref))))
print(f"[{mode}] {reps} reps: jvp mismatches {bad_j}")
print(f"[{mode}] {reps} reps: matvec mismatches {bad_m}")
