"""A/B check of two library option settings on one Gramian matvec (bitwise and relative diff)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch, bench
import paper_2505_11638_b200 as ngd
from paper_2505_11638_b200 import _lib
cfg, key = sys.argv[1], sys.argv[2]
vals = [int(x) for x in sys.argv[3:5]]
out = []
for v in vals:
    with _lib.option(key, v):
        prob, quad, theta0, _ = bench.make_problem(ngd, cfg)
        gop = ngd.GramianOperator.from_problem(prob, theta0, quad)
        x = np.random.default_rng(0).standard_normal(gop.dim)
        out.append(gop.matvec(x))
d = np.abs(out[0] - out[1])
print(f"{cfg} {key} {vals}: max|diff| {d.max():.3e} rel {np.linalg.norm(out[0]-out[1])/np.linalg.norm(out[0]):.3e} "
      f"bitwise-equal {np.array_equal(out[0], out[1])}")
