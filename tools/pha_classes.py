"""Per-class device time of Gramian matvecs at a config (phase A / B engines)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2505_11638_b200 as ngd  # noqa: E402
from paper_2505_11638_b200 import _lib  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
for kv in sys.argv[2:]:
    k, v = kv.split("=")
    _lib.set_option(k, int(v))
prob, quad, theta0, _ = bench.make_problem(ngd, cfg)
gop = ngd.GramianOperator.from_problem(prob, theta0, quad)
v = torch.randn(gop.dim, dtype=torch.float64, device="cuda")
out = torch.empty_like(v)
gop.matvec_device(v, 0.0, out)
torch.cuda.synchronize()
lib = _lib.load()
cls = bench.probe_all(_lib, lib, lambda: ([gop.matvec_device(v, 0.0, out) for _ in range(5)], torch.cuda.synchronize()))
print(cfg, sys.argv[2:], {k: (round(t / 5, 3), n // 5) for k, (t, n) in cls.items()})
