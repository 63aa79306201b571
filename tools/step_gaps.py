"""Per-phase device time of NGD steps (CUDA events at phase boundaries) vs the outer step time,
averaged over K steps, to expose host gaps inside a step."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import bench
import paper_2505_11638_b200 as ngd
from paper_2505_11638_b200.optim import NystromNgdRunner, _StepTimer

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 10
prob, quad, theta0, c = bench.make_problem(ngd, cfg)
runner = NystromNgdRunner(prob, theta0, c, quad)
for _ in range(3):
    runner.step()
torch.cuda.synchronize()
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
acc, tot, its = {}, [], []
for _ in range(K):
    flush.zero_()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tm = _StepTimer(True)
    s.record()
    rec = runner.step(timer=tm)
    e.record()
    e.synchronize()
    ev = tm.events
    for i in range(len(ev) - 1):
        acc.setdefault(ev[i + 1][0], []).append(ev[i][1].elapsed_time(ev[i + 1][1]))
    acc.setdefault("pre", []).append(s.elapsed_time(ev[0][1]))
    acc.setdefault("post", []).append(ev[-1][1].elapsed_time(e))
    tot.append(s.elapsed_time(e))
    its.append(rec.pcg_iters)
print(cfg, "step %.3f ms" % np.mean(tot), {k: round(float(np.mean(v)), 3) for k, v in acc.items()}, "pcg its", its)
