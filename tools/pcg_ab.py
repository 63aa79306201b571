"""Per-phase NGD step timing at a BASELINE config with a library option toggled (A/B)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import bench
import paper_2505_11638_b200 as ngd
from paper_2505_11638_b200 import _lib
from paper_2505_11638_b200.optim import NystromNgdRunner, _StepTimer

cfg_name = sys.argv[1]
for kv in sys.argv[2:]:
    k, v = kv.split("=")
    _lib.set_option(k, int(v))
prob, quad, theta0, cfg = bench.make_problem(ngd, cfg_name)
runner = NystromNgdRunner(prob, theta0, cfg, quad)
for _ in range(3):
    runner.step()
torch.cuda.synchronize()
acc = {}
for _ in range(5):
    tm = _StepTimer(True)
    runner.step(timer=tm)
    torch.cuda.synchronize()
    ev = tm.events
    for i in range(len(ev) - 1):
        acc[ev[i + 1][0]] = acc.get(ev[i + 1][0], 0.0) + ev[i][1].elapsed_time(ev[i + 1][1]) / 5
print(cfg_name, sys.argv[2:], json.dumps({k: round(v, 3) for k, v in acc.items()}), "total", round(sum(acc.values()), 3))
