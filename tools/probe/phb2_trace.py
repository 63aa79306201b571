"""Read the NGD_PHB2_TRACE counters after one matvec (variant build): per-CTA consumer wait /
compute / total cycles and producer empty-slot wait."""
import os, sys, ctypes
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch, bench
import paper_2505_11638_b200 as ngd
from paper_2505_11638_b200 import _lib
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
prob, quad, theta0, _ = bench.make_problem(ngd, cfg, 1, 0)
gop = ngd.GramianOperator.from_problem(prob, theta0, quad)
v = torch.randn(gop.dim, dtype=torch.float64, device="cuda"); out = torch.empty_like(v)
gop.matvec_device(v, 0.0, out); torch.cuda.synchronize()
lib = _lib.load()
cudart = ctypes.CDLL("libcudart.so.12") if False else None
# read the symbol through the library's exported helper
buf = (ctypes.c_ulonglong * 4096)()
lib.ngd_debug_read_p2tr(buf)
a = np.array(buf[:], dtype=np.float64).reshape(1024, 4)
lib.ngd_debug_read_p2tr(buf)  # (second read clears nothing; counters accumulate over launches)
n = int(np.count_nonzero(a[:, 2]))
print(f"{cfg}: CTAs with work {n}")
for i in range(0, min(n, 400), 37):
    print(f"cta {i:3d}: wait {a[i,0]:9.0f} compute {a[i,1]:9.0f} total {a[i,2]:9.0f} producer-empty-wait {a[i,3]:9.0f}")
sm = a[:n, 0].astype(int)
heavy = a[:n, 2] > 15000
from collections import Counter
hc = Counter(sm[heavy])
print("SMs with 2 heavy CTAs:", sum(1 for v in hc.values() if v >= 2), "SMs with heavy:", len(hc),
      "SMs used:", len(set(sm)))
st = a[:n, 1]; en = a[:n, 3]; t0 = st.min()
print("start ns: min 0 max %.0f ; end ns: min %.0f max %.0f" % (st.max() - t0, en.min() - t0, en.max() - t0))
order = np.argsort(st)
for i in list(order[:4]) + list(order[-6:]):
    print(f"cta {i:3d} sm {int(a[i,0]):3d} start {st[i]-t0:8.0f} end {en[i]-t0:8.0f}")
