"""NGD_PHA2_TRACE counters after one matvec (variant build): per-CTA start/end, units, wait cycles."""
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
buf = (ctypes.c_ulonglong * 4096)()
_lib.load().ngd_debug_read_a2tr(buf)
a = np.array(buf[:], dtype=np.float64).reshape(1024, 4)
n = int(np.count_nonzero(a[:, 1]))
st, en = a[:n, 0], a[:n, 1]; t0 = st.min()
print(f"{cfg}: CTAs {n}; start spread {st.max()-t0:.0f} ns; end min {en.min()-t0:.0f} max {en.max()-t0:.0f} ns")
for i in range(0, n, 21):
    print(f"cta {i:3d}: start {st[i]-t0:7.0f} end {en[i]-t0:7.0f} units {int(a[i,2])} wait {a[i,3]:8.0f} cyc")
