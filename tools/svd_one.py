"""One Jacobi SVD launch at ell (for ncu): R from a graded synthetic Nystrom-like matrix."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2505_11638_b200 import _lib
from paper_2505_11638_b200.gramian import utility_context

n = int(sys.argv[1]) if len(sys.argv) > 1 else 300
method = int(sys.argv[2]) if len(sys.argv) > 2 else 3
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
ctx = utility_context()
rng = np.random.default_rng(n)
s = np.maximum(np.exp(-np.arange(n) / (n / 15)), 1.5e-8 * (1 + 0.01 * rng.random(n)))
qa, _ = np.linalg.qr(rng.standard_normal((n, n))); qb, _ = np.linalg.qr(rng.standard_normal((n, n)))
r = np.linalg.qr((qa * s) @ qb.T)[1]
A = torch.as_tensor(r.T.copy(), device="cuda")
U = torch.empty((n, n), dtype=torch.float64, device="cuda"); S = torch.empty(n, dtype=torch.float64, device="cuda")
sw = _lib.ctypes.c_int32()
for _ in range(reps):
    ctx.call("ngd_small_svd", _lib.ptr(A), n, _lib.ptr(U), _lib.ptr(S), method, _lib.ctypes.byref(sw))
torch.cuda.synchronize()
print("sweeps", sw.value, "err", np.max(np.abs(S.cpu().numpy() - np.linalg.svd(r, compute_uv=False))) / s[0])
