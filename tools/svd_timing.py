"""Time the ell x ell SVD options of the Nystrom factor on the GPU (R from a real C1/C2 sketch)."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2505_11638_b200 import _lib
from paper_2505_11638_b200.gramian import utility_context

ctx = utility_context()
for n in (100, 160, 300, 400):
    rng = np.random.default_rng(n)
    s = np.maximum(np.exp(-np.arange(n) / (n / 15)), 1.5e-8 * (1 + 0.01 * rng.random(n)))
    qa, _ = np.linalg.qr(rng.standard_normal((n, n))); qb, _ = np.linalg.qr(rng.standard_normal((n, n)))
    r = np.linalg.qr((qa * s) @ qb.T)[1]
    A = torch.as_tensor(r.T.copy(), device="cuda")
    U = torch.empty((n, n), dtype=torch.float64, device="cuda"); S = torch.empty(n, dtype=torch.float64, device="cuda")
    for method in (3, 2, 1):
        sw = _lib.ctypes.c_int32()
        try:
            ctx.call("ngd_small_svd", _lib.ptr(A), n, _lib.ptr(U), _lib.ptr(S), method, _lib.ctypes.byref(sw))
        except ValueError as e:
            print(n, method, "skip", e); continue
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            ctx.call("ngd_small_svd", _lib.ptr(A), n, _lib.ptr(U), _lib.ptr(S), method, _lib.ctypes.byref(sw))
        dt = (time.perf_counter() - t0) / 3
        err = np.max(np.abs(S.cpu().numpy() - np.linalg.svd(r, compute_uv=False))) / s[0]
        print(f"n={n} method={method} {1e3*dt:8.3f} ms sweeps={sw.value} abs_err/s1={err:.2e}")
