"""Time the ell x ell Cholesky options (cuSOLVER / one-CTA / cluster) on the GPU."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2505_11638_b200 import _lib
from paper_2505_11638_b200.gramian import utility_context

ctx = utility_context()
for n in (100, 160, 300, 512):
    g = np.random.default_rng(n).standard_normal((3 * n, n))
    a = g.T @ g
    A0 = torch.as_tensor(a.T.copy(), device="cuda")
    for method in (0, 1, 2):
        if method == 1 and n > 160:
            continue
        A = A0.clone()
        info = _lib.ctypes.c_int32()
        ctx.call("ngd_small_cholesky", _lib.ptr(A), n, method, _lib.ctypes.byref(info))
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        reps = 20
        As = [A0.clone() for _ in range(reps)]
        torch.cuda.synchronize()
        s.record(torch.cuda.current_stream())
        for i in range(reps):
            ctx.call("ngd_small_cholesky", _lib.ptr(As[i]), n, method, _lib.ctypes.byref(info))
        e.record(torch.cuda.current_stream())
        e.synchronize()
        print(f"n={n} method={method} {1e3 * s.elapsed_time(e) / reps:8.1f} us/call (incl. host sync) info={info.value}")
