"""Blocked Cholesky (n > 512) reproduction for compute-sanitizer."""
import sys

import numpy as np
import torch

from paper_2505_11638_b200 import _lib
from paper_2505_11638_b200.gramian import utility_context

n = int(sys.argv[1]) if len(sys.argv) > 1 else 513
rng = np.random.default_rng(100 + n)
g = rng.standard_normal((2 * n + 5, n))
a = g.T @ g + 1e-3 * np.eye(n)
ctx = utility_context()
A = torch.as_tensor(a.T.copy(), device="cuda")
info = _lib.ctypes.c_int32()
ctx.call("ngd_small_cholesky", _lib.ptr(A), n, 0, _lib.ctypes.byref(info))
u = np.triu(A.cpu().numpy().T)
print("info", info.value, "err", np.linalg.norm(u - np.linalg.cholesky(a).T) / np.linalg.norm(u))
