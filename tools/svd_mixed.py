"""FP64 block Jacobi (small_svd method 3) vs FP32 pre-sweeps + FP64 finish (method 4) on the C2
sketch's R (tools/probe/R_c2.bin) and a graded synthetic R: time, sweeps, accuracy against LAPACK,
and the preconditioner-apply error P^{-1} v at several mu (the quantity PCG parity depends on)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2505_11638_b200 import _lib
from paper_2505_11638_b200.gramian import utility_context

ctx = utility_context()


def load_c2():
    with open(os.path.join(ROOT, "tools", "probe", "R_c2.bin"), "rb") as f:
        n = int(np.fromfile(f, dtype=np.int32, count=1)[0])
        r = np.fromfile(f, dtype=np.float64, count=n * n).reshape(n, n).T
    return r


def graded(n):
    rng = np.random.default_rng(n)
    s = np.maximum(np.exp(-np.arange(n) / (n / 15)), 1.5e-8 * (1 + 0.01 * rng.random(n)))
    qa, _ = np.linalg.qr(rng.standard_normal((n, n)))
    qb, _ = np.linalg.qr(rng.standard_normal((n, n)))
    return np.linalg.qr((qa * s) @ qb.T)[1]


def run(r, method, reps=10):
    n = r.shape[0]
    A = torch.as_tensor(r.T.copy(), device="cuda")
    U = torch.empty((n, n), dtype=torch.float64, device="cuda")
    S = torch.empty(n, dtype=torch.float64, device="cuda")
    sw = _lib.ctypes.c_int32()
    ctx.call("ngd_small_svd", _lib.ptr(A), n, _lib.ptr(U), _lib.ptr(S), method, _lib.ctypes.byref(sw))
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.call("ngd_small_svd", _lib.ptr(A), n, _lib.ptr(U), _lib.ptr(S), method, _lib.ctypes.byref(sw))
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return U.cpu().numpy().T, S.cpu().numpy(), sw.value, float(np.median(ts))


cases = (("c2", load_c2()), ("graded300", graded(300)), ("graded160", graded(160)))
methods = (3, 4)
if "big" in sys.argv[1:]:  # ell above the FP64 shared-memory limit: polar SVD vs mixed (V in global)
    cases = tuple((f"graded{n}", graded(n)) for n in (320, 400, 500, 512))
    methods = (1, 4)
for name, r in cases:
    n = r.shape[0]
    u0, s0, _ = np.linalg.svd(r)
    nu = 2.2e-16 * s0[0] ** 2 * 10
    eig0 = np.maximum(s0 ** 2 - nu, 0)
    v = np.random.default_rng(0).standard_normal(n)
    for m in methods:
        u, s, sw, ms = run(r, m)
        eig = np.maximum(s ** 2 - nu, 0)
        line = f"{name} method {m}: {ms:.3f} ms sweeps {sw} sig_abs {np.max(np.abs(s - s0)) / s0[0]:.1e}"
        line += f" orth {np.linalg.norm(u.T @ u - np.eye(n)):.1e}"
        for mu in (1e-4, 1e-8, 1e-11):
            mu_ = mu * s0[0] ** 2
            pinv = lambda uu, e: v + uu @ ((((e[-1] + mu_) / (e + mu_)) - 1) * (uu.T @ v))
            p0 = pinv(u0, eig0)
            line += f" P(mu={mu:.0e}) {np.linalg.norm(pinv(u, eig) - p0) / np.linalg.norm(p0):.1e}"
        print(line, flush=True)
