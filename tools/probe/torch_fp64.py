"""Probe: cuBLAS DGEMM (torch.matmul fp64) peak and cuSOLVER-ish timings at NGD sizes."""
import torch, time, json
dev = torch.device("cuda:0")
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        s.record(); fn(); e.record(); e.synchronize(); best = min(best, s.elapsed_time(e))
    return best
res = {}
for n in (2048, 4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device=dev); b = torch.randn(n, n, dtype=torch.float64, device=dev)
    ms = t(lambda: a @ b)
    res[f"dgemm_{n}"] = 2 * n**3 / ms / 1e9
# tall-skinny shapes of the sketch
for (m, k, n) in ((4608, 8577, 300), (8577, 4608, 300), (65536, 132609 // 8, 512)):
    a = torch.randn(m, k, dtype=torch.float64, device=dev); b = torch.randn(k, n, dtype=torch.float64, device=dev)
    ms = t(lambda: a @ b)
    res[f"dgemm_{m}x{k}x{n}"] = (ms, 2 * m * k * n / ms / 1e9)
for (p, l) in ((1185, 100), (8577, 300), (33921, 500)):
    x = torch.randn(p, l, dtype=torch.float64, device=dev)
    res[f"qr_{p}x{l}_ms"] = t(lambda: torch.linalg.qr(x))
    r = torch.linalg.qr(x)[1]
    for drv in ("gesvd", "gesvdj", "gesvda"):
        try:
            res[f"svd_{drv}_{l}x{l}_ms"] = t(lambda: torch.linalg.svd(r, full_matrices=False, driver=drv))
        except Exception as ex:
            res[f"svd_{drv}_{l}x{l}_ms"] = str(ex)[:80]
    for drv in ("gesvd", "gesvdj"):
        try:
            res[f"svd_{drv}_{p}x{l}_ms"] = t(lambda: torch.linalg.svd(x, full_matrices=False, driver=drv), reps=2)
        except Exception as ex:
            res[f"svd_{drv}_{p}x{l}_ms"] = str(ex)[:80]
    m = r.T @ r + torch.eye(l, dtype=torch.float64, device=dev)
    res[f"chol_{l}_ms"] = t(lambda: torch.linalg.cholesky(m))
    res[f"eigh_{l}_ms"] = t(lambda: torch.linalg.eigh(m))
print(json.dumps(res, indent=1))
