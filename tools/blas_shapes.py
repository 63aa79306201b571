import torch, time
p, l = 8577, 300
d = torch.device("cuda")
A = torch.randn(p, l, dtype=torch.float64, device=d)
B = torch.randn(p, l, dtype=torch.float64, device=d)
R = torch.linalg.cholesky(A.T @ A).T.contiguous()
J = torch.randn(4608, p, dtype=torch.float64, device=d)
def t(fn, n=20):
    fn(); torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n): fn()
    e.record(); e.synchronize()
    return s.elapsed_time(e) / n
res = {}
res["gram A^T A (gemm)"] = t(lambda: A.T @ A)
res["A^T B (gemm K=p)"] = t(lambda: A.T @ B)
res["A @ R (p x l x l)"] = t(lambda: A @ R)
res["trsm A R^-1"] = t(lambda: torch.linalg.solve_triangular(R, A, upper=True, left=False))
res["chol l"] = t(lambda: torch.linalg.cholesky(A.T @ A))
res["sketch J @ Om (4608 x p x l)"] = t(lambda: J @ A)
S = J @ A
res["sketch J^T S (p x 4608 x l)"] = t(lambda: J.T @ S)
for k, v in res.items():
    flops = {"gram A^T A (gemm)": 2*p*l*l, "A^T B (gemm K=p)": 2*p*l*l, "A @ R (p x l x l)": 2*p*l*l, "trsm A R^-1": p*l*l,
             "chol l": 2*p*l*l + l**3/3, "sketch J @ Om (4608 x p x l)": 2*4608*p*l, "sketch J^T S (p x 4608 x l)": 2*4608*p*l}[k]
    print(f"{k:32s} {v*1e3:8.1f} us  {flops/v/1e9:6.1f} TFLOP/s")
