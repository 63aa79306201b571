"""Regenerate tools/probe/R_c2.bin (the C2 Nystrom sketch's triangular factor R and its singular
values, from the CPU oracle) for tools/probe/jsvd_acc.cu.  Takes ~1 min on CPU."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import ngd_oracle as O

widths = (2, 64, 64, 64, 1)
prob = O.PoissonProblem(widths)
quad = prob.sample_quadrature(4096, 512, 0)
theta = O.init_theta(widths, 0)
p, ell = len(theta), 300
gop = O.GramianOracle(prob, theta, quad)
om = np.linalg.qr(np.random.default_rng(7).standard_normal((p, ell)))[0]
Y = gop.matmat(om)
nu = np.finfo(float).eps * np.linalg.norm(Y)
Yn = Y + nu * om
C = np.linalg.cholesky(om.T @ Yn).T
B = np.linalg.solve(C.T, Yn.T).T
R = np.linalg.qr(B)[1]
s = np.linalg.svd(R, compute_uv=False)
with open(os.path.join(ROOT, "tools", "probe", "R_c2.bin"), "wb") as f:
    np.array([ell], dtype=np.int32).tofile(f)
    R.T.ravel().tofile(f)  # column-major R
    s.tofile(f)
print("wrote tools/probe/R_c2.bin", R.shape, s[0], s[-1])
