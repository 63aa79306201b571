"""How sensitive is the reference's 20-step NGD loss trajectory (C1, fixed rank 100)
to 1-ulp-level rounding noise?  Runs the CPU oracle with its Gramian matvec
output multiplied by (1 + eps_rel * N(0,1)) and reports the per-step relative
loss deviation from the golden reference trajectory (tests/golden/c1.npz).
CPU only; test infrastructure (imports the oracle)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import ngd_oracle as O

G = dict(np.load(os.path.join(ROOT, "tests", "golden", "c1.npz")))
eps_rel = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-16
prob = O.PoissonProblem((2, 32, 32, 1))
quad = prob.sample_quadrature(900, 120, 0)
theta = O.init_theta((2, 32, 32, 1), 0)
noise = np.random.default_rng(12345)
orig = O.GramianOracle.matvec
def noisy(self, v):
    out = orig(self, v)
    return out * (1.0 + eps_rel * noise.standard_normal(out.shape))
O.GramianOracle.matvec = noisy
cfg = O.NgdConfigOracle(ell0=100, ell_max=100, cg_maxit=20, kappa=1e-300, mu_floor_mode="grad-power",
                        mu_floor_coeff=1e-6, mu_floor_exponent=1.0, iterations=20, seed=0, fixed_rank=True)
_, recs = O.nystrom_ngd_run(prob, theta, cfg, quad)
for r, rl in zip(recs, G["traj_loss"]):
    print(r.iteration, f"rel {abs(r.loss - rl) / abs(rl):.2e}")
