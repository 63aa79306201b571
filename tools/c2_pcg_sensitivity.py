"""Rounding sensitivity of the PCG breakdown iteration on the C2 trajectory: the oracle run 5 steps
unperturbed and with a relative 1-ulp perturbation of every Gramian matvec output (profiles/r02_c2_pcg_breakdown_sensitivity.txt)."""
import numpy as np, time
from oracle import ngd_oracle as O
widths = (2, 64, 64, 64, 1)
prob = O.PoissonProblem(widths)
quad = prob.sample_quadrature(4096, 512, 0)
theta = O.init_theta(widths, 0)
orig = O.GramianOracle.matvec
for run in range(3):
    prng = np.random.default_rng(2000 + run)
    def mv(self, v, _p=prng):
        y = orig(self, v)
        return y * (1.0 + 2.220446049250313e-16 * _p.uniform(-1, 1, y.shape)) if run > 0 else y
    O.GramianOracle.matvec = mv
    cfg = O.NgdConfigOracle(ell0=300, ell_max=300, cg_maxit=50, kappa=1e-300, mu_floor_mode="grad-power",
                            mu_floor_coeff=1e-6, mu_floor_exponent=1.0, iterations=5, seed=0, fixed_rank=True)
    t0 = time.time()
    _, recs = O.nystrom_ngd_run(prob, theta, cfg, quad)
    print(run, [r.pcg_iters for r in recs], [r.loss for r in recs], time.time() - t0, flush=True)
