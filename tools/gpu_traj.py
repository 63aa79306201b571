"""Per-step trajectory comparison vs the golden reference run (GPU box)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2505_11638_b200 as ngd

G = dict(np.load(os.path.join(ROOT, "tests", "golden", "c1.npz")))
top = ngd.MlpTopology((2, 32, 32, 1))
prob = ngd.Poisson2D(top)
quad = prob.sample_quadrature(900, 120, 0)
theta = ngd.init(top, 0).values
cfg = ngd.NystromNgdConfig(ell0=100, ell_max=100, cg_maxit=20, kappa=1e-300, mu_floor_mode="grad-power",
                           mu_floor_coeff=1e-6, mu_floor_exponent=1.0, iterations=20, seed=0, fixed_rank=True)
info = []
th, recs = ngd.nystrom_ngd_run(prob, theta, cfg, quad, step_hook=lambda k, d: info.append((d["alpha"], d["mu"], d["report"].relative_residual, d["report"].breakdown)))
for r, rl, (a, mu, rr, bd), rmu in zip(recs, G["traj_loss"], info, G["traj_mu"]):
    print(r.iteration, f"{r.loss:.16e} {rl:.16e} rel {abs(r.loss-rl)/abs(rl):.2e} mu {mu:.6e}/{rmu:.6e} alpha {a} relres {rr:.2e} bd {bd}")
