"""The C2 5-step trajectory of tests/test_gpu_parity.py::test_c2_trajectory with the per-step PCG reports."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2505_11638_b200 as ngd

G = dict(np.load(os.path.join(ROOT, "tests", "golden", "c2_step.npz")))
top = ngd.MlpTopology((2, 64, 64, 64, 1))
prob = ngd.Poisson2D(top)
quad = prob.sample_quadrature(4096, 512, 0)
theta = ngd.init(top, 0).values
cfg = ngd.NystromNgdConfig(ell0=300, ell_max=300, cg_maxit=50, kappa=1e-300, mu_floor_mode="grad-power",
                           mu_floor_coeff=1e-6, mu_floor_exponent=1.0, iterations=5, seed=0, fixed_rank=True)
def hook(k, info):
    rep = info["report"]
    print("step", k, {a: getattr(rep, a) for a in ("iterations", "matvecs", "breakdown", "converged", "relative_residual") if hasattr(rep, a)},
          "alpha", info["alpha"], "mu", info["mu"])


_, recs = ngd.nystrom_ngd_run(prob, theta, cfg, quad, step_hook=hook)
print("its", [r.pcg_iters for r in recs], "ref", G["traj_pcg"].tolist())
print("matvecs/step", np.diff(np.concatenate([[0], [r.matvecs for r in recs]])).tolist())
for r in recs:
    print({k: getattr(r, k) for k in dir(r) if not k.startswith("_") and not callable(getattr(r, k))})
