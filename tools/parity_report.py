"""Parity table for DESIGN.md section 5: relative deviation of the CUDA path from the live-reference
golden fixtures (tests/golden) per configuration and quantity, plus full-size checks against the
oracle.  Run on the GPU box:  python tools/parity_report.py > profiles/r02_parity_table.json"""

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2505_11638_b200 as ngd  # noqa: E402
from oracle import ngd_oracle as O  # noqa: E402


def gold(name):
    return dict(np.load(os.path.join(ROOT, "tests", "golden", f"{name}.npz")))


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def omega8(p, seed=123):
    return np.linalg.qr(np.random.default_rng(seed).standard_normal((p, 8)), mode="reduced")[0]


out = {}
# C1: full step pieces + 20-step trajectory vs the reference and its 1-ulp ensemble
G = gold("c1")
top = ngd.MlpTopology((2, 32, 32, 1))
prob = ngd.Poisson2D(top)
quad = prob.sample_quadrature(900, 120, 0)
theta = ngd.init(top, 0).values
gop = ngd.GramianOperator.from_problem(prob, theta, quad)
fac = ngd.nystrom_approximate(gop, 100, seed=7, omega_source="host")
keep = G["eig100"] > 1e-8 * G["eig100"][0]
pre = ngd.NystromPreconditioner(fac, float(G["mu"]))
r = {"loss": abs(prob.loss_value(theta, quad) / float(G["loss"]) - 1), "grad": rel(prob.loss_grad(theta, quad), G["grad"]),
     "Gv": rel(gop.matvec(G["v"]), G["gv"]), "Y8": rel(gop.matmat(G["omega8"]), G["y8"]),
     "eig (> 1e-8 l1)": rel(fac.eig_host[keep], G["eig100"][keep]), "P^-1 v": rel(pre.apply(G["v"]), G["pinv_v"])}
for k in (1, 5, 20):
    rep = ngd.pcg(ngd.ShiftedOperator(gop, float(G["mu"])), G["grad"], 1e-300, k, precond=pre)
    r[f"PCG x_{k}"] = rel(rep.solution, G[f"pcg{k}_x"])
cfg = ngd.NystromNgdConfig(ell0=100, ell_max=100, cg_maxit=20, kappa=1e-300, mu_floor_mode="grad-power",
                           mu_floor_coeff=1e-6, mu_floor_exponent=1.0, iterations=20, seed=0, fixed_rank=True)
_, recs = ngd.nystrom_ngd_run(prob, theta, cfg, quad)
dev = np.abs(np.array([x.loss for x in recs]) - G["traj_loss"]) / np.abs(G["traj_loss"])
E = gold("c1_ensemble")
ens = np.max(np.abs(E["ens_loss"] - G["traj_loss"]) / np.abs(G["traj_loss"]), axis=0)
r["trajectory loss, steps 1-13 (max)"] = float(dev[:13].max())
r["trajectory loss, steps 14-20 / ensemble max (max ratio)"] = float(np.max(dev[13:] / ens[13:]))
r["trajectory loss per step"] = dev.tolist()
r["reference 1-ulp ensemble max per step"] = ens.tolist()
out["c1"] = r

# C2: the benchmarked step's pieces (rank 300, host Omega)
G = gold("c2_step")
top = ngd.MlpTopology((2, 64, 64, 64, 1))
prob = ngd.Poisson2D(top)
quad = prob.sample_quadrature(4096, 512, 0)
theta = ngd.init(top, 0).values
g2 = gold("c2")
gop = ngd.GramianOperator.from_problem(prob, theta, quad)
fac = ngd.nystrom_approximate(gop, 300, seed=11, omega_source="host")
keep = G["eig300"] > 1e-8 * G["eig300"][0]
pre = ngd.NystromPreconditioner(fac, float(G["mu"]))
g = prob.loss_grad(theta, quad)
r = {"loss": abs(prob.loss_value(theta, quad) / float(g2["loss"]) - 1), "grad": rel(g, g2["grad"]),
     "Gv": rel(gop.matvec(g2["v"]), g2["gv"]), "eig (> 1e-8 l1)": rel(fac.eig_host[keep], G["eig300"][keep]),
     "P^-1 v": rel(pre.apply(G["v"]), G["pinv_v"])}
for k in (5, 20, 50):
    rep = ngd.pcg(ngd.ShiftedOperator(gop, float(G["mu"])), g, 1e-300, k, precond=pre)
    r[f"PCG x_{k}"] = rel(rep.solution, G[f"pcg{k}_x"])
    r[f"PCG x_{k} iterations (ours, ref)"] = [rep.iterations, int(G[f"pcg{k}_meta"][0])]
cfg = ngd.NystromNgdConfig(ell0=300, ell_max=300, cg_maxit=50, kappa=1e-300, mu_floor_mode="grad-power",
                           mu_floor_coeff=1e-6, mu_floor_exponent=1.0, iterations=5, seed=0, fixed_rank=True)
_, recs = ngd.nystrom_ngd_run(prob, theta, cfg, quad)
r["trajectory loss (5 steps, max)"] = float(np.max(np.abs(np.array([x.loss for x in recs]) - G["traj_loss"])
                                                   / np.abs(G["traj_loss"])))
r["trajectory PCG iterations (ours, ref)"] = [[x.pcg_iters for x in recs], G["traj_pcg"].astype(int).tolist()]
out["c2"] = r

# C3 / C5 1024 + 256-point subsets, C4 1024 points: matvec + 8 sketch columns
for name, widths, kind in (("c3_1k", (5, 128, 128, 128, 1), "sinsum"), ("c5_1k", (10, 256, 256, 256, 256, 1), "gauss")):
    G = gold(name)
    top = ngd.MlpTopology(widths)
    prob = ngd.PoissonND(top, kind)
    quad = prob.sample_quadrature(1024, 256, 0)
    theta = ngd.init(top, 0).values
    p = len(theta)
    gop = ngd.GramianOperator.from_problem(prob, theta, quad)
    out[name] = {"loss": abs(prob.loss_value(theta, quad) / float(G["loss"]) - 1),
                 "grad": rel(prob.loss_grad(theta, quad), G["grad"]),
                 "Gv": rel(gop.matvec(np.random.default_rng(1).standard_normal(p)), G["gv"]),
                 "Y8": rel(gop.matmat(omega8(p)), G["y8"])}
G = gold("c4_1k")
top = ngd.MlpTopology((2, 256, 256, 256, 1))
prob = ngd.LaplacianStack(top)
n = G["x"].shape[0]
quad = ngd.QuadratureSet(G["x"], np.full(n, 1.0 / n), np.zeros((0, 2)), np.zeros(0))
theta = ngd.init(top, 0).values
p = len(theta)
gop = ngd.GramianOperator.from_problem(prob, theta, quad)
out["c4_1k"] = {"Gv": rel(gop.matvec(np.random.default_rng(1).standard_normal(p)), G["gv"]),
                "Y8": rel(gop.matmat(omega8(p)), G["y8"])}

# full-size C3 / C4 / C5 against the oracle (host cores of the GPU box)
import bench  # noqa: E402

for name, ncols in (("c3", 4), ("c4", 2), ("c5", 1)):
    widths, kind, nint, nbnd, ell, maxit = bench.CONFIGS[name]
    prob, quad, theta, _ = bench.make_problem(ngd, name)
    p = len(theta)
    okind = "sin2d" if kind == "lap" else kind
    oprob = O.PoissonProblem(widths, kind=okind, interior_only=(kind == "lap"))
    oq = O.Quadrature(quad.interior_points, quad.interior_weights, quad.boundary_points, quad.boundary_weights)
    v = np.random.default_rng(9).standard_normal(p)
    om = omega8(p, 10)[:, :ncols]
    gop = ngd.GramianOperator.from_problem(prob, theta, quad)
    ogop = O.GramianOracle(oprob, theta, oq)
    out[f"{name} full ({nint + nbnd} points) vs oracle"] = {
        "loss": abs(prob.loss_value(theta, quad) / oprob.loss_value(theta, oq) - 1),
        "Gv": rel(gop.matvec(v), ogop.matvec(v)), f"Y ({ncols} columns)": rel(gop.matmat(om), ogop.matmat(om))}
    del ogop
print(json.dumps(out, indent=1))
