"""Print parity diagnostics of the CUDA path against the golden fixtures (GPU box)."""
import os
import sys
import time
import traceback

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2505_11638_b200 as ngd  # noqa: E402
from oracle import ngd_oracle as O  # noqa: E402


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def g(name):
    return dict(np.load(os.path.join(ROOT, "tests", "golden", f"{name}.npz")))


def c1():
    G = g("c1")
    top = ngd.MlpTopology((2, 32, 32, 1))
    prob = ngd.Poisson2D(top)
    quad = prob.sample_quadrature(900, 120, 0)
    theta = ngd.init(top, 0).values
    print("loss", prob.loss_value(theta, quad), float(G["loss"]), rel(prob.loss_value(theta, quad), G["loss"]))
    print("metric rel", rel(prob.metric_stack(theta, None, quad), G["metric"]))
    print("grad rel", rel(prob.loss_grad(theta, quad), G["grad"]))
    gop = ngd.GramianOperator.from_problem(prob, theta, quad)
    print("Gv rel", rel(gop.matvec(G["v"]), G["gv"]))
    print("Y8 rel", rel(gop.matmat(G["omega8"]), G["y8"]))
    for src in ("host", "device"):
        fac = ngd.nystrom_approximate(gop, 100, seed=7, omega_source=src)
        e = fac.eig_host
        top_ = G["eig100"] > 1e-8 * G["eig100"][0]
        print(src, "eig rel (top)", rel(e[top_], G["eig100"][top_]), "n top", top_.sum(), "lam1", e[0], G["eig100"][0])
    fac = ngd.nystrom_approximate(gop, 100, seed=7, omega_source="host")
    pre = ngd.NystromPreconditioner(fac, float(G["mu"]))
    print("Pinv v rel", rel(pre.apply(G["v"]), G["pinv_v"]))
    for k in (1, 5, 20):
        rep = ngd.pcg(ngd.ShiftedOperator(gop, float(G["mu"])), G["grad"], 1e-300, k, precond=pre)
        m = G[f"pcg{k}_meta"]
        print(f"pcg{k} x rel", rel(rep.solution, G[f"pcg{k}_x"]), "its", rep.iterations, int(m[0]), "mv", rep.matvecs,
              int(m[1]), "relres", rep.relative_residual, m[2], "bd", rep.breakdown, bool(m[4]))
    cfg = ngd.NystromNgdConfig(ell0=100, ell_max=100, cg_maxit=20, kappa=1e-300, mu_floor_mode="grad-power",
                               mu_floor_coeff=1e-6, mu_floor_exponent=1.0, iterations=20, seed=0, fixed_rank=True)
    t0 = time.time()
    th, recs = ngd.nystrom_ngd_run(prob, theta, cfg, quad)
    dt = time.time() - t0
    loss = np.array([r.loss for r in recs])
    print("traj loss max rel", np.max(np.abs(loss - G["traj_loss"]) / np.abs(G["traj_loss"])), f"{dt:.2f}s")
    print("traj pcg", [r.pcg_iters for r in recs] == list(G["traj_pcg"].astype(int)),
          "matvecs", [r.matvecs for r in recs][-1], int(G["traj_matvecs"][-1]))
    print("final theta rel", rel(th, G["traj_theta"]))


def nd(name, widths, kind, nint, nbnd):
    G = g(name)
    top = ngd.MlpTopology(widths)
    prob = ngd.make_problem("poisson2d", topology=top) if kind == "sin2d" else ngd.PoissonND(top, kind)
    quad = prob.sample_quadrature(nint, nbnd, 0)
    theta = ngd.init(top, 0).values
    print(name, "loss rel", rel(prob.loss_value(theta, quad), G["loss"]), "grad rel",
          rel(prob.loss_grad(theta, quad), G["grad"]))
    gop = ngd.GramianOperator.from_problem(prob, theta, quad)
    print(name, "Gv rel", rel(gop.matvec(G["v"]), G["gv"]))


def main():
    for fn in (c1, lambda: nd("c2", (2, 64, 64, 64, 1), "sin2d", 4096, 512),
               lambda: nd("c3_sub", (5, 128, 128, 128, 1), "sinsum", 256, 64),
               lambda: nd("c5_sub", (10, 256, 256, 256, 256, 1), "gauss", 24, 8)):
        try:
            fn()
        except Exception:
            traceback.print_exc()


if __name__ == "__main__" and "--sweeps" not in sys.argv:
    main()


def sweeps():
    """Jacobi sweep counts of the real Nystrom factorisations at C1/C2."""
    from paper_2505_11638_b200 import _lib
    for widths, nint, nbnd, ell in (((2, 32, 32, 1), 900, 120, 100), ((2, 64, 64, 64, 1), 4096, 512, 300)):
        top = ngd.MlpTopology(widths)
        prob = ngd.Poisson2D(top)
        quad = prob.sample_quadrature(nint, nbnd, 0)
        gop = ngd.GramianOperator.from_problem(prob, ngd.init(top, 0).values, quad)
        import time as _t
        for src in ("host", "device"):
            ngd.nystrom_approximate(gop, ell, seed=1, omega_source=src)
            _lib.torch_mod().cuda.synchronize()
            t0 = _t.perf_counter()
            fac = ngd.nystrom_approximate(gop, ell, seed=2, omega_source=src)
            dt = _t.perf_counter() - t0
            out = _lib.ctypes.c_int64()
            gop.ctx.call("ngd_get_stat", b"jacobi_sweeps", _lib.ctypes.byref(out))
            print(f"ell={ell} {src}: jacobi sweeps {out.value}, nystrom {1e3 * dt:.2f} ms, "
                  f"unclamped {(fac.eig_host > 0).sum()}")


if __name__ == "__main__" and "--sweeps" in sys.argv:
    sweeps()
