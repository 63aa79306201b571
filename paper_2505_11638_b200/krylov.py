"""Preconditioned conjugate gradient on the GPU (mirror of nystromngd/krylov.py:12-88).

For the operators this package builds (Gramian / shifted Gramian / dense) the
whole solve runs inside ``ngd_pcg``: device-resident scalars, device-side
breakdown / convergence flags, the reference's recompute-every-50 true
residual and final true-residual matvec, no per-iteration host round trip.
Arbitrary callables fall back to a host-driven loop over CUDA tensors.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .gramian import DenseOperator, GramianOperator, ShiftedOperator, utility_context
from .sketch import NystromPreconditioner

__all__ = ["SolveReport", "pcg"]


@dataclass
class SolveReport:
    """Outcome of one (P)CG solve (krylov.py:12-21)."""

    solution: object
    iterations: int
    relative_residual: float
    matvecs: int
    converged: bool
    breakdown: bool = False


def _unwrap(op):
    mu = 0.0
    base = op
    if isinstance(op, ShiftedOperator):
        mu, base = op.mu, op.base
    return base, mu


def pcg(op, b, rel_tol, maxit, precond=None, recompute_every=50):
    """Solve op x = b from x0 = 0 (krylov.py:24-88)."""
    torch = _lib.torch_mod()
    if not 0.0 < rel_tol < 1.0:
        raise ValueError(f"rel_tol must be in (0, 1), got {rel_tol}")
    if maxit < 1:
        raise ValueError("maxit must be >= 1")
    base, mu = _unwrap(op)
    if isinstance(base, (np.ndarray,)):
        base = DenseOperator(base)
    fast_op = isinstance(base, (GramianOperator, DenseOperator))
    fast_pre = precond is None or isinstance(precond, NystromPreconditioner)
    if fast_op and fast_pre:
        bt = _lib.to_device(b)
        x = torch.empty_like(bt)
        rep = _lib.SolveReportC()
        U = eig = None
        ell = 0
        pmu = 0.0
        if precond is not None:
            U, eig, ell = precond.factor.basis, precond.factor.eigenvalues, precond.factor.rank
            if U.stride(0) != 1:
                U = U.t().contiguous().t()
            pmu = precond.mu
        if isinstance(base, GramianOperator):
            base._ensure()
            ctx, dense, p = base.ctx, None, base.dim
        else:
            ctx, dense, p = base.ctx, base.matrix, base.dim
        if bt.shape != (p,):
            raise ValueError(f"expected vector of length {p}, got {tuple(bt.shape)}")
        ctx.call("ngd_pcg", _lib.ptr(dense) if dense is not None else None, p, _lib.ptr(bt), float(mu),
                 _lib.ptr(U), _lib.ptr(eig), int(ell), float(pmu), float(rel_tol), int(maxit),
                 int(recompute_every), _lib.ptr(x), _lib.ctypes.byref(rep))
        base.matvec_count += int(rep.matvecs)
        return SolveReport(_lib.like_input(x, b), int(rep.iterations), float(rep.relative_residual),
                           int(rep.matvecs), bool(rep.converged), bool(rep.breakdown))
    return _pcg_generic(op, b, rel_tol, maxit, precond, recompute_every)


def _pcg_generic(op, b, rel_tol, maxit, precond, recompute_every):
    """Host-driven PCG over CUDA tensors for arbitrary callables (same control flow)."""
    torch = _lib.torch_mod()
    matvec = op.matvec if hasattr(op, "matvec") else op
    apply_p = (precond.apply if hasattr(precond, "apply") else precond) if precond else None
    as_numpy = not _lib.is_device_array(b)

    def mv(v):
        out = matvec(v.cpu().numpy() if as_numpy else v)
        return _lib.to_device(out)

    def pp(v):
        if not apply_p:
            return v
        return _lib.to_device(apply_p(v.cpu().numpy() if as_numpy else v))

    bt = _lib.to_device(b)
    norm_b = float(torch.linalg.norm(bt))
    x = torch.zeros_like(bt)
    if norm_b == 0.0:
        return SolveReport(_lib.like_input(x, b), 0, 0.0, 0, True)
    r = bt.clone()
    z = pp(r)
    d = z.clone()
    rz = float(r @ z)
    matvecs = iterations = 0
    breakdown = False
    for it in range(1, maxit + 1):
        ad = mv(d)
        matvecs += 1
        dad = float(d @ ad)
        if dad <= 0.0:
            breakdown = True
            break
        alpha = rz / dad
        x = x + alpha * d
        iterations = it
        if it % recompute_every == 0:
            r = bt - mv(x)
            matvecs += 1
        else:
            r = r - alpha * ad
        if float(torch.linalg.norm(r)) / norm_b <= rel_tol:
            break
        z = pp(r)
        rz_new = float(r @ z)
        beta = rz_new / rz
        rz = rz_new
        d = z + beta * d
    r_true = bt - mv(x)
    matvecs += 1
    rel_res = float(torch.linalg.norm(r_true)) / norm_b
    return SolveReport(_lib.like_input(x, b), iterations, rel_res, matvecs, (not breakdown) and rel_res <= rel_tol,
                       breakdown)
