"""Randomized Nystrom approximation and preconditioner on the GPU (mirror of
nystromngd/sketch.py:23-121).

``nystrom_approximate`` follows Alg. 1 (sketch.py:58-90):
Gaussian test matrix -> orthonormalise (Cholesky-QR2 on tensor cores; same
basis as the reference's Householder QR up to column signs) -> Y = G Omega
(one batched sketch call) -> shift nu = eps ||Y||_F -> Cholesky of Omega^T Y_nu
(retry with a fresh Omega from the same rng on failure) -> B = Y_nu C^{-1} ->
thin SVD of B (Householder QR + Jacobi SVD of R) -> Lambda = max(s^2 - nu, 0).

Test matrix source (``omega_source``):
  * ``"host"``   -- numpy ``default_rng(seed).standard_normal((p, rank))``, the
                    reference's exact draws (bit-identical Omega; parity mode);
  * ``"device"`` -- counter-based Philox4x32-10 Gaussians generated on the GPU
                    from the same seed (throughput mode; statistically
                    equivalent, not bit-comparable).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .gramian import DenseOperator, GramianOperator, utility_context

__all__ = ["NystromFactor", "NystromPreconditioner", "nystrom_approximate", "effective_dimension", "SketchFailure"]

OMEGA_SOURCE = "host"


class SketchFailure(RuntimeError):
    """The shifted sketch was numerically indefinite for all retry seeds (sketch.py:23-24)."""


@dataclass(frozen=True)
class NystromFactor:
    """G ~= U diag(eigenvalues) U^T (sketch.py:27-49).  ``basis`` is a (p, l)
    CUDA tensor view of column-major storage (each basis vector contiguous);
    ``eigenvalues`` a (l,) CUDA tensor."""

    basis: object
    eigenvalues: object
    eig_host: np.ndarray = field(default=None, repr=False)
    shift: float = 0.0

    def __post_init__(self):
        eh = self.eig_host
        if eh is None:
            eh = np.asarray(_lib.like_input(_lib.to_device(self.eigenvalues), np.zeros(1)))
            object.__setattr__(self, "eig_host", eh)
        if np.any(eh < 0):
            raise ValueError("eigenvalue estimates must be nonnegative")
        if np.any(np.diff(eh) > 0):
            raise ValueError("eigenvalue estimates must be sorted descending")

    @property
    def rank(self):
        return int(self.basis.shape[1])

    def dense(self, k=None):
        """Dense reconstruction (test oracle; small p only)."""
        k = self.rank if k is None else k
        u = np.asarray(_lib.like_input(self.basis, np.zeros(1)))[:, :k]
        return (u * self.eig_host[:k]) @ u.T


def _operator(op):
    if isinstance(op, np.ndarray) or _lib.is_device_array(op):
        return DenseOperator(op)
    return op


def _draw_omega(rng, p, rank, source, seed, attempt):
    torch = _lib.torch_mod()
    if source == "host":
        om = rng.standard_normal((p, rank))  # sketch.py:74
        return _lib.to_device(np.ascontiguousarray(om.T))  # (rank, p) == p x rank column-major
    if source == "device":
        om = torch.empty((rank, p), dtype=torch.float64, device=_lib.device())
        ctx = utility_context()
        philox_seed = (int(seed) * 0x9E3779B97F4A7C15 + attempt) & ((1 << 64) - 1)
        ctx.call("ngd_fill_gaussian", _lib.ctypes.c_uint64(philox_seed), _lib.ptr(om), p * rank)
        return om
    raise ValueError(f"unknown omega source {source!r}")


def nystrom_approximate(op, rank, seed, max_retries=3, omega_source=None, omega_hook=None):
    """Stable randomized Nystrom approximation of an SPSD operator (sketch.py:58-90)."""
    torch = _lib.torch_mod()
    op = _operator(op)
    p = op.dim
    if not 1 <= rank <= p:
        raise ValueError(f"rank must be in [1, {p}], got {rank}")
    source = omega_source or OMEGA_SOURCE
    rng = np.random.default_rng(seed)
    ctx = op.ctx if hasattr(op, "ctx") else utility_context()
    last_err = None
    for attempt in range(max_retries):
        omega = _draw_omega(rng, p, rank, source, seed, attempt)
        ctx.call("ngd_nystrom_prepare", _lib.ptr(omega), p, rank)
        if omega_hook is not None:
            omega_hook(omega.t())
        Y = torch.empty_like(omega)
        if hasattr(op, "matmat_colmajor"):
            op.matmat_colmajor(omega, Y)
        else:  # generic operator with a (p, l) matmat
            Y.copy_(_lib.to_device(op.matmat(omega.t().cpu().numpy())).t())
        Ucm = torch.empty((rank, p), dtype=torch.float64, device=omega.device)  # p x rank column-major
        eig = torch.empty(rank, dtype=torch.float64, device=omega.device)
        shift = _lib.ctypes.c_double()
        try:
            ctx.call("ngd_nystrom_finish", _lib.ptr(omega), _lib.ptr(Y), p, rank, _lib.ptr(Ucm), _lib.ptr(eig),
                     _lib.ctypes.byref(shift))
        except _lib.CholeskyFailure as err:
            last_err = err
            continue
        eh = eig.cpu().numpy()
        return NystromFactor(Ucm.t(), eig, eh, float(shift.value))
    raise SketchFailure(f"sketch Cholesky failed after {max_retries} attempts") from last_err


class NystromPreconditioner:
    """P^{-1} v = (lam_l + mu) U (Lam + mu I)^{-1} U^T v + (v - U U^T v) (sketch.py:93-121),
    applied on the GPU in two fused passes over U."""

    def __init__(self, factor, mu):
        if factor.eig_host[-1] + mu <= 0:
            raise ValueError("need smallest eigenvalue estimate + mu > 0")
        self.factor = factor
        self.mu = float(mu)
        self._scale = factor.eig_host[-1] + mu
        self.ctx = utility_context()

    def apply_device(self, v, out=None):
        torch = _lib.torch_mod()
        if out is None:
            out = torch.empty_like(v)
        U = self.factor.basis
        if U.stride(0) != 1:  # caller-built factor: make it column-major
            U = U.t().contiguous().t()
        self.ctx.call("ngd_precond_apply", _lib.ptr(U), _lib.ptr(self.factor.eigenvalues), U.shape[1], self.mu,
                      _lib.ptr(v), _lib.ptr(out), U.shape[0])
        return out

    def apply(self, v):
        t = _lib.to_device(v)
        return _lib.like_input(self.apply_device(t), v)

    def __call__(self, v):
        return self.apply(v)

    def dense_inverse(self):
        """Dense P^{-1} (test oracle), one device apply per column."""
        p = self.factor.basis.shape[0]
        eye = np.eye(p)
        return np.column_stack([self.apply(eye[:, i]) for i in range(p)])


def effective_dimension(eigs, mu):
    """sum lam_i / (lam_i + mu) (sketch.py:124-131; host utility)."""
    eigs = np.asarray(eigs, dtype=float)
    if mu <= 0:
        raise ValueError("mu must be positive")
    if np.any(eigs < 0):
        raise ValueError("eigenvalues must be nonnegative")
    return float(np.sum(eigs / (eigs + mu)))
