"""Matrix-free Gramian operators on the GPU (mirror of nystromngd/gramian.py).

``GramianOperator.from_problem(problem, theta, quad)`` linearises the metric
stack once on the device (forward jet sweep + reverse jet sweep, caching the
per-layer jet factors); ``matvec`` is then two dense contraction passes on FP64
tensor cores (phase A: J v, phase B: J^T(w o Jv)), and ``matmat`` is the
J-chunk sketch (explicit Jacobian rows + two DGEMMs).  Operator protocol
(SPEC.md:12): ``dim``, ``matvec``, ``matmat``, ``matvec_count``, ``__call__``.
"""

from __future__ import annotations

import numpy as np

from . import _lib

DENSE_GUARD = 2000


class GramianOperator:
    """SPSD operator v -> J^T diag(w) J v, accessed only via matvecs (gramian.py:20-64)."""

    def __init__(self, problem, theta, quad):
        self.problem = problem
        self.quad = quad
        self.theta = _lib.to_device(theta).clone()
        self.ctx = problem.context(quad)
        self.dim = self.ctx.p
        self.weights = problem.metric_weights(quad)
        self.matvec_count = 0
        self.loss = problem.linearize(self.theta, quad, owner=self)

    @classmethod
    def from_problem(cls, problem, theta, quad):
        """Gramian of a problem at theta (gramian.py:33-41)."""
        return cls(problem, theta, quad)

    def _ensure(self):
        # the context holds one linearisation; restore ours if another operator replaced it
        if self.ctx.lin_owner is not self:
            self.problem.context(self.quad)
            self.problem.linearize(self.theta, self.quad, owner=self)

    def _vec(self, v):
        t = _lib.to_device(v)
        if t.shape != (self.dim,):
            raise ValueError(f"expected vector of length {self.dim}, got {tuple(t.shape)}")
        return t

    def matvec_device(self, v, mu=0.0, out=None):
        """(G + mu I) v for a CUDA tensor v; counts one matvec."""
        torch = _lib.torch_mod()
        self._ensure()
        if out is None:
            out = torch.empty(self.dim, dtype=torch.float64, device=self.ctx.device)
        self.ctx.call("ngd_gram_matvec", _lib.ptr(v), float(mu), _lib.ptr(out))
        self.matvec_count += 1
        return out

    def matvec(self, v):  # gramian.py:48-53
        t = self._vec(v)
        return _lib.like_input(self.matvec_device(t), v)

    def matmat(self, vmat):
        """Y = G V for a (p, ell) block (gramian.py:55-61); counts ell matvecs."""
        torch = _lib.torch_mod()
        self._ensure()
        V = vmat if _lib.is_device_array(vmat) else _lib.to_device(vmat)
        if V.dim() != 2 or V.shape[0] != self.dim:
            raise ValueError(f"expected ({self.dim}, ell) block, got {tuple(V.shape)}")
        ell = V.shape[1]
        Vcm = V.to(torch.float64).t().contiguous()  # (ell, p) row-major == p x ell column-major
        Ycm = torch.empty_like(Vcm)
        self.ctx.call("ngd_gram_matmat", _lib.ptr(Vcm), ell, self.dim, _lib.ptr(Ycm), self.dim)
        self.matvec_count += ell
        return _lib.like_input(Ycm.t(), vmat)

    def matmat_colmajor(self, Vcm, Ycm):
        """Y = G V with both blocks stored column-major as (ell, p) CUDA tensors."""
        self._ensure()
        ell = Vcm.shape[0]
        self.ctx.call("ngd_gram_matmat", _lib.ptr(Vcm), ell, self.dim, _lib.ptr(Ycm), self.dim)
        self.matvec_count += ell
        return Ycm

    def __call__(self, v):
        return self.matvec(v)


_util_ctx = None


def utility_context():
    """A topology-free context for dense operators and vector helpers."""
    global _util_ctx
    if _util_ctx is None:
        _util_ctx = _lib.Context((1, 1))
    return _util_ctx


class DenseOperator:
    """Matvec wrapper around an explicit matrix held on the device (gramian.py:101-120)."""

    def __init__(self, matrix):
        m = matrix if _lib.is_device_array(matrix) else np.asarray(matrix, dtype=float)
        if m.ndim != 2 or m.shape[0] != m.shape[1]:
            raise ValueError("expected a square matrix")
        self.matrix = _lib.to_device(m)  # C-order (row-major)
        self.dim = int(self.matrix.shape[0])
        self.matvec_count = 0
        self.ctx = utility_context()

    def matvec_device(self, v, mu=0.0, out=None):
        torch = _lib.torch_mod()
        out = self.matmat_device(v.reshape(1, -1)).reshape(-1)
        if mu:
            out = out + mu * v
        self.matvec_count -= 0  # counted in matmat_device (1 column)
        return out

    def matmat_device(self, Vcm):
        """Vcm: (ell, p) CUDA tensor = p x ell column-major; returns same layout."""
        torch = _lib.torch_mod()
        ell = Vcm.shape[0]
        Y = torch.empty_like(Vcm)
        self.ctx.call("ngd_dense_matmat", _lib.ptr(self.matrix), self.dim, _lib.ptr(Vcm), ell, _lib.ptr(Y))
        self.matvec_count += ell
        return Y

    def matvec(self, v):
        t = _lib.to_device(v)
        return _lib.like_input(self.matvec_device(t), v)

    def matmat(self, vmat):
        torch = _lib.torch_mod()
        V = _lib.to_device(vmat)
        Y = self.matmat_device(V.t().contiguous())
        return _lib.like_input(Y.t(), vmat)

    def matmat_colmajor(self, Vcm, Ycm):
        Ycm.copy_(self.matmat_device(Vcm))
        return Ycm

    def __call__(self, v):
        return self.matvec(v)


class ShiftedOperator:
    """v -> A v + mu v; matvec counting delegates to the base operator (gramian.py:123-135)."""

    def __init__(self, base, mu):
        self.base = base
        self.mu = float(mu)
        self.dim = base.dim

    def matvec_device(self, v, out=None):
        if hasattr(self.base, "matvec_device"):
            if isinstance(self.base, GramianOperator):
                return self.base.matvec_device(v, mu=self.mu, out=out)
            return self.base.matvec_device(v, mu=self.mu)
        raise TypeError("base operator has no device matvec")

    def matvec(self, v):
        if hasattr(self.base, "matvec_device"):
            t = _lib.to_device(v)
            return _lib.like_input(self.matvec_device(t), v)
        return self.base.matvec(v) + self.mu * v

    def __call__(self, v):
        return self.matvec(v)


def assemble_dense(op, guard=DENSE_GUARD):
    """Assemble an operator densely (gramian.py:138-145).  A Gramian is formed as
    J^T diag(w) J from explicit Jacobian rows with one DSYRK per row chunk
    (ngd_gram_dense); other operators by one matmat of I.  numpy in -> numpy out."""
    p = op.dim
    if p > guard:
        raise ValueError(f"dense assembly guard: p={p} exceeds {guard}")
    if isinstance(op, GramianOperator):
        torch = _lib.torch_mod()
        op._ensure()
        G = torch.empty((p, p), dtype=torch.float64, device=op.ctx.device)
        op.ctx.call("ngd_gram_dense", _lib.ptr(G), p)
        op.matvec_count += p
        return G.cpu().numpy()
    if hasattr(op, "matmat"):
        return np.asarray(_lib.like_input(_lib.to_device(op.matmat(np.eye(p))), np.eye(1)))
    return np.column_stack([op.matvec(np.eye(p)[:, i]) for i in range(p)])


def normalized_spectrum(matrix, top=None):
    """Descending eigenvalues of an SPSD matrix over the largest (harness.py:237-248)."""
    eigs = np.clip(np.linalg.eigvalsh(np.asarray(matrix, dtype=float))[::-1], 0.0, None)
    if eigs[0] == 0.0:
        raise ZeroDivisionError("matrix is identically zero; cannot normalize")
    ratios = eigs / eigs[0]
    return ratios if top is None else ratios[:top]


def gramian_spectrum(problem, theta, quad, top=None):
    """Top normalised eigenvalues of the Gramian (harness.py:249-252), assembled on the device as
    J^T diag(w) J from Jacobian-row chunks on the DMMA GEMM (ngd_gram_dense)."""
    return normalized_spectrum(assemble_dense(GramianOperator.from_problem(problem, theta, quad)), top=top)
