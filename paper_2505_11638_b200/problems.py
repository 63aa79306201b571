"""Poisson problems with device-resident quadrature (mirror of nystromngd/problems.py).

The quadrature sampling and the data offsets (source f, Dirichlet g) are host
numpy -- seeded INPUT generation, reproducing the reference's RNG streams bit
for bit (problems.py:122-125, 210-232).  Everything evaluated per NGD step --
metric stack, residual, loss, gradient, Gramian -- runs on the GPU through
libngd_b200 (no CPU fallback).

Shipped problems: ``poisson2d`` (problems.py:190-219) and the N-D Poisson
problems of BASELINE C3/C5 (``poisson_nd``: sin-sum or Gaussian exact
solution), plus the interior-only Laplacian stack of BASELINE C4.
"""

from __future__ import annotations

import weakref
from dataclasses import dataclass

import numpy as np

from . import _lib
from .model import MlpTopology


@dataclass(frozen=True)
class QuadratureSet:
    """Fixed Monte-Carlo quadrature (problems.py:34-48)."""

    interior_points: np.ndarray
    interior_weights: np.ndarray
    boundary_points: np.ndarray
    boundary_weights: np.ndarray
    initial_points: np.ndarray | None = None
    initial_weights: np.ndarray | None = None

    def __post_init__(self):
        for w in (self.interior_weights, self.boundary_weights, self.initial_weights):
            if w is not None and np.any(np.asarray(w) <= 0):
                raise ValueError("quadrature weights must be positive")


def _uniform_box(rng, n, lo, hi):  # problems.py:122-125
    lo = np.asarray(lo, dtype=float)
    hi = np.asarray(hi, dtype=float)
    return lo + (hi - lo) * rng.random((n, lo.shape[0]))


def _unit_square_boundary(rng, n):  # problems.py:222-232
    s = 4.0 * rng.random(n)
    pts = np.empty((n, 2))
    side = np.minimum(s.astype(int), 3)
    t = s - side
    pts[side == 0] = np.stack([t[side == 0], np.zeros(np.sum(side == 0))], axis=1)
    pts[side == 1] = np.stack([np.ones(np.sum(side == 1)), t[side == 1]], axis=1)
    pts[side == 2] = np.stack([1.0 - t[side == 2], np.ones(np.sum(side == 2))], axis=1)
    pts[side == 3] = np.stack([np.zeros(np.sum(side == 3)), 1.0 - t[side == 3]], axis=1)
    return pts


def _hypercube_boundary(rng, n, d):
    """Uniform on the 2d faces of [0,1]^d (random face, normal coordinate pinned)."""
    face = rng.integers(0, 2 * d, size=n)
    pts = rng.random((n, d))
    pts[np.arange(n), face // 2] = (face % 2).astype(float)
    return pts


class PdeProblem:
    """Least-squares PDE problem whose metric stack is [Lap u]_int ++ [u]_bnd.

    Device contexts are cached per quadrature object; ``shard=(rank, nranks)``
    selects a contiguous slice of interior and boundary points.
    """

    name = "abstract"
    metric_kind = "least-squares"
    has_initial = False
    input_dim = None
    interior_only = False

    def __init__(self, topology):
        self.topology = topology
        if self.input_dim is not None and topology.input_dim != self.input_dim:
            raise ValueError(f"{self.name} needs input dim {self.input_dim}, topology has {topology.input_dim}")
        if topology.output_dim != 1:
            raise ValueError("scalar-output networks only")
        self._ctx = None
        self._ctx_quad = None
        self.shard = (0, 1)
        self.comm = None  # set by distributed.attach

    # -- data (host, per quadrature) ------------------------------------------
    def exact(self, x):
        raise NotImplementedError

    def exact_grad(self, x):
        raise NotImplementedError

    def source(self, x):
        raise NotImplementedError

    def dirichlet(self, x):
        return self.exact(x)

    def metric_weights(self, quad):  # problems.py:174-177
        return np.concatenate([quad.interior_weights, quad.boundary_weights])

    residual_weights = metric_weights

    def data_offsets(self, quad):
        """residual - metric = [f]_int ++ [-g]_bnd (problems.py:161-166)."""
        return np.concatenate([self.source(quad.interior_points), -self.dirichlet(quad.boundary_points)])

    # -- device context --------------------------------------------------------
    def context(self, quad):
        """The libngd context holding this quadrature's points (cached)."""
        if self._ctx is not None and self._ctx_quad is not None and self._ctx_quad() is quad:
            return self._ctx
        if self._ctx is None:
            self._ctx = _lib.Context(self.topology.widths)
            if self.comm is not None:
                self.comm.bind(self._ctx)
        rank, nranks = self.shard
        xi, wi = quad.interior_points, quad.interior_weights
        xb, wb = quad.boundary_points, quad.boundary_weights
        fi = self.source(xi) if len(xi) else np.zeros(0)
        gb = -self.dirichlet(xb) if len(xb) else np.zeros(0)
        if nranks > 1:
            from .distributed import shard_slices

            si, sb = shard_slices(len(xi), len(xb), self.topology.input_dim + 2, rank, nranks)
            xi, wi, fi = xi[si], wi[si], fi[si]
            xb, wb, gb = xb[sb], wb[sb], gb[sb]
        d = self.topology.input_dim
        t = [_lib.to_device(np.asarray(a, dtype=float).reshape(shape)) for a, shape in (
            (xi, (-1, d)), (wi, (-1,)), (fi, (-1,)), (xb, (-1, d)), (wb, (-1,)), (gb, (-1,)))]
        self._ctx.call("ngd_set_points", len(xi), _lib.ptr(t[0]), _lib.ptr(t[1]), _lib.ptr(t[2]),
                       len(xb), _lib.ptr(t[3]), _lib.ptr(t[4]), _lib.ptr(t[5]))
        self._ctx.stream.synchronize()
        self._ctx._keep = t
        self._ctx_quad = weakref.ref(quad)
        self._ctx.lin_owner = None
        return self._ctx

    # -- loss / gradient (problems.py:92-102) -----------------------------------
    def loss_value(self, theta, quad):
        ctx = self.context(quad)
        th = _lib.to_device(theta)
        out = _lib.ctypes.c_double()
        ctx.call("ngd_loss", _lib.ptr(th), _lib.ctypes.byref(out))
        return float(out.value)

    def linearize(self, theta, quad, owner=None):
        """Linearise the metric stack at theta on the device; returns the loss."""
        ctx = self.context(quad)
        th = _lib.to_device(theta)
        out = _lib.ctypes.c_double()
        ctx.call("ngd_linearize", _lib.ptr(th), _lib.ctypes.byref(out), None)
        ctx.lin_token += 1
        ctx.lin_owner = owner
        return float(out.value)

    def loss_grad(self, theta, quad):
        torch = _lib.torch_mod()
        ctx = self.context(quad)
        self.linearize(theta, quad)
        g = torch.empty(ctx.p, dtype=torch.float64, device=ctx.device)
        ctx.call("ngd_loss_grad", _lib.ptr(g))
        return _lib.like_input(g, theta)

    def metric_stack(self, theta, theta_bar, quad):
        torch = _lib.torch_mod()
        ctx = self.context(quad)
        th = _lib.to_device(theta)
        n = len(quad.interior_points) + len(quad.boundary_points)
        if self.shard[1] > 1:
            raise NotImplementedError("metric_stack on a sharded problem")
        out = torch.empty(n, dtype=torch.float64, device=ctx.device)
        loss = _lib.ctypes.c_double()
        ctx.call("ngd_linearize", _lib.ptr(th), _lib.ctypes.byref(loss), _lib.ptr(out))
        ctx.lin_token += 1
        ctx.lin_owner = None
        return _lib.like_input(out, theta)

    def residual_stack(self, theta, quad):
        m = self.metric_stack(theta, None, quad)
        off = self.data_offsets(quad)
        if _lib.is_device_array(m):
            return m + _lib.to_device(off)
        return m + off


class Poisson2D(PdeProblem):
    """-Laplace(u) = f on (0,1)^2; u* = sin(pi x) sin(pi y) (problems.py:190-219)."""

    name = "poisson2d"
    input_dim = 2

    def exact(self, x):
        return np.sin(np.pi * x[:, 0]) * np.sin(np.pi * x[:, 1])

    def exact_grad(self, x):
        sx, cx = np.sin(np.pi * x[:, 0]), np.cos(np.pi * x[:, 0])
        sy, cy = np.sin(np.pi * x[:, 1]), np.cos(np.pi * x[:, 1])
        return np.pi * np.stack([cx * sy, sx * cy], axis=1)

    def source(self, x):
        return 2.0 * np.pi**2 * self.exact(x)

    def sample_quadrature(self, n_interior, n_boundary, seed):
        rng = np.random.default_rng(seed)
        pts = _uniform_box(rng, n_interior, [0.0, 0.0], [1.0, 1.0])
        bnd = _unit_square_boundary(rng, n_boundary)
        return QuadratureSet(pts, np.full(n_interior, 1.0 / n_interior), bnd, np.full(n_boundary, 4.0 / n_boundary))


class PoissonND(PdeProblem):
    """-Laplace(u) = f on (0,1)^d (BASELINE C3/C5; not in the reference).

    kind='sinsum': u* = sum_i sin(pi x_i);  kind='gauss': u* = exp(-|x|^2/10).
    Boundary points uniform on the 2d faces, weights 2d/N_bnd.
    """

    name = "poisson_nd"

    def __init__(self, topology, kind="sinsum"):
        if kind not in ("sinsum", "gauss"):
            raise ValueError(f"unknown exact solution {kind!r}")
        self.kind = kind
        self.input_dim = topology.input_dim
        super().__init__(topology)

    def exact(self, x):
        if self.kind == "sinsum":
            return np.sum(np.sin(np.pi * x), axis=1)
        return np.exp(-np.sum(x * x, axis=1) / 10.0)

    def exact_grad(self, x):
        if self.kind == "sinsum":
            return np.pi * np.cos(np.pi * x)
        return -x / 5.0 * self.exact(x)[:, None]

    def source(self, x):
        if self.kind == "sinsum":
            return np.pi**2 * np.sum(np.sin(np.pi * x), axis=1)
        r2 = np.sum(x * x, axis=1)
        return (self.input_dim / 5.0 - r2 / 25.0) * self.exact(x)

    def sample_quadrature(self, n_interior, n_boundary, seed):
        d = self.input_dim
        rng = np.random.default_rng(seed)
        pts = _uniform_box(rng, n_interior, np.zeros(d), np.ones(d))
        bnd = _hypercube_boundary(rng, n_boundary, d) if n_boundary else np.zeros((0, d))
        return QuadratureSet(pts, np.full(n_interior, 1.0 / n_interior), bnd,
                             np.full(n_boundary, 2.0 * d / max(n_boundary, 1)))


class LaplacianStack(Poisson2D):
    """Interior-only metric [Lap u(x_r)] with weights 1/N (BASELINE C4 microbench;
    the reference builds it with GramianOperator.from_stack, gramian.py:43-46)."""

    name = "laplacian2d"
    interior_only = True

    def sample_quadrature(self, n_interior, n_boundary=0, seed=0):
        x = np.random.default_rng(seed).random((n_interior, 2))
        return QuadratureSet(x, np.full(n_interior, 1.0 / n_interior), np.zeros((0, 2)), np.zeros(0))


_PROBLEMS = {cls.name: cls for cls in (Poisson2D, LaplacianStack)}
PROBLEM_NAMES = tuple(sorted(_PROBLEMS)) + ("poisson_nd",)


def make_problem(name, topology=None, hidden_width=32, hidden_depth=2, kind="sinsum", input_dim=5):
    """Instantiate a problem by name with a default tanh MLP (problems.py:395-403)."""
    if name == "poisson_nd":
        if topology is None:
            topology = MlpTopology((input_dim,) + (hidden_width,) * hidden_depth + (1,))
        return PoissonND(topology, kind)
    if name not in _PROBLEMS:
        raise KeyError(f"unknown problem {name!r}; available: {PROBLEM_NAMES}")
    cls = _PROBLEMS[name]
    if topology is None:
        topology = MlpTopology((cls.input_dim,) + (hidden_width,) * hidden_depth + (1,))
    return cls(topology)
