"""Poisson problems with device-resident quadrature (mirror of nystromngd/problems.py).

The quadrature sampling and the data offsets (source f, Dirichlet g) are host
numpy -- seeded INPUT generation, reproducing the reference's RNG streams bit
for bit (problems.py:122-125, 210-232).  Everything evaluated per NGD step --
metric stack, residual, loss, gradient, Gramian -- runs on the GPU through
libngd_b200 (no CPU fallback).

Shipped problems: every problem of the reference registry -- ``poisson1d``,
``poisson2d``, ``heat1p1d``, ``nlpoisson2d`` (problems.py:128-385) -- plus the
N-D Poisson problems of BASELINE C3/C5 (``poisson_nd``: sin-sum or Gaussian
exact solution) and the interior-only Laplacian stack of BASELINE C4.
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


@dataclass(frozen=True)
class DeviceRows:
    """The row set one context evaluates (see ngd_set_rows in include/ngd.h): head rows at
    the interior points, value rows (F = u) at ``x_val``; per row a metric weight ``wm``
    (Gramian), a residual weight ``wr`` (loss / gradient) and a residual offset ``off``.
    ``metric_index`` / ``residual_index`` select each stack's rows, in the reference's
    row order, from the device row order [interior ++ value rows] (None = all rows)."""

    x_int: np.ndarray
    wm_int: np.ndarray
    wr_int: np.ndarray
    off_int: np.ndarray
    x_val: np.ndarray
    wm_val: np.ndarray
    wr_val: np.ndarray
    off_val: np.ndarray
    metric_index: np.ndarray | None = None
    residual_index: np.ndarray | None = None


class PdeProblem:
    """Least-squares PDE problem (problems.py:50-119) evaluated on the device.

    A problem states its stacks as device rows (``device_rows``) plus an output
    head (``head``: coefficients over the output jet channels, the cubic
    coefficient kappa and the second-derivative coordinate mask); the default is
    the Poisson metric [Lap u]_int ++ [u]_bnd.  Device contexts are cached per
    quadrature object (two at a time: training + evaluation quadrature);
    ``shard=(rank, nranks)`` selects a contiguous slice of both row sets.
    """

    name = "abstract"
    metric_kind = "least-squares"
    has_initial = False
    input_dim = None
    interior_only = False
    _MAX_CONTEXTS = 2

    def __init__(self, topology):
        self.topology = topology
        if self.input_dim is not None and topology.input_dim != self.input_dim:
            raise ValueError(f"{self.name} needs input dim {self.input_dim}, topology has {topology.input_dim}")
        if topology.output_dim != 1:
            raise ValueError("scalar-output networks only")
        self._ctxs = []  # [(weakref(quad), Context, DeviceRows)], most recent last
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
        """residual - metric = [f]_int ++ [-g]_bnd (problems.py:161-166); linear problems only."""
        return np.concatenate([self.source(quad.interior_points), -self.dirichlet(quad.boundary_points)])

    def head(self):
        """(coef over output channels [u, d_1 u..d_d u, Lambda], kappa, Lambda coordinate mask)."""
        d = self.topology.input_dim
        coef = np.zeros(d + 2)
        coef[-1] = 1.0
        return coef, 0.0, (1 << d) - 1

    def device_rows(self, quad):
        """Poisson-type stacks: metric and residual share the rows (problems.py:161-177)."""
        xi, xb = quad.interior_points, quad.boundary_points
        wi, wb = quad.interior_weights, quad.boundary_weights
        fi = self.source(xi) if len(xi) else np.zeros(0)
        gb = -self.dirichlet(xb) if len(xb) else np.zeros(0)
        return DeviceRows(xi, wi, wi, fi, xb, wb, wb, gb)

    # -- device context --------------------------------------------------------
    def _entry(self, quad):
        for i, (ref, ctx, rows) in enumerate(self._ctxs):
            if ref() is quad:
                if i != len(self._ctxs) - 1:
                    self._ctxs.append(self._ctxs.pop(i))
                return ctx, rows
        return None

    def context(self, quad):
        """The libngd context holding this quadrature's rows (cached)."""
        hit = self._entry(quad)
        if hit is not None:
            return hit[0]
        live = [e for e in self._ctxs if e[0]() is not None]
        if len(live) >= self._MAX_CONTEXTS or len(live) < len(self._ctxs):
            # reuse the least recently used (or orphaned) context's workspace
            dead = [e for e in self._ctxs if e[0]() is None]
            victim = dead[0] if dead else self._ctxs[0]
            self._ctxs.remove(victim)
            ctx = victim[1]
        else:
            ctx = _lib.Context(self.topology.widths)
            if self.comm is not None:
                self.comm.bind(ctx)
        rows = self.device_rows(quad)
        rank, nranks = self.shard
        xi, wmi, wri, oi = rows.x_int, rows.wm_int, rows.wr_int, rows.off_int
        xv, wmv, wrv, ov = rows.x_val, rows.wm_val, rows.wr_val, rows.off_val
        ctx._int_slice = slice(0, len(xi))
        if nranks > 1:
            from .distributed import shard_slices

            si, sv = shard_slices(len(xi), len(xv), rank, nranks)
            ctx._int_slice = si
            xi, wmi, wri, oi = xi[si], wmi[si], wri[si], oi[si]
            xv, wmv, wrv, ov = xv[sv], wmv[sv], wrv[sv], ov[sv]
        d = self.topology.input_dim
        t = [_lib.to_device(np.asarray(a, dtype=float).reshape(shape)) for a, shape in (
            (xi, (-1, d)), (wmi, (-1,)), (wri, (-1,)), (oi, (-1,)),
            (xv, (-1, d)), (wmv, (-1,)), (wrv, (-1,)), (ov, (-1,)))]
        ctx.call("ngd_set_rows", len(xi), *[_lib.ptr(x) for x in t[:4]], len(xv), *[_lib.ptr(x) for x in t[4:]])
        coef, kappa, mask = self.head()
        hc = (_lib.ctypes.c_double * len(coef))(*[float(c) for c in coef])
        ctx.call("ngd_set_head", hc, len(coef), float(kappa), int(mask))
        ctx.stream.synchronize()
        ctx._keep = t
        ctx.lin_owner = None
        self._ctxs.append((weakref.ref(quad), ctx, rows))
        return ctx

    def _rows(self, quad):
        self.context(quad)
        return self._entry(quad)[1]

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

    def _stacks(self, theta, theta_bar, quad):
        torch = _lib.torch_mod()
        ctx = self.context(quad)
        rows = self._rows(quad)
        if self.shard[1] > 1:
            raise NotImplementedError("stack values on a sharded problem")
        th = _lib.to_device(theta)
        tb = None
        if theta_bar is not None:
            tb = _lib.to_device(theta_bar)
            if tb.data_ptr() == th.data_ptr() or torch.equal(tb, th):
                tb = None
        n = len(rows.x_int) + len(rows.x_val)
        metric = torch.empty(n, dtype=torch.float64, device=ctx.device)
        resid = torch.empty(n, dtype=torch.float64, device=ctx.device)
        loss = _lib.ctypes.c_double()
        ctx.call("ngd_linearize_ex", _lib.ptr(th), _lib.ptr(tb), _lib.ctypes.byref(loss), _lib.ptr(metric),
                 _lib.ptr(resid))
        ctx.lin_token += 1
        ctx.lin_owner = None
        return rows, metric, resid

    def metric_stack(self, theta, theta_bar, quad):
        """Metric rows at theta, nonlinear coefficients frozen at theta_bar (gramian.py:36-40)."""
        rows, metric, _ = self._stacks(theta, theta_bar, quad)
        if rows.metric_index is not None:
            metric = metric[_lib.to_device(rows.metric_index).long()]
        return _lib.like_input(metric, theta)

    def residual_stack(self, theta, quad):
        rows, _, resid = self._stacks(theta, None, quad)
        if rows.residual_index is not None:
            resid = resid[_lib.to_device(rows.residual_index).long()]
        return _lib.like_input(resid, theta)

    def h1_relative_error(self, theta, quad):
        """Relative H1 error at the interior points (problems.py:104-119), on the device; on a
        sharded problem each rank sums its interior shard and the C-ABI all-reduces both sums."""
        ctx = self.context(quad)
        key = "_h1_exact"
        ex = getattr(ctx, key, None)
        if ex is None or ex[0] is not quad:
            x = quad.interior_points[ctx._int_slice]
            tab = np.concatenate([self.exact(x)[:, None], self.exact_grad(x).reshape(len(x), -1)], axis=1)
            ex = (quad, _lib.to_device(tab))
            setattr(ctx, key, ex)
        out = _lib.ctypes.c_double()
        ctx.call("ngd_h1_error", _lib.ptr(_lib.to_device(theta)), _lib.ptr(ex[1]), _lib.ctypes.byref(out))
        return float(out.value)


class Poisson1D(PdeProblem):
    """-u'' = f on (0,1), u = 0 at the endpoints; u* = sin(pi x) (problems.py:128-177)."""

    name = "poisson1d"
    input_dim = 1

    def exact(self, x):
        return np.sin(np.pi * x[:, 0])

    def exact_grad(self, x):
        return np.pi * np.cos(np.pi * x[:, 0])[:, None]

    def source(self, x):
        return np.pi**2 * np.sin(np.pi * x[:, 0])

    def sample_quadrature(self, n_interior, n_boundary, seed):
        # the 1D boundary is the two endpoints with unit counting weights (n_boundary unused)
        rng = np.random.default_rng(seed)
        pts = _uniform_box(rng, n_interior, [0.0], [1.0])
        return QuadratureSet(pts, np.full(n_interior, 1.0 / n_interior), np.array([[0.0], [1.0]]), np.ones(2))


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


class Heat1p1D(PdeProblem):
    """u_t - u_xx = f on (t,x) in (0,1)^2; u* = cos(pi x) exp(-pi^2 t / 4) (problems.py:235-331).

    Residual [u_t - u_xx - f]_int ++ [u - g]_lateral ++ [u - u0]_initial; metric
    [u_t - u_xx]_int ++ [u]_int (bulk) ++ [u]_initial.  Device rows: head rows
    (coef = e_{d_t} - e_Lambda, Lambda over {x}) at the interior points; value rows
    [bulk | lateral | initial] with metric weights [w_int | 0 | w_0] and residual
    weights [0 | w_b | w_0].
    """

    name = "heat1p1d"
    input_dim = 2
    has_initial = True

    def exact(self, x):
        return np.cos(np.pi * x[:, 1]) * np.exp(-np.pi**2 * x[:, 0] / 4.0)

    def exact_grad(self, x):
        u = self.exact(x)
        dt = -np.pi**2 / 4.0 * u
        dx = -np.pi * np.sin(np.pi * x[:, 1]) * np.exp(-np.pi**2 * x[:, 0] / 4.0)
        return np.stack([dt, dx], axis=1)

    def source(self, x):
        return 0.75 * np.pi**2 * self.exact(x)

    def initial_value(self, x):
        return np.cos(np.pi * x[:, 1])

    def sample_quadrature(self, n_interior, n_boundary, seed):  # problems.py:266-287
        rng = np.random.default_rng(seed)
        pts = _uniform_box(rng, n_interior, [0.0, 0.0], [1.0, 1.0])
        t = rng.random(n_boundary)
        side = rng.integers(0, 2, n_boundary).astype(float)
        bnd = np.stack([t, side], axis=1)
        n_init = max(n_boundary // 2, 1)
        xi = rng.random(n_init)
        init = np.stack([np.zeros(n_init), xi], axis=1)
        return QuadratureSet(pts, np.full(n_interior, 1.0 / n_interior), bnd, np.full(n_boundary, 2.0 / n_boundary),
                             init, np.full(n_init, 1.0 / n_init))

    def residual_weights(self, quad):
        return np.concatenate([quad.interior_weights, quad.boundary_weights, quad.initial_weights])

    def metric_weights(self, quad):
        return np.concatenate([quad.interior_weights, quad.interior_weights, quad.initial_weights])

    def data_offsets(self, quad):
        raise TypeError("heat1p1d: metric and residual stacks have different rows")

    def head(self):
        # channels [u, d_t u, d_x u, Lambda]; Lambda = d_xx u (mask: coordinate 1)
        return np.array([0.0, 1.0, 0.0, -1.0]), 0.0, 0b10

    def device_rows(self, quad):
        xi, wi = quad.interior_points, quad.interior_weights
        xb, wb = quad.boundary_points, quad.boundary_weights
        x0, w0 = quad.initial_points, quad.initial_weights
        ni, nb, n0 = len(xi), len(xb), len(x0)
        x_val = np.concatenate([xi, xb, x0])
        wm_val = np.concatenate([wi, np.zeros(nb), w0])
        wr_val = np.concatenate([np.zeros(ni), wb, w0])
        off_val = np.concatenate([np.zeros(ni), -self.dirichlet(xb), -self.initial_value(x0)])
        head = np.arange(ni)
        metric_index = np.concatenate([head, ni + np.arange(ni), ni + ni + nb + np.arange(n0)])
        residual_index = np.concatenate([head, ni + ni + np.arange(nb + n0)])
        return DeviceRows(xi, wi, wi, -self.source(xi), x_val, wm_val, wr_val, off_val, metric_index, residual_index)


class NonlinearPoisson2D(Poisson2D):
    """-Laplace(u) + u^3 = f on (0,1)^2 with a Gauss-Newton metric (problems.py:334-385).

    Residual Lap u - u^3 + f; metric row Lap u - 3 ubar^2 u with ubar frozen at
    the linearisation point (head kappa = -1)."""

    name = "nlpoisson2d"
    metric_kind = "gauss-newton"

    def source(self, x):
        u = self.exact(x)
        return 2.0 * np.pi**2 * u + u**3

    def head(self):
        return np.array([0.0, 0.0, 0.0, 1.0]), -1.0, 0b11

    def data_offsets(self, quad):
        raise TypeError("nlpoisson2d: the residual is not metric + offsets")


_PROBLEMS = {cls.name: cls for cls in (Poisson1D, Poisson2D, Heat1p1D, NonlinearPoisson2D, LaplacianStack)}
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
