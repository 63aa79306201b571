"""CPU oracle for the NystromNGD inner solve -- TEST INFRASTRUCTURE ONLY.

This module is the *checker*, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference``
legs of ``bench.py`` may import it.  The shipped path
(``paper_2505_11638_b200``) must never import, call or fall back to it.

It is a numpy/scipy restatement of the reference algorithm
(``/root/reference/pkg/src/nystromngd``, "the reference" below), written from
the reference's equations, vectorised over collocation points.  Each function
cites the reference file:line it follows.  Parity is PINNED: the fixtures in
``tests/golden/`` were produced by running the live reference
(``tests/golden/make_golden.py``) and ``tests/test_oracle_golden.py`` checks
this module against them.

Restated pieces
* MLP layout / init / forward / second-order input jets
  (model.py:34-60, 94-124; autodiff.py:621-666)
* Poisson metric & residual stacks, weights, loss (problems.py:92-99, 161-232)
  plus the N-D Poisson problems BASELINE configs C3/C5 need
* Linearised metric map: JVP (tangent sweep) and VJP (adjoint sweep) through
  the jets -- the arithmetic the reference's tape performs
  (autodiff.py:81-125, 587-613; gramian.py:48-61)
* nystrom_approximate / NystromPreconditioner (sketch.py:58-112)
* pcg (krylov.py:24-88)
* adapt_mu / adapt_rank / Armijo line search / nystrom_ngd_run (optim.py:86-270)
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np
import scipy.linalg

EPS = np.finfo(float).eps  # optim.py:19, sketch.py:77


# ---------------------------------------------------------------------------
# Model (model.py)
# ---------------------------------------------------------------------------


class Topology:
    """Layer widths (n0, ..., n_{L+1}); tanh on hidden layers (model.py:12-51)."""

    def __init__(self, widths):
        self.widths = tuple(int(w) for w in widths)
        if len(self.widths) < 2 or min(self.widths) < 1:
            raise ValueError("bad widths")

    @property
    def input_dim(self):
        return self.widths[0]

    @property
    def param_count(self):  # model.py:34-39
        return sum(o * i + o for i, o in zip(self.widths[:-1], self.widths[1:]))

    def layer_slices(self):  # model.py:41-51: per layer W (n_out, n_in) row-major, then b
        out, off = [], 0
        for n_in, n_out in zip(self.widths[:-1], self.widths[1:]):
            ws = slice(off, off + n_out * n_in)
            off += n_out * n_in
            bs = slice(off, off + n_out)
            off += n_out
            out.append((ws, bs, n_out, n_in))
        return out

    def unflatten(self, theta):  # model.py:53-60
        return [(theta[ws].reshape(n_out, n_in), theta[bs]) for ws, bs, n_out, n_in in self.layer_slices()]


def init_theta(widths, seed):
    """Weights ~ N(0, 1/fan_in) drawn layer by layer, biases 0 (model.py:94-100)."""
    top = Topology(widths)
    rng = np.random.default_rng(seed)
    theta = np.zeros(top.param_count)
    for ws, _, n_out, n_in in top.layer_slices():
        theta[ws] = rng.standard_normal(n_out * n_in) / np.sqrt(n_in)
    return theta


def mlp_forward(widths, theta, x):
    """u(x) for x (q, d) (model.py:103-124)."""
    layers = Topology(widths).unflatten(theta)
    z = np.asarray(x, dtype=float)
    for k, (w, b) in enumerate(layers):
        z = z @ w.T + b
        if k < len(layers) - 1:
            z = np.tanh(z)
    return z.reshape(z.shape[0])


def mlp_jets(widths, theta, x):
    """Value, input gradient and per-coordinate second derivatives
    (autodiff.py:621-666, same operation order)."""
    layers = Topology(widths).unflatten(theta)
    x = np.asarray(x, dtype=float)
    q, d = x.shape
    z = x
    g = [np.broadcast_to(np.eye(d)[i], (q, d)).copy() for i in range(d)]
    h = [np.zeros((q, d)) for _ in range(d)]
    for k, (w, b) in enumerate(layers):
        z = z @ w.T + b
        g = [gi @ w.T for gi in g]
        h = [hi @ w.T for hi in h]
        if k < len(layers) - 1:
            t = np.tanh(z)
            d1 = 1.0 - t * t
            d2 = -2.0 * t * d1
            h = [d2 * gi * gi + d1 * hi for gi, hi in zip(g, h)]
            g = [d1 * gi for gi in g]
            z = t
    value = z.reshape(q)
    grad = np.stack([gi.reshape(q) for gi in g], axis=1)
    second = np.stack([hi.reshape(q) for hi in h], axis=1)
    return value, grad, second


# ---------------------------------------------------------------------------
# Problems (problems.py)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class Quadrature:
    """Fixed Monte-Carlo quadrature (problems.py:34-48)."""

    interior_points: np.ndarray
    interior_weights: np.ndarray
    boundary_points: np.ndarray
    boundary_weights: np.ndarray
    initial_points: np.ndarray | None = None
    initial_weights: np.ndarray | None = None


def _uniform_box(rng, n, d):  # problems.py:122-125 on the unit box
    lo = np.zeros(d)
    hi = np.ones(d)
    return lo + (hi - lo) * rng.random((n, d))


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
    """Uniform on the 2d faces of [0,1]^d: a random face, its normal coordinate
    pinned to 0/1 (not in the reference, D6)."""
    face = rng.integers(0, 2 * d, size=n)
    pts = rng.random((n, d))
    pts[np.arange(n), face // 2] = (face % 2).astype(float)
    return pts


@dataclass
class StackRows:
    """A metric or residual stack in the two row kinds every reference problem uses.

    * head rows at ``x_int``: F = alpha*u + sum_i beta_i d_i u + sum_i gamma_i d_ii u
      (Laplacian: gamma = 1; heat operator u_t - u_xx: beta = e_t, gamma = -e_x;
      nonlinear Poisson Gauss-Newton row: gamma = 1, alpha = -3 ubar^2 per point),
    * value rows at ``x_val``: F = u.
    """

    x_int: np.ndarray
    alpha: np.ndarray | float
    beta: np.ndarray
    gamma: np.ndarray
    x_val: np.ndarray


class StackProblem:
    """Least-squares problem from a residual stack (problems.py:50-119)."""

    has_initial = False

    def residual_stack(self, theta, quad):
        raise NotImplementedError

    def stack_rows(self, theta, theta_bar, quad, which):
        raise NotImplementedError

    def metric_stack(self, theta, quad, theta_bar=None):  # gramian.py:33-41 (metric frozen at theta_bar)
        return Linearization(self, theta, quad, "metric", theta_bar).value

    def loss_value(self, theta, quad):  # problems.py:92-99
        r = self.residual_stack(theta, quad)
        w = self.residual_weights(quad)
        return float(0.5 * np.sum(w * r * r))

    def loss_grad(self, theta, quad):  # problems.py:101-102: grad of the loss = J_res^T (w * r)
        lin = Linearization(self, theta, quad, "residual")
        return lin.vjp(self.residual_weights(quad) * self.residual_stack(theta, quad))

    def h1_relative_error(self, theta, quad):  # problems.py:104-119 (space-time gradient for heat)
        x, w = quad.interior_points, quad.interior_weights
        u, gu, _ = mlp_jets(self.widths, theta, x)
        ue, ge = self.exact(x), self.exact_grad(x)
        num = np.sum(w * (u - ue) ** 2) + np.sum(w * np.sum((gu - ge) ** 2, axis=1))
        den = np.sum(w * ue**2) + np.sum(w * np.sum(ge**2, axis=1))
        if den == 0.0:
            raise ZeroDivisionError("exact solution has zero H1 norm")
        return float(np.sqrt(num / den))


class PoissonProblem(StackProblem):
    """-Laplace(u) = f on (0,1)^d with Dirichlet data.

    kind = 'sin2d'  : Poisson2D, u* = sin(pi x) sin(pi y)        (problems.py:190-219)
    kind = 'sin1d'  : Poisson1D, u* = sin(pi x), boundary = the two endpoints with
                      unit weights                                (problems.py:128-177)
    kind = 'sinsum' : u* = sum_i sin(pi x_i)                     (BASELINE C3)
    kind = 'gauss'  : u* = exp(-|x|^2/10)                          (BASELINE C5)
    interior_only   : metric/residual stack without boundary rows (BASELINE C4,
                      the reference's GramianOperator.from_stack, gramian.py:43-46)

    Metric stack [Lap u(x_r)]_int ++ [u(x_s)]_bnd, residual [Lap u + f] ++ [u - g],
    weights 1/N_int ++ |dOmega|/N_bnd (problems.py:161-177).
    """

    def __init__(self, widths, kind="sin2d", interior_only=False):
        self.topology = Topology(widths)
        self.widths = self.topology.widths
        self.d = self.widths[0]
        self.kind = kind
        self.interior_only = interior_only
        if kind == "sin2d" and self.d != 2:
            raise ValueError("sin2d needs d = 2")
        if kind == "sin1d" and self.d != 1:
            raise ValueError("sin1d needs d = 1")

    # exact solution and data ------------------------------------------------
    def exact(self, x):
        if self.kind == "sin2d":
            return np.sin(np.pi * x[:, 0]) * np.sin(np.pi * x[:, 1])
        if self.kind in ("sinsum", "sin1d"):
            return np.sum(np.sin(np.pi * x), axis=1)
        return np.exp(-np.sum(x * x, axis=1) / 10.0)

    def exact_grad(self, x):
        if self.kind == "sin2d":
            sx, cx = np.sin(np.pi * x[:, 0]), np.cos(np.pi * x[:, 0])
            sy, cy = np.sin(np.pi * x[:, 1]), np.cos(np.pi * x[:, 1])
            return np.pi * np.stack([cx * sy, sx * cy], axis=1)
        if self.kind in ("sinsum", "sin1d"):
            return np.pi * np.cos(np.pi * x)
        return -x / 5.0 * self.exact(x)[:, None]

    def source(self, x):
        if self.kind == "sin2d":
            return 2.0 * np.pi**2 * self.exact(x)  # problems.py:211-212
        if self.kind in ("sinsum", "sin1d"):
            return np.pi**2 * np.sum(np.sin(np.pi * x), axis=1)  # problems.py:147-148 for d = 1
        r2 = np.sum(x * x, axis=1)
        return (self.d / 5.0 - r2 / 25.0) * self.exact(x)

    def dirichlet(self, x):
        return self.exact(x)

    def boundary_measure(self):
        return 4.0 if self.d == 2 else 2.0 * self.d

    def sample_quadrature(self, n_interior, n_boundary, seed):
        """problems.py:210-219 for d=2, 150-159 for d=1; the hypercube analogue otherwise."""
        rng = np.random.default_rng(seed)
        pts = _uniform_box(rng, n_interior, self.d)
        if self.kind == "sin1d":
            return Quadrature(pts, np.full(n_interior, 1.0 / n_interior), np.array([[0.0], [1.0]]), np.ones(2))
        if self.interior_only or n_boundary == 0:
            bnd = np.zeros((0, self.d))
            wb = np.zeros(0)
        else:
            bnd = _unit_square_boundary(rng, n_boundary) if self.d == 2 else _hypercube_boundary(rng, n_boundary, self.d)
            wb = np.full(n_boundary, self.boundary_measure() / n_boundary)
        return Quadrature(pts, np.full(n_interior, 1.0 / n_interior), bnd, wb)

    # stacks ------------------------------------------------------------------
    def metric_weights(self, quad):  # problems.py:174-177
        return np.concatenate([quad.interior_weights, quad.boundary_weights])

    residual_weights = metric_weights

    def stack_rows(self, theta, theta_bar, quad, which):  # problems.py:161-172: same rows both stacks
        return StackRows(quad.interior_points, 0.0, np.zeros(self.d), np.ones(self.d), quad.boundary_points)

    def data_offsets(self, quad):
        """Residual minus metric stack: [f]_int ++ [-g]_bnd (problems.py:161-166)."""
        return np.concatenate([self.source(quad.interior_points), -self.dirichlet(quad.boundary_points)])

    def residual_stack(self, theta, quad):  # problems.py:161-166
        _, _, sec = mlp_jets(self.widths, theta, quad.interior_points)
        interior = np.sum(sec, axis=1) + self.source(quad.interior_points)
        if len(quad.boundary_points):
            boundary = mlp_forward(self.widths, theta, quad.boundary_points) - self.dirichlet(quad.boundary_points)
        else:
            boundary = np.zeros(0)
        return np.concatenate([interior, boundary])

    def loss_grad(self, theta, quad):  # linear stack: residual = metric + offsets
        lin = Linearization(self, theta, quad)
        r = lin.value + self.data_offsets(quad)
        return lin.vjp(self.residual_weights(quad) * r)


class NonlinearPoissonProblem(PoissonProblem):
    """-Laplace(u) + u^3 = f on (0,1)^2, Gauss-Newton metric (problems.py:334-385).

    Residual [Lap u - u^3 + f]_int ++ [u - g]_bnd; metric rows
    [Lap u - 3 ubar^2 u]_int ++ [u]_bnd with ubar = u_{theta_bar} frozen.
    """

    def __init__(self, widths):
        super().__init__(widths, kind="sin2d")

    def source(self, x):  # problems.py:350-352
        u = self.exact(x)
        return 2.0 * np.pi**2 * u + u**3

    def residual_stack(self, theta, quad):  # problems.py:354-362
        _, _, sec = mlp_jets(self.widths, theta, quad.interior_points)
        u = mlp_forward(self.widths, theta, quad.interior_points)
        interior = np.sum(sec, axis=1) - u**3 + self.source(quad.interior_points)
        boundary = mlp_forward(self.widths, theta, quad.boundary_points) - self.dirichlet(quad.boundary_points)
        return np.concatenate([interior, boundary])

    def stack_rows(self, theta, theta_bar, quad, which):  # problems.py:364-373
        # the residual's Jacobian at theta is the metric row frozen at theta_bar = theta
        ref = theta if which == "residual" else theta_bar
        ubar = mlp_forward(self.widths, ref, quad.interior_points)
        return StackRows(quad.interior_points, -3.0 * ubar**2, np.zeros(2), np.ones(2), quad.boundary_points)

    def data_offsets(self, quad):
        raise TypeError("the nonlinear Poisson residual is not metric + offsets")

    loss_grad = StackProblem.loss_grad


class HeatProblem(StackProblem):
    """u_t - u_xx = f on (t,x) in (0,1)^2, u* = cos(pi x) exp(-pi^2 t/4) (problems.py:235-331).

    Residual [u_t - u_xx - f]_int ++ [u - g]_lateral ++ [u - u0]_initial with weights
    [1/N, 2/N_b, 1/N_0]; metric [u_t - u_xx]_int ++ [u]_int (bulk) ++ [u]_initial with
    weights [1/N, 1/N, 1/N_0] -- the two stacks have different row sets.
    """

    has_initial = True

    def __init__(self, widths):
        self.topology = Topology(widths)
        self.widths = self.topology.widths
        self.d = 2
        if self.widths[0] != 2:
            raise ValueError("heat1p1d needs input dim 2 (t, x)")

    def exact(self, x):
        return np.cos(np.pi * x[:, 1]) * np.exp(-np.pi**2 * x[:, 0] / 4.0)

    def exact_grad(self, x):
        u = self.exact(x)
        dt = -np.pi**2 / 4.0 * u
        dx = -np.pi * np.sin(np.pi * x[:, 1]) * np.exp(-np.pi**2 * x[:, 0] / 4.0)
        return np.stack([dt, dx], axis=1)

    def source(self, x):
        return 0.75 * np.pi**2 * self.exact(x)

    def dirichlet(self, x):
        return self.exact(x)

    def initial_value(self, x):
        return np.cos(np.pi * x[:, 1])

    def sample_quadrature(self, n_interior, n_boundary, seed):  # problems.py:266-287
        rng = np.random.default_rng(seed)
        pts = _uniform_box(rng, n_interior, 2)
        t = rng.random(n_boundary)
        side = rng.integers(0, 2, n_boundary).astype(float)
        bnd = np.stack([t, side], axis=1)
        n_init = max(n_boundary // 2, 1)
        xi = rng.random(n_init)
        init = np.stack([np.zeros(n_init), xi], axis=1)
        return Quadrature(pts, np.full(n_interior, 1.0 / n_interior), bnd, np.full(n_boundary, 2.0 / n_boundary),
                          init, np.full(n_init, 1.0 / n_init))

    def residual_weights(self, quad):
        return np.concatenate([quad.interior_weights, quad.boundary_weights, quad.initial_weights])

    def metric_weights(self, quad):
        return np.concatenate([quad.interior_weights, quad.interior_weights, quad.initial_weights])

    def stack_rows(self, theta, theta_bar, quad, which):  # problems.py:294-311
        beta, gamma = np.array([1.0, 0.0]), np.array([0.0, -1.0])
        second = quad.interior_points if which == "metric" else quad.boundary_points
        return StackRows(quad.interior_points, 0.0, beta, gamma, np.concatenate([second, quad.initial_points]))

    def residual_stack(self, theta, quad):  # problems.py:294-301
        _, g, sec = mlp_jets(self.widths, theta, quad.interior_points)
        interior = g[:, 0] - sec[:, 1] - self.source(quad.interior_points)
        boundary = mlp_forward(self.widths, theta, quad.boundary_points) - self.dirichlet(quad.boundary_points)
        initial = mlp_forward(self.widths, theta, quad.initial_points) - self.initial_value(quad.initial_points)
        return np.concatenate([interior, boundary, initial])


# ---------------------------------------------------------------------------
# Linearised metric map (autodiff.py:81-125, 587-613)
# ---------------------------------------------------------------------------


class Linearization:
    """A stack (metric by default, or the residual's) traced at theta: cached
    primal jets, then JVP (tangent sweep) and VJP (adjoint sweep) through the
    same arithmetic the reference tape records for mlp_input_derivatives /
    forward (autodiff.py:164-328).  Head rows follow StackRows."""

    def __init__(self, problem, theta, quad, which="metric", theta_bar=None):
        self.widths = problem.widths
        self.top = problem.topology
        self.theta = np.asarray(theta, dtype=float)
        self.layers = self.top.unflatten(self.theta)
        rows = problem.stack_rows(self.theta, self.theta if theta_bar is None else np.asarray(theta_bar, float),
                                  quad, which)
        self.xi = np.asarray(rows.x_int, dtype=float)
        self.xb = np.asarray(rows.x_val, dtype=float)
        self.alpha = rows.alpha
        self.beta = np.asarray(rows.beta, dtype=float)
        self.gamma = np.asarray(rows.gamma, dtype=float)
        self.nl = len(self.layers)
        d = self.widths[0]
        q = self.xi.shape[0]
        # interior jets cache: inputs (z, g_i, h_i) and pre-activation jets per layer
        z = self.xi
        g = [np.broadcast_to(np.eye(d)[i], (q, d)).copy() for i in range(d)]
        h = [np.zeros((q, d)) for _ in range(d)]
        self.cache_i = []
        for k, (w, b) in enumerate(self.layers):
            a = z @ w.T + b
            ga = [gi @ w.T for gi in g]
            ha = [hi @ w.T for hi in h]
            ent = {"z": z, "g": g, "h": h, "a": a, "ga": ga, "ha": ha}
            if k < self.nl - 1:
                t = np.tanh(a)
                d1 = 1.0 - t * t
                d2 = -2.0 * t * d1
                ent.update(t=t, d1=d1, d2=d2)
                h = [d2 * gai * gai + d1 * hai for gai, hai in zip(ga, ha)]
                g = [d1 * gai for gai in ga]
                z = t
            self.cache_i.append(ent)
        last = self.cache_i[-1]
        head = self._head(q, last["a"], last["ga"], last["ha"])
        # value rows: plain forward cache
        zb = self.xb
        self.cache_b = []
        for k, (w, b) in enumerate(self.layers):
            a = zb @ w.T + b
            ent = {"z": zb, "a": a}
            if k < self.nl - 1:
                t = np.tanh(a)
                ent.update(t=t, d1=1.0 - t * t)
                zb = t
            self.cache_b.append(ent)
        ub = self.cache_b[-1]["a"].reshape(self.xb.shape[0]) if self.xb.shape[0] else np.zeros(0)
        self.value = np.concatenate([head, ub])
        self.n_int = q
        self.n_bnd = self.xb.shape[0]

    def _head(self, q, a, ga, ha):
        """alpha*u + beta . grad + gamma . second at the output layer (zero coefficients skipped)."""
        out = np.zeros(q)
        for gi, hai in zip(self.gamma, ha):
            if gi != 0.0:
                out = out + (hai.reshape(q) if gi == 1.0 else gi * hai.reshape(q))
        for bi, gai in zip(self.beta, ga):
            if bi != 0.0:
                out = out + bi * gai.reshape(q)
        if np.any(np.asarray(self.alpha) != 0.0):
            out = out + self.alpha * a.reshape(q)
        return out

    def jvp(self, v):
        """Tangent sweep: d/de stack(theta + e v) at e = 0."""
        vl = self.top.unflatten(np.asarray(v, dtype=float))
        d = self.widths[0]
        q = self.n_int
        dz = np.zeros_like(self.xi)
        dg = [np.zeros((q, d)) for _ in range(d)]
        dh = [np.zeros((q, d)) for _ in range(d)]
        for k, ((w, _), (vw, vb)) in enumerate(zip(self.layers, vl)):
            c = self.cache_i[k]
            da = dz @ w.T + c["z"] @ vw.T + vb
            dga = [dgi @ w.T + gi @ vw.T for dgi, gi in zip(dg, c["g"])]
            dha = [dhi @ w.T + hi @ vw.T for dhi, hi in zip(dh, c["h"])]
            if k < self.nl - 1:
                t, d1, d2 = c["t"], c["d1"], c["d2"]
                dt = d1 * da
                dd1 = -2.0 * t * dt
                dd2 = -2.0 * (dt * d1 + t * dd1)
                dh = [dd2 * gai * gai + d2 * 2.0 * gai * dgai + dd1 * hai + d1 * dhai
                      for gai, dgai, hai, dhai in zip(c["ga"], dga, c["ha"], dha)]
                dg = [dd1 * gai + d1 * dgai for gai, dgai in zip(c["ga"], dga)]
                dz = dt
            else:
                dhead = self._head(q, da, dga, dha)
        # value rows
        if self.n_bnd:
            dzb = np.zeros_like(self.xb)
            for k, ((w, _), (vw, vb)) in enumerate(zip(self.layers, vl)):
                c = self.cache_b[k]
                da = dzb @ w.T + c["z"] @ vw.T + vb
                dzb = c["d1"] * da if k < self.nl - 1 else da
            dub = dzb.reshape(self.n_bnd)
        else:
            dub = np.zeros(0)
        return np.concatenate([dhead, dub])

    def vjp(self, cot):
        """Adjoint sweep: J^T cot for the stack."""
        cot = np.asarray(cot, dtype=float)
        ci, cb = cot[: self.n_int], cot[self.n_int:]
        d = self.widths[0]
        grads = [(np.zeros_like(w), np.zeros_like(b)) for w, b in self.layers]
        # head rows: seeds alpha (value), beta_i (gradient), gamma_i (second derivative)
        ones = np.ones_like(self.cache_i[-1]["a"])
        ci2 = ci[:, None]
        alpha = np.asarray(self.alpha, dtype=float)
        abar = (ci * alpha)[:, None] * ones if alpha.ndim else ci2 * alpha * ones
        gabar = [ci2 * bi * ones for bi in self.beta]
        habar = [ci2 * ones if gi == 1.0 else ci2 * gi * ones for gi in self.gamma]
        for k in range(self.nl - 1, -1, -1):
            w, _ = self.layers[k]
            c = self.cache_i[k]
            if k < self.nl - 1:
                # adjoints arriving at this layer's outputs (z, g_i, h_i) -> pre-activation
                t, d1, d2 = c["t"], c["d1"], c["d2"]
                zbar, gbar, hbar = zbar_in, gbar_in, hbar_in
                d2bar = sum(hb * ga * ga for hb, ga in zip(hbar, c["ga"]))
                d1bar = sum(hb * ha for hb, ha in zip(hbar, c["ha"])) + sum(gb * ga for gb, ga in zip(gbar, c["ga"]))
                gabar = [hb * d2 * 2.0 * ga + gb * d1 for hb, gb, ga in zip(hbar, gbar, c["ga"])]
                habar = [hb * d1 for hb in hbar]
                tbar = zbar - 2.0 * d1 * d2bar
                d1bar = d1bar - 2.0 * t * d2bar
                tbar = tbar - 2.0 * t * d1bar
                abar = tbar * d1
            gw = abar.T @ c["z"]
            for gab, gi in zip(gabar, c["g"]):
                gw = gw + gab.T @ gi
            for hab, hi in zip(habar, c["h"]):
                gw = gw + hab.T @ hi
            grads[k] = (grads[k][0] + gw, grads[k][1] + abar.sum(axis=0))
            zbar_in = abar @ w
            gbar_in = [gab @ w for gab in gabar]
            hbar_in = [hab @ w for hab in habar]
        # value rows: u = last-layer value
        if self.n_bnd:
            abar = cb[:, None] * np.ones((self.n_bnd, 1))
            for k in range(self.nl - 1, -1, -1):
                w, _ = self.layers[k]
                c = self.cache_b[k]
                if k < self.nl - 1:
                    abar = zbar_b * c["d1"]
                grads[k] = (grads[k][0] + abar.T @ c["z"], grads[k][1] + abar.sum(axis=0))
                zbar_b = abar @ w
        return np.concatenate([np.concatenate([gw.reshape(-1), gb]) for gw, gb in grads])


class GramianOracle:
    """v -> J^T diag(w) J v at a fixed linearisation (gramian.py:20-61)."""

    def __init__(self, problem, theta, quad):
        self.lin = Linearization(problem, theta, quad)
        self.weights = problem.metric_weights(quad)
        self.dim = problem.topology.param_count
        self.matvec_count = 0

    def matvec(self, v):  # gramian.py:48-53
        v = np.asarray(v, dtype=float)
        if v.shape != (self.dim,):
            raise ValueError(f"expected vector of length {self.dim}, got {v.shape}")
        self.matvec_count += 1
        return self.lin.vjp(self.weights * self.lin.jvp(v))

    def matmat(self, vmat):  # gramian.py:55-61: column loop, fixed order
        vmat = np.asarray(vmat, dtype=float)
        out = np.empty_like(vmat)
        for j in range(vmat.shape[1]):
            out[:, j] = self.matvec(vmat[:, j])
        return out

    __call__ = matvec


class DenseOracle:
    """Explicit matrix operator (gramian.py:101-120)."""

    def __init__(self, matrix):
        self.matrix = np.asarray(matrix, dtype=float)
        self.dim = self.matrix.shape[0]
        self.matvec_count = 0

    def matvec(self, v):
        self.matvec_count += 1
        return self.matrix @ v

    def matmat(self, vmat):
        self.matvec_count += vmat.shape[1]
        return self.matrix @ vmat

    __call__ = matvec


class ShiftedOracle:
    """v -> A v + mu v (gramian.py:123-135)."""

    def __init__(self, base, mu):
        self.base, self.mu, self.dim = base, float(mu), base.dim

    def matvec(self, v):
        return self.base.matvec(v) + self.mu * v

    __call__ = matvec


# ---------------------------------------------------------------------------
# Nystrom sketch and preconditioner (sketch.py)
# ---------------------------------------------------------------------------


class SketchFailure(RuntimeError):
    pass


@dataclass(frozen=True)
class NystromFactorOracle:
    basis: np.ndarray
    eigenvalues: np.ndarray


def nystrom_approximate(op, rank, seed, max_retries=3, omega_hook=None):
    """Alg. 1 of the paper as in sketch.py:58-90.  ``omega_hook`` (tests) sees
    each post-QR Omega."""
    if isinstance(op, np.ndarray):
        op = DenseOracle(op)
    p = op.dim
    if not 1 <= rank <= p:
        raise ValueError(f"rank must be in [1, {p}], got {rank}")
    rng = np.random.default_rng(seed)
    for _ in range(max_retries):
        omega = rng.standard_normal((p, rank))
        omega, _ = np.linalg.qr(omega, mode="reduced")
        if omega_hook is not None:
            omega_hook(omega)
        y = op.matmat(omega)
        shift = EPS * np.linalg.norm(y, "fro")
        y_shifted = y + shift * omega
        try:
            chol = scipy.linalg.cholesky(omega.T @ y_shifted, lower=False)
        except (np.linalg.LinAlgError, scipy.linalg.LinAlgError):
            continue
        b = scipy.linalg.solve_triangular(chol, y_shifted.T, lower=False, trans="T").T
        u, s, _ = np.linalg.svd(b, full_matrices=False)
        return NystromFactorOracle(u, np.maximum(s**2 - shift, 0.0))
    raise SketchFailure(f"sketch Cholesky failed after {max_retries} attempts")


class PreconditionerOracle:
    """P^{-1} v = (lam_l+mu) U (Lam+mu)^{-1} U^T v + (v - U U^T v) (sketch.py:93-112)."""

    def __init__(self, factor, mu):
        if factor.eigenvalues[-1] + mu <= 0:
            raise ValueError("need smallest eigenvalue estimate + mu > 0")
        self.u = factor.basis
        self.scale = factor.eigenvalues[-1] + mu
        self.inv = 1.0 / (factor.eigenvalues + mu)

    def apply(self, v):
        utv = self.u.T @ v
        return self.scale * (self.u @ (self.inv * utv)) + (v - self.u @ utv)

    __call__ = apply


# ---------------------------------------------------------------------------
# PCG (krylov.py:24-88)
# ---------------------------------------------------------------------------


@dataclass
class SolveReportOracle:
    solution: np.ndarray
    iterations: int
    relative_residual: float
    matvecs: int
    converged: bool
    breakdown: bool = False


def pcg(op, b, rel_tol, maxit, precond=None, recompute_every=50):
    if not 0.0 < rel_tol < 1.0:
        raise ValueError(f"rel_tol must be in (0, 1), got {rel_tol}")
    if maxit < 1:
        raise ValueError("maxit must be >= 1")
    matvec = op.matvec if hasattr(op, "matvec") else op
    apply_p = (precond.apply if hasattr(precond, "apply") else precond) if precond else None
    b = np.asarray(b, dtype=float)
    norm_b = np.linalg.norm(b)
    x = np.zeros_like(b)
    if norm_b == 0.0:
        return SolveReportOracle(x, 0, 0.0, 0, True)
    r = b.copy()
    z = apply_p(r) if apply_p else r
    d = z.copy()
    rz = float(r @ z)
    matvecs = iterations = 0
    breakdown = False
    for it in range(1, maxit + 1):
        ad_ = matvec(d)
        matvecs += 1
        dad = float(d @ ad_)
        if dad <= 0.0:
            breakdown = True
            break
        alpha = rz / dad
        x = x + alpha * d
        iterations = it
        if it % recompute_every == 0:
            r = b - matvec(x)
            matvecs += 1
        else:
            r = r - alpha * ad_
        if np.linalg.norm(r) / norm_b <= rel_tol:
            break
        z = apply_p(r) if apply_p else r
        rz_new = float(r @ z)
        beta = rz_new / rz
        rz = rz_new
        d = z + beta * d
    r_true = b - matvec(x)
    matvecs += 1
    rel_res = float(np.linalg.norm(r_true) / norm_b)
    return SolveReportOracle(x, iterations, rel_res, matvecs, (not breakdown) and rel_res <= rel_tol, breakdown)


# ---------------------------------------------------------------------------
# Outer loop (optim.py)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class NgdConfigOracle:
    """optim.py:40-69 plus ``fixed_rank`` (pin ell for benchmarks)."""

    ell0: int = 10
    ell_max: int | None = None
    gamma: float | None = None
    cg_maxit: int = 20
    kappa: float = 0.1
    rank_ratio: float = 10.0
    mu_floor_mode: str = "loss-power"
    mu_floor_coeff: float = 1e-4
    mu_floor_exponent: float = 2.0
    ls_shrink: float = 0.5
    ls_max_backtracks: int = 30
    ls_sufficient_decrease: float = 1e-4
    iterations: int = 300
    seed: int = 0
    fixed_rank: bool = False


@dataclass(frozen=True)
class RecordOracle:
    iteration: int
    loss: float
    h1_rel_error: float
    mu: float
    ell: int
    pcg_iters: int
    matvecs: int
    seconds: float


def adapt_mu(lam1, gamma, loss, grad_norm, mode, coeff, exponent):  # optim.py:86-103
    if lam1 < 0 or gamma <= 0:
        raise ValueError("need lam1 >= 0 and gamma > 0")
    base = gamma * EPS * lam1
    if mode == "loss-power":
        floor = coeff * abs(loss) ** exponent
    elif mode == "grad-power":
        floor = coeff * grad_norm**exponent
    elif mode == "constant":
        floor = coeff
    else:
        raise ValueError(f"unknown mu floor mode {mode!r}")
    return max(base, floor)


def adapt_rank(eigenvalues, mu, ell, ell_max, ratio=10.0):  # optim.py:106-118
    eigenvalues = np.asarray(eigenvalues, dtype=float)
    threshold = ratio * mu
    if eigenvalues[-1] > threshold:
        return min(2 * ell, ell_max)
    first_below = int(np.argmax(eigenvalues < threshold)) + 1
    return min(first_below + 1, ell_max)


def backtracking_linesearch(theta, direction, loss_fn, grad_dot_dir, shrink=0.5,
                            max_backtracks=30, sufficient_decrease=1e-4):  # optim.py:121-146
    loss0 = loss_fn(theta)
    alpha = 1.0
    for _ in range(max_backtracks + 1):
        loss_new = loss_fn(theta - alpha * direction)
        if not np.isfinite(loss_new):
            loss_new = np.inf
        if loss_new <= loss0 - sufficient_decrease * alpha * grad_dot_dir:
            return alpha, loss_new
        alpha *= shrink
    return 0.0, loss0


def cg_rel_tol(kappa, grad_norm):  # optim.py:183-185
    return min(max(min(kappa, grad_norm), 1e-300), 1.0 - 1e-16)


def resolve_ell_max(config, p):  # optim.py:169-174
    if config.ell_max is not None:
        return min(config.ell_max, p)
    return max(min(500, p // 2), min(config.ell0, p))


def nystrom_ngd_run(problem, theta0, config, quad, quad_eval=None, step_hook=None):
    """optim.py:188-270.  ``step_hook(k, dict)`` exposes per-step internals to tests."""
    theta = np.asarray(theta0, dtype=float)
    p = theta.shape[0]
    gamma = float(config.gamma) if config.gamma is not None else float(p)
    ell_max = resolve_ell_max(config, p)
    ell = min(config.ell0, ell_max)
    rng = np.random.default_rng(config.seed)
    loss_fn = lambda th: problem.loss_value(th, quad)
    records = []
    total = 0
    boost = 1.0
    for k in range(config.iterations):
        tic = time.perf_counter()
        loss = loss_fn(theta)
        if not np.isfinite(loss):
            raise ArithmeticError(f"non-finite loss at iteration {k}")
        g = problem.loss_grad(theta, quad)
        gnorm = float(np.linalg.norm(g))
        gop = GramianOracle(problem, theta, quad)
        factor = nystrom_approximate(gop, ell, seed=int(rng.integers(2**63)))
        mu = adapt_mu(factor.eigenvalues[0], gamma, loss, gnorm, config.mu_floor_mode,
                      config.mu_floor_coeff * boost, config.mu_floor_exponent)
        if mu <= 0.0:
            mu = gamma * EPS
        pre = PreconditionerOracle(factor, mu)
        rep = pcg(ShiftedOracle(gop, mu), g, cg_rel_tol(config.kappa, gnorm), config.cg_maxit, precond=pre)
        alpha, _ = backtracking_linesearch(theta, rep.solution, loss_fn, float(g @ rep.solution),
                                           config.ls_shrink, config.ls_max_backtracks,
                                           config.ls_sufficient_decrease)
        if step_hook is not None:
            step_hook(k, {"theta": theta, "grad": g, "direction": rep.solution, "alpha": alpha,
                          "eigenvalues": factor.eigenvalues, "mu": mu})
        if alpha == 0.0:
            boost *= 10.0
        else:
            theta = theta - alpha * rep.solution
            boost = 1.0
        total += gop.matvec_count
        h1 = problem.h1_relative_error(theta, quad_eval) if quad_eval is not None else float("nan")
        records.append(RecordOracle(k, loss, h1, mu, ell, rep.iterations, total, time.perf_counter() - tic))
        if not config.fixed_rank:
            ell = adapt_rank(factor.eigenvalues, mu, ell, ell_max, ratio=config.rank_ratio)
    return theta, records
