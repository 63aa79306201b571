"""NystromNGD outer loop on the GPU (mirror of nystromngd/optim.py:19-270).

The host keeps only the scalar policy of the reference -- ``adapt_mu``,
``adapt_rank``, the Armijo backtracking control flow, the rng that seeds each
sketch -- restated here with the same names and semantics.  theta, the
gradient, the sketch, the Nystrom factor and the PCG iterates stay on the
device; the host reads back the scalars the policy needs (loss, ||g||, top
eigenvalue, g.d, PCG report, candidate losses).
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .gramian import GramianOperator, ShiftedOperator
from .krylov import pcg
from .sketch import NystromPreconditioner, nystrom_approximate

EPS_MACH = np.finfo(float).eps  # optim.py:19

__all__ = ["NystromNgdConfig", "RunRecord", "adapt_mu", "adapt_rank", "backtracking_linesearch", "nystrom_ngd_run"]


@dataclass(frozen=True)
class NystromNgdConfig:
    """optim.py:40-69, plus two build-specific knobs:
    ``fixed_rank`` pins ell = ell0 (benchmark configs) and
    ``omega_source`` picks host-numpy ("host", bit-identical to the reference)
    or on-device Philox ("device") Gaussian test matrices."""

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
    omega_source: str = "host"

    def __post_init__(self):
        if self.ell0 < 1:
            raise ValueError("need ell0 >= 1")
        if self.ell_max is not None and self.ell0 > self.ell_max:
            raise ValueError("need 1 <= ell0 <= ell_max")
        if self.gamma is not None and self.gamma <= 0:
            raise ValueError("gamma must be positive")
        if not 0.0 < self.kappa < 1.0:
            raise ValueError("kappa must be in (0, 1)")
        if self.mu_floor_mode not in ("loss-power", "grad-power", "constant"):
            raise ValueError(f"unknown mu floor mode {self.mu_floor_mode!r}")
        if self.omega_source not in ("host", "device"):
            raise ValueError(f"unknown omega source {self.omega_source!r}")


@dataclass(frozen=True)
class RunRecord:
    """One optimizer iteration in the trace (optim.py:72-83)."""

    iteration: int
    loss: float
    h1_rel_error: float
    mu: float
    ell: int
    pcg_iters: int
    matvecs: int
    seconds: float


def adapt_mu(lam1, gamma, loss, grad_norm, mode, coeff, exponent):
    """mu = max(gamma * eps * lam1, floor) (optim.py:86-103)."""
    if lam1 < 0 or gamma <= 0:
        raise ValueError("need lam1 >= 0 and gamma > 0")
    base = gamma * EPS_MACH * lam1
    if mode == "loss-power":
        floor = coeff * abs(loss) ** exponent
    elif mode == "grad-power":
        floor = coeff * grad_norm**exponent
    elif mode == "constant":
        floor = coeff
    else:
        raise ValueError(f"unknown mu floor mode {mode!r}")
    return max(base, floor)


def adapt_rank(eigenvalues, mu, ell, ell_max, ratio=10.0):
    """Next sketch rank from the estimated spectrum (optim.py:106-118)."""
    eigenvalues = np.asarray(eigenvalues, dtype=float)
    threshold = ratio * mu
    if eigenvalues[-1] > threshold:
        return min(2 * ell, ell_max)
    first_below = int(np.argmax(eigenvalues < threshold)) + 1
    return min(first_below + 1, ell_max)


def backtracking_linesearch(theta, direction, loss_fn, grad_dot_dir, shrink=0.5, max_backtracks=30,
                            sufficient_decrease=1e-4, loss0=None):
    """Armijo backtracking along theta - alpha * direction (optim.py:121-146).

    ``loss_fn(theta, alpha, direction)`` evaluates the loss at the candidate
    (on the device); ``loss0`` may be supplied when the caller already holds
    the (bitwise identical, deterministic) loss at theta."""
    if loss0 is None:
        loss0 = loss_fn(theta, 0.0, direction)
    alpha = 1.0
    for _ in range(max_backtracks + 1):
        try:
            loss_new = loss_fn(theta, alpha, direction)
        except _lib.NonFiniteError:
            loss_new = np.inf
        if loss_new <= loss0 - sufficient_decrease * alpha * grad_dot_dir:
            return alpha, loss_new
        alpha *= shrink
    return 0.0, loss0


def _resolve_gamma(config, p):
    return float(config.gamma) if config.gamma is not None else float(p)


def _resolve_ell_max(config, p):  # optim.py:169-174
    if config.ell_max is not None:
        return min(config.ell_max, p)
    return max(min(500, p // 2), min(config.ell0, p))


def _cg_rel_tol(kappa, grad_norm):  # optim.py:183-185
    return min(max(min(kappa, grad_norm), 1e-300), 1.0 - 1e-16)


class _StepTimer:
    """Optional per-phase CUDA-event timing (bench.py)."""

    def __init__(self, enabled):
        self.enabled = enabled
        self.events = []

    def mark(self, name):
        if self.enabled:
            torch = _lib.torch_mod()
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            self.events.append((name, e))


class NystromNgdRunner:
    """Step-wise form of ``nystrom_ngd_run`` (optim.py:188-270): one ``step()`` is
    one NGD iteration (linearise, gradient, sketch, damping, PCG, line search,
    update, rank adaptation).  State (theta, rng, ell, floor boost, matvec
    total) lives here so benchmarks can time single steps."""

    def __init__(self, problem, theta0, config, quad, quad_eval=None):
        torch = _lib.torch_mod()
        self.problem, self.config, self.quad, self.quad_eval = problem, config, quad, quad_eval
        self.theta = _lib.to_device(theta0).clone()
        p = self.theta.shape[0]
        self.p = p
        self.gamma = _resolve_gamma(config, p)
        self.ell_max = _resolve_ell_max(config, p)
        self.ell = min(config.ell0, self.ell_max)
        self.rng = np.random.default_rng(config.seed)
        self.ctx = problem.context(quad)
        if self.ctx.p != p:
            raise ValueError(f"expected {self.ctx.p} parameters, got {p}")
        self.cand = torch.empty_like(self.theta)
        self.grad = torch.empty_like(self.theta)
        self.total_matvecs = 0
        self.floor_boost = 1.0
        self.k = 0

    def _loss_at(self, th, alpha, direction):
        out = _lib.ctypes.c_double()
        self.ctx.call("ngd_loss_at", _lib.ptr(th), float(alpha), _lib.ptr(direction), _lib.ctypes.byref(out))
        return float(out.value)

    def _dot(self, a, b):
        out = _lib.ctypes.c_double()
        self.ctx.call("ngd_dot", _lib.ptr(a), _lib.ptr(b), self.p, _lib.ctypes.byref(out))
        return float(out.value)

    def step(self, step_hook=None, timer=None):
        config, problem, quad = self.config, self.problem, self.quad
        k = self.k
        tic = time.perf_counter()
        if timer:
            timer.mark("start")
        gop = GramianOperator.from_problem(problem, self.theta, quad)  # linearise once: loss, jets, adjoints
        loss = gop.loss
        if not np.isfinite(loss):
            raise _lib.NonFiniteError(f"non-finite loss at iteration {k}")
        self.ctx.call("ngd_loss_grad", _lib.ptr(self.grad))
        grad = self.grad
        if timer:
            timer.mark("linearize+grad")
        factor = nystrom_approximate(gop, self.ell, seed=int(self.rng.integers(2**63)),
                                     omega_source=config.omega_source)
        # |grad| is read after the sketch (same value as before it: deterministic kernels), so the
        # host does not stall on the gradient while the sketch could already be queued
        grad_norm = float(np.sqrt(self._dot(grad, grad)))
        if timer:
            timer.mark("sketch")
        mu = adapt_mu(factor.eig_host[0], self.gamma, loss, grad_norm, config.mu_floor_mode,
                      config.mu_floor_coeff * self.floor_boost, config.mu_floor_exponent)
        if mu <= 0.0:
            mu = self.gamma * EPS_MACH
        precond = NystromPreconditioner(factor, mu)
        report = pcg(ShiftedOperator(gop, mu), grad, _cg_rel_tol(config.kappa, grad_norm), config.cg_maxit,
                     precond=precond)
        if timer:
            timer.mark("pcg")
        d = report.solution
        alpha, _ = backtracking_linesearch(self.theta, d, self._loss_at, self._dot(grad, d),
                                           shrink=config.ls_shrink, max_backtracks=config.ls_max_backtracks,
                                           sufficient_decrease=config.ls_sufficient_decrease, loss0=loss)
        if step_hook is not None:
            step_hook(k, {"theta": self.theta.clone(), "grad": grad.clone(), "direction": d.clone(),
                          "alpha": alpha, "eigenvalues": factor.eig_host, "mu": mu, "report": report})
        if alpha == 0.0:
            self.floor_boost *= 10.0
        else:
            self.ctx.call("ngd_axpy", _lib.ptr(self.theta), float(alpha), _lib.ptr(d), _lib.ptr(self.cand), self.p)
            self.theta, self.cand = self.cand, self.theta
            self.floor_boost = 1.0
        if timer:
            timer.mark("linesearch")
        self.total_matvecs += gop.matvec_count
        h1 = float("nan")
        if self.quad_eval is not None:
            h1 = h1_relative_error(problem, self.theta, self.quad_eval)
        rec = RunRecord(k, loss, h1, mu, self.ell, report.iterations, self.total_matvecs, time.perf_counter() - tic)
        if not config.fixed_rank:
            self.ell = adapt_rank(factor.eig_host, mu, self.ell, self.ell_max, ratio=config.rank_ratio)
        self.k += 1
        self.last_matvecs = gop.matvec_count
        return rec


def nystrom_ngd_run(problem, theta0, config, quad, quad_eval=None, h1_stop=None, step_hook=None, timer=None):
    """Natural gradient descent with a randomized Nystrom preconditioner (optim.py:188-270).

    Returns (theta_final, [RunRecord, ...]); theta_final is a CUDA tensor if
    theta0 was one, else a numpy array."""
    runner = NystromNgdRunner(problem, theta0, config, quad, quad_eval)
    records = []
    for _ in range(config.iterations):
        records.append(runner.step(step_hook=step_hook, timer=timer))
        if h1_stop is not None and records[-1].h1_rel_error <= h1_stop:
            break
    return _lib.like_input(runner.theta, theta0), records


def h1_relative_error(problem, theta, quad):
    """Relative H1 error (problems.py:104-119), evaluated on the device (ngd_h1_error)."""
    return problem.h1_relative_error(theta, quad)


# ---------------------------------------------------------------------------
# NGD-CG baseline of the reference's comparison protocol (optim.py:273-327):
# unpreconditioned CG on the same device Gramian.
# ---------------------------------------------------------------------------


def _baseline_mu(loss, cap=1e-5):  # optim.py:273-275
    return max(min(cap, loss), 1e-14)


class _DeviceIterate:
    """theta on the device plus the context helpers the baselines share with the runner."""

    def __init__(self, problem, theta0, quad):
        torch = _lib.torch_mod()
        self.problem, self.quad = problem, quad
        self.theta = _lib.to_device(theta0).clone()
        self.p = self.theta.shape[0]
        self.ctx = problem.context(quad)
        self.grad = torch.empty_like(self.theta)
        self.cand = torch.empty_like(self.theta)

    def loss_at(self, th, alpha, direction):
        out = _lib.ctypes.c_double()
        self.ctx.call("ngd_loss_at", _lib.ptr(th), float(alpha), _lib.ptr(direction), _lib.ctypes.byref(out))
        return float(out.value)

    def dot(self, a, b):
        out = _lib.ctypes.c_double()
        self.ctx.call("ngd_dot", _lib.ptr(a), _lib.ptr(b), self.p, _lib.ctypes.byref(out))
        return float(out.value)

    def linearize(self):
        """Gramian operator at theta (one linearisation), loss and gradient."""
        gop = GramianOperator.from_problem(self.problem, self.theta, self.quad)
        if not np.isfinite(gop.loss):
            raise _lib.NonFiniteError("non-finite loss")
        self.ctx.call("ngd_loss_grad", _lib.ptr(self.grad))
        return gop, gop.loss, self.grad

    def step(self, direction, grad_dot_dir, loss0):
        """Armijo line search along -direction and update (default line-search knobs, optim.py:121)."""
        alpha, _ = backtracking_linesearch(self.theta, direction, self.loss_at, grad_dot_dir, loss0=loss0)
        if alpha > 0.0:
            self.ctx.call("ngd_axpy", _lib.ptr(self.theta), float(alpha), _lib.ptr(direction), _lib.ptr(self.cand),
                          self.p)
            self.theta, self.cand = self.cand, self.theta
        return alpha


def _h1(problem, theta, quad_eval):
    return float("nan") if quad_eval is None else problem.h1_relative_error(theta, quad_eval)


def ngd_cg_step(problem, theta, quad, mu, kappa, maxit_total, loss_fn=None):
    """One matrix-free NGD step solved with plain CG, no preconditioner (optim.py:278-292).
    Returns (theta_next, SolveReport, matvecs)."""
    it = _DeviceIterate(problem, theta, quad)
    gop, loss, g = it.linearize()
    gnorm = float(np.sqrt(it.dot(g, g)))
    report = pcg(ShiftedOperator(gop, mu), g, _cg_rel_tol(kappa, gnorm), maxit_total)
    d = _lib.to_device(report.solution)
    it.step(d, it.dot(g, d), loss)
    return _lib.like_input(it.theta, theta), report, gop.matvec_count


def ngd_cg_run(problem, theta0, config, quad, quad_eval=None, matvec_budget=None):
    """Unpreconditioned NGD-CG baseline (optim.py:295-327): CG capped at cg_maxit + ell_max."""
    it = _DeviceIterate(problem, theta0, quad)
    maxit_total = config.cg_maxit + _resolve_ell_max(config, it.p)
    records, total = [], 0
    for k in range(config.iterations):
        tic = time.perf_counter()
        gop, loss, g = it.linearize()
        mu = _baseline_mu(loss)
        gnorm = float(np.sqrt(it.dot(g, g)))
        report = pcg(ShiftedOperator(gop, mu), g, _cg_rel_tol(config.kappa, gnorm), maxit_total)
        d = _lib.to_device(report.solution)
        it.step(d, it.dot(g, d), loss)
        total += gop.matvec_count
        records.append(RunRecord(k, loss, _h1(problem, it.theta, quad_eval), mu, 0, report.iterations, total,
                                 time.perf_counter() - tic))
        if matvec_budget is not None and total >= matvec_budget:
            break
    return _lib.like_input(it.theta, theta0), records


# The hot path's optimizer and the one baseline SURVEY 8f #4 keeps (NGD-CG, the paper's comparison
# protocol); gradient descent, dense BFGS and dense NGD (optim.py:330-438) are off the path.
OPTIMIZER_NAMES = ("nystrom_ngd", "ngd_cg")

_RUNNERS = {
    "nystrom_ngd": nystrom_ngd_run,
    "ngd_cg": ngd_cg_run,
}


def run_optimizer(name, problem, theta0, config, quad, quad_eval=None):
    """Dispatch by name (optim.py:441-455), for the two optimizers built on the device path."""
    if name not in _RUNNERS:
        raise KeyError(f"unknown optimizer {name!r}; available: {OPTIMIZER_NAMES}")
    return _RUNNERS[name](problem, theta0, config, quad, quad_eval=quad_eval)
