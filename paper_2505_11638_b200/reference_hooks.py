"""Drive the reference's own experiment harness with the B200 runner injected.

The reference harness (``nystromngd/harness.py:199-234``) calls
``optim.run_optimizer`` (dispatch table ``optim._RUNNERS``, ``optim.py:441-455``)
and, for the spectrum dump, ``harness.gramian_spectrum`` (``harness.py:249-252``).
``install(nystromngd)`` swaps those entries for wrappers that rebuild the
reference problem on this package (same class name, topology and quadrature),
run the device path, and hand back the reference's own ``RunRecord`` objects and
numpy arrays -- so the reference's CSV traces, summary JSON and spectrum file are
written by the reference code from GPU results.  ``uninstall()`` restores the
originals.  The reference package is passed in by the caller; nothing here
imports it.
"""

from __future__ import annotations

import numpy as np

from . import problems as _problems
from .gramian import gramian_spectrum as _gramian_spectrum
from .model import MlpTopology
from .optim import NystromNgdConfig, run_optimizer

# optimizers the device path provides (the rest of the reference's table stays on the CPU)
INJECTED = ("nystrom_ngd", "ngd_cg")

_saved = {}


def device_problem(ref_problem):
    """The package's problem of the same class and topology as a reference problem
    (problems.py:128-385: Poisson1D, Poisson2D, Heat1p1D, NonlinearPoisson2D)."""
    cls = getattr(_problems, type(ref_problem).__name__, None)
    if cls is None or not isinstance(cls, type) or not issubclass(cls, _problems.PdeProblem):
        raise TypeError(f"no device problem for {type(ref_problem).__name__}")
    return cls(MlpTopology(tuple(ref_problem.topology.widths)))


def device_quadrature(ref_quad):
    return _problems.QuadratureSet(np.asarray(ref_quad.interior_points), np.asarray(ref_quad.interior_weights),
                                   np.asarray(ref_quad.boundary_points), np.asarray(ref_quad.boundary_weights))


def device_config(ref_config):
    """NystromNgdConfig (optim.py:40-69) field by field; the reference's rank adaptation is kept."""
    fields = {k: getattr(ref_config, k) for k in NystromNgdConfig.__dataclass_fields__ if hasattr(ref_config, k)}
    return NystromNgdConfig(**fields)


def _runner(name, ref_optim):
    def run(problem, theta0, config, quad, quad_eval=None):
        q = device_quadrature(quad)
        qe = None if quad_eval is None else (q if quad_eval is quad else device_quadrature(quad_eval))
        theta, recs = run_optimizer(name, device_problem(problem), np.asarray(theta0, dtype=float),
                                    device_config(config), q, quad_eval=qe)
        return np.asarray(theta), [ref_optim.RunRecord(**r.__dict__) for r in recs]

    run.__name__ = f"b200_{name}_run"
    return run


def install(nystromngd):
    """Route the reference harness's NystromNGD / NGD-CG runs and its spectrum dump to the B200 path."""
    ref_optim, ref_harness = nystromngd.optim, nystromngd.harness
    if _saved:
        uninstall()
    _saved["runners"] = (ref_optim, dict(ref_optim._RUNNERS))
    _saved["spectrum"] = (ref_harness, ref_harness.gramian_spectrum)
    for name in INJECTED:
        ref_optim._RUNNERS[name] = _runner(name, ref_optim)

    def spectrum(problem, theta, quad, top=None):
        return _gramian_spectrum(device_problem(problem), np.asarray(theta, dtype=float), device_quadrature(quad),
                                 top=top)

    ref_harness.gramian_spectrum = spectrum


def uninstall():
    if "runners" in _saved:
        ref_optim, table = _saved.pop("runners")
        ref_optim._RUNNERS.clear()
        ref_optim._RUNNERS.update(table)
    if "spectrum" in _saved:
        ref_harness, fn = _saved.pop("spectrum")
        ref_harness.gramian_spectrum = fn
