"""B200-native NystromNGD inner solve (arXiv 2505.11638) -- drop-in for the
reference's operator / sketch / PCG / NGD-step API (nystromngd), computing on
sm_100a CUDA kernels through the C-ABI library libngd_b200.so."""

from . import _lib
from ._lib import NonFiniteError
from .gramian import DenseOperator, GramianOperator, ShiftedOperator, assemble_dense, gramian_spectrum, normalized_spectrum
from .krylov import SolveReport, pcg
from .model import MlpTopology, ParamVector, init
from .optim import (OPTIMIZER_NAMES, NystromNgdConfig, RunRecord, adapt_mu, adapt_rank, backtracking_linesearch,
                    ngd_cg_run, ngd_cg_step, nystrom_ngd_run, run_optimizer)
from .problems import (PROBLEM_NAMES, Heat1p1D, LaplacianStack, NonlinearPoisson2D, Poisson1D, Poisson2D, PoissonND,
                       QuadratureSet, make_problem)
from .sketch import NystromFactor, NystromPreconditioner, SketchFailure, effective_dimension, nystrom_approximate

__all__ = [
    "NonFiniteError", "DenseOperator", "GramianOperator", "ShiftedOperator", "assemble_dense", "SolveReport", "pcg",
    "MlpTopology", "ParamVector", "init", "NystromNgdConfig", "RunRecord", "adapt_mu", "adapt_rank",
    "backtracking_linesearch", "nystrom_ngd_run", "LaplacianStack", "Poisson2D", "PoissonND", "QuadratureSet",
    "make_problem", "NystromFactor", "NystromPreconditioner", "SketchFailure", "effective_dimension",
    "nystrom_approximate", "OPTIMIZER_NAMES", "run_optimizer", "ngd_cg_run", "ngd_cg_step", "PROBLEM_NAMES",
    "Poisson1D", "Heat1p1D", "NonlinearPoisson2D", "gramian_spectrum", "normalized_spectrum",
]
