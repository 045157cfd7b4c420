"""B200-native online loop of the history-aware iSVD adaptive ROM.

Drop-in for the hot path of the reference package ``adrom``
(/root/reference/pkg/src/adrom, arXiv 2605.28684): same names, argument
meaning and error behaviour for the functions on that path, computed by
hand-written sm_100a CUDA kernels behind the C-ABI in
``include/adrom_b200.h`` (``lib/libadrom_b200.so``).  No CPU fallback.
"""

from .errors import DenseError, RomStepError
from .fom import (
    BurgersProblem,
    FomProblem,
    NewtonResult,
    ReactingEulerProblem,
    SodProblem,
    TimeStepper,
    coarse_step,
    fd_jacobian,
    fd_jacobian_blocks,
    implicit_step,
    reacting_mechanism,
    rusanov_flux,
    sod_initial_state,
)
from .dense import (SvdResult, least_squares, max_principal_angle, newton_solve, orth, pivoted_qr,
                    principal_angles, thin_svd)
from .tracking import (ReducedBasis, SnapshotWindow, UpdateRule, direct_update, grouse_update,
                       isvd_update, oja_update, onestep_update, wsvd_update)

__version__ = "0.1.0"

from .sampling import (  # noqa: F401
    FeatureMap, SamplingPlan, SamplingSet, build_deim_operator, fgs_sample, qdeim_sample,
    stencil_closure)
from .snapshots import ScalingTransform, fit_scaling, pod  # noqa: F401
from .projection import (  # noqa: F401
    ReducedState, RomOperator, RomStepResult, build_rom_operator, decode, encode,
    galerkin_step, lspg_objective, lspg_step, rom_step)
from .driver import (  # noqa: F401
    ExperimentConfig, RunResult, acceleration, make_problem, relative_error,
    run_adaptive_rom, run_fom, run_static_rom)
