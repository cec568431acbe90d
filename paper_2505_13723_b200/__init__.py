"""B200-native ADASAP (arXiv 2505.13723) -- drop-in for the reference ``sapgp``
hot path: kernel oracle, partitioned block products, randomised Nystrom
preconditioning and the accelerated approximate sketch-and-project solver,
with the block-row product K[B,:] W in hand-written sm_100a CUDA
(``csrc/``, C ABI in ``include/sapgp_b200.h``).

Public names mirror pkg/src/sapgp/__init__.py:24-73 for the hot path.
Nothing here falls back to the CPU: without ``_lib/libsapgp_b200.so`` or a
CUDA device every product raises ``WorkerError``.
"""

__version__ = "0.1.0"

from .baselines import pcg_solve, sap_solve, sdd_solve  # noqa: F401
from .config import RunConfig, kernel_from_dict  # noqa: F401
from .dist import WorkerPool, col_dist_matmul, row_dist_matmul  # noqa: F401
from .errors import (  # noqa: F401
    ConfigError,
    ContractError,
    NumericalError,
    ParseError,
    SapgpError,
    ValidationError,
    WorkerError,
)
from .gp import (  # noqa: F401
    ExactPrior,
    PosteriorMean,
    PosteriorSampleSet,
    RandomFeatureMap,
    RandomFeaturePrior,
    mean_nll,
    pathwise_sample,
    posterior_mean,
    rmse,
    sample_prior,
)
from .kernels import (  # noqa: F401
    KernelOracle,
    KernelSpec,
    block_block,
    block_rows_times,
    cross_kernel,
    kernel_eval,
)
from .randnla import (  # noqa: F401
    NystromFactor,
    apply_inv,
    apply_inv_plain,
    apply_inv_sqrt,
    rand_nystrom,
    rand_nystrom_retry,
    rand_power_stepsize,
)
from .solvers import (  # noqa: F401
    NO_ACCELERATION,
    AccelParams,
    AdasapEngine,
    ConvergenceTrace,
    RawAccel,
    SolveResult,
    SolverState,
    adasap_solve,
    adasap_step,
    make_state,
    nesterov_update,
    resolve_accel,
    solve,
    tail_average,
)
