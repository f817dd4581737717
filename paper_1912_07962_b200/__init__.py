"""B200-native slimLS: the sampled limited-memory row-action LS iteration.

Drop-in for the reference package's slimLS path (``slimsolve.solvers.run``
with its operator, sampler, schedule and Trajectory types); the per-step
work runs as hand-written sm_100a CUDA kernels behind the C-ABI in
``include/slimb200.h``.
"""

from .linops import (
    DenseBlockOperator,
    GeneratedBlockOperator,
    RowBlockOperator,
    SampleBlock,
    SinglePassAdapter,
    SparseBlockOperator,
    StreamOrderError,
    device_operator,
)
from .sampling import Sampler
from .solvers import (
    DIVERGENCE_FACTOR,
    METHODS,
    DivergenceError,
    Schedule,
    Trajectory,
    dual_step,
    potrf,
    run,
)

__version__ = "0.1.0"
