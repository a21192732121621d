"""B200-native randomized complete pivoting (RCP) block LDL^T factor/solve.

Drop-in for the reference ``randldl`` factor/solve path (arXiv 1710.00125):
``factor``, ``factor_robust``, ``solve``, ``solve_many``, ``reconstruct`` with
the reference's ``FactorConfig`` / ``Factorization`` / ``BlockDiag`` /
``GrowthStats`` / ``SolveReport`` types.  All arithmetic runs in the sm_100a
CUDA library ``librcp_b200.so`` (see ``include/rcp_b200.h``).
"""

from .api import (  # noqa: F401
    PAT_DEFICIENT,
    PAT_PAIR_END,
    PAT_PAIR_START,
    PAT_SINGLE,
    SBKP_ALPHA,
    BlockDiag,
    DeviceFactorization,
    FactorConfig,
    Factorization,
    GrowthStats,
    GrowthTracking,
    NumericalError,
    OpCounters,
    SolveReport,
    Strategy,
    factor,
    factor_device,
    factor_robust,
    reconstruct,
    reconstruct_device,
    solve,
    solve_device,
    solve_many,
)
from ._native import NativeUnavailable  # noqa: F401
from .batched import (  # noqa: F401
    BatchedDeviceFactorization,
    factor_batched,
    factor_batched_device,
    factor_batched_sharded,
    shard_range,
    solve_batched,
    solve_batched_device,
)

from . import grid  # noqa: F401,E402

__version__ = "0.2.0"
