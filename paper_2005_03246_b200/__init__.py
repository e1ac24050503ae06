"""B200-native generalized ECDF / ESF / Laplacian-KDE (arXiv 2005.03246) — drop-in for the
reference package ``fastcdf``'s hot path (fastcdf/__init__.py:6-62 names).

Host side: Python + PyTorch (device memory, streams, torch.distributed).  Compute: the sm_100a
C-ABI library ``libfastcdf_b200.so`` (include/fastcdf_b200.h) loaded with ctypes.  There is
no CPU fallback.
"""

from .core import (
    EXP_OVERFLOW_GUARD,
    GRID_ALIGNED,
    POINT_ALIGNED,
    Bandwidth,
    DegenerateRangeError,
    DeltaVector,
    EvalResult,
    OverflowGuardError,
    ParameterError,
    RectilinearGrid,
    Sample,
    ShapeError,
    TieError,
    ValidationError,
    all_deltas,
    build_grid_auto,
    generate_gaussian_sample,
    read_result_csv,
    read_sample_csv,
    validate_sample,
    write_result_csv,
    write_sample_csv,
)
from .fastsum import (
    CumulativeTensor,
    directional_sweep,
    ecdf_fastsum,
    ecdf_fastsum_counts,
    esf_fastsum,
    kde_fastsum,
)
from .histogram import LocalSumTensor, local_sums, local_sums_sorted, local_sums_uniform
from .kernels import (
    KernelSpec,
    gaussian,
    laplacian,
    matern32_additive,
    matern32_product,
    parse_kernel_spec,
    uniform,
)

from .dnc import DeltaTermTable, ecdf_dnc, kde_dnc, kde_terms_dnc, rank_tiebreak
from .points import (
    ecdf_at_points,
    ecdf_esf_at_points,
    esf_at_points,
    kde_numerators,
    kernel_regression,
    rank_f64,
)
from .interp import multilinear_interp

__version__ = "0.1.0"
