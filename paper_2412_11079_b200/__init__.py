"""B200-native fused Sinkhorn-UOT (MAP-UOT, arxiv 2412.11079) behind the
reference solver API. See DESIGN.md; the C ABI is include/uot_cuda.h."""
from .uot import (  # noqa: F401
    ConfigError, CudaError, CudaExtensionMissing, DegenerateSum, Error, FusedState,
    InvalidParameter, PartitionError, Problem, RankPartition, ScalingFactors, Session,
    SolveReport, SolveResult, compute_fi, convergence_error, fused_iterate, fused_solve,
    gen_problem_t, init_col_sums, lib, rescale_factor,
)
