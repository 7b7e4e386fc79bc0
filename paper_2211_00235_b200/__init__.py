"""B200-native Parallel Evoformer block + Branch Parallelism (arXiv
2211.00235), drop-in for the reference package's block and train-step
API (src/__init__.py:1-40).  Compute runs only through the sm_100a CUDA
library (include/evo_b200.h); there is no CPU fallback."""

from .errors import (BranchparError, CollectiveError, ComparisonError, ConfigError,
                     ContractError, DimensionError, NumericsError, WorldError)
from .evoformer import (EvoConfig, ParamStore, col_attn, evoformer_block, evoformer_stack,
                        get_precision, init_params, msa_track, msa_transition, opm,
                        pair_track, pair_transition, param_count, row_attn, seeded_inputs,
                        set_precision, tri_attn, tri_mult)
from .schedules import (ParallelLayout, RunResult, compare_runs, expected_comm_volume,
                        make_batch, run_single, trace_volume)
from .distributed import CommRecord, CommTrace, run_bp, run_dap, run_distributed, run_dp

__version__ = "0.1.0"
