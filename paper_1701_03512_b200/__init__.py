"""paper_1701_03512_b200 -- B200-native engine for arXiv 1701.03512.

Drop-in for the hot path of the reference ``binpaths`` package: exact
expected values of path-dependent payoffs over all 2^N paths of a
recombinant binomial tree, and the stratified ("partitioned") Monte Carlo
estimators.  The Python layer mirrors the reference API (same names,
arguments and exceptions); the work runs in hand-written sm_100a CUDA
kernels behind the C ABI in include/binpaths_b200.h.
"""
from .errors import (DeviceError, EnumerationGuard, InfeasibleAllocation, InvalidInput, InvalidWorkerCount,
                     LengthMismatch, NonConstantProbs, PathDependentPayoff, PricingError, ProbabilityOutOfRange,
                     RankOutOfRange)
from .model import (MAX_DEPTH, MarketInputs, TreeParams, asset_path, classic_crr, derive_crr, leaf_prices,
                    with_custom_probs)
from .paths import (BernoulliPath, PathPartition, block_code_ranges, block_probability, codes_to_bits, iter_block,
                    make_partition, path_probability)
from .payoffs import (ASIAN_CALL, FLOATING_LOOKBACK, GpuPayoff, PayoffKind, kind_bit, parse_payoff, payoff,
                      payoff_batch, resolve_kind)
from .mc import (Estimate, McConfig, PhiloxStream, RepetitionSummary, allocate_strata, estimate_basic,
                 estimate_partitioned, estimate_partitioned_equal, estimate_shared, mc_stream, run_repetitions,
                 sample_path)
from .exact import (LARGE_DEPTH, ExactResult, ValuationRequest, price_batch, value_exact, value_exact_batch,
                    value_exact_parallel, value_exact_serial, value_leaf_formula)

from .bench import BENCH_CSV_HEADER, BenchRecord, records_to_csv, records_to_tables, run_bench

__version__ = "0.1.0"
