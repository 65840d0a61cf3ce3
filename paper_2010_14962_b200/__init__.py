"""B200-native sliced tensor-network contraction engine (arXiv 2010.14962 hot path).

The engine replaces the reference's per-slice path sum_range -> apply_cut ->
execute_plan -> contract_pair (proj/core/src/executor.cpp:45-68) with
hand-written sm_100a CUDA behind a C-ABI (include/qcut_gpu.h).
"""
from .engine import Engine, RankGuardError, contract_pair, contract_pair_bench, load_library  # noqa: F401
from .shard import aggregate, round_count, shard_range  # noqa: F401

__all__ = ["Engine", "RankGuardError", "contract_pair", "contract_pair_bench", "load_library", "aggregate", "round_count", "shard_range"]
