"""paper_1508_03167_b200: B200-native MergeShuffle (arXiv 1508.03167).

Drop-in for the reference shufflekit's MergeShuffle path: same entry points,
bit-identical permutations and bit counts, computed by hand-written sm_100a
CUDA kernels behind a C ABI (include/shufflekit_b200.h).
"""
from .bitstream import BitSource, advance_state, mix64, substream_seed
from .shufflers import (MERGE_CUTOFF_DEFAULT, MergeRange, ShuffleConfig, ShuffleReport, batched_shuffle,
                        fisher_yates, merge, merge_plan, merge_rounds, merge_shuffle, merge_shuffle_parallel,
                        merge_task_indices)
from .balanced import balanced_shuffle
from .splitshuffle import RS_CUTOFF_DEFAULT, rs_shuffle, rs_shuffle_parallel
from .verify import ChiSquareResult, chi_counts, chi_square_threshold, chi_square_uniformity, permutation_rank

__version__ = "0.1.0"

__all__ = [
    "BitSource", "mix64", "substream_seed", "advance_state", "MergeRange", "ShuffleConfig", "ShuffleReport", "MERGE_CUTOFF_DEFAULT", "fisher_yates",
    "merge", "merge_plan", "merge_rounds", "merge_task_indices", "merge_shuffle", "merge_shuffle_parallel",
    "batched_shuffle", "ChiSquareResult", "chi_counts", "chi_square_threshold", "chi_square_uniformity",
    "permutation_rank", "balanced_shuffle", "RS_CUTOFF_DEFAULT", "rs_shuffle", "rs_shuffle_parallel",
]
