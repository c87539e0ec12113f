"""rtk-b200: B200-native (sm_100a) radix top-k with the reference's rtk:: interface.

The compute path is librtk_b200.so (hand-written CUDA behind the C-ABI in include/rtk_c.h);
this package is the thin host mirror of /root/reference/proj/include/rtk/.
"""
from .rtk import (BatchInput, BatchOptions, BatchRunInfo, BufferPolicy, EngineConfig,
                  Instrumentation, ScaleInfo, ScaleMode, ScalePolicy, SelectionOrder, TopKResult,
                  batch_topk, batch_topk_dense, empty_input_error, invariant_violation, last_stats, merge_shards,
                  rank_out_of_range, scaled_topk, set_option, topk, topk_sample)

__all__ = [
    "BatchInput", "BatchOptions", "BatchRunInfo", "BufferPolicy", "EngineConfig",
    "Instrumentation", "ScaleInfo", "ScaleMode", "ScalePolicy", "SelectionOrder", "TopKResult",
    "batch_topk", "batch_topk_dense", "empty_input_error", "invariant_violation", "last_stats", "merge_shards",
    "rank_out_of_range", "scaled_topk", "set_option", "topk", "topk_sample",
]
