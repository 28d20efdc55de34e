"""B200-native Global-QSGD compressed gradient sync (arxiv 2305.18627).

The product is libgq_b200.so (sm_100a CUDA kernels behind the C-ABI in
include/gq_b200.h); `gqsgd` mirrors the reference's gqsgd:: API on top of it.
"""
from .gqsgd import (CommEvent, GqsgdConfig, InprocSync, IntSumOps, LevelKind,  # noqa: F401
                    MeanResult, NormSpec, PayloadOps, Schedule, TokenReduceOps, TopologyKind,
                    TrafficReport, allreduce_inproc, allreduce_schedule, baseline_mean, check_width,
                    chunk_lane_range, make_schedule, ring_schedule, tree_schedule,
                    combine_norm_stats, decode, global_norm, gqsgd_mean, lane_bytes,
                    local_norm_stats, plan_path, prescale_shift, quantize_shard,
                    standard_lane_width)
from ._lib import DomainError, InvalidArgument, LaneOverflow, RuntimeFailure  # noqa: F401
