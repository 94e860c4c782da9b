"""B200-native Flash3D hot path: PSH bucketing, bucket-swin attention,
in-bucket pooling, and the row scatter/gather around them.

Drop-in for the reference package ``bucketswin`` (same module names,
signatures, defaults and exception classes) — ``import
paper_2412_16481_b200 as bucketswin``.  Compute runs in hand-written sm_100a
CUDA (libf3d.so, include/f3d.h); there is no CPU fallback.
"""

from .attention import (AttentionParams, CopyMeter, ScopeSchedule, build_schedule,
                        copy_meter, logical_gather, lowest_period, positional_encoding,
                        reference_attention, tiled_attention)
from .bucketing import (BucketAssignment, ProbeSchedule, assign_buckets,
                        assign_buckets_two_stage, claim_slot, compute_bucket_base,
                        default_probe_schedule, gather, optimistic_race, scatter)
from .errors import (ConfigError, EmptyInputError, IntegrityError, NumericError,
                     ParseError, RangeError)
from .geometry import PointCloud, VoxelGrid, synth_cloud, voxelize
from .hashing import (HASH_KINDS, HashConfig, hash_bucket, morton_encode,
                      remap_nonnegative)
from .pooling import (SubBucketAssignment, build_subbuckets, pool_features,
                      pool_stage, pool_stage_map, unpool)
from .stage import StageParams, gelu, init_params, layer_norm, stage_forward

__version__ = "0.1.0"
