"""B200-native PAT decode attention: pack -> multi-tile forward -> merge.

Drop-in for the hot path of the reference ``prefixpack`` package
(``/root/reference/pkg/src/prefixpack/__init__.py:10-86``): the same public
names for the pack stage, the forward/merge entry point and the domain types;
the work runs in libpatb200.so (``include/pat.h``) -- a host C++ / CUDA packer
and hand-written sm_100a kernels.  The reference's analytical cost model,
simulator and CLI are out of scope.
"""

from .errors import (CoverageGap, EmptyFeasibleSet, EmptyPartialList, EmptySpan, InvalidChildIndex,
                     InvalidSpec, MissingRegisterEntry, NativeError, NoFeasibleConfig, NonPositiveDenominator,
                     PrefixpackError, ShapeMismatch)
from .workload import (BlockTable, CtaPack, Partition, WorkloadSpec, assemble_partition, generate_workload,
                       validate_partition)
from .packer import (CtaTask, PackCache, baseline_query_centric, naive_per_node, pack_batch, pack_batch_async,
                     split_long_kv)
from .plan import PatPlan
from .attention import PatDecoder, PatDeviceDecoder, PatLayerGraph, kv_pool_from_store, pat_attention, run_packed_attention
from .metrics import (TrafficReport, account_traffic, distinct_block_census, intermediate_round_trip_bytes,
                      kv_token_bytes, theoretical_min_kv_bytes)
from .forest import PrefixForest, PrefixNode, build_forest, flatten_forest, pack_forest, tree_heuristic
from .numerics import (PartialBatch, PartialResult, cta_partial, dump_tensors, full_attention, gather_kv,
                       generate_qkv, load_tensors, max_rel_error, merge_partials)
from .schedule import TileConfig, assign_streams, plan_tasks
from .calibration import CostModel, get_cost_model, load_profile, set_cost_model
from .torch_op import decode_attention  # registers torch.ops.patb200.decode_attention

__version__ = "0.1.0"
