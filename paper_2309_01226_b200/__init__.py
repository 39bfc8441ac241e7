"""B200-native batched SPASE plan evaluation and search (arXiv 2309.01226, "Saturn").

The product is libsaturn.so (C ABI in include/saturn.h, sm_100a kernels in csrc/);
this package is its thin binding.  See DESIGN.md.
"""
from .saturn import (  # noqa: F401
    Plan, SearchConfig, SaturnError, Placement, PLACEMENT_DTYPE, EXPORTS, LIB_PATH, BASELINES,
    load_library, partition, get_unique_id, broadcast_unique_id, attach_distributed, attach_peers, peer_name, q32,
    plan_create, load_runtime_table, evaluate, enumerate, search, search_group, best_plan,
    DECODER_AUTO, DECODER_THREAD, DECODER_WARP, DECODER_NODE_SMEM, EVENT_STOP, EVENT_ARRIVE, PROVEN_OPTIMAL, INCUMBENT, PREFIX_SHARED, SYMMETRY_REDUCED, ENUM_SYMMETRY,
    OK, EINVAL, EUNSCHEDULABLE, ELIMIT, ECUDA, ENCCL, ESTATE,
)
