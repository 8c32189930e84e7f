"""B200-native TABI atlas packer (arxiv 2602.07782).

The product path is ``libtabi.so`` (hand-written sm_100a CUDA kernels behind
the C ABI in ``include/tabi.h``); this package is its thin Python binding.
"""
from .tabi import (CAND_DTYPE, EINVAL, ECAPACITY, ECUDA, EXPORTS, F_ADJACENT_LOCKS_ONLY, PENDING,  # noqa
                   F_EXACT_TAIL, F_NO_BALANCE, F_NO_HC, F_NO_OBB, F_PREROTATE, NO_FIT, OK, PLACEMENT_DTYPE,
                   PROXY_DTYPE, ABLATIONS, Context, Validation,
                   BatchInfo, Info, Spec, TabiError, concat_chart_sets, latency_floor, lib, make_spec,
                   pack_batch,
                   shard_plan, spec_of)
