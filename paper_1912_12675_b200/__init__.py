"""paper_1912_12675_b200 -- pipelined backpropagation with stale weights on B200.

Thin ctypes binding over libpst.so (include/pst.h, include/pst_ops.h):
argument marshalling only; every step of the training path runs in the
library's sm_100a kernels.  There is no CPU fallback: if libpst.so is missing
or cannot be loaded this package raises at import of `lib()`.
"""
from .binding import (PstError, Pipeline, lib, build_info, schedule, partition_ranges, ring_slots,
                      param_count, nccl_unique_id, ops, net_struct, W_PARAMS, W_MOMENTUM,
                      W_BNSTATS)

__all__ = ["PstError", "Pipeline", "lib", "build_info", "schedule", "partition_ranges", "ring_slots",
           "param_count", "nccl_unique_id", "ops", "net_struct", "W_PARAMS", "W_MOMENTUM",
           "W_BNSTATS"]
