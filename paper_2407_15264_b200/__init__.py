"""B200-native LSM-GNN feature-gather hot path (arXiv 2407.15264).

The product is liblsmgnn.so (paper_2407_15264_b200/csrc, C-ABI in include/lsmgnn.h);
this package is its thin ctypes binding. See DESIGN.md.
"""
from .binding import (BF16, F16, F32, POLICY, STATS_FIELDS, LsmGnn, LsmGnnError, Sampler, load_library,  # noqa: F401
                      check_handles, last_error, plan_handle, prefetch_dev)
