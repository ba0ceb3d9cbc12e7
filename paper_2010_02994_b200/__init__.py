"""B200-native Hawkes log-likelihood + location-gradient hot path (arXiv 2010.02994).

The product is the C-ABI library ``libhawkes_b200.so`` (include/hawkes.h, sources in
``csrc/``); ``hawkes`` is its thin Python binding.
"""
from .hawkes import HawkesContext, HawkesError, diag_exp, diag_fp64_peak, nccl_unique_id  # noqa: F401
from .sharding import init_distributed_context  # noqa: F401
