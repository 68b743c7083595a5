"""B200-native (sm_100a) hot path of AWRTRD / SAWRTRD (arXiv 2305.09044).

The product is libtrd.so (C ABI in include/trd.h); ``trd`` is its ctypes binding.
"""
from .trd import (TRD, TrdError, load_library, declared_symbols, nccl_unique_id,  # noqa: F401
                  TRD_SIGMA_FIXED, TRD_SIGMA_INF, TRD_SIGMA_RMS)
