"""B200-native PHub parameter-exchange hot path (arXiv 1805.07891).

libphub.so (sm_100a CUDA + C++ host core, C ABI in include/phub.h) does the
work; this package is the thin ctypes binding (`capi`, same names as the C
entry points), a marshalling-only handle (`PHub`), and the multi-GPU plumbing
over torch.distributed (`sharded`).  Importing it loads libphub.so and fails
loudly if the library is missing -- there is no CPU fallback.
"""
from .capi import (  # noqa: F401
    PHUB_ALL_KEYS, PHUB_BORROW, PHUB_COPY, PhubError, EXPORTS, LIB_PATH,
)
from .phub import PHub  # noqa: F401
