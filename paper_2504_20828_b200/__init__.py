"""B200-native (sm_100a) Ascendra urgency scheduler and batch-level serving simulator.

The hot path lives in libasc.so (include/asc.h); `asc` is its thin ctypes binding.
"""
from . import asc  # noqa: F401
