"""B200-native µop decode engine (VDCores decoupled µop model on sm_100a).

Host side: the uopsim C++ builder (isa / workload / costmodel / generator,
include/uopsim/*.hpp) behind the C-ABI in include/vdc.h. Device side: one
persistent sm_100a kernel executing µop streams (memory virtual cores feeding
shared-memory slots with bulk copies, compute virtual cores running the
handlers, device-side dependency counters/queues).
"""
from ._native import KvPages, Program, VdcError, lib  # noqa: F401
