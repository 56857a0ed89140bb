"""B200-native heterogeneous-compatible KV transmission path (arXiv 2509.17542, III-B).

Gather a finished prefill's paged KV, convert layout / block size / dtype / TP sharding
to the decode instance's, and deliver it into the decode pool -- on one GPU or across
NVLink.  The product is ``libkvx.so`` (include/kvx.h); this package is its thin binding.
Importing it without the built library raises (no CPU fallback).
"""
from .kv import *  # noqa: F401,F403
from .kv import __all__  # noqa: F401
