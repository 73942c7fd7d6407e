"""B200-native KVQuant decode hot path (arXiv 2401.18079).

The product is libkvq.so (C ABI in include/kvq.h, sm_100a kernels in csrc/); this
package holds its thin Python binding (``kvq``), the sequence-sharding glue
(``sharding``) and layout byte accounting (``accounting``).
"""
from .kvq import KVQCache, KVQError, merge_partials, version  # noqa: F401
