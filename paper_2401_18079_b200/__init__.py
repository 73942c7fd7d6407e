"""B200-native KVQuant decode hot path (arXiv 2401.18079).

The product is libkvq.so (C ABI in include/kvq.h, sm_100a kernels in csrc/); this
package holds its thin Python binding (``kvq``), the sequence-sharding glue
(``sharding``) and layout byte accounting (``accounting``).  The binding is imported
lazily so that ``paper_2401_18079_b200._build`` can (re)build the library first.
"""
__all__ = ["KVQCache", "KVQError", "merge_partials", "version"]


def __getattr__(name):
    if name in __all__:
        from . import kvq
        return getattr(kvq, name)
    raise AttributeError(name)
