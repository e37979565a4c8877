"""B200-native frontier traversal + batch updates (BYO graphbench hot path).

The product is the CUDA library ``libgbg.so`` behind the C ABI in
``include/gbg_c.h``; ``graph`` is its Python host mirror.  Attributes are
resolved lazily so ``python -m paper_2405_11671_b200.build`` works before the
library exists.
"""
import importlib

__all__ = ["graph"]


def __getattr__(name):
    mod = importlib.import_module(__name__ + ".graph")
    if name == "graph":
        return mod
    try:
        return getattr(mod, name)
    except AttributeError:
        raise AttributeError(name) from None
