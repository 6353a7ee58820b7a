"""B200-native time step of the meshfree ALE scheme for the BGK equation (arXiv 2408.02350).

The method runs in hand-written sm_100a CUDA kernels behind the C ABI in
``include/bgk.h`` (library ``libbgk_b200.so``, built in-tree); this package is
the thin Python binding.  There is no CPU fallback: ``Bgk`` raises if the
library is missing.
"""
from ._lib import EXPORTED, BgkError, load  # noqa: F401

__all__ = ["Bgk", "BgkError", "load", "EXPORTED", "make_config"]


def __getattr__(name):
    # torch is imported lazily so that `import paper_2408_02350_b200` stays light
    if name in ("Bgk", "make_config"):
        from . import api
        return getattr(api, name)
    raise AttributeError(name)
