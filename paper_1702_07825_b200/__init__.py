"""B200-native autoregressive WaveNet sample generation (Deep Voice, arXiv 1702.07825).

The product is libdvw.so (C ABI in include/dvw.h, CUDA kernels for sm_100a in
csrc/).  ``Model`` is its thin ctypes binding (``_lib``); ``synth`` holds the
seeded synthetic input generators.  Importing ``Model`` without a built
libdvw.so raises -- there is no CPU fallback.
"""
from . import synth  # noqa: F401

__all__ = ["synth", "Model", "DvwError"]


def __getattr__(name):
    if name in ("Model", "DvwError", "weights_numel"):
        from . import _lib
        return getattr(_lib, name)
    raise AttributeError(name)
