"""B200-native (sm_100a) spike-wave step of SpykeTorch (arxiv 1903.02440).

``snn``      thin ctypes binding of libsnn.so (include/snn.h, the C ABI)
``pipeline`` per-config compositions of the ABI calls (the paper's forward / training passes)
``build``    nvcc build of libsnn.so in-tree
"""
from . import snn  # noqa: F401

__all__ = ["snn"]
