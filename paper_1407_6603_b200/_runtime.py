"""Per-thread default device handle for the reference-shaped Python API.

The reference's compiled kernel may be called from several threads on
disjoint stores at once (engine.py:89 ``nogil=True``). Each Python thread
therefore gets its own ``Handle`` (own CUDA stream and buffers); ctypes
releases the GIL around every library call.
"""

from __future__ import annotations

import os
import threading

from ._native import Handle

_tls = threading.local()


def device_index() -> int:
    return int(os.environ.get("WSORT_DEVICE", "0"))


def default_handle() -> Handle:
    h = getattr(_tls, "handle", None)
    if h is None:
        h = Handle(device_index())
        _tls.handle = h
    return h
