"""B200-native exhaustive retrieval for Recurrent Binary Embeddings (arXiv 1802.06466).

Drop-in for the reference's ``rbe._core`` retrieval surface (pack, make_embedding,
build_index, save_index/load_index, ScanGeometry, thread_assignment, search) plus
``DeviceIndex`` (the HBM-resident store) and ``search_batch``.  Retrieval runs
only on sm_100a kernels through the C ABI in include/rbe_cuda.h; importing works
without a GPU, but every search raises RuntimeError when no B200 is usable.
There is no CPU fallback.
"""
from __future__ import annotations

import os as _os

_LIB = _os.path.join(_os.path.dirname(_os.path.abspath(__file__)), "_lib")

try:
    from ._lib import _core  # noqa: F401
except ImportError as _e:  # fail loudly: the native extension is the product
    raise ImportError(
        "paper_1802_06466_b200 native extension is not built "
        "(run `python -m paper_1802_06466_b200.build`): " + str(_e)
    ) from _e

from ._lib._core import *  # noqa: F401,F403,E402

LIB_DIR = _LIB
CUDA_LIBRARY = _os.path.join(_LIB, "librbe_cuda.so")


def pinned_empty(shape, dtype=float):
    """numpy array in page-locked host memory (rbe_cuda_host_alloc).  Used as the ``out=``
    arrays of ``DeviceIndex.search_words``, results are DMA'd straight into it."""
    import ctypes
    import weakref

    import numpy as np

    lib = ctypes.CDLL(CUDA_LIBRARY)
    dt = np.dtype(dtype)
    count = int(np.prod(shape)) if not isinstance(shape, int) else shape
    nbytes = max(count * dt.itemsize, 1)
    ptr = ctypes.c_void_p()
    if lib.rbe_cuda_host_alloc(ctypes.c_size_t(nbytes), ctypes.byref(ptr)) != 0:
        lib.rbe_cuda_last_error.restype = ctypes.c_char_p
        raise RuntimeError(lib.rbe_cuda_last_error().decode())
    buf = (ctypes.c_char * nbytes).from_address(ptr.value)
    weakref.finalize(buf, lib.rbe_cuda_host_free, ctypes.c_void_p(ptr.value))
    return np.frombuffer(buf, dtype=dt, count=count).reshape(shape)
