"""Shared test helpers (no pytest fixtures)."""
import ctypes


def _cuda_available():
    try:
        import ctypes

        lib = ctypes.CDLL("libcuda.so.1")
        n = ctypes.c_int(0)
        if lib.cuInit(0) != 0:
            return False
        return lib.cuDeviceGetCount(ctypes.byref(n)) == 0 and n.value > 0
    except OSError:
        return False


HAS_GPU = _cuda_available()
