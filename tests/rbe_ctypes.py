"""The reference-side ctypes binding of the C ABI (include/rbe_cuda.h) that a
maintainer of the reference would add -- shown in INTEGRATION.md and exercised
as-is by tests/test_gpu_abi.py (GPU) and tests/test_abi.py (symbols, CPU).
Every entry point gets its argtypes/restype, so 64-bit sizes are never passed as
C ints."""
import ctypes as C
import os

import numpy as np

LIB_PATH = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1802_06466_b200", "_lib",
                        "librbe_cuda.so")


class Geometry(C.Structure):  # rbe::ScanGeometry, reference include/rbe/search.hpp:12-21
    _fields_ = [("blocks", C.c_uint32), ("threads_per_block", C.c_uint32), ("items_per_thread", C.c_uint32),
                ("queue_length", C.c_uint32)]


class Shape(C.Structure):  # KeywordIndex header, reference include/rbe/index.hpp:23-27
    _fields_ = [("dim", C.c_uint32), ("keyword_planes", C.c_uint32), ("residual_weights", C.c_uint32)]


class Stats(C.Structure):  # rbe_search_stats
    _fields_ = [("scored", C.c_uint64), ("variant", C.c_uint32), ("fallback", C.c_uint32),
                ("candidates", C.c_uint64), ("survivors", C.c_uint64), ("scan_ms", C.c_double),
                ("total_ms", C.c_double), ("launches", C.c_uint32), ("reserved", C.c_uint32 * 3)]


class LoadStats(C.Structure):  # rbe_load_stats
    _fields_ = [("file_bytes_read", C.c_uint64), ("seconds", C.c_double)]


def _ptr(t):
    return np.ctypeslib.ndpointer(dtype=t, flags="C_CONTIGUOUS")


def load(path=LIB_PATH):
    lib = C.CDLL(path)
    vp, u32, u64, i32 = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int
    lib.rbe_cuda_last_error.restype = C.c_char_p
    lib.rbe_cuda_last_error.argtypes = []
    lib.rbe_cuda_version.restype = C.c_char_p
    lib.rbe_cuda_version.argtypes = []
    lib.rbe_cuda_index_create.restype = i32
    lib.rbe_cuda_index_create.argtypes = [C.POINTER(Shape), u32, _ptr(np.uint32), _ptr(np.uint64), i32,
                                          C.POINTER(vp)]
    lib.rbe_cuda_index_upload_partition.restype = i32
    lib.rbe_cuda_index_upload_partition.argtypes = [vp, u32, _ptr(np.uint64), _ptr(np.float32), _ptr(np.uint64)]
    lib.rbe_cuda_index_destroy.restype = i32
    lib.rbe_cuda_index_destroy.argtypes = [vp]
    lib.rbe_cuda_index_bytes.restype = i32
    lib.rbe_cuda_index_bytes.argtypes = [vp, C.POINTER(u64), C.POINTER(u64)]
    lib.rbe_cuda_search.restype = i32
    lib.rbe_cuda_search.argtypes = [vp, _ptr(np.uint64), u32, u32, C.POINTER(Geometry), u64, vp,
                                    _ptr(np.float64), _ptr(np.uint64), _ptr(np.uint32), _ptr(np.int64),
                                    _ptr(np.uint64), C.POINTER(Stats)]
    # RBEI v1 straight into HBM (replaces load_index + upload, reference src/index.cpp:170-208)
    lib.rbe_cuda_rbei_header.restype = i32
    lib.rbe_cuda_rbei_header.argtypes = [C.c_char_p, C.POINTER(Shape), C.POINTER(u32), _ptr(np.uint64), u32]
    lib.rbe_cuda_index_open_rbei.restype = i32
    lib.rbe_cuda_index_open_rbei.argtypes = [C.c_char_p, vp, u32, i32, u32, C.POINTER(vp), C.POINTER(LoadStats)]
    return lib


class Index:
    """One device index built from reference-layout partitions [(planes[kp][count*wpp] u64,
    magnitudes f32, ids u64)] -- what the reference's KeywordIndex holds (index.hpp:16-34)."""

    def __init__(self, lib, dim, kp, rw, partitions, device=0):
        self.lib, self.dim = lib, dim
        counts = np.array([len(p[2]) for p in partitions], dtype=np.uint64)
        ords = np.arange(len(partitions), dtype=np.uint32)
        self.h = C.c_void_p()
        self._ck(lib.rbe_cuda_index_create(C.byref(Shape(dim, kp, int(rw))), len(partitions), ords, counts, device,
                                           C.byref(self.h)))
        for i, (planes, mags, ids) in enumerate(partitions):
            self._ck(lib.rbe_cuda_index_upload_partition(
                self.h, i, np.ascontiguousarray(planes, np.uint64).reshape(-1), np.ascontiguousarray(mags, np.float32),
                np.ascontiguousarray(ids, np.uint64)))

    @classmethod
    def open_rbei(cls, lib, path, device=0):
        """The whole RBEI file on one device (rbe_cuda_index_open_rbei, partitions = all)."""
        self = cls.__new__(cls)
        self.lib = lib
        shape, P = Shape(), C.c_uint32()
        self._ck(lib.rbe_cuda_rbei_header(str(path).encode(), C.byref(shape), C.byref(P), np.zeros(1, np.uint64), 0))
        self.dim = shape.dim
        self.h = C.c_void_p()
        self.stats = LoadStats()
        self._ck(lib.rbe_cuda_index_open_rbei(str(path).encode(), None, 0, device, 0, C.byref(self.h),
                                              C.byref(self.stats)))
        return self

    def _ck(self, rc):
        if rc != 0:
            msg = self.lib.rbe_cuda_last_error().decode()
            raise {1: ValueError, 2: IndexError}.get(rc, RuntimeError)(msg)

    def search(self, query_words, geometry, n):
        """query_words [Q][qp][wpp] u64 -> list of [(score, id, partition)] per query, plus stats."""
        q = np.ascontiguousarray(query_words, np.uint64)
        Q, qp = q.shape[0], q.shape[1]
        scores = np.zeros(Q * n, np.float64)
        ids = np.zeros(Q * n, np.uint64)
        parts = np.zeros(Q * n, np.uint32)
        accs = np.zeros(Q * n, np.int64)
        cnt = np.zeros(Q, np.uint64)
        st = Stats()
        self._ck(self.lib.rbe_cuda_search(self.h, q.reshape(-1), Q, qp, C.byref(Geometry(*geometry)), n, None, scores,
                                          ids, parts, accs, cnt, C.byref(st)))
        out = [list(zip(scores[k * n:k * n + int(cnt[k])].tolist(), ids[k * n:k * n + int(cnt[k])].tolist(),
                        parts[k * n:k * n + int(cnt[k])].tolist())) for k in range(Q)]
        return out, st

    def close(self):
        if self.h:
            self._ck(self.lib.rbe_cuda_index_destroy(self.h))
            self.h = C.c_void_p()
