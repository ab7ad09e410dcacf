"""ctypes front-end to the parity checkers (TEST INFRASTRUCTURE ONLY).

Two checkers, both CPU:
  * ``Ref``    -- the reference's own hot-path sources compiled unmodified
                  (oracle/_ref/librbe_ref.so, see oracle/Makefile): rbe::search,
                  rbe::local_select/global_select, rbe::binary_dot, ... .
  * ``Port``   -- the plain-C restatement oracle/rbe_oracle.c
                  (oracle/_build/librbe_oracle.so), pinned against ``Ref`` and
                  the SPEC.md KATs by tests/test_oracle.py.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "librbe_ref.so")
PORT_SO = os.path.join(HERE, "_build", "librbe_oracle.so")

U64P = C.POINTER(C.c_uint64)
F32P = C.POINTER(C.c_float)
F64P = C.POINTER(C.c_double)
U32P = C.POINTER(C.c_uint32)
I64P = C.POINTER(C.c_int64)

GAMMA = 0x9E3779B97F4A7C15
MASK64 = (1 << 64) - 1


def _p(a, t):
    return a.ctypes.data_as(t)


def wpp_of(dim: int) -> int:
    return (dim + 63) // 64


# ----------------------------------------------------------------------------
# numpy restatement of the counter-based generator; used for
# vectorised fixture generation, cross-checked against rbo_splitmix64_at.
def splitmix64_at(seed: int, j: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + (j.astype(np.uint64) + np.uint64(1)) * np.uint64(GAMMA)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def pad_mask(dim: int) -> int:
    return MASK64 if dim % 64 == 0 else (1 << (dim % 64)) - 1


def gen_partition_planes(seed, n_total, dim, kp, n_partitions, p):
    """[kp][count*wpp] u64 plane blocks of partition p (global doc i -> i%P)."""
    wpp = wpp_of(dim)
    count = (n_total - p + n_partitions - 1) // n_partitions if p < n_total else 0
    slots = np.arange(count, dtype=np.uint64)
    i = slots * np.uint64(n_partitions) + np.uint64(p)
    out = np.empty((kp, count, wpp), dtype=np.uint64)
    for t in range(kp):
        for w in range(wpp):
            j = (np.uint64(t) * np.uint64(n_total) + i) * np.uint64(wpp) + np.uint64(w)
            v = splitmix64_at(seed, j)
            if w == wpp - 1:
                v &= np.uint64(pad_mask(dim))
            out[t, :, w] = v
    return out.reshape(kp, count * wpp), count, i


def gen_queries(seed, n_queries, dim, qp):
    """[Q][qp][wpp] u64 query planes."""
    wpp = wpp_of(dim)
    j = np.arange(n_queries * qp * wpp, dtype=np.uint64)
    v = splitmix64_at(seed, j)
    v = v.reshape(n_queries, qp, wpp)
    v[:, :, -1] &= np.uint64(pad_mask(dim))
    return np.ascontiguousarray(v)


# ----------------------------------------------------------------------------
class RefError(Exception):
    pass


_STATUS_EXC = {1: ValueError, 2: IndexError, 3: RuntimeError}


class Ref:
    """The compiled reference (unmodified proj/src/*.cpp + ref_shim.cpp)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        L = C.CDLL(path)
        self.L = L
        L.ref_last_error.restype = C.c_char_p
        L.ref_index_new.restype = C.c_void_p
        L.ref_index_new.argtypes = [C.c_uint32, C.c_uint32, C.c_int, C.c_uint32]
        L.ref_index_free.argtypes = [C.c_void_p]
        L.ref_index_set_partition.argtypes = [C.c_void_p, C.c_uint32, C.c_uint64, U64P, F32P, U64P]
        L.ref_index_build.restype = C.c_void_p
        L.ref_index_build.argtypes = [C.c_uint32, C.c_uint32, C.c_int, C.c_uint32, C.c_uint64, U64P, U64P,
                                      C.POINTER(C.c_int)]
        L.ref_index_count.restype = C.c_uint64
        L.ref_index_count.argtypes = [C.c_void_p, C.c_uint32]
        L.ref_index_get_partition.argtypes = [C.c_void_p, C.c_uint32, U64P, F32P, U64P]
        L.ref_save_index.argtypes = [C.c_void_p, C.c_char_p]
        L.ref_load_index.restype = C.c_void_p
        L.ref_load_index.argtypes = [C.c_char_p, C.POINTER(C.c_int), U32P, U32P, C.POINTER(C.c_int), U32P]
        L.ref_search_batch.argtypes = [C.c_void_p, U64P, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                       C.c_uint32, C.c_uint32, C.c_uint64, F64P, U64P, U32P, U64P, U64P,
                                       C.c_uint32]
        L.ref_partition_select.argtypes = [C.c_void_p, U64P, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                           C.c_uint32, C.c_uint32, C.c_uint64, F64P, U64P, U32P, U64P, U64P]
        L.ref_local_select.argtypes = [C.c_void_p, U64P, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                       C.c_uint32, C.c_uint32, C.c_uint32, F64P, U64P, U32P, U64P]
        L.ref_pack.argtypes = [C.POINTER(C.c_int), C.c_uint32, U64P, U32P]
        L.ref_binary_dot.argtypes = [U64P, C.c_uint32, U64P, C.c_uint32, I64P]
        L.ref_combine_plane_dots.restype = C.c_double
        L.ref_combine_plane_dots.argtypes = [I64P, C.c_uint32, C.c_uint32, C.c_int]
        L.ref_make_embedding.argtypes = [U64P, C.c_uint32, C.c_uint32, C.c_int, F64P]
        L.ref_rbe_score.argtypes = [U64P, C.c_uint32, U64P, C.c_uint32, C.c_uint32, C.c_int, C.c_int, F64P]
        L.ref_thread_assignment.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64,
                                            C.c_uint32, C.c_uint32, U64P, U32P]
        L.ref_scan_benchmark.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                         C.c_uint64, F64P, F64P]

    def _check(self, st):
        if st != 0:
            raise _STATUS_EXC.get(st, RuntimeError)(self.L.ref_last_error().decode())

    # -- leaf functions
    def pack(self, values):
        v = np.ascontiguousarray(values, dtype=np.int32)
        words = np.zeros(max(1, wpp_of(len(v))), dtype=np.uint64)
        dim = C.c_uint32()
        self._check(self.L.ref_pack(v.ctypes.data_as(C.POINTER(C.c_int)), len(v), _p(words, U64P), C.byref(dim)))
        return words, dim.value

    def binary_dot(self, x, xdim, y, ydim):
        x = np.ascontiguousarray(x, dtype=np.uint64)
        y = np.ascontiguousarray(y, dtype=np.uint64)
        out = C.c_int64()
        self._check(self.L.ref_binary_dot(_p(x, U64P), xdim, _p(y, U64P), ydim, C.byref(out)))
        return out.value

    def combine_plane_dots(self, dots, qp, kp, rw):
        d = np.ascontiguousarray(dots, dtype=np.int64)
        return self.L.ref_combine_plane_dots(_p(d, I64P), qp, kp, int(rw))

    def magnitude(self, words, n_planes, dim, rw=True):
        w = np.ascontiguousarray(words, dtype=np.uint64)
        out = C.c_double()
        self._check(self.L.ref_make_embedding(_p(w, U64P), n_planes, dim, int(rw), C.byref(out)))
        return out.value

    def rbe_score(self, qwords, qp, kwords, kp, dim, rw=True, normalize=True):
        q = np.ascontiguousarray(qwords, dtype=np.uint64)
        k = np.ascontiguousarray(kwords, dtype=np.uint64)
        out = C.c_double()
        self._check(self.L.ref_rbe_score(_p(q, U64P), qp, _p(k, U64P), kp, dim, int(rw), int(normalize),
                                         C.byref(out)))
        return out.value

    def expected_recall(self, candidates, relevant, items_per_thread):
        """Appendix A prediction (src/analysis.cpp:143-184): (recall@N, expected misses)."""
        r, m = C.c_double(), C.c_double()
        self._check(self.L.ref_expected_recall(C.c_uint64(candidates), C.c_uint64(relevant),
                                               C.c_uint64(items_per_thread), C.byref(r), C.byref(m)))
        return r.value, m.value

    def thread_assignment(self, geometry, count, block, thread):
        b, t, i, q = geometry
        out = np.zeros(max(i, 1), dtype=np.uint64)
        n = C.c_uint32()
        self._check(self.L.ref_thread_assignment(b, t, i, q, count, block, thread, _p(out, U64P), C.byref(n)))
        return [int(x) for x in out[: n.value]]

    def scan_benchmark(self, count, dim, qp, kp, repeats=1, seed=1):
        b, f = C.c_double(), C.c_double()
        self._check(self.L.ref_scan_benchmark(count, dim, qp, kp, repeats, seed, C.byref(b), C.byref(f)))
        return b.value, f.value

    # -- index
    def index(self, dim, kp, rw, partitions):
        """partitions: list of (planes[kp][count*wpp] u64, mags f32[count], ids u64[count])."""
        return RefIndex(self, dim, kp, rw, partitions)

    def build_index(self, dim, kp, rw, n_partitions, words, ids):
        """Through rbe::IndexBuilder; words [N][kp][wpp]."""
        w = np.ascontiguousarray(words, dtype=np.uint64)
        i = np.ascontiguousarray(ids, dtype=np.uint64)
        st = C.c_int()
        h = self.L.ref_index_build(dim, kp, int(rw), n_partitions, len(i), _p(w, U64P), _p(i, U64P), C.byref(st))
        self._check(st.value)
        return RefIndex(self, dim, kp, rw, None, handle=h, n_partitions=n_partitions)

    def load_index(self, path):
        st = C.c_int()
        dim, kp, npart = C.c_uint32(), C.c_uint32(), C.c_uint32()
        rw = C.c_int()
        h = self.L.ref_load_index(str(path).encode(), C.byref(st), C.byref(dim), C.byref(kp), C.byref(rw),
                                  C.byref(npart))
        self._check(st.value)
        return RefIndex(self, dim.value, kp.value, bool(rw.value), None, handle=h, n_partitions=npart.value)


class RefIndex:
    def __init__(self, ref, dim, kp, rw, partitions, handle=None, n_partitions=None):
        self.ref, self.dim, self.kp, self.rw = ref, dim, kp, rw
        if handle is None:
            handle = ref.L.ref_index_new(dim, kp, int(rw), len(partitions))
            self._keep = []
            for p, (planes, mags, ids) in enumerate(partitions):
                planes = np.ascontiguousarray(planes, dtype=np.uint64)
                mags = np.ascontiguousarray(mags, dtype=np.float32)
                ids = np.ascontiguousarray(ids, dtype=np.uint64)
                ref._check(ref.L.ref_index_set_partition(handle, p, len(ids), _p(planes, U64P), _p(mags, F32P),
                                                         _p(ids, U64P)))
            n_partitions = len(partitions)
        self.h = handle
        self.n_partitions = n_partitions

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.L.ref_index_free(self.h)
            self.h = None

    def partition(self, p):
        wpp = wpp_of(self.dim)
        n = self.ref.L.ref_index_count(self.h, p)
        planes = np.zeros(self.kp * n * wpp, dtype=np.uint64)
        mags = np.zeros(n, dtype=np.float32)
        ids = np.zeros(n, dtype=np.uint64)
        self.ref._check(self.ref.L.ref_index_get_partition(self.h, p, _p(planes, U64P), _p(mags, F32P),
                                                           _p(ids, U64P)))
        return planes.reshape(self.kp, n * wpp), mags, ids

    def save(self, path):
        self.ref._check(self.ref.L.ref_save_index(self.h, str(path).encode()))

    def search(self, queries, geometry, n, threads=1):
        """queries [Q][qp][wpp]; returns (list of [(score, id, partition)], scored)."""
        q = np.ascontiguousarray(queries, dtype=np.uint64)
        Q, qp = q.shape[0], q.shape[1]
        b, t, i, ql = geometry
        nn = max(int(n), 1)
        scores = np.zeros(Q * nn, dtype=np.float64)
        ids = np.zeros(Q * nn, dtype=np.uint64)
        parts = np.zeros(Q * nn, dtype=np.uint32)
        cnt = np.zeros(Q, dtype=np.uint64)
        scored = C.c_uint64()
        self.ref._check(self.ref.L.ref_search_batch(self.h, _p(q, U64P), Q, qp, b, t, i, ql, n, _p(scores, F64P),
                                                    _p(ids, U64P), _p(parts, U32P), _p(cnt, U64P),
                                                    C.byref(scored), threads))
        out = []
        for k in range(Q):
            m = int(cnt[k])
            s = slice(k * nn, k * nn + m)
            out.append(list(zip(scores[s].tolist(), ids[s].tolist(), parts[s].tolist())))
        return out, scored.value

    def local_select(self, query, p, geometry):
        """rbe::local_select -> (scores[threads][ql], slots[threads][ql], counts[threads], scored),
        ql = min(queue_length, items_per_thread)."""
        q = np.ascontiguousarray(query, dtype=np.uint64)
        b, t, i, ql = geometry
        qle = min(ql, i)
        threads = b * t
        scores = np.zeros((threads, qle), dtype=np.float64)
        slots = np.zeros((threads, qle), dtype=np.uint64)
        counts = np.zeros(threads, dtype=np.uint32)
        scored = C.c_uint64()
        self.ref._check(self.ref.L.ref_local_select(self.h, _p(q, U64P), q.shape[0], p, b, t, i, ql, qle,
                                                    _p(scores, F64P), _p(slots, U64P), _p(counts, U32P),
                                                    C.byref(scored)))
        return scores, slots, counts, scored.value

    def partition_select(self, query, p, geometry, n):
        q = np.ascontiguousarray(query, dtype=np.uint64)
        b, t, i, ql = geometry
        nn = max(int(n), 1)
        scores = np.zeros(nn, dtype=np.float64)
        ids = np.zeros(nn, dtype=np.uint64)
        parts = np.zeros(nn, dtype=np.uint32)
        cnt, ns = C.c_uint64(), C.c_uint64()
        self.ref._check(self.ref.L.ref_partition_select(self.h, _p(q, U64P), q.shape[0], p, b, t, i, ql, n,
                                                        _p(scores, F64P), _p(ids, U64P), _p(parts, U32P),
                                                        C.byref(cnt), C.byref(ns)))
        m = cnt.value
        return list(zip(scores[:m].tolist(), ids[:m].tolist(), parts[:m].tolist())), ns.value


# ----------------------------------------------------------------------------
class _Entry(C.Structure):
    _fields_ = [("score", C.c_double), ("id", C.c_uint64), ("partition", C.c_uint32), ("acc", C.c_int64)]


class Port:
    """The plain-C restatement (oracle/rbe_oracle.c)."""

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle oracle`")
        L = C.CDLL(path)
        self.L = L
        L.rbo_splitmix64_at.restype = C.c_uint64
        L.rbo_splitmix64_at.argtypes = [C.c_uint64, C.c_uint64]
        L.rbo_gen_partition_planes.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                               C.c_uint32, C.c_uint64, U64P]
        L.rbo_gen_queries.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, U64P]
        L.rbo_binary_dot_words.restype = C.c_int64
        L.rbo_binary_dot_words.argtypes = [U64P, U64P, C.c_uint64, C.c_uint32]
        L.rbo_combine_plane_dots.restype = C.c_double
        L.rbo_combine_plane_dots.argtypes = [I64P, C.c_uint32, C.c_uint32, C.c_int, I64P]
        L.rbo_magnitude.restype = C.c_double
        L.rbo_magnitude.argtypes = [U64P, C.c_uint64, C.c_uint32, C.c_uint32, C.c_int]
        L.rbo_partition_magnitudes.argtypes = [U64P, C.c_uint64, C.c_uint32, C.c_uint32, C.c_int, F32P]
        L.rbo_gen_partition_planes_range.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                                     C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint64, U64P]
        L.rbo_partition_magnitudes_range.argtypes = [U64P, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32,
                                                     C.c_uint32, C.c_int, F32P]
        L.rbo_thread_assignment.restype = C.c_uint32
        L.rbo_thread_assignment.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint32,
                                            C.c_uint32, U64P]
        EP = C.POINTER(_Entry)
        L.rbo_partition_select.restype = C.c_int64
        L.rbo_partition_select.argtypes = [U64P, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int, U64P, F32P, U64P,
                                           C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                           C.c_uint32, C.c_uint64, EP, U64P]
        L.rbo_merge.restype = C.c_uint64
        L.rbo_merge.argtypes = [EP, C.c_uint64, C.c_uint64]

    def splitmix64_at(self, seed, j):
        return self.L.rbo_splitmix64_at(seed, j)

    def gen_partition_planes(self, seed, n_total, dim, kp, n_partitions, p):
        wpp = wpp_of(dim)
        count = (n_total - p + n_partitions - 1) // n_partitions if p < n_total else 0
        out = np.zeros(kp * count * wpp, dtype=np.uint64)
        self.L.rbo_gen_partition_planes(seed, n_total, dim, kp, n_partitions, p, count, _p(out, U64P))
        return out.reshape(kp, count * wpp)

    def gen_partition_prefix(self, seed, n_total, dim, kp, n_partitions, p, count, threads=1):
        """The first `count` slots of partition p (reference layout planes, exact magnitudes,
        ids): a bounded sample of a large synthetic corpus, generated with `threads` threads."""
        from concurrent.futures import ThreadPoolExecutor

        wpp = wpp_of(dim)
        planes = np.empty(kp * count * wpp, dtype=np.uint64)
        mags = np.empty(count, dtype=np.float32)
        step = -(-count // max(threads, 1))

        def chunk(b):
            e = min(b + step, count)
            self.L.rbo_gen_partition_planes_range(seed, n_total, dim, kp, n_partitions, p, count, b, e,
                                                  _p(planes, U64P))
            self.L.rbo_partition_magnitudes_range(_p(planes, U64P), count, b, e, dim, kp, int(True), _p(mags, F32P))

        with ThreadPoolExecutor(max_workers=max(threads, 1)) as ex:  # ctypes releases the GIL
            list(ex.map(chunk, range(0, count, step)))
        ids = np.arange(count, dtype=np.uint64) * np.uint64(n_partitions) + np.uint64(p)
        return planes.reshape(kp, count * wpp), mags, ids

    def gen_queries(self, seed, Q, dim, qp):
        out = np.zeros(Q * qp * wpp_of(dim), dtype=np.uint64)
        self.L.rbo_gen_queries(seed, Q, dim, qp, _p(out, U64P))
        return out.reshape(Q, qp, wpp_of(dim))

    def binary_dot_words(self, x, y, dim):
        x = np.ascontiguousarray(x, dtype=np.uint64)
        y = np.ascontiguousarray(y, dtype=np.uint64)
        return self.L.rbo_binary_dot_words(_p(x, U64P), _p(y, U64P), len(x), dim)

    def combine_plane_dots(self, dots, qp, kp, rw):
        d = np.ascontiguousarray(dots, dtype=np.int64)
        acc = C.c_int64()
        v = self.L.rbo_combine_plane_dots(_p(d, I64P), qp, kp, int(rw), C.byref(acc))
        return v, acc.value

    def magnitudes(self, planes, count, dim, kp, rw=True):
        p = np.ascontiguousarray(planes, dtype=np.uint64)
        out = np.zeros(count, dtype=np.float32)
        self.L.rbo_partition_magnitudes(_p(p, U64P), count, dim, kp, int(rw), _p(out, F32P))
        return out

    def thread_assignment(self, geometry, count, block, thread):
        b, t, i, _ = geometry
        out = np.zeros(max(i, 1), dtype=np.uint64)
        n = self.L.rbo_thread_assignment(b, t, i, count, block, thread, _p(out, U64P))
        return [int(x) for x in out[:n]]

    def search(self, query, dim, kp, rw, partitions, geometry, n):
        """query [qp][wpp]; partitions list of (planes, mags, ids).  Returns
        ([(score, id, partition, acc)], scored)."""
        q = np.ascontiguousarray(query, dtype=np.uint64)
        b, t, i, ql = geometry
        nn = max(int(n), 1)
        buf = (_Entry * (nn * max(len(partitions), 1)))()
        total = 0
        scored = C.c_uint64(0)
        for p, (planes, mags, ids) in enumerate(partitions):
            planes = np.ascontiguousarray(planes, dtype=np.uint64)
            mags = np.ascontiguousarray(mags, dtype=np.float32)
            ids = np.ascontiguousarray(ids, dtype=np.uint64)
            m = self.L.rbo_partition_select(_p(q, U64P), q.shape[0], dim, kp, int(rw), _p(planes, U64P),
                                            _p(mags, F32P), _p(ids, U64P), len(ids), p, b, t, i, ql, n,
                                            C.cast(C.byref(buf, total * C.sizeof(_Entry)), C.POINTER(_Entry)),
                                            C.byref(scored))
            if m < 0:
                raise ValueError("invalid search arguments")
            total += m
        m = self.L.rbo_merge(buf, total, n)
        return [(e.score, e.id, e.partition, e.acc) for e in buf[:m]], scored.value


def synthetic_partitions(seed, n_total, dim, kp, n_partitions, rw=True, port=None):
    """Reference-layout partitions of the synthetic corpus with exact magnitudes."""
    port = port or Port()
    parts = []
    for p in range(n_partitions):
        planes, count, gids = gen_partition_planes(seed, n_total, dim, kp, n_partitions, p)
        mags = port.magnitudes(planes, count, dim, kp, rw)
        parts.append((planes, mags, gids.astype(np.uint64)))
    return parts


def synthetic_prefix(seed, n_total, count, dim, kp, rw=True, port=None):
    """The first `count` slots of the single-partition (P=1) synthetic corpus of
    n_total docs -- a bounded sample of the bench workload for the CPU arm."""
    port = port or Port()
    wpp = wpp_of(dim)
    i = np.arange(count, dtype=np.uint64)
    planes = np.empty((kp, count, wpp), dtype=np.uint64)
    for t in range(kp):
        for w in range(wpp):
            j = (np.uint64(t) * np.uint64(n_total) + i) * np.uint64(wpp) + np.uint64(w)
            v = splitmix64_at(seed, j)
            if w == wpp - 1:
                v &= np.uint64(pad_mask(dim))
            planes[t, :, w] = v
    planes = planes.reshape(kp, count * wpp)
    mags = port.magnitudes(planes, count, dim, kp, rw)
    return planes, mags, i.copy()
