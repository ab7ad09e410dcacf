"""Pin the CPU oracle (oracle/rbe_oracle.c) before trusting it: against the
SPEC.md KATs, the golden fixtures produced by the compiled reference, and the
compiled reference itself (oracle/_ref) on seeded sweeps."""
import json
import os

import numpy as np
import pytest

from oracle.oracle import gen_partition_planes, gen_queries, splitmix64_at, synthetic_partitions

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def test_generator_counter_form(port):
    # numpy restatement == C restatement == sequential splitmix64 (bench.cpp:15-21)
    state, seq = 0x1234, []
    for _ in range(5):
        state = (state + 0x9E3779B97F4A7C15) & ((1 << 64) - 1)
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & ((1 << 64) - 1)
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & ((1 << 64) - 1)
        seq.append(z ^ (z >> 31))
    assert [port.splitmix64_at(0x1234, j) for j in range(5)] == seq
    assert [int(v) for v in splitmix64_at(0x1234, np.arange(5))] == seq
    a = port.gen_partition_planes(7, 999, 65, 3, 4, 2)
    b, _, _ = gen_partition_planes(7, 999, 65, 3, 4, 2)
    assert np.array_equal(a, b)
    assert np.array_equal(port.gen_queries(9, 3, 130, 2), gen_queries(9, 3, 130, 2))


def test_spec_kats(port, ref):
    k = load("spec_kats.json")
    for case in k["binary_dot"]:
        wx, dx = ref.pack(case["x"])
        wy, _ = ref.pack(case["y"])
        assert port.binary_dot_words(wx, wy, dx) == case["dot"]
    for case in k["magnitude"]:
        w = np.array([ref.pack(p)[0][0] for p in case["planes"]], np.uint64)
        got = port.L.rbo_magnitude(w.ctypes.data_as(__import__("ctypes").POINTER(__import__("ctypes").c_uint64)), 1,
                                   2, len(case["planes"]), int(case["rw"]))
        assert got == case["magnitude"]
        assert got == float(np.sqrt(np.sum(np.square(case["refined"]))))
    for case in k["thread_assignment"]:
        assert port.thread_assignment(tuple(case["geometry"]), case["count"], case["block"],
                                      case["thread"]) == case["items"]
    t = k["tie"]
    doc = np.array([t["doc_word"]], np.uint64)
    for ql, want in ((1, t["ql1_ids"]), (4, t["ql4_ids"])):
        planes = np.tile(doc, 4).reshape(1, 4)
        mags = np.full(4, 8.0, np.float32)
        res, _ = port.search(doc.reshape(1, 1), 64, 1, True, [(planes, mags, np.array(t["ids"], np.uint64))],
                             (1, 1, 4, ql), 10)
        assert [e[1] for e in res] == want


def test_combine_plane_dots_matches_reference(port, ref):
    rng = np.random.default_rng(0)
    for qp in range(1, 5):
        for kp in range(1, 5):
            for rw in (True, False):
                dots = rng.integers(-512, 513, qp * kp)
                v, acc = port.combine_plane_dots(dots, qp, kp, rw)
                assert v == ref.combine_plane_dots(dots, qp, kp, rw)
                L = qp + kp - 2 if rw else 0
                assert acc == sum(int(dots[s * kp + t]) << ((L - s - t) if rw else 0)
                                  for s in range(qp) for t in range(kp))


def test_golden_search_cases(port):
    for c in load("search_cases.json"):
        parts = synthetic_partitions(c["seed"], c["n_docs"], c["dim"], c["kp"], c["partitions"],
                                     c["residual_weights"], port)
        qs = gen_queries(c["query_seed"], c["n_queries"], c["dim"], c["qp"])
        for q in range(c["n_queries"]):
            res, scored = port.search(qs[q], c["dim"], c["kp"], c["residual_weights"], parts,
                                      tuple(c["geometry"]), c["n"])
            assert scored == c["n_docs"]
            assert [[s.hex(), i, p] for s, i, p, _ in res] == c["results"][q], c["name"]


SWEEP = [
    # N, dim, kp, qp, P, geometry, n, rw
    (3000, 1, 1, 1, 1, (1, 16, 256, 1), 20, True),
    (3000, 63, 2, 2, 2, (2, 32, 32, 2), 30, True),
    (3000, 64, 1, 4, 1, (1, 64, 64, 1), 30, True),
    (3000, 65, 4, 2, 3, (1, 128, 16, 3), 100, True),
    (2000, 128, 3, 3, 8, (1, 8, 32, 1), 50, False),
    (1500, 512, 2, 3, 1, (3, 32, 16, 16), 40, True),
    (2500, 100, 3, 1, 2, (5, 33, 9, 1), 70, True),
]


@pytest.mark.parametrize("case", SWEEP)
def test_port_matches_reference(port, ref, case):
    N, dim, kp, qp, P, geo, n, rw = case
    parts = synthetic_partitions(11, N, dim, kp, P, rw, port)
    ri = ref.index(dim, kp, rw, parts)
    qs = gen_queries(13, 3, dim, qp)
    rres, scored = ri.search(qs, geo, n)
    assert scored == 3 * N
    for q in range(3):
        pres, _ = port.search(qs[q], dim, kp, rw, parts, geo, n)
        assert [(s, i, p) for s, i, p, _ in pres] == rres[q]


def test_reference_errors(ref):
    parts = synthetic_partitions(1, 100, 64, 2, 1, True)
    ri = ref.index(64, 2, True, parts)
    q = gen_queries(2, 1, 64, 2)
    with pytest.raises(ValueError, match="queue_length"):
        ri.search(q, (1, 256, 256, 0), 5)
    with pytest.raises(ValueError, match="does not cover"):
        ri.search(q, (1, 4, 4, 1), 5)
