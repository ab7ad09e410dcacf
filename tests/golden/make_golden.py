"""Generate the golden fixtures under tests/golden/ from the REFERENCE itself.

Run in the build container (needs oracle/_ref/librbe_ref.so, i.e. the
reference's unmodified proj/src/*.cpp compiled by oracle/Makefile):

    make -C oracle && python tests/golden/make_golden.py

* spec_kats.json    -- the SPEC.md known-answer tests of the hot path
                       (SPEC.md:60-62, 70-72, 80-82, 310, 343-345, 353-355,
                       363-365, 373-375), each asserted against the SPEC value
                       AND recorded as the compiled reference's output.
* search_cases.json -- small seeded search cases (synthetic corpus of
                       SURVEY.md §8(d)) with the reference's rbe::search
                       output; scores stored as float.hex() (bit-exact).
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import Port, Ref, gen_queries, synthetic_partitions  # noqa: E402


def words_of(ref, values):
    w, dim = ref.pack(values)
    return [int(x) for x in w], dim


def spec_kats(ref):
    k = {}
    # pack
    k["pack"] = []
    for vals in ([1, 1, 1, 1], [-1, -1, -1, -1], [1, -1, 1, -1, 1]):
        w, dim = words_of(ref, vals)
        k["pack"].append({"values": vals, "words": w, "dim": dim})
    assert k["pack"][0]["words"] == [0b1111] and k["pack"][1]["words"] == [0] and k["pack"][2]["words"] == [0b10101]
    # binary_dot
    x = [1] * 64
    k["binary_dot"] = []
    for a, b, want in (
        (x, x, 64),
        (x, [-1] * 64, -64),
        ([1, 1, 1, 1, -1, -1, -1, -1], [1, -1, 1, -1, 1, -1, 1, -1], 0),
    ):
        wa, da = words_of(ref, a)
        wb, db = words_of(ref, b)
        got = ref.binary_dot(np.array(wa, np.uint64), da, np.array(wb, np.uint64), db)
        assert got == want
        k["binary_dot"].append({"x": a, "y": b, "dot": got})
    # rbe_score u=v=0
    wq, _ = words_of(ref, [1, 1, 1, 1])
    wk, _ = words_of(ref, [1, 1, -1, -1])
    s = ref.rbe_score(np.array(wq, np.uint64), 1, np.array(wk, np.uint64), 1, 4, True, False)
    assert s == 0.0
    k["rbe_score"] = [{"q": [1, 1, 1, 1], "k": [1, 1, -1, -1], "qp": 1, "kp": 1, "score": s}]
    # self cosine = 1, 2+2 planes dim 8
    rng = np.random.default_rng(5)
    planes = [[int(v) for v in rng.choice([-1, 1], 8)] for _ in range(2)]
    w = np.array([words_of(ref, p)[0][0] for p in planes], np.uint64)
    s_self = ref.rbe_score(w, 2, w, 2, 8, True, True)
    assert abs(s_self - 1.0) < 1e-12
    k["rbe_score"].append({"q_planes": planes, "k_planes": planes, "qp": 2, "kp": 2, "normalize": True,
                           "score": s_self})
    # refined_vector / magnitude
    w2 = np.array([words_of(ref, [1, 1])[0][0], words_of(ref, [1, -1])[0][0]], np.uint64)
    k["magnitude"] = [
        {"planes": [[1, 1], [1, -1]], "rw": True, "magnitude": ref.magnitude(w2, 2, 2, True),
         "refined": [1.5, 0.5]},
        {"planes": [[1, 1], [1, -1]], "rw": False, "magnitude": ref.magnitude(w2, 2, 2, False),
         "refined": [2.0, 0.0]},
        {"planes": [[1, -1]], "rw": True, "magnitude": ref.magnitude(w2[:1], 1, 2, True), "refined": [1.0, -1.0]},
    ]
    assert k["magnitude"][0]["magnitude"] == (1.5 ** 2 + 0.5 ** 2) ** 0.5
    # thread_assignment
    ta0 = ref.thread_assignment((1, 256, 256, 1), 1 << 20, 0, 0)
    assert ta0 == list(range(0, 65281, 256))
    ta1 = ref.thread_assignment((2, 4, 2, 1), 16, 1, 3)
    assert ta1 == [11, 15]
    cover = sorted(z for b in range(2) for t in range(4) for z in ref.thread_assignment((2, 4, 2, 1), 16, b, t))
    assert cover == list(range(16))
    k["thread_assignment"] = [
        {"geometry": [1, 256, 256, 1], "count": 1 << 20, "block": 0, "thread": 0, "items": ta0},
        {"geometry": [2, 4, 2, 1], "count": 16, "block": 1, "thread": 3, "items": ta1},
    ]
    # memory claim: n=64, v=1 -> 16 B/keyword
    k["memory"] = {"dim": 64, "keyword_planes": 2, "bytes_per_keyword": 16, "keywords": 10 ** 6,
                   "payload_bytes": 16 * 10 ** 6}
    # tie KAT: 4 equal docs ids [40,30,20,10] in one thread
    doc = np.array([0x0F0F0F0F0F0F0F0F], np.uint64)
    words = np.tile(doc, (4, 1, 1))
    ix = ref.build_index(64, 1, True, 1, words, np.array([40, 30, 20, 10], np.uint64))
    q = doc.reshape(1, 1, 1)
    r1, _ = ix.search(q, (1, 1, 4, 1), 10)
    r4, _ = ix.search(q, (1, 1, 4, 4), 10)
    assert [e[1] for e in r1[0]] == [40] and [e[1] for e in r4[0]] == [10, 20, 30, 40]
    k["tie"] = {"doc_word": int(doc[0]), "ids": [40, 30, 20, 10], "ql1_ids": [e[1] for e in r1[0]],
                "ql4_ids": [e[1] for e in r4[0]], "score_hex": r1[0][0][0].hex()}
    # self-retrieval: the query's own embedding ranks first
    parts = synthetic_partitions(0x5E1F, 2000, 64, 2, 1, True)
    planes, mags, ids = parts[0]
    slot = 777
    qw = planes.reshape(2, 2000, 1)[:, slot, :].reshape(1, 2, 1)
    ri = ref.index(64, 2, True, parts)
    rs, _ = ri.search(qw, (1, 2000, 1, 1), 5)
    assert rs[0][0][1] == int(ids[slot])
    k["self_retrieval"] = {"seed": 0x5E1F, "n_docs": 2000, "dim": 64, "kp": 2, "slot": slot,
                           "top_id": rs[0][0][1], "top_score_hex": rs[0][0][0].hex()}
    return k


CASES = [
    # name, seed, N, dim, kp, qp, P, geometry, n, rw, Q
    ("c1_small", 0xD0C5, 20000, 64, 2, 2, 1, (1, 256, 256, 1), 100, True, 3),
    ("dim65_qp2kp3_P3", 0xA1, 6000, 65, 3, 2, 3, (2, 32, 40, 2), 40, True, 3),
    ("dim128_3x3_P2_unweighted", 0xB2, 6000, 128, 3, 3, 2, (3, 64, 16, 1), 50, False, 2),
    ("dim1_lossless", 0xC3, 300, 1, 1, 1, 1, (1, 8, 64, 64), 30, True, 2),
    ("dim512_qp1kp4", 0xD4, 3000, 512, 4, 1, 2, (2, 64, 16, 1), 25, True, 2),
    ("dim63_P8_ql4", 0xE5, 5000, 63, 2, 3, 8, (1, 16, 64, 4), 60, True, 2),
]


def search_cases(ref):
    port = Port()
    out = []
    for name, seed, N, dim, kp, qp, P, geo, n, rw, Q in CASES:
        parts = synthetic_partitions(seed, N, dim, kp, P, rw, port)
        ri = ref.index(dim, kp, rw, parts)
        qs = gen_queries(seed ^ 0x0E1, Q, dim, qp)
        res, scored = ri.search(qs, geo, n)
        assert scored == Q * N
        out.append({
            "name": name, "seed": seed, "query_seed": seed ^ 0x0E1, "n_docs": N, "dim": dim, "kp": kp, "qp": qp,
            "partitions": P, "geometry": list(geo), "n": n, "residual_weights": rw, "n_queries": Q,
            "results": [[[s.hex(), i, p] for s, i, p in r] for r in res],
        })
    return out


def main():
    ref = Ref()
    with open(os.path.join(HERE, "spec_kats.json"), "w") as f:
        json.dump(spec_kats(ref), f, indent=1)
    with open(os.path.join(HERE, "search_cases.json"), "w") as f:
        json.dump(search_cases(ref), f)
    print("wrote", os.listdir(HERE))


if __name__ == "__main__":
    main()
