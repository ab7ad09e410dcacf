"""Recall@N of the lossy scan vs the Appendix A prediction at a given scale (SURVEY.md §8(f)4,
PAPER.md:327-329 reports 99.99% recall@1000 over 1.2B keywords).  Validation tool: the
prediction comes from the reference's own analysis code (oracle/_ref).  Prints one JSON line.

    python tools/recall_validation.py --docs 100000000 --partitions 1 --queries 16 --n 1000

The lossless ground truth (one item per logical thread) keeps a survivor slot per document and
query, so the measured scale is bounded by device memory (C x Q x 32 B); the prediction at
the headline scale (C = 1B) is printed alongside.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--docs", type=int, default=100_000_000)
    ap.add_argument("--partitions", type=int, default=1)
    ap.add_argument("--queries", type=int, default=16)
    ap.add_argument("--n", type=int, default=1000)
    ap.add_argument("--items-per-thread", type=int, default=256)
    args = ap.parse_args()
    import paper_1802_06466_b200 as rbe
    from oracle.oracle import Ref, gen_queries

    dix = rbe.DeviceIndex.synthetic(128, 3, True, args.docs, args.partitions, 0xD0C5)
    per_part = -(-args.docs // args.partitions)
    qs = gen_queries(0x5EC, args.queries, 128, 3)

    def geo(ipt):
        g = rbe.ScanGeometry()
        g.items_per_thread = ipt
        g.blocks = -(-per_part // (256 * ipt))
        return g

    t = time.perf_counter()
    exact = dix.search_words(qs, geo(1), args.n)[1]
    t_exact = time.perf_counter() - t
    t = time.perf_counter()
    lossy = dix.search_words(qs, geo(args.items_per_thread), args.n)[1]
    t_lossy = time.perf_counter() - t
    rec = [len(set(exact[q].tolist()) & set(lossy[q].tolist())) / args.n for q in range(args.queries)]
    want, misses = Ref().expected_recall(args.docs, args.n, args.items_per_thread)
    want_1b, _ = Ref().expected_recall(1_000_000_000, args.n, args.items_per_thread)
    print(json.dumps({"docs": args.docs, "partitions": args.partitions, "queries": args.queries, "n": args.n,
                      "items_per_thread": args.items_per_thread, "measured_recall_mean": float(np.mean(rec)),
                      "measured_recall_min": float(np.min(rec)), "predicted_recall_appendix_a": want,
                      "predicted_misses": misses, "predicted_recall_at_1B": want_1b, "paper_recall_at_1000_1p2B": 0.9999,
                      "lossless_pass_s": round(t_exact, 3), "lossy_pass_s": round(t_lossy, 3)}))


if __name__ == "__main__":
    main()
