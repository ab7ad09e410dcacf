"""GPU float32 / bf16 dense scan vs the RBE scan (the reference's `bench`
subcommand compares its bitwise scan with a float32 scan, src/bench.cpp:75-87, and the paper
reports full precision about ten times slower than rbe*).  The dense baseline is
the library path on the same GPU: torch.matmul (cuBLAS) of the query batch against an
N x 128 embedding matrix, then torch.topk per query.  Prints one JSON line.

    python tools/float_scan_compare.py --docs 100000000 --queries 64 --k 1000
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--docs", type=int, default=100_000_000)
    ap.add_argument("--queries", type=int, default=64)
    ap.add_argument("--k", type=int, default=1000)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import torch

    import paper_1802_06466_b200 as rbe
    from oracle.oracle import gen_queries

    N, Q, D = args.docs, args.queries, 128
    out = {"docs": N, "queries": Q, "k": args.k, "dim": D}

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / args.reps

    # RBE scan (tensor variant, top-k per query, exact FP64 scores)
    dix = rbe.DeviceIndex.synthetic(D, 3, True, N, 1, 0xD0C5)
    g = rbe.ScanGeometry()
    g.blocks = -(-N // 65536)
    qs = gen_queries(0x0E1, Q, D, 3)
    st = dix.search_words(qs, g, args.k)[5]
    rbe_ms = min(dix.search_words(qs, g, args.k)[5]["device_ms"] for _ in range(args.reps))
    out["rbe_ms_per_batch"] = round(rbe_ms, 3)
    del dix
    for name, dt in (("float32", torch.float32), ("bfloat16", torch.bfloat16)):
        try:
            corpus = torch.randn(N, D, device="cuda", dtype=dt)
            qv = torch.randn(Q, D, device="cuda", dtype=dt)
            ms = timed(lambda: torch.topk(qv @ corpus.T, args.k, dim=1))
            out[f"{name}_ms_per_batch"] = round(ms, 3)
            out[f"{name}_over_rbe"] = round(ms / rbe_ms, 2)
            del corpus, qv
            torch.cuda.empty_cache()
        except RuntimeError as e:  # out of memory at very large N
            out[f"{name}_ms_per_batch"] = f"not measured ({str(e).splitlines()[0]})"
    out["rbe_stats"] = {k: v for k, v in st.items() if k in ("variant", "candidates", "survivors")}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
