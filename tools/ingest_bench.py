"""RBEI ingest throughput: DeviceIndex.from_rbei (pread by host threads ->
page-locked staging -> H2D -> on-device repack) against the reference path it replaces
(load_index into host memory, then upload).  Writes a synthetic RBEI v1 file of --docs
documents (128-dim, 3 planes, --partitions partitions) from the device generator, then times
both paths on it; prints one JSON line.  Run under gpurun:

    python tools/ingest_bench.py --docs 100000000 --partitions 8 --dir /tmp
"""
import argparse
import json
import os
import struct
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def write_rbei(path, dix, dim, kp, P):
    """RBEI v1: header, counts, then per partition planes, mags, ids."""
    counts = [dix.partition_size(p) for p in range(P)]
    with open(path, "wb") as f:
        f.write(b"RBEI" + struct.pack("<5I", 1, dim, kp, 1, P) + struct.pack(f"<{P}Q", *counts))
        for p in range(P):
            planes, mags, ids = dix.download_partition(p)
            np.ascontiguousarray(planes, dtype=np.uint64).tofile(f)
            np.ascontiguousarray(mags, dtype=np.float32).tofile(f)
            np.ascontiguousarray(ids, dtype=np.uint64).tofile(f)
    return os.path.getsize(path)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--docs", type=int, default=100_000_000)
    ap.add_argument("--partitions", type=int, default=8)
    ap.add_argument("--dir", default="/tmp")
    ap.add_argument("--io-threads", type=int, default=0)
    ap.add_argument("--skip-host-path", action="store_true")
    ap.add_argument("--rbee", action="store_true", help="also time the RBEE -> device index build")
    args = ap.parse_args()
    import paper_1802_06466_b200 as rbe

    dim, kp, P = 128, 3, args.partitions
    path = os.path.join(args.dir, f"ingest_{args.docs}_{P}.rbei")
    src = rbe.DeviceIndex.synthetic(dim, kp, True, args.docs, P, 0xD0C5, [0])
    t = time.perf_counter()
    size = write_rbei(path, src, dim, kp, P)
    t_write = time.perf_counter() - t
    del src
    out = {"docs": args.docs, "partitions": P, "file_bytes": size, "write_s": round(t_write, 2)}
    # warm page cache (the file was just written)
    dix = rbe.DeviceIndex.from_rbei(path, [0], args.io_threads)
    st = dix.load_stats
    out["from_rbei_warm"] = {"seconds": round(st["seconds"], 3), "gb_per_s": round(st["gb_per_s"], 2)}
    # check against the host path on one partition (ids and magnitudes)
    p0 = dix.download_partition(0)
    del dix
    # cold: drop the page cache when permitted (root on the GPU box)
    try:
        os.sync()
        with open("/proc/sys/vm/drop_caches", "w") as f:
            f.write("3\n")
        dix = rbe.DeviceIndex.from_rbei(path, [0], args.io_threads)
        st = dix.load_stats
        out["from_rbei_cold"] = {"seconds": round(st["seconds"], 3), "gb_per_s": round(st["gb_per_s"], 2)}
        del dix
    except OSError as e:
        out["from_rbei_cold"] = f"not measured ({e.strerror})"
    if not args.skip_host_path:
        # the path it replaces: load_index (whole file into host memory) + DeviceIndex upload
        t = time.perf_counter()
        host = rbe.load_index(path)
        t_load = time.perf_counter() - t
        t = time.perf_counter()
        dix = rbe.DeviceIndex(host, [0])
        t_up = time.perf_counter() - t
        q0 = dix.download_partition(0)
        assert all(np.array_equal(np.asarray(a).reshape(-1), np.asarray(b).reshape(-1)) for a, b in zip(p0, q0))
        out["load_index_then_upload"] = {"load_s": round(t_load, 3), "upload_s": round(t_up, 3),
                                         "gb_per_s": round(size / (t_load + t_up) / 1e9, 2)}
        del dix, host
    os.remove(path)
    if args.rbee:
        # RBEE bulk embeddings (magnitudes 0: every one recomputed on the device) -> build_rbee
        rpath = os.path.join(args.dir, f"ingest_{args.docs}.rbee")
        src = rbe.DeviceIndex.synthetic(dim, kp, True, args.docs, 1, 0xD0C5, [0])
        planes, _, ids = src.download_partition(0)
        del src
        n = args.docs
        rec = np.zeros(n, dtype=[("id", "<u8"), ("w", "<u8", (kp * 2,)), ("m", "<f4")])
        rec["id"] = ids
        rec["w"] = np.asarray(planes).reshape(kp, n, 2).transpose(1, 0, 2).reshape(n, kp * 2)
        with open(rpath, "wb") as f:
            f.write(b"RBEE" + struct.pack("<4I", 1, dim, kp, 1))
            rec.tofile(f)
        del rec, planes, ids
        dix = rbe.DeviceIndex.build_rbee(rpath, P, [0], args.io_threads)
        st = dix.load_stats
        out["build_rbee_warm"] = {"seconds": round(st["seconds"], 3), "gb_per_s": round(st["gb_per_s"], 2),
                                  "docs_per_s": round(n / st["seconds"])}
        del dix
        # the reference's IndexBuilder (make_embedding per keyword) on a 1M-doc sample, 1 thread
        from oracle.oracle import Port, Ref

        m = min(n, 1_000_000)
        w = Port().gen_partition_prefix(0xD0C5, m, dim, kp, 1, 0, m, 16)[0]
        words = np.asarray(w).reshape(kp, m, 2).transpose(1, 0, 2).copy()
        t = time.perf_counter()
        Ref().build_index(dim, kp, True, P, words, np.arange(m, dtype=np.uint64))
        dt = time.perf_counter() - t
        out["reference_index_builder_1thread"] = {"sample_docs": m, "seconds": round(dt, 3), "docs_per_s": round(m / dt)}
        os.remove(rpath)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
