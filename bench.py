#!/usr/bin/env python
"""Benchmark of the B200 exhaustive RBE retrieval path (BASELINE.json metric:
"queries/s & p50 latency, top-1000 over 1B RBE docs; HBM GB/s vs peak").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE config 3, the metric's own): 1B synthetic docs, 128-dim RBE
with 3 bit-planes (qp = kp = 3, residual weights), P = 8 partitions (doc i ->
partition i mod 8, slot i div 8), a 64-query batch, top-1000, default geometry
(T_b=256, I=256, queue length 1, auto blocks = ceil(125M / 65536) = 1908).
It fits one B200 (60 GB with ids).  A step = one batch of 64 queries scanned
over the whole corpus + selection (+ NCCL gather and device merge for N > 1).

Strong scaling: partition p lives on rank p mod N (N in {1, 2, 4, 8}); every N
computes the identical merged top-1000 (its sha256 is in the JSON line as
`result_sha256`, so runs at different N can be compared).

`value`  queries/s with the query batch already in HBM (CUDA events on the
         launching stream, max over ranks).
`e2e`    the same with host buffers: N=1 through the public API
         (DeviceIndex.search_words -> rbe_cuda_search, page-locked out arrays);
         N>1 H2D of the query words on every rank + the sharded device path +
         D2H of the merged records on rank 0, host-timed, max over ranks.
The corpus (52 GB) is far larger than L2 (126 MB): no flush is needed.

`--impl reference` times the reference's own CPU rbe::search (its unmodified
sources compiled into oracle/_ref) on the host cores on a bounded sample of the
same workload: the first --sample-docs slots of partition 0 of the 1B-doc
corpus, one query per host thread (query-parallel), scaled linearly to the
whole corpus (the scan is O(N)); plus the reference "as
shipped" (one rbe::search per query, sequentially, P=1 and P=nproc partitions
of the sample -- std::async per partition).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DIM, KP, QP = 128, 3, 3
SEED_DOCS, SEED_QUERIES = 0xD0C5, 0x0E1
METRIC = "queries/s & p50 latency, top-1000 over 1B RBE docs; HBM GB/s vs peak"
UNIT = "queries/s"
BYTES_PER_DOC = KP * ((DIM + 63) // 64) * 8 + 4  # plane words + f32 magnitude


def env_rank():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(
        os.environ.get("LOCAL_RANK", "0"))


def part_count(n_docs, P, p):
    return (n_docs - p + P - 1) // P if p < n_docs else 0


def workload(args, n_gpus):
    per_part = part_count(args.docs, args.partitions, 0)
    name = "BASELINE config 3" if args.docs == 1_000_000_000 and args.partitions == 8 else "custom"
    return {
        "workload": f"{name}: {args.docs / 1e9:g}B docs x {DIM}-dim RBE, {KP}+{QP} bit-planes (residual weights), "
                    f"P={args.partitions} partitions (partition p on GPU p mod N), Q={args.queries}, k={args.k}, "
                    f"geometry 256/256/1 auto blocks",
        "docs": args.docs, "partitions": args.partitions, "docs_per_partition": per_part, "dim": DIM,
        "keyword_planes": KP, "query_planes": QP, "queries_per_batch": args.queries, "k": args.k,
        "geometry": {"threads_per_block": 256, "items_per_thread": 256, "queue_length": 1,
                     "blocks": -(-per_part // 65536)},
        "seeds": {"docs": SEED_DOCS, "queries": SEED_QUERIES},
        "parallelism": f"shard{n_gpus} (partitions over GPUs, NCCL gather + device merge)",
        "l2": f"corpus {args.docs * BYTES_PER_DOC / 1e9:.0f} GB > 126 MB L2: inputs larger than L2, no flush",
    }


class ClockSampler:
    """nvidia-smi equivalent via NVML, sampled every 20 ms during the timed region."""

    REASONS = {
        0x0000000000000004: "sw_power_cap", 0x0000000000000008: "hw_slowdown",
        0x0000000000000020: "sw_thermal_slowdown", 0x0000000000000040: "hw_thermal_slowdown",
        0x0000000000000080: "hw_power_brake_slowdown", 0x0000000000000002: "applications_clocks_setting",
    }

    def __init__(self, device_index):
        self.samples, self.reasons, self.ok = [], set(), False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:  # noqa: BLE001
            self.max_mhz = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic():
    """dram bytes per main-scan launch from the committed `ncu --set full` summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "scan_traffic.json")) as f:
            return json.load(f)
    except Exception:  # noqa: BLE001
        return None


def host_cpu():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "cpu"


# --------------------------------------------------------------------------- CPU reference arm
def cpu_reference(args, steps, warmup, as_shipped=True):
    """The reference's rbe::search (oracle/_ref, its unmodified sources) on a bounded sample
    of the workload: the first `sample_docs` slots of partition 0 of the corpus."""
    import numpy as np

    from oracle.oracle import Port, Ref, gen_queries

    threads = os.cpu_count() or 1
    full = part_count(args.docs, args.partitions, 0)
    S = min(args.sample_docs, full) if args.sample_docs else full
    ref = Ref()
    planes, mags, ids = Port().gen_partition_prefix(SEED_DOCS, args.docs, DIM, KP, args.partitions, 0, S, threads)
    ix = ref.index(DIM, KP, True, [(planes, mags, ids)])
    geo = (-(-S // 65536), 256, 256, 1)
    qs = gen_queries(SEED_QUERIES, max(threads, 1), DIM, QP)
    scale = S / args.docs  # the scan is O(N): sample docs / whole corpus
    times, cpu_times = [], []
    for s in range(warmup + steps):
        t0, c0 = time.perf_counter(), time.process_time()
        ix.search(qs, geo, args.k, threads=threads)
        dt, dc = time.perf_counter() - t0, time.process_time() - c0
        if s >= warmup:
            times.append(dt)
            cpu_times.append(dc)
    per_step = statistics.median(times)
    qps = qs.shape[0] / per_step * scale
    info = {"value": qps, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"{qs.shape[0]} queries per step (one per host thread, query-parallel rbe::search) over "
                      + (f"all {S:,} slots of partition 0, one of the {args.partitions} equal partitions"
                         if S == full else f"the first {S:,} slots of partition 0")
                      + f" of the {args.docs:,}-doc corpus ({S * BYTES_PER_DOC / 1e9:.2f} "
                      f"GB, >> LLC), scaled x{scale:g} to the whole corpus; {len(times)} steps, median "
                      f"{per_step * 1e3:.0f} ms wall / {statistics.median(cpu_times) * 1e3:.0f} ms process CPU per step; "
                      f"reference sources compiled unmodified (oracle/_ref); host {host_cpu()}",
            "ms_per_step_sample": per_step * 1e3, "cpu_ms_per_step_sample": statistics.median(cpu_times) * 1e3,
            "sample_docs": S, "ns_per_doc_query_thread": per_step * 1e9 / S}
    if as_shipped:
        # the reference as shipped: one rbe::search per query, sequentially (CLI semantics,
        # tools/rbe_main.cpp:185-199), P=1 and P=nproc partitions (std::async per partition)
        shipped = {}
        for P in (1, threads):
            if P == 1:
                pix = ix
            else:
                w = planes.reshape(KP, S, -1)
                pparts = []
                for p in range(P):
                    sel = np.arange(p, S, P)
                    pparts.append((np.ascontiguousarray(w[:, sel]).reshape(KP, -1), mags[sel], ids[sel]))
                pix = ref.index(DIM, KP, True, pparts)
            pgeo = (-(-(-(-S // P)) // 65536), 256, 256, 1)
            t0, c0 = time.perf_counter(), time.process_time()
            nq = 1
            for q in range(nq):
                pix.search(qs[q:q + 1], pgeo, args.k, threads=1)
            dt, dc = time.perf_counter() - t0, time.process_time() - c0
            shipped[f"P={P}"] = {"value": nq / dt * scale, "unit": UNIT, "wall_ms_per_query_sample": dt / nq * 1e3,
                                 "cpu_ms_per_query_sample": dc / nq * 1e3}
        info["as_shipped"] = shipped
    return qps, info, times


def run_reference_arm(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    qps, info, times = cpu_reference(args, args.steps, args.warmup)
    line = {
        "metric": METRIC, "value": qps, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": statistics.median(times) * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u64 popcnt -> s64 acc, f64 score",
        "data": "synthetic (counter-based splitmix64 corpus, SURVEY.md §8(d))",
        "config": workload(args, args.gpus), "cpu_baseline": info,
        "e2e": {"value": qps, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- our arm
def run_ours(args):
    import numpy as np
    import torch

    import paper_1802_06466_b200 as rbe
    from oracle.oracle import gen_queries  # the query generator (same counter stream as the corpus)
    from paper_1802_06466_b200.distributed import RESULT_BYTES, gather_and_merge

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    dev = f"cuda:{local}"
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device(dev))
    Q, K = args.queries, args.k
    t_build = time.perf_counter()
    # partitions p with p % world == rank, generated on this GPU
    dix = rbe.DeviceIndex.synthetic(DIM, KP, True, args.docs, args.partitions, SEED_DOCS, [local], rank, world)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t_build
    geo = rbe.ScanGeometry()
    geo.blocks = -(-part_count(args.docs, args.partitions, 0) // 65536)
    qs = gen_queries(SEED_QUERIES, Q, DIM, QP)
    d_words = torch.from_numpy(qs.view(np.int64).copy()).to(dev)
    # a dedicated stream (the legacy default stream's handle is 0, which the C ABI reads as
    # "the index's own stream"): every kernel, copy and event of a step is ordered on it
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    out = torch.empty(Q * K * RESULT_BYTES, dtype=torch.uint8, device=dev)
    merged = torch.empty_like(out)
    gathered = torch.empty(world * Q * K * RESULT_BYTES, dtype=torch.uint8, device=dev) if rank == 0 else None
    has_docs = dix.total_keywords > 0

    def merge(blocks):
        if len(blocks) == 1:
            return blocks[0]
        torch.cat(blocks, out=gathered)
        rbe.merge_device(local, gathered.data_ptr(), len(blocks), Q, K, merged.data_ptr(), stream.cuda_stream)
        return merged

    def step(with_stats):
        # with_stats=False: the batch is only enqueued (no host sync), so consecutive
        # steps run back to back on the GPU
        st = None
        if has_docs:
            st = rbe.search_device(dix.handle(0), d_words.data_ptr(), Q, QP, geo, K, out.data_ptr(),
                                   stream.cuda_stream, args.variant, with_stats)
        else:
            out.zero_()
        return st, gather_and_merge(out, rank, world, merge, dist)

    stats = []
    for _ in range(args.warmup):
        st, _ = step(True)  # warm-up steps also collect the per-batch counters
        if st:
            stats.append(st)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        ev[0].record(stream)
        res = None
        for s in range(args.steps):
            _, res = step(False)
            ev[s + 1].record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    per = [ev[s].elapsed_time(ev[s + 1]) for s in range(args.steps)]
    total_ms = ev[0].elapsed_time(ev[args.steps])
    if has_docs:
        rbe.last_batch_ms(dix.handle(0))  # surfaces a sticky error of any asynchronous batch
    if dist:
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = Q * args.steps / (total_ms / 1e3)

    # identical-results check across N: sha256 of the merged records (score, id, partition)
    digest = None
    if rank == 0:
        rec = np.frombuffer(res.cpu().numpy().tobytes(), dtype=np.dtype(
            [("score", "<f8"), ("id", "<u8"), ("acc", "<i8"), ("partition", "<u4"), ("valid", "<u4")]))
        digest = hashlib.sha256(rec[["score", "id", "partition", "valid"]].tobytes()).hexdigest()
        n_valid = int(rec["valid"].sum())

    # roofline of the dominant kernel (the scan): this rank's algorithmic bytes / the scan
    # kernels' device time (CUDA events around probe + threshold + main scan on the launching
    # stream), averaged over `steps` further batches with per-batch statistics
    scan_ms = []
    if has_docs:
        for _ in range(args.steps):
            st, _ = step(True)
            scan_ms.append(st["scan_ms"])
    scan_ms = statistics.mean(scan_ms) if scan_ms else float("nan")
    scan_bytes = dix.scan_bytes
    peak, peak_src = measured_peak()
    achieved = scan_bytes / (scan_ms / 1e3) / 1e9 if has_docs else 0.0
    if dist:
        t = torch.tensor([achieved, scan_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)  # the slowest rank
        achieved, scan_ms = float(t[0].item()), float(t[1].item())
    traffic = ncu_traffic()
    launches = (int(stats[-1]["launches"]) if stats else 0) * args.steps + (2 * args.steps if world > 1 and rank == 0
                                                                            else 0)

    # e2e with host buffers
    e2e = None
    if world == 1:
        # a serving loop through the public API: the result arrays are allocated once
        # (page-locked) and reused (out=); the query words come from host memory and the
        # results land in host memory every batch
        pe = rbe.pinned_empty
        outs = (pe((Q, K), np.float64), pe((Q, K), np.uint64), pe((Q, K), np.uint32), pe((Q, K), np.int64),
                pe(Q, np.uint64))
        for _ in range(2):
            dix.search_words(qs, geo, K, args.variant, 0, False, outs)
        e2e_times = []
        t0 = time.perf_counter()
        for _ in range(args.steps):
            t1 = time.perf_counter()
            dix.search_words(qs, geo, K, args.variant, 0, False, outs)
            e2e_times.append(time.perf_counter() - t1)
        e2e_total = time.perf_counter() - t0
        e2e = {"value": Q * args.steps / e2e_total, "unit": UNIT, "h2d_bytes_per_step": int(qs.nbytes),
               "d2h_bytes_per_step": Q * K * (8 + 8 + 4 + 8) + Q * 8, "p50_ms": statistics.median(e2e_times) * 1e3,
               "api": "DeviceIndex.search_words(out=reused page-locked host arrays) -> rbe_cuda_search"}
    else:
        h_words = torch.from_numpy(qs.view(np.int64).copy()).pin_memory()
        h_res = torch.empty(Q * K * RESULT_BYTES, dtype=torch.uint8).pin_memory()

        def e2e_step():
            d_words.copy_(h_words, non_blocking=True)
            _, r = step(False)
            if rank == 0:
                h_res.copy_(r, non_blocking=True)
            stream.synchronize()

        for _ in range(2):
            e2e_step()
        dist.barrier()
        e2e_times = []
        t0 = time.perf_counter()
        for _ in range(args.steps):
            t1 = time.perf_counter()
            e2e_step()
            e2e_times.append(time.perf_counter() - t1)
        e2e_total = time.perf_counter() - t0
        t = torch.tensor([e2e_total, statistics.median(e2e_times)], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e = {"value": Q * args.steps / float(t[0].item()), "unit": UNIT,
               "h2d_bytes_per_step": int(qs.nbytes) * world, "d2h_bytes_per_step": Q * K * RESULT_BYTES,
               "p50_ms": float(t[1].item()) * 1e3,
               "api": "per rank: H2D query words -> rbe_cuda_search_device; NCCL gather; rbe_cuda_merge_device; "
                      "D2H of the merged records on rank 0"}

    # C4 latency / throughput of the query batch size (Q in [1, 256]) on the
    # same corpus: device time per batch through the same call (CUDA events on the stream)
    sweep = None
    if world == 1 and has_docs and not args.no_q_sweep:
        sweep = []
        for nq in (1, 2, 8, 16, 64, 128, 256):
            qw = gen_queries(SEED_QUERIES + nq, nq, DIM, QP)
            dw = torch.from_numpy(qw.view(np.int64).copy()).to(dev)
            ob = torch.empty(nq * K * RESULT_BYTES, dtype=torch.uint8, device=dev)
            for _ in range(2):
                rbe.search_device(dix.handle(0), dw.data_ptr(), nq, QP, geo, K, ob.data_ptr(), stream.cuda_stream,
                                  args.variant, False)
            reps = 5
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
            evs[0].record(stream)
            for r in range(reps):
                rbe.search_device(dix.handle(0), dw.data_ptr(), nq, QP, geo, K, ob.data_ptr(), stream.cuda_stream,
                                  args.variant, False)
                evs[r + 1].record(stream)
            torch.cuda.synchronize()
            b = [evs[r].elapsed_time(evs[r + 1]) for r in range(reps)]
            sweep.append({"queries": nq, "batch_ms_p50": statistics.median(b),
                          "queries_per_s": nq / (statistics.median(b) / 1e3),
                          "scan_passes": -(-nq // 64)})
        rbe.last_batch_ms(dix.handle(0))

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            _, cpu, _ = cpu_reference(args, steps=1, warmup=0)
        except Exception as ex:  # noqa: BLE001
            cpu = {"value": None, "unit": UNIT, "kind": "reference", "error": str(ex)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "p50_ms": statistics.median(per),
            "p99_ms": sorted(per)[max(0, -(-99 * len(per) // 100) - 1)],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "s8xu8->s32 tensor / u32 popc->s64; f64 scores" if stats and stats[0]["variant"] == "tensor"
            else "u32 popc -> s64 acc, f64 score",
            "data": "synthetic (counter-based splitmix64 corpus generated on device, SURVEY.md §8(d))",
            "config": dict(workload(args, world), variant=stats[0]["variant"] if stats else None),
            "e2e": e2e,
            "gpu_launches": launches,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic.get("dram_bytes_per_launch") if traffic else None,
                         "traffic_config": traffic.get("config") if traffic else None,
                         "kernel": "scan (" + (stats[0]["variant"] if stats else "-") + "): probe + threshold + main",
                         "scan_ms": scan_ms, "algorithmic_bytes_per_launch": scan_bytes,
                         "bytes_per_doc": BYTES_PER_DOC, "peak_source": peak_src,
                         "aggregate_frac": (args.docs * BYTES_PER_DOC / (ms_per_step / 1e3) / 1e9) / (peak * world)},
            "cpu_baseline": cpu,
            "clocks": clocks.summary(),
            "result_sha256": digest, "result_entries": n_valid, "q_sweep": sweep,
            "doc_queries_per_s": value * args.docs,
            "index_build_s": build_s,
            "candidates_per_batch": statistics.mean(s["candidates"] for s in stats) if stats else None,
            "survivors_per_batch": statistics.mean(s["survivors"] for s in stats) if stats else None,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--variant", default="auto", choices=["auto", "exact", "tensor"])
    ap.add_argument("--docs", type=int, default=1_000_000_000)
    ap.add_argument("--partitions", type=int, default=8)
    ap.add_argument("--queries", type=int, default=64)
    ap.add_argument("--k", type=int, default=1000)
    ap.add_argument("--sample-docs", type=int, default=0,
                    help="CPU reference sample: the first N slots of partition 0 (0 = the whole partition)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-q-sweep", action="store_true", help="skip the C4 query-batch sweep table")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
