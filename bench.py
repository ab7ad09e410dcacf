#!/usr/bin/env python
"""Benchmark of the B200 exhaustive RBE retrieval path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (N=1): BASELINE config 2 -- 100M synthetic docs, 128-dim RBE with 3
bit-planes (qp = kp = 3, residual weights), a 64-query batch, top-1000, one
partition, default geometry (T_b=256, I=256, queue length 1, auto blocks).
A step = one batch of 64 queries scanned over the whole corpus + selection.
N>1 (torchrun, one process per GPU, NCCL): weak scaling, 100M docs per GPU
(partition p on rank p), per-rank top-1000 gathered to rank 0 with one NCCL
gather and merged on its GPU.

`value`  queries/s with the query batch already in HBM (device-timed, CUDA
         events on the launching stream, max over ranks).
`e2e`    the same through the public host API (DeviceIndex.search_words ->
         rbe_cuda_search) with host buffers: H2D of the query words and D2H of
         the result records inside the timed region.
The corpus (5.2 GB per GPU) is larger than L2 (126 MB), so no L2 flush is
needed between steps.

`--impl reference` times the reference's own CPU rbe::search (compiled
unmodified into oracle/_ref) on the host cores, query-parallel over all
threads, on a bounded sample (a prefix of the same corpus), scaled linearly to
the full corpus (the scan is O(N)).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DIM, KP, QP, Q, K_TOP = 128, 3, 3, 64, 1000
DOCS_PER_GPU = 100_000_000
SEED_DOCS, SEED_QUERIES = 0xD0C5, 0x0E1
METRIC = "queries/s & p50 latency, top-1000 over 1B RBE docs; HBM GB/s vs peak"
UNIT = "queries/s"
BYTES_PER_DOC = KP * ((DIM + 63) // 64) * 8 + 4  # plane words + f32 magnitude


def env_rank():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(
        os.environ.get("LOCAL_RANK", "0"))


def workload(n_gpus, docs_per_gpu):
    return {
        "workload": f"BASELINE config 2 per GPU: {docs_per_gpu // 1_000_000}M docs x {DIM}-dim RBE, "
                    f"{KP}+{QP} bit-planes (residual weights), Q={Q}, k={K_TOP}, geometry 256/256/1 auto blocks",
        "docs": docs_per_gpu * n_gpus, "docs_per_gpu": docs_per_gpu, "dim": DIM, "keyword_planes": KP,
        "query_planes": QP, "queries_per_batch": Q, "k": K_TOP, "partitions": n_gpus,
        "geometry": {"threads_per_block": 256, "items_per_thread": 256, "queue_length": 1,
                     "blocks": -(-docs_per_gpu // 65536)},
        "seeds": {"docs": SEED_DOCS, "queries": SEED_QUERIES},
        "l2": "corpus 5.2 GB/GPU > 126 MB L2: inputs larger than L2, no flush",
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
    """dram bytes per scan launch from the committed `ncu --set full` summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "scan_traffic.json")) as f:
            return json.load(f)
    except Exception:  # noqa: BLE001
        return None


# --------------------------------------------------------------------------- CPU reference arm
def cpu_reference(steps, warmup, sample_docs=None, threads=None):
    """The reference's rbe::search (oracle/_ref, unmodified sources) on a
    bounded prefix sample; returns (qps scaled to the full 100M corpus, info)."""
    import numpy as np

    from oracle.oracle import Port, Ref, gen_queries, synthetic_prefix

    threads = threads or os.cpu_count() or 1
    sample_docs = sample_docs or 1_000_000
    ref = Ref()
    planes, mags, ids = synthetic_prefix(SEED_DOCS, DOCS_PER_GPU, sample_docs, DIM, KP, True, Port())
    ix = ref.index(DIM, KP, True, [(planes, mags, ids)])
    geo = (-(-sample_docs // 65536), 256, 256, 1)
    qs = gen_queries(SEED_QUERIES, max(threads, 1), DIM, QP)
    times = []
    for s in range(warmup + steps):
        t0 = time.perf_counter()
        ix.search(qs, geo, K_TOP, threads=threads)
        dt = time.perf_counter() - t0
        if s >= warmup:
            times.append(dt)
    per_step = statistics.median(times)
    qps_sample = qs.shape[0] / per_step
    qps_full = qps_sample * sample_docs / DOCS_PER_GPU
    import platform

    cpu = platform.processor() or "cpu"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                cpu = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    info = {"value": qps_full, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"{qs.shape[0]} queries per step (one per thread) over the first {sample_docs:,} docs of the "
                      f"100M-doc corpus (P=1, same geometry rule), scaled x{sample_docs / DOCS_PER_GPU:g} to the full "
                      f"corpus; {steps} steps, median {per_step * 1e3:.1f} ms/step; rbe::search from the reference's "
                      f"own sources (oracle/_ref), query-parallel std::threads; host {cpu}",
            "ms_per_step_sample": per_step * 1e3, "sample_docs": sample_docs}
    return qps_full, info, times


def run_reference_arm(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    qps, info, times = cpu_reference(args.steps, args.warmup, args.sample_docs)
    line = {
        "metric": METRIC, "value": qps, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": statistics.median(times) * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64 popcnt -> s64 acc, f64 score",
        "data": "synthetic (counter-based splitmix64 corpus, SURVEY.md §8(d))",
        "config": workload(args.gpus, DOCS_PER_GPU), "cpu_baseline": info,
        "e2e": {"value": qps, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- our arm
def run_ours(args):
    import numpy as np
    import torch

    import paper_1802_06466_b200 as rbe
    from oracle.oracle import gen_queries  # the query generator (same as the corpus stream)

    rank, world, local = env_rank()
    n_gpus = world
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    docs_per_gpu = args.docs_per_gpu
    n_docs = docs_per_gpu * world
    t_build = time.perf_counter()
    dix = rbe.DeviceIndex.synthetic(DIM, KP, True, n_docs, world, SEED_DOCS, [local], rank, world)
    build_s = time.perf_counter() - t_build
    geo = rbe.ScanGeometry()
    geo.blocks = -(-dix.max_partition_count // 65536)
    qs = gen_queries(SEED_QUERIES, Q, DIM, QP)
    d_words = torch.from_numpy(qs.view(np.int64).copy()).to(f"cuda:{local}")
    from paper_1802_06466_b200.distributed import RESULT_BYTES, gather_and_merge

    # a dedicated stream (the legacy default stream's handle is 0, which the C ABI reads as
    # "the index's own stream"): every kernel, copy and event of a step is ordered on it
    stream = torch.cuda.Stream(device=f"cuda:{local}")
    torch.cuda.set_stream(stream)
    out = torch.empty(Q * K_TOP * RESULT_BYTES, dtype=torch.uint8, device=f"cuda:{local}")

    def merge(blocks):
        if len(blocks) == 1:
            return blocks[0]
        cat = torch.cat(blocks)
        merged = torch.empty_like(blocks[0])
        rbe.merge_device(local, cat.data_ptr(), len(blocks), Q, K_TOP, merged.data_ptr(), stream.cuda_stream)
        return merged

    def step(with_stats):
        # with_stats=False: the batch is only enqueued (no host sync), so consecutive
        # steps run back to back on the GPU
        st = rbe.search_device(dix.handle(0), d_words.data_ptr(), Q, QP, geo, K_TOP, out.data_ptr(),
                               stream.cuda_stream, args.variant, with_stats)
        gather_and_merge(out, rank, world, merge, dist)
        return st

    stats = []
    for _ in range(args.warmup):
        stats.append(step(True))  # warm-up steps also collect the per-batch counters
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    scan_ms_timed = []
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        ev[0].record(stream)
        for s in range(args.steps):
            step(False)
            ev[s + 1].record(stream)
        torch.cuda.synchronize()
        scan_ms_timed.append(rbe.last_batch_ms(dix.handle(0))[0])  # the last timed batch's scan kernels
    if dist:
        dist.barrier()
    per = [ev[s].elapsed_time(ev[s + 1]) for s in range(args.steps)]
    total_ms = ev[0].elapsed_time(ev[args.steps])
    if dist:
        t = torch.tensor([total_ms], device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = Q * args.steps / (total_ms / 1e3)

    # roofline of the dominant kernel (the scan): algorithmic bytes / its event time, from the
    # CUDA events the library records around the scan kernels of the last timed batch
    scan_ms = statistics.mean(scan_ms_timed)
    scan_bytes = dix.scan_bytes  # this rank's docs x 52 B
    peak, peak_src = measured_peak()
    achieved = scan_bytes / (scan_ms / 1e3) / 1e9
    traffic = ncu_traffic()
    launches = int(stats[-1]["launches"]) * args.steps + (args.steps if world > 1 and rank == 0 else 0)

    # e2e through the public host API with host buffers (N=1: rbe_cuda_search)
    e2e = None
    if world == 1:
        # a serving loop: the result arrays are allocated once and reused (out=), the query
        # words come from host memory and the results land in host memory every batch
        pe = rbe.pinned_empty  # page-locked, as a serving loop would hold them
        out = (pe((Q, K_TOP), np.float64), pe((Q, K_TOP), np.uint64), pe((Q, K_TOP), np.uint32),
               pe((Q, K_TOP), np.int64), pe(Q, np.uint64))
        for _ in range(2):
            dix.search_words(qs, geo, K_TOP, args.variant, 0, False, out)
        t0 = time.perf_counter()
        e2e_times = []
        for _ in range(args.steps):
            t1 = time.perf_counter()
            dix.search_words(qs, geo, K_TOP, args.variant, 0, False, out)
            e2e_times.append(time.perf_counter() - t1)
        e2e_total = time.perf_counter() - t0
        e2e = {"value": Q * args.steps / e2e_total, "unit": UNIT, "h2d_bytes_per_step": int(qs.nbytes),
               "d2h_bytes_per_step": Q * K_TOP * (8 + 8 + 4 + 8) + Q * 8, "p50_ms": statistics.median(e2e_times) * 1e3,
               "api": "DeviceIndex.search_words(out=reused page-locked host arrays) -> rbe_cuda_search"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            _, cpu, _ = cpu_reference(steps=2, warmup=0, sample_docs=args.sample_docs * 4)
        except Exception as ex:  # noqa: BLE001
            cpu = {"value": None, "unit": UNIT, "kind": "reference", "error": str(ex)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n_gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "p50_ms": statistics.median(per),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "s8xu8->s32 tensor / u32 popc->s64; f64 scores" if stats[0]["variant"] == "tensor"
            else "u32 popc -> s64 acc, f64 score",
            "data": "synthetic (counter-based splitmix64 corpus generated on device, SURVEY.md §8(d))",
            "config": dict(workload(n_gpus, docs_per_gpu), parallelism=f"shard{n_gpus}", variant=stats[0]["variant"]),
            "e2e": e2e,
            "gpu_launches": launches,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic.get("dram_bytes_per_launch") if traffic else None,
                         "kernel": "scan (" + stats[0]["variant"] + ")", "scan_ms": scan_ms,
                         "algorithmic_bytes_per_launch": scan_bytes, "peak_source": peak_src,
                         "aggregate_frac": (scan_bytes * n_gpus / (ms_per_step / 1e3) / 1e9) / (peak * n_gpus)},
            "cpu_baseline": cpu,
            "clocks": clocks.summary(),
            "doc_queries_per_s": value * n_docs,
            "index_build_s": build_s,
            "candidates_per_batch": statistics.mean(s["candidates"] for s in stats),
            "survivors_per_batch": statistics.mean(s["survivors"] for s in stats),
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--variant", default="auto", choices=["auto", "exact", "tensor"])
    ap.add_argument("--docs-per-gpu", type=int, default=DOCS_PER_GPU)
    ap.add_argument("--sample-docs", type=int, default=1_000_000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
