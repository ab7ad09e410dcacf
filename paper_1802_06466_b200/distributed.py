"""Multi-GPU sharding of the search (one process per GPU, torch.distributed).

Replaces the reference's in-process partition fan-out (``std::async`` per
partition, src/search.cpp:148-157) and merge (search.cpp:160-167):

* partition p of the corpus lives on rank ``p % world`` (``owned_partitions``);
* every rank scans its partitions into a device-resident top-n per query
  (``rbe_cuda_search_device`` via ``_core.search_device``);
* the per-rank lists (rbe_result records, 32 B each) are gathered to rank 0
  with one NCCL gather over NVLink, and rank 0 merges them on the GPU under
  (score desc, id asc) (``rbe_cuda_merge_device``).

Because top-n over the union of per-rank top-n lists equals top-n over all
survivors, results are identical for any world size with the partition count
fixed (tests/test_distributed.py checks this orchestration with gloo on CPU).
"""
from __future__ import annotations

from typing import Callable, List

RESULT_BYTES = 32  # sizeof(rbe_result)


def owned_partitions(n_partitions: int, rank: int, world: int) -> List[int]:
    """Partition p lives on rank p % world (round-robin, like IndexBuilder's
    doc -> partition rule, src/index.cpp:53)."""
    return [p for p in range(n_partitions) if p % world == rank]


def gather_and_merge(local_results, rank: int, world: int, merge: Callable, dist=None, dst: int = 0):
    """Gather each rank's [Q][n] result block to `dst` and merge there.

    local_results: a tensor holding this rank's [Q][n] records (any dtype/
    layout the `merge` callable understands); `merge(list_of_blocks)` returns
    the merged [Q][n] block.  Returns the merged block on `dst`, None elsewhere.
    """
    if dist is None:
        import torch.distributed as dist  # noqa: F811
    if world == 1:
        return merge([local_results])
    if rank == dst:
        import torch

        bufs = [torch.empty_like(local_results) for _ in range(world)]
        dist.gather(local_results, gather_list=bufs, dst=dst)
        return merge(bufs)
    dist.gather(local_results, gather_list=None, dst=dst)
    return None
