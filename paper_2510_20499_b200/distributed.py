"""Multi-GPU probing-cache construction, one process per GPU: candidates are sharded
across ranks with no data-path collective; each rank probes its slice on its own GPU (problem
replicated per GPU), packs it (bp_cache_pack), and the slices are gathered to rank 0 over
torch.distributed (NCCL over NVLink on GPUs; gloo in the CPU tests):

  1. all_gather of the per-rank packed byte counts (int64, 8 bytes per rank)
  2. one batch of point-to-point sends to rank 0 (ncclGroupStart / ncclSend / ncclRecv under
     batch_isend_irecv) -- a gather: only rank 0 receives the slices

Rank 0 merges the slices (bp_cache_merge_packed). Entries are deterministic per variable, so any
partition gives the same cache. The single-process variant over several GPUs is the C-ABI
bp_build_cache_multi (probing.build_cache_multi).
"""
from __future__ import annotations

import numpy as np


def shard(items, rank: int, world: int):
    """Strided interleave of a priority-ordered candidate list (balances skewed probe costs)."""
    if isinstance(items, np.ndarray):
        return np.ascontiguousarray(items[rank::world])
    return list(items[rank::world])


def gather_packed(buf: np.ndarray, device=None, group=None) -> list | None:
    """Gathers every rank's packed slice to rank 0; returns the list of slices there, None elsewhere."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = device if device is not None else torch.device("cpu")
    n = torch.tensor([int(buf.size)], dtype=torch.int64, device=dev)
    sizes = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    mine = torch.from_numpy(np.ascontiguousarray(buf, dtype=np.uint8)).to(dev)
    if rank != 0:
        if sizes[rank]:
            ops = [dist.P2POp(dist.isend, mine, dist.get_global_rank(group, 0) if group else 0, group)]
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        return None
    recv = {r: torch.empty(sizes[r], dtype=torch.uint8, device=dev) for r in range(1, world) if sizes[r]}
    ops = [dist.P2POp(dist.irecv, t, dist.get_global_rank(group, r) if group else r, group)
           for r, t in recv.items()]
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    out = [np.ascontiguousarray(buf, dtype=np.uint8)]
    for r in range(1, world):
        out.append(recv[r].cpu().numpy() if r in recv else np.zeros(0, np.uint8))
    return out


def build_cache_sharded(p, vars_, root=None, device=None, group=None):
    """Probes ``vars_`` sharded over the ranks of ``group``; returns the merged ProbingCache on
    rank 0 (None on other ranks) and this rank's local device time (ms)."""
    import torch.distributed as dist

    from .probing import probe_variables

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    local = probe_variables(p, root, shard(vars_, rank, world))
    if world == 1:  # nothing to gather: the local cache is the cache
        return local, local.probe_ms
    # rank 0 keeps its own slice in place and merges the others' into it (entries are per
    # variable, so the merge order does not change the cache)
    slices = gather_packed(local.pack() if rank != 0 else np.zeros(0, np.uint8), device=device, group=group)
    if rank != 0:
        return None, local.probe_ms
    for s in slices[1:]:
        if s.size:
            local.merge_packed(s)
    return local, local.probe_ms
