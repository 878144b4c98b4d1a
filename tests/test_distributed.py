"""CPU (gloo, world size 2): the host-side logic of the sharded probing-cache build — candidate
sharding, the packed-slice gather, and rank-0 merging of packed slices into one cache. The probe
kernels themselves are covered by the GPU tests; here slices are packed by hand in the documented
bp_cache_pack layout, and the merge runs in libbp without touching a device."""
import os
import socket
import struct

import numpy as np
import pytest
import torch.multiprocessing as mp


def pack_slice(entries):
    """bp_cache_pack layout: header {ne, nd, n_fallback, certified} then per entry
    {i32 var, i32 kind, u8 feas[2], u8 force[2], f64 branch[4], i64 count[2]}, then deltas SoA."""
    hdr = struct.pack("<4q", len(entries), sum(len(e["d0"]) + len(e["d1"]) for e in entries), 0, 1)
    body = b""
    dv, dl, du = [], [], []
    for e in entries:
        body += struct.pack("<ii2B2B4d2q", e["var"], e["kind"], *e["feas"], *e["force"], *e["br"],
                            len(e["d0"]), len(e["d1"]))
        for d in (e["d0"], e["d1"]):
            for v, lo, up in d:
                dv.append(v)
                dl.append(lo)
                du.append(up)
    tail = np.array(dv, np.int32).tobytes() + np.array(dl).tobytes() + np.array(du).tobytes()
    return np.frombuffer(hdr + body + tail, dtype=np.uint8).copy()


def entry(v):
    return {"var": v, "kind": 0, "feas": (1, v % 3 != 0), "force": (int(v % 3 == 0), 0),
            "br": (0.0, 0.0, 1.0, 1.0), "d0": [(v, 0.0, 0.0)], "d1": [(v, 1.0, 1.0), (v + 1, 0.0, 0.5)]}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    import torch.distributed as dist

    from paper_2510_20499_b200.distributed import gather_packed, shard
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = shard(list(range(10)), rank, world)
    slices = gather_packed(pack_slice([entry(v) for v in mine]))
    if rank == 0:
        out.put([s.tobytes() for s in slices])
    dist.destroy_process_group()


def test_gloo_gather_and_merge():
    from paper_2510_20499_b200 import _lib
    if not _lib.LIB_PATH.exists():
        pytest.skip("libbp.so not built")
    from paper_2510_20499_b200.probing import ProbingCache
    from paper_2510_20499_b200.propagation import BoundsState

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    slices = q.get(timeout=120)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert len(slices) == 2
    root = BoundsState(raw=np.tile([0.0, 1.0], 12))
    merged = ProbingCache.empty(root)
    for s in slices:
        merged.merge_packed(np.frombuffer(s, dtype=np.uint8))
    assert merged.n_probed == 10
    assert merged.n_infeasible_branches == sum(1 for v in range(10) if v % 3 == 0)
    for v in range(10):
        e = merged.at(v)
        assert e.var == v and e.up.feasible == (v % 3 != 0) and e.forces_down == (v % 3 == 0)
        assert [(d.var, d.new_lower, d.new_upper) for d in e.up.deltas] == [(v, 1.0, 1.0), (v + 1, 0.0, 0.5)]
    # merging the same slice again overwrites (entries are deterministic per variable)
    merged.merge_packed(np.frombuffer(slices[0], dtype=np.uint8))
    assert merged.n_probed == 10


def test_shard_is_a_partition():
    from paper_2510_20499_b200.distributed import shard
    items = list(range(103))
    parts = [shard(items, r, 4) for r in range(4)]
    assert sorted(sum(parts, [])) == items
    assert max(len(x) for x in parts) - min(len(x) for x in parts) <= 1
