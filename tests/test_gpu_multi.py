"""Multi-GPU probing-cache construction: the candidates sharded over GPUs (one process
driving several devices through the C-ABI bp_build_cache_multi, or one process per GPU through
torch.distributed), the packed slices gathered to rank 0 and merged there, must give exactly the
single-GPU cache (entries are deterministic per variable; probing.hpp:243-281)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2510_20499_b200 import synth
from paper_2510_20499_b200.probing import build_cache, build_cache_multi, probe_variables

pytestmark = pytest.mark.gpu


def caches_equal(a, b, vars_):
    """Bitwise equality of two engine caches over vars_ (kind, flags, branch bounds, deltas)."""
    for v in vars_:
        ra, rb = a._entry_raw(v), b._entry_raw(v)
        if (ra is None) != (rb is None):
            return False, v
        if ra is None:
            continue
        if not (np.array_equal(ra[0], rb[0]) and np.array_equal(ra[1].view(np.uint64), rb[1].view(np.uint64))):
            return False, v
        for side in range(2):
            for x, y in zip(a.deltas(v, side), b.deltas(v, side)):
                if not np.array_equal(np.asarray(x).view(np.uint8), np.asarray(y).view(np.uint8)):
                    return False, v
    return True, None


def _devices():
    import torch
    return list(range(torch.cuda.device_count()))


def test_build_cache_multi_equals_single_gpu():
    """bp_build_cache_multi over every visible GPU (one host thread per device, NCCL gather to
    device 0) == the single-GPU cache of the same candidates; and build_cache's budgeted mode."""
    p = synth.c3(n_bin=20_000, n_cont=30_000, n_cover=40_000, n_link=10_000)
    vars_ = np.arange(20_000, dtype=np.int32)
    single = probe_variables(p, None, vars_)
    devs = _devices()
    multi, ms = build_cache_multi(p, devs, vars_)
    assert multi.n_probed == single.n_probed == 20_000 and len(ms) == len(devs)
    assert multi.n_infeasible_branches == single.n_infeasible_branches
    ok, v = caches_equal(multi, single, range(20_000))
    assert ok, v
    q = synth.c1(n=3000, m=3000)  # uncertified root: prioritized candidates, full coverage
    a, _ = build_cache_multi(q, devs, None, 1e9)
    b = build_cache(q, 1e9)
    assert a.n_probed == b.n_probed > 0
    ok, v = caches_equal(a, b, range(q.n_vars))
    assert ok, v


def test_build_cache_multi_two_devices_if_available():
    devs = _devices()
    if len(devs) < 2:
        pytest.skip("one GPU on this box: the NCCL gather path runs with 2+ devices")
    p = synth.c3(n_bin=20_000, n_cont=30_000, n_cover=40_000, n_link=10_000)
    vars_ = np.arange(20_000, dtype=np.int32)
    multi, _ = build_cache_multi(p, devs[:2], vars_)
    ok, v = caches_equal(multi, probe_variables(p, None, vars_), range(20_000))
    assert ok, v


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank(rank, world, port, out):
    import torch.distributed as dist

    from paper_2510_20499_b200.distributed import build_cache_sharded
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p = synth.c3(n_bin=20_000, n_cont=30_000, n_cover=40_000, n_link=10_000)
    merged, _ = build_cache_sharded(p, np.arange(20_000, dtype=np.int32))
    if rank == 0:
        single = probe_variables(p, None, np.arange(20_000, dtype=np.int32))
        ok, v = caches_equal(merged, single, range(20_000))
        out.put((ok, v, merged.n_probed))
    dist.destroy_process_group()


def test_world2_sharded_build_on_one_gpu():
    """Two processes (ranks) on this GPU over gloo run build_cache_sharded end to end: each probes
    its strided half on the device, packs it, sends it to rank 0 (batch_isend_irecv), and rank 0's
    merged cache equals the single-rank cache bit for bit."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    ok, v, n = q.get(timeout=600)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    assert ok, v
    assert n == 20_000
