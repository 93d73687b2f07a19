"""CPU (gloo, world_size 2) tests of the partitioned path's host protocol —
what bench.py and the NCCL transport do across processes: the NCCL unique id
travels rank 0 -> all as a pickled object, every rank derives the same
2048-aligned row blocks, and per-rank local matching + an allgather of the
aggregate counts reproduces the global aggregate numbering of the
partition-aware oracle (oracle/partition.py)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1810_04221_b200 as pkg
        from oracle import partition as PA
        from oracle.oracle import Ref
        ref = Ref()
        # 1. unique-id broadcast (bench.py run_partitioned)
        obj = [pkg.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
        # 2. identical level-0 blocks on every rank
        A = ref.gen_randk3d(24, 24, 24, 1.0, 5)
        bounds = pkg.partition_bounds(A.nrows, world)
        assert bounds == PA.partition_bounds(A.nrows, world)
        # 3. local matching on my block + allgather of the counts
        g0, g1 = bounds[rank], bounds[rank + 1]
        Am = PA.mask_cross(A, bounds)
        xadj, adj, wt, z = ref.build_weights(Am, np.ones(A.nrows))
        mate = ref.suitor(xadj, adj, wt)
        local_mate = mate[g0:g1].copy()
        local_mate[local_mate >= 0] -= g0
        agg, nc, _, _ = ref.pairwise_aggregate(local_mate)
        counts = [None] * world
        dist.all_gather_object(counts, int(nc))
        off = sum(counts[:rank])
        q.put((rank, bytes(uid), bounds, (agg + off).tolist(), counts))
    finally:
        dist.destroy_process_group()


def test_partition_protocol_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=240) for _ in range(world)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    uids = {r[1] for r in res}
    assert len(uids) == 1 and len(next(iter(uids))) == 128
    assert res[0][2] == res[1][2]
    # global numbering from the per-rank pieces == the partition-aware oracle
    from oracle import partition as PA
    from oracle.oracle import Ref
    ref = Ref()
    A = ref.gen_randk3d(24, 24, 24, 1.0, 5)
    bounds = res[0][2]
    Am = PA.mask_cross(A, bounds)
    g = ref.build_weights(Am, np.ones(A.nrows))
    agg, nc, _, _ = ref.pairwise_aggregate(ref.suitor(*g[:3]))
    assert res[0][3] + res[1][3] == agg.tolist()
    assert sum(res[0][4]) == nc
