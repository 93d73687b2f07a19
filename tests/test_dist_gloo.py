"""CPU (gloo, world_size 2) tests of the partitioned path's host protocol —
the product code that runs on the host across processes, no GPU needed:

  * the NCCL unique id travels rank 0 -> all as a pickled object (bench.py
    run_partitioned) and every rank derives the same 2048-aligned row blocks
    from the product's mamg_dist_bounds;
  * the NCCL-free multi-process transport's host collective
    (mamg_shm_allgather: the POSIX shared-memory segment with its
    sense-reversing barrier, shm_comm.cu) returns exactly what gloo's
    all_gather returns, including payloads larger than one slot (chunked);
  * a rank whose peer never arrives fails with a timeout instead of hanging.

The device half of that transport (CUDA-IPC exchange blocks, peer mailboxes,
peer reductions, the peer-memory Suitor) runs in tests/test_gpu_dist_mp.py."""
import os
import socket
import uuid

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
    os.environ["MAMG_SHM_TIMEOUT"] = "60"
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1810_04221_b200 as pkg
        # 1. unique-id broadcast + identical level-0 blocks
        obj = [(pkg.nccl_unique_id(), "mamg_gloo_" + uuid.uuid4().hex[:12]) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid, name = obj[0]
        bounds = pkg.partition_bounds(13824, world)
        all_bounds = [None] * world
        dist.all_gather_object(all_bounds, bounds)
        # 2. shm allgather vs gloo allgather: a small and a chunked payload
        rng = np.random.default_rng(100 + rank)
        out = []
        for ln in (1, 7, 4096 * 2 + 3):
            mine = rng.integers(-2**62, 2**62, ln, dtype=np.int64)
            got = pkg.shm_allgather(f"{name}_{ln}", world, rank, mine)
            ref = [None] * world
            dist.all_gather_object(ref, mine)
            out.append(bool(np.array_equal(got, np.stack(ref))))
        q.put((rank, bytes(uid), all_bounds, out))
    finally:
        dist.destroy_process_group()


def test_partition_host_protocol_world2():
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
    from oracle import partition as PA
    for r in res:
        assert r[2][0] == r[2][1] == PA.partition_bounds(13824, world)
        assert r[3] == [True, True, True]


def test_shm_collective_times_out_without_peer(monkeypatch):
    import paper_1810_04221_b200 as pkg
    monkeypatch.setenv("MAMG_SHM_TIMEOUT", "1")
    with pytest.raises(pkg.MamgError, match="timed out"):
        pkg.shm_allgather("mamg_lonely_" + uuid.uuid4().hex[:12], 2, 0, [1, 2, 3])
