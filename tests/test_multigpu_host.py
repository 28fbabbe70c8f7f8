"""Host-side logic of the multi-GPU path, on CPU with torch.distributed (gloo, world 2):
the NCCL unique-id bootstrap the library uses and the row-block partition every rank
computes (the products of the main loop split across GPUs)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1707_01007_b200 import cfpq as C
    # bootstrap: rank 0 draws the NCCL unique id, every rank receives the same 128 bytes
    if rank == 0:
        try:
            uid = C.nccl_unique_id()
        except C.CfpqError as e:          # no usable NCCL on this host: still test the broadcast
            uid = bytes(range(128))
        t = torch.tensor(list(uid), dtype=torch.uint8)
    else:
        t = torch.zeros(128, dtype=torch.uint8)
    dist.broadcast(t, src=0)
    got = [torch.zeros(128, dtype=torch.uint8) for _ in range(world)]
    dist.all_gather(got, t)
    same = all(torch.equal(got[0], g) for g in got)
    # row blocks: every rank computes its own block, the blocks tile [0, n)
    blocks = {}
    for n in (0, 1, 127, 128, 129, 1000, 16384, 65537):
        lo, hi = C.shard_rows(n, world, rank)
        lo_t = torch.tensor([lo, hi], dtype=torch.int64)
        allb = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allb, lo_t)
        blocks[n] = [tuple(b.tolist()) for b in allb]
    # 2-D grids (tensor engine, SUMMA-style blocks): every rank its block, all tile [0,n)^2
    grids = {}
    for n in (1, 300, 1025, 16384):
        for gr, gc in ((1, 2), (2, 1)):
            blk = torch.tensor(C.shard_block(n, gr, gc, rank), dtype=torch.int64)
            allb = [torch.zeros(4, dtype=torch.int64) for _ in range(world)]
            dist.all_gather(allb, blk)
            grids[(n, gr, gc)] = [tuple(b.tolist()) for b in allb]
    # bench.py's whole-job numbers: max time over ranks, work once (sharded) or summed (replicas)
    import bench
    t = 10.0 + rank
    sh = bench.job_totals(dist, world, True, t, 100.0, 1000.0, "cpu")
    rp = bench.job_totals(dist, world, False, t, 100.0 + rank, 1000.0, "cpu")
    dist.destroy_process_group()
    q.put((rank, same, blocks, grids, sh, rp))


def test_bootstrap_and_partition_gloo_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, same, blocks, grids, sh, rp in res:
        assert same
        assert sh == (11.0, 100.0, 1000.0)
        assert rp == (11.0, 201.0, 2000.0)
        for (n, gr, gc), bl in grids.items():
            cover = np.zeros((n, n), np.int32) if n <= 1025 else None
            for r0, r1, c0, c1 in bl:
                assert 0 <= r0 <= r1 <= n and 0 <= c0 <= c1 <= n
                if cover is not None:
                    cover[r0:r1, c0:c1] += 1
            if cover is not None:
                assert (cover == 1).all(), (n, gr, gc)
        for n, bl in blocks.items():
            # contiguous, ordered, disjoint, covering [0, n), boundaries on 128-row tiles
            cur = 0
            for lo, hi in bl:
                assert lo == cur and hi >= lo
                assert lo % 128 == 0 or lo == n
                cur = hi
            assert cur == n


def test_partition_many_ranks():
    from paper_1707_01007_b200 import cfpq as C
    for n in (1, 300, 4096, 16385):
        for world in (1, 2, 3, 4, 8):
            cur = 0
            for r in range(world):
                lo, hi = C.shard_rows(n, world, r)
                assert lo == cur
                cur = hi
            assert cur == n
