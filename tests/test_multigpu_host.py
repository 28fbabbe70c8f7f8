"""Host-side logic of the multi-GPU path, on CPU with torch.distributed (gloo, world 2):
the NCCL unique-id bootstrap the library uses and the row-block partition every rank
computes (the products of the main loop split across GPUs)."""
import os
import socket

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
    dist.destroy_process_group()
    q.put((rank, same, blocks))


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
    for rank, same, blocks in res:
        assert same
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
