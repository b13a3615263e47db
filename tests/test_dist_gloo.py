"""N > 1 host path on CPU: world_size-2 gloo process groups exercise the sharding and the
result gather of paper_2311_00591_b200.dist (the NCCL path uses the same code with
all_gather_into_tensor).  Per-shard results come from the oracle on small pools, so the
gathered set must be byte-identical to a single-process run."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from gen import pools as G
        from oracle import oracle as O
        from paper_2311_00591_b200 import dist as D
        # batched search shards (weak scaling): each rank owns its own pools
        P, n = 40, 32
        lo, hi = D.pool_range(P, rank)
        ss, c, s, r = G.bench_pools_host(G.MODE_SMALL, 9, lo, P, n)
        res = O.search_many(ss, c, s, r, P, n, n)
        allr = D.gather_bytes(torch.from_numpy(res.view(np.uint8).copy()), world)
        # replay sweep cells, cyclic
        n_cells = 7
        mine = D.cyclic_cells(n_cells, rank, world)
        rec = np.array([c * 1000 + rank * 0 for c in mine], np.int64).view(np.uint8)
        cells = D.gather_cells(torch.from_numpy(rec.copy()), n_cells, 8, world)
        if rank == 0:
            q.put((allr.numpy().copy(), cells.numpy().copy()))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_world2_gather_matches_single_process():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    allr, cells = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    from gen import pools as G
    from oracle import oracle as O
    ss, c, s, r = G.bench_pools_host(G.MODE_SMALL, 9, 0, 80, 32)
    want = O.search_many(ss, c, s, r, 80, 32, 32).view(np.uint8)
    assert allr.reshape(-1).tobytes() == want.tobytes()
    assert cells.view(np.int64).reshape(-1).tolist() == [c * 1000 for c in range(7)]


def test_sharding_helpers():
    from paper_2311_00591_b200 import dist as D
    assert D.pool_range(10, 3) == (30, 40)
    got = sorted(c for r in range(3) for c in D.cyclic_cells(8, r, 3))
    assert got == list(range(8))
