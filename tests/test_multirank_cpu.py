"""N > 1 host logic on CPU with gloo (world_size 2 and 3): the row-shard plan of the C library
covers [0, n) exactly once with equal staging blocks, and the all-gather + unpack layout used by
the sharded E pass (dme.cu: epass) reconstructs E @ Z exactly (numpy stands in for the kernels)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, k, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    import paper_1805_08990_b200 as dme
    row0, rows, nloc = dme.shard_rows(n, world, rank)
    # every rank computes its local rows of Y = E Z into a (nloc x k) column-major staging block
    rng = np.random.default_rng(0)
    E = rng.standard_normal((n, n))
    Z = rng.standard_normal((n, k))
    stage = np.zeros((k, nloc))          # column-major n_loc x k == row-major k x n_loc
    if rows > 0:
        stage[:, :rows] = (E[row0:row0 + rows] @ Z).T
    gathered = [torch.zeros(k * nloc, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(gathered, torch.from_numpy(stage.ravel().copy()))
    # unpack: block g holds rows [g*nloc, min(n, (g+1)*nloc))
    Y = np.zeros((n, k))
    for g, blk in enumerate(gathered):
        r0, rr, nl = dme.shard_rows(n, world, g)
        b = blk.numpy().reshape(k, nl)
        Y[r0:r0 + rr] = b[:, :rr].T
    ok = np.array_equal(Y, E @ Z) or np.allclose(Y, E @ Z, rtol=1e-14, atol=1e-12)
    spans = [torch.zeros(3, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(spans, torch.tensor([row0, rows, nloc]))
    if rank == 0:
        out.put((bool(ok), [tuple(int(v) for v in s) for s in spans]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 100), (3, 101), (2, 1000), (8, 10000)])
def test_shard_and_allgather_plan(world, n):
    if world > 4:
        # plan only (no processes): coverage of [0, n) by the 8-rank shards
        import paper_1805_08990_b200 as dme
        spans = [dme.shard_rows(n, world, g) for g in range(world)]
    else:
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        port = _free_port()
        procs = [ctx.Process(target=_worker, args=(r, world, port, n, 5, q)) for r in range(world)]
        for p in procs:
            p.start()
        ok, spans = q.get(timeout=120)
        for p in procs:
            p.join(timeout=60)
            assert p.exitcode == 0
        assert ok
    nlocs = {s[2] for s in spans}
    assert len(nlocs) == 1 and list(nlocs)[0] % 16 == 0
    covered = sorted((s[0], s[0] + s[1]) for s in spans if s[1] > 0)
    assert covered[0][0] == 0 and covered[-1][1] == n
    for (a0, a1), (b0, b1) in zip(covered, covered[1:]):
        assert a1 == b0
