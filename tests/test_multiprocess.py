"""Multi-process (N > 1) host logic on CPU with the gloo backend, world_size 2.

The data path has no collective: each rank decodes a contiguous block range chosen by gomp_plan_shards; the only
inter-rank operations are the barrier and the max-over-ranks of the timed region. Here each rank plans the
shards of the same file, takes its range, checks the ranges tile the file, and reduces a per-rank time with MAX
exactly as bench.py does. The decode itself runs on the GPU (tests/test_gpu_parity.py::test_blocks_range...)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import datagen
    import oracle
    import paper_1606_00519_b200 as gomp
    x = datagen.wiki(1_500_000, seed=4)
    c = gomp.compress(x, mode="bit", block_size=65536)
    info = gomp.get_info(c)
    first = gomp.plan_shards(c, world)
    b0, b1 = first[rank], first[rank + 1]
    # this rank's shard, decoded by the oracle here (CPU test of the planning/ownership logic)
    y = oracle.decompress_blocks(c.numpy(), b0, b1, info.block_size) if b1 > b0 else np.zeros(0, np.uint8)
    lo = b0 * info.block_size
    ok = torch.tensor([int(np.array_equal(y, x[lo: lo + len(y)]))])
    n = torch.tensor([len(y)], dtype=torch.int64)
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    dist.all_reduce(n, op=dist.ReduceOp.SUM)
    t = torch.tensor([1.0 + rank], dtype=torch.float64)       # bench.py: max over ranks of the timed region
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    gathered = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(gathered, torch.tensor([b0, b1]))
    if rank == 0:
        out.put((int(ok.item()), int(n.item()), float(t.item()), [g.tolist() for g in gathered], info.uncompressed_len,
                 info.n_blocks))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_shards_over_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ok, n, t, ranges, total, nb = res
    assert ok == 1 and n == total and t == float(world)
    assert ranges[0][0] == 0 and ranges[-1][1] == nb
    assert all(ranges[i][1] == ranges[i + 1][0] for i in range(world - 1))
