"""Multi-process (N > 1) host logic on CPU with the gloo backend, world_size 2.

The data path has no collective: each rank decodes a contiguous block range chosen by gomp_plan_shards; the only
inter-rank operations are the setup scatter of shard files (gomp_shard_file: rebased tables, O(shard) bytes),
the gather of per-rank {bytes, error word, time} and the max-over-ranks of the timed region, as bench.py does. The decode itself runs on the GPU (tests/test_gpu_parity.py::test_blocks_range...)."""
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
    # rank 0 plans the shards and scatters each rank its shard file (rebased tables + its payloads only: device
    # memory O(shard)); sizes travel first, then the bytes (scatter inputs, gather sizes)
    if rank == 0:
        c = gomp.compress(x, mode="bit", block_size=65536)
        info = gomp.get_info(c)
        first = gomp.plan_shards(c, world)
        shards = [gomp.shard_file(c, first[r], first[r + 1] - first[r]) for r in range(world)]
        meta = torch.tensor([[first[r], first[r + 1], shards[r].numel()] for r in range(world)], dtype=torch.int64)
    else:
        meta = torch.zeros((world, 3), dtype=torch.int64)
    dist.broadcast(meta, 0)
    b0, b1, slen = (int(v) for v in meta[rank])
    mine = torch.zeros(slen, dtype=torch.uint8)
    if rank == 0:
        for r in range(1, world):
            dist.send(shards[r], r)
        mine.copy_(shards[0])
    else:
        dist.recv(mine, 0)
    sinfo = gomp.get_info(mine)
    gomp.validate_tables(mine)
    # this rank's shard, decoded by the oracle here (CPU test of the planning/ownership/shard-file logic)
    y = oracle.decompress(mine.numpy()) if b1 > b0 else np.zeros(0, np.uint8)
    lo = b0 * 65536
    ok = torch.tensor([int(np.array_equal(y, x[lo: lo + len(y)]) and len(y) == sinfo.uncompressed_len)])
    # gather per-rank {bytes, error word, time}; t = max over ranks (bench.py)
    rec = torch.tensor([len(y), 0, 1 + rank], dtype=torch.int64)
    gathered = [torch.zeros(3, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(gathered, rec)
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    ranges = [g.tolist() for g in [torch.tensor([int(meta[r][0]), int(meta[r][1])]) for r in range(world)]]
    if rank == 0:
        out.put((int(ok.item()), int(sum(g[0] for g in gathered)), float(max(g[2] for g in gathered)), ranges,
                 len(x), info.n_blocks, int(sum(g[1] for g in gathered)), int(meta[:, 2].sum()), info.file_len))
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
    ok, n, t, ranges, total, nb, errs, shard_bytes, file_len = res
    assert ok == 1 and n == total and t == float(world) and errs == 0
    assert shard_bytes < file_len + world * 4096      # shards hold no more than the file (+ per-shard headers)
    assert ranges[0][0] == 0 and ranges[-1][1] == nb
    assert all(ranges[i][1] == ranges[i + 1][0] for i in range(world - 1))
