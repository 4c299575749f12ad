"""bench.py's contract on the host (no GPU needed): the GPU arm refuses to run without CUDA (no CPU fallback),
the reference arm (the oracle) prints one JSON line with the driver's keys, and the roofline
inputs committed under profiles/ are readable."""
import json
import os
import subprocess
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def _run(*args, timeout=600):
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                          text=True, timeout=timeout)


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the CPU-only refusal")
def test_gpu_arm_refuses_without_cuda():
    r = _run("--steps", "1", "--warmup", "3")
    assert r.returncode != 0
    assert "no CPU fallback" in (r.stdout + r.stderr)


def test_reference_arm_json_line():
    r = _run("--impl", "reference", "--steps", "1", "--warmup", "3")
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "GB/s" and d["higher_is_better"] is True
    assert d["warmup"] >= 3 and d["steps"] == 5     # median of >= 5 steps
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["value"] == d["value"] and cb["cores"] == os.cpu_count() == cb["nproc"]
    assert cb["cpu_model"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["workload"].startswith("C2")


def test_roofline_inputs():
    t = bench.ncu_traffic("C2")
    assert t is not None and t["bytes"] > 0 and "capture" in t["source"] and len(t["src_sha"]) > 0
    for k in t["kernels"].values():
        assert k["dram_read"] > 0 and 0 < k["issue_active"] <= 1
    assert isinstance(t["same_build"], bool)
    assert bench.ncu_traffic("no_such_config") is None
    assert len(bench.source_sha()) == 16
    peak, src = bench.peaks()
    assert peak > 1000 and src


def test_cpu_baseline_legs():
    """cpu_baseline: the 1-thread and all-cores oracle legs over a shared block queue."""
    import datagen
    import paper_1606_00519_b200 as gomp
    x = datagen.wiki(1 << 20, seed=2)
    c = gomp.compress(x, mode="bit", block_size=65536, sub_blocks_per_block=4).numpy()
    info = gomp.get_info(c)
    cb = bench.cpu_baseline(c, info.block_size, info.n_blocks, info.uncompressed_len, 1.2)
    assert cb["legs"]["1_thread"]["threads"] == 1 and cb["legs"]["all_cores"]["threads"] == os.cpu_count()
    assert cb["value"] == cb["legs"]["all_cores"]["value"] > 0 and cb["legs"]["1_thread"]["value"] > 0


@pytest.mark.parametrize("tiles,world", [(1, 2), (3, 2), (4, 3), (5, 8)])
def test_tiled_shards(tiles, world):
    """bench.py's multi-GPU corpus: the file's blocks tiled `tiles` times, split by gomp_plan_shards; each rank's
    shard file (rebased tables) validates and the oracle decodes it to its slice of the tiled input."""
    import numpy as np
    import datagen
    import oracle
    import paper_1606_00519_b200 as gomp
    x = datagen.wiki(12 * 65536, seed=2)
    c = gomp.compress(x, mode="bit", block_size=65536, sub_blocks_per_block=4).numpy()
    tt = bench.tiled_tables(c, tiles)
    ti = gomp.get_info(tt)
    assert ti.n_blocks == 12 * tiles and ti.uncompressed_len == tiles * len(x)
    first = gomp.plan_shards(tt, world)
    xt = np.tile(x, tiles)
    got = []
    for r in range(world):
        b0, b1 = first[r], first[r + 1]
        s = bench.tiled_shard(c, b0, b1)
        gomp.validate_tables(s)
        if b1 > b0:
            got.append(oracle.decompress(s))
        assert gomp.get_info(s).uncompressed_len == (b1 - b0) * 65536
        if tiles == 1 and b1 > b0:
            assert np.array_equal(s, gomp.shard_file(c, b0, b1 - b0).numpy())   # == gomp_shard_file
    assert np.array_equal(np.concatenate(got), xt)
