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
    assert d["warmup"] >= 3 and d["steps"] == 1
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["workload"].startswith("C2")


def test_roofline_inputs():
    for k in ("huff_warp_kernel", "lz77_batch_kernel"):
        t = bench.ncu_traffic(k, "C2")
        assert t is not None and t["bytes"] > 0 and "capture" in t["source"]
        assert 0 < t["issue"]["issue_active"] <= 1 and 0 < t["issue"]["alu_pipe"] <= 1
    assert bench.ncu_traffic("no_such_kernel", "C2") is None
    peak, src = bench.peaks()
    assert peak > 1000 and src
