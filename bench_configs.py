#!/usr/bin/env python
"""bench_configs.py — the BASELINE.json configurations beside the headline bench line.

    python bench_configs.py [--only C1,C3,C4,C5] [--steps K] > profiles/r01_configs.jsonl

One JSON line per measured point, same timing rules as bench.py (CUDA events on the launching stream, W >= 3
untimed warm-up steps, the 126 MB L2 flushed by a 512 MiB write between timed steps, device-resident inputs),
every point checked against its input byte for byte before it is timed. value = uncompressed bytes / median step
time (GB/s, 1e9); roofline_frac = (compressed + uncompressed bytes) / step time / HBM peak.

  C1  1 MiB English-like text, Byte, 64 KiB blocks, DE: single-launch latency and steady state (CUDA graph of
      32 back-to-back decompressions), the oracle beside it on 1 core.
  C3  256 MiB nesting-depth-D data (D = 1..32), Byte and Bit, MRR on the non-DE file vs DE on the DE
      file, with the MRR rounds histogram measured on the GPU (GOMP_FLAG_STATS run, untimed).
  C4  16 GiB Wikipedia-shaped corpus on one B200 = the C2 file's blocks tiled 64x (blocks are
      independent and the window is 8 KiB, so tiling keeps per-block statistics).
  C5  4 GiB MatrixMarket-shaped numeric text (a 256 MiB file's blocks tiled 16x), Bit, DE: block size x
      sub-blocks-per-block sweep on one GPU (BASELINE names 8 GPUs: 1/8 of the blocks each, no exchange).
  f2  the GPU compressor (gomp_compress_device) beside the host compressor, identical files required.
  f4  the paper's host-link modes at C2: "In/Out" and "In" through gomp_decompress_host.
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import datagen  # noqa: E402
import paper_1606_00519_b200 as gomp  # noqa: E402

DEV = torch.device("cuda", 0)
FLUSH = None


def timed(fn, k, w):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
    for _ in range(w):
        FLUSH.fill_(1)
        fn()
    torch.cuda.synchronize()
    for i in range(k):
        FLUSH.fill_(i & 0xff)
        ev[i][0].record()
        fn()
        ev[i][1].record()
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in ev]


def point(tag, c, x_check, steps, strategy="auto", extra=None, stats=False):
    """Time device-resident decompression of file c (host uint8 tensor); x_check(out) -> bool."""
    info = gomp.get_info(c)
    U, C = info.uncompressed_len, info.file_len
    d = c.to(DEV)
    out = torch.empty(U, dtype=torch.uint8, device=DEV)
    ws = torch.empty(gomp.workspace_size(info), dtype=torch.uint8, device=DEV)
    gomp.decompress_into(info, d, out, ws, strategy)
    e = gomp.read_error(ws)
    ok = e.status == 0 and bool(x_check(out))
    ms = timed(lambda: gomp.decompress_into(info, d, out, ws, strategy), steps, 3)
    t = statistics.median(ms)
    P, _ = bench.peaks()
    line = {"config": tag, "value": round(U / (t * 1e-3) / 1e9, 3), "unit": "GB/s", "ms_per_step": round(t, 4),
            "uncompressed_bytes": U, "compressed_bytes": C, "ratio": round(U / C, 4), "strategy": strategy,
            "mode": "bit" if info.mode else "byte", "de_file": bool(info.de), "block_size": info.block_size,
            "n_blocks": info.n_blocks, "n_sub_total": info.n_sub_total,
            "roofline_frac": round((U + C) / (t * 1e-3) / 1e9 / P, 4), "peak_gbs": P, "steps": steps,
            "parity": ok}
    if info.mode == 1:
        kd = statistics.median(timed(lambda: gomp.decompress_into(info, d, out, ws, strategy, phase="decode"), 5, 3))
        kl = statistics.median(timed(lambda: gomp.decompress_into(info, d, out, ws, strategy, phase="lz77"), 5, 3))
        line["kernels_ms"] = {"huff_" + gomp.huff_variant(info): round(kd, 4), "lz77": round(kl, 4)}
    if stats:
        gomp.decompress_into(info, d, out, ws, strategy, stats=True)
        st = gomp.read_stats(ws)
        groups = sum(st["rounds"])
        line["rounds_hist"] = {str(r): n for r, n in enumerate(st["rounds"]) if n}
        line["mean_rounds"] = round(sum(r * n for r, n in enumerate(st["rounds"])) / max(groups, 1), 3)
        line["de_fallback_groups"] = st["de_fallback_groups"]
    if extra:
        line.update(extra)
    print(json.dumps(line), flush=True)
    del d, out, ws
    torch.cuda.empty_cache()
    return line


def run_c1(steps):
    import oracle
    x = datagen.text(1 << 20, seed=1)
    c = gomp.compress(x, mode="byte", de=True, block_size=65536)
    info = gomp.get_info(c)
    xd = torch.from_numpy(x).to(DEV)
    line = point("C1", c, lambda o: torch.equal(o, xd), steps, extra={"workload": bench.CONFIGS["C1"][4]})
    # single-launch latency (host enqueue + kernel, synchronised) and steady state through a CUDA graph
    d = c.to(DEV)
    out = torch.empty(info.uncompressed_len, dtype=torch.uint8, device=DEV)
    ws = torch.empty(gomp.workspace_size(info), dtype=torch.uint8, device=DEV)
    lat = []
    for i in range(23):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        gomp.decompress_into(info, d, out, ws)
        torch.cuda.synchronize()
        if i >= 3:
            lat.append((time.perf_counter() - t0) * 1e6)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        gomp.decompress_into(info, d, out, ws, stream=s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(32):
            gomp.decompress_into(info, d, out, ws, stream=s)
    g.replay()
    torch.cuda.synchronize()
    ok = bool(torch.equal(out, xd))
    ms = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b) / 32)
    t0 = time.perf_counter()
    reps = 0
    while time.perf_counter() - t0 < 3.0:
        oracle.decompress(c.numpy())
        reps += 1
    cpu = info.uncompressed_len * reps / (time.perf_counter() - t0) / 1e9
    print(json.dumps({"config": "C1-latency", "single_launch_us_median": round(statistics.median(lat), 1),
                      "graph_steady_state_us": round(1e3 * statistics.median(ms), 2),
                      "graph_steady_state_gbs": round(info.uncompressed_len / (statistics.median(ms) * 1e-3) / 1e9, 3),
                      "oracle_1core_gbs": round(cpu, 4), "parity": ok and line["parity"]}), flush=True)


def run_c3(steps):
    for D in (1, 2, 4, 8, 16, 32):
        x = datagen.nested(256 << 20, D, seed=3)
        xd = torch.from_numpy(x).to(DEV)
        for mode in ("byte", "bit"):
            kw = dict(mode=mode, block_size=262144)
            if mode == "bit":
                kw.update(sub_block_seqs=16)
            for de, strat in ((False, "mrr"), (True, "de")):
                c = gomp.compress(x, de=de, **kw)
                point(f"C3-D{D}-{mode}-{strat}", c, lambda o: torch.equal(o, xd), steps, strategy=strat, stats=True,
                      extra={"depth": D, "workload": f"256 MiB nesting-depth-{D} data, Gompresso/{mode.capitalize()}, "
                                                     f"{'DE file, DE' if de else 'non-DE file, MRR'}"})
        del xd
        torch.cuda.empty_cache()


def tile_file(c, times):
    """A valid file whose blocks are the blocks of c repeated `times` times (c's last block must be full): bench.py's
    tiled shard of the whole tiled range."""
    a = c.numpy()
    return torch.from_numpy(bench.tiled_shard(a, 0, gomp.get_info(a).n_blocks * times))


def run_c4(steps):
    kind, n, seed, ckw = bench.CONFIGS["C2"][:4]
    x = bench.gen(kind, n, seed)
    c = tile_file(gomp.compress(x, **ckw), 64)
    xd = torch.from_numpy(x).to(DEV)

    def check(o):
        return all(torch.equal(o[i * n:(i + 1) * n], xd) for i in range(64))

    point("C4-1gpu", c, check, max(3, steps // 4),
          extra={"workload": "C4: 16 GiB Wikipedia-shaped corpus (C2 blocks tiled 64x), Gompresso/Bit, 256 KiB "
                             "blocks, 16 sub-blocks/block, DE, 1 B200 (the driver's scaling run covers 2/4/8)"})


def run_c5(steps):
    """C5 at its BASELINE size: 4 GiB of MatrixMarket-shaped text = a 256 MiB matrix file's blocks tiled 16x (blocks
    are independent, so tiling keeps every block's statistics), every block size x sub-block point on one B200
    (BASELINE names 8 GPUs: each would hold 1/8 of the blocks, no exchange)."""
    tiles = 16
    x = datagen.matrix(256 << 20, seed=5)
    xd = torch.from_numpy(x).to(DEV)
    n = len(x)

    def check(o):
        return all(torch.equal(o[i * n:(i + 1) * n], xd) for i in range(tiles))

    for bs in (65536, 131072, 262144, 524288, 1 << 20):
        for sub in (4, 8, 16, 32, 64, "S16"):
            kw = dict(mode="bit", de=True, block_size=bs)
            kw.update(dict(sub_block_seqs=16) if sub == "S16" else dict(sub_blocks_per_block=sub))
            c = tile_file(gomp.compress(x, **kw), tiles)
            point(f"C5-4GiB-bs{bs // 1024}k-{'S16' if sub == 'S16' else f'k{sub}'}", c, check, max(3, steps // 2),
                  extra={"workload": "4 GiB MatrixMarket-shaped numeric text (256 MiB file tiled 16x), "
                                     "Gompresso/Bit, DE, 1 B200", "sub_blocks": sub})
            del c


def run_f2(steps):
    """GPU compressor: C2-shaped and C3/C5 inputs compressed on the device (input and file
    resident), wall time of the gomp_compress_device call (it synchronises: the file layout needs the block
    sizes), beside the host compressor on all host threads; the files must be identical."""
    import os as _os
    for tag, kind, n, seed, kw in [
            ("f2-C2", "wiki", 256 << 20, 2, dict(mode="bit", de=True, block_size=262144, sub_blocks_per_block=16)),
            ("f2-C2-byte", "wiki", 256 << 20, 2, dict(mode="byte", de=True, block_size=262144)),
            ("f2-C5", "matrix", 256 << 20, 5, dict(mode="bit", de=True, block_size=262144, sub_blocks_per_block=16)),
            ("f2-C3-D8", "nested8", 256 << 20, 3, dict(mode="bit", de=True, block_size=262144, sub_block_seqs=16))]:
        x = bench.gen(kind, n, seed)
        xd = torch.from_numpy(x).to(DEV)
        g = gomp.compress_device(xd, **kw)
        torch.cuda.synchronize()
        ts = []
        for _ in range(max(3, steps // 3)):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            g = gomp.compress_device(xd, **kw)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        t0 = time.perf_counter()
        h = gomp.compress(x, **kw)
        th = time.perf_counter() - t0
        same = bool(np.array_equal(g.cpu().numpy(), h.numpy()))
        print(json.dumps({"config": tag, "gpu_compress_gbs": round(n / statistics.median(ts) / 1e9, 3),
                          "gpu_compress_ms": round(1e3 * statistics.median(ts), 2),
                          "host_compress_gbs": round(n / th / 1e9, 3), "host_threads": _os.cpu_count(),
                          "ratio": round(n / g.numel(), 4), "identical_to_host": same}), flush=True)
        del xd, g
        torch.cuda.empty_cache()


def run_f4(steps):
    """Host-link modes of the paper at C2: "In/Out" (compressed file in, output out: the bench's e2e)
    and "In" (compressed file in, output stays on the device), both through gomp_decompress_host with pinned
    buffers; the copy engines' own ceiling measured beside them."""
    kind, n, seed, ckw = bench.CONFIGS["C2"][:4]
    x = bench.gen(kind, n, seed)
    c = gomp.compress(x, **ckw).pin_memory()
    info = gomp.get_info(c)
    bufs = (torch.empty(info.file_len, dtype=torch.uint8, device=DEV),
            torch.empty(info.uncompressed_len, dtype=torch.uint8, device=DEV),
            torch.empty(gomp.workspace_size(info), dtype=torch.uint8, device=DEV))
    out_h = torch.empty(info.uncompressed_len, dtype=torch.uint8, pin_memory=True)
    res = {}
    for mode in ("in_out", "in"):
        ts = []
        for i in range(3 + steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            y = gomp.decompress_host(c, out_host=out_h, device=DEV, bufs=bufs, info=info, in_mode=mode == "in")
            torch.cuda.synchronize()
            if i >= 3:
                ts.append(time.perf_counter() - t0)
        ok = bool(np.array_equal((y.cpu() if y.is_cuda else y).numpy(), x))
        res[mode] = (round(n / statistics.median(ts) / 1e9, 2), ok)
    h2d = torch.empty(info.file_len, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(info.file_len, dtype=torch.uint8, device=DEV)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        d.copy_(h2d, non_blocking=True)
    torch.cuda.synchronize()
    h2d_gbs = 5 * info.file_len / (time.perf_counter() - t0) / 1e9
    print(json.dumps({"config": "f4-C2", "in_out_gbs": res["in_out"][0], "in_gbs": res["in"][0],
                      "h2d_copy_gbs": round(h2d_gbs, 1), "in_mode_ceiling_gbs": round(h2d_gbs * n / info.file_len, 1),
                      "parity": res["in_out"][1] and res["in"][1],
                      "note": "uncompressed GB/s through gomp_decompress_host, wall clock incl. synchronisation"}),
          flush=True)


def main():
    global FLUSH
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="C1,C3,C4,C5")
    ap.add_argument("--steps", type=int, default=10)
    args = ap.parse_args()
    if not torch.cuda.is_available():
        raise SystemExit("bench_configs.py needs a CUDA device (no CPU fallback)")
    FLUSH = torch.empty(512 << 20, dtype=torch.uint8, device=DEV)
    for name in args.only.split(","):
        {"C1": run_c1, "C3": run_c3, "C4": run_c4, "C5": run_c5, "f2": run_f2, "f4": run_f4}[name](args.steps)


if __name__ == "__main__":
    main()
