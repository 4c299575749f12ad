#!/usr/bin/env python
"""bench.py — Gompresso decompression throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

A step = one decompression of the whole configured file through gomp_decompress (every hot-path step of
SURVEY.md §8(a): tables, sub-block scans, LUT build, Huffman decode, LZ77 with DE/MRR). Default workload =
BASELINE.json configs[1] (C2): 256 MiB Wikipedia-shaped synthetic text, Gompresso/Bit, 256 KiB blocks,
16 sub-blocks per block, DE. Under torchrun (N > 1) every rank decodes its own 256 MiB file (weak scaling:
data blocks are independent; no data-path collective), timing = max over ranks.

Timing: CUDA events on the launching stream around each step; the L2 (126 MB) is flushed by writing a 512 MiB
buffer between steps (outside the events). value = uncompressed bytes / mean step time (GB/s, 1e9).
e2e = the same through gomp_decompress_host with pinned host buffers (H2D + kernels + D2H inside the events).
roofline: algorithmic bytes (compressed + uncompressed) / kernel time vs the measured HBM
copy bandwidth in MEASURED_PEAKS.json. cpu_baseline: the oracle (oracle/, test infrastructure) timed on a
bounded sample on rank 0. --impl reference times the oracle as the reference arm.
"""
import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (generator, n_bytes, seed, compression kwargs, workload string)
    "C1": ("text", 1 << 20, 1, dict(mode="byte", de=True, block_size=65536),
           "C1: 1 MiB English-like text, Gompresso/Byte, 64 KiB blocks, DE"),
    "C2": ("wiki", 256 << 20, 2, dict(mode="bit", de=True, block_size=262144, sub_blocks_per_block=16),
           "C2: 256 MiB Wikipedia-shaped text, Gompresso/Bit, 256 KiB blocks, 16 sub-blocks/block, DE"),
    "C2-g128": ("wiki", 256 << 20, 2, dict(mode="bit", de=True, block_size=262144, sub_blocks_per_block=16,
                                         de_group=128),
                "256 MiB Wikipedia-shaped text, Gompresso/Bit, 256 KiB blocks, 16 sub-blocks/block, DE over "
                "128-sequence groups (SURVEY 8(f) f3)"),
    "C2-byte": ("wiki", 256 << 20, 2, dict(mode="byte", de=True, block_size=262144),
                "256 MiB Wikipedia-shaped text, Gompresso/Byte, 256 KiB blocks, DE"),
    "C2-S16": ("wiki", 256 << 20, 2, dict(mode="bit", de=True, block_size=262144, sub_block_seqs=16),
               "256 MiB Wikipedia-shaped text, Gompresso/Bit, 256 KiB blocks, 16-sequence sub-blocks (P:556), DE"),
    "C3-mrr": ("nested8", 256 << 20, 3, dict(mode="byte", de=False, block_size=262144),
               "C3: 256 MiB nesting-depth-8 data, Gompresso/Byte, MRR"),
    "C3-de": ("nested8", 256 << 20, 3, dict(mode="byte", de=True, block_size=262144),
              "C3: 256 MiB nesting-depth-8 data, Gompresso/Byte, DE"),
    "C5": ("matrix", 256 << 20, 5, dict(mode="bit", de=True, block_size=262144, sub_blocks_per_block=16),
           "256 MiB MatrixMarket-shaped numeric text, Gompresso/Bit, 256 KiB blocks, 16 sub-blocks/block, DE"),
}
METRIC = "decompression GB/s (uncompressed bytes) at 1/2/4/8 B200; % of HBM roofline"


def gen(kind, n, seed):
    import datagen
    if kind.startswith("nested"):
        return datagen.nested(n, int(kind[6:]), seed=seed)
    return datagen.GENERATORS[kind](n, seed=seed)


def ncu_traffic(kernel, config):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` from the committed ncu --set full
    summary (profiles/ncu_traffic.json, written from the capture named there), or None."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "ncu_traffic.json")
    try:
        with open(path) as fh:
            t = json.load(fh)
        e = t[config][kernel]
        r = {"bytes": int(e["dram_read"] + e["dram_write"]), "source": e["source"]}
        if "issue_active" in e:
            r["issue"] = {"issue_active": e["issue_active"], "alu_pipe": e["alu_pipe"], "source": e["source"]}
        return r
    except (OSError, KeyError, ValueError):
        return None


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting"}

    def __init__(self, index):
        self.samples, self.reasons, self.ok = [], set(), False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def oracle_rate(c_np, block_size, n_blocks, budget_s, total):
    """Time the oracle (single thread) on whole blocks until ~budget_s of CPU work; returns GB/s + sample."""
    import oracle
    t0 = time.perf_counter()
    done, b = 0, 0
    while True:
        nb = min(4, n_blocks - b)
        oracle.decompress_blocks(c_np, b, b + nb, block_size)
        done += min((b + nb) * block_size, total) - b * block_size
        b = (b + nb) % n_blocks
        if time.perf_counter() - t0 >= budget_s:
            break
    dt = time.perf_counter() - t0
    return done / dt / 1e9, done, dt


def run_reference(args, cfg):
    """Reference arm: the oracle as it stands, single-threaded on the host (no GPU work)."""
    import numpy as np
    import paper_1606_00519_b200 as gomp
    kind, n, seed, ckw, workload = CONFIGS[cfg]
    x = gen(kind, n, seed)
    c = gomp.compress(x, **ckw).numpy()
    info = gomp.get_info(c)
    import oracle
    # bounded sample per step: the whole run within ~90 s of CPU time
    t0 = time.perf_counter()
    oracle.decompress_blocks(c, 0, 1, info.block_size)
    per_block = max(time.perf_counter() - t0, 1e-4)
    budget = 90.0 / max(args.steps + args.warmup, 1)
    blocks = int(max(1, min(info.n_blocks, budget / per_block)))
    times = []
    for s in range(args.warmup + args.steps):
        b0 = (s * blocks) % max(info.n_blocks - blocks + 1, 1)
        t = time.perf_counter()
        y = oracle.decompress_blocks(c, b0, b0 + blocks, info.block_size)
        dt = time.perf_counter() - t
        if s >= args.warmup:
            times.append(dt)
        assert np.array_equal(y, x[b0 * info.block_size: b0 * info.block_size + len(y)])
    nbytes = min(blocks * info.block_size, info.uncompressed_len)
    val = nbytes / statistics.mean(times) / 1e9
    sample = f"{blocks} consecutive blocks ({nbytes} B) of the {cfg} file per step, single thread"
    line = {"metric": METRIC, "impl": "reference", "value": round(val, 4), "unit": "GB/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * statistics.mean(times), 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": workload, "bytes_per_step": nbytes, "l2": "n/a (CPU)"},
            "cpu_baseline": {"value": round(val, 4), "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": round(val, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2", choices=sorted(CONFIGS))
    ap.add_argument("--strategy", default="auto")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=12.0, help="seconds of oracle work for cpu_baseline")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank == 0:
            run_reference(args, args.config)
        return

    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_1606_00519_b200 as gomp

    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    kind, n, seed, ckw, workload = CONFIGS[args.config]
    x = gen(kind, n, seed + rank)
    t0 = time.time()
    c = gomp.compress(x, **ckw)
    t_compress = time.time() - t0
    info = gomp.get_info(c)
    U, C = info.uncompressed_len, info.file_len
    d_src = c.to(dev)
    out = torch.empty(U, dtype=torch.uint8, device=dev)
    ws = torch.empty(gomp.workspace_size(info), dtype=torch.uint8, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    launches_per_step = 1 if info.mode == 0 else 2

    def step():
        gomp.decompress_into(info, d_src, out, ws, args.strategy, stream)

    # correctness of the timed configuration (parity in every timed run)
    step()
    e = gomp.read_error(ws, stream)
    if e.status:
        raise SystemExit(f"device error {gomp.STATUS.get(e.status)} block {e.block}")
    ok = bool(torch.equal(out, torch.from_numpy(x).to(dev)))
    if not ok:
        raise SystemExit("GPU output differs from the input")

    def timed(fn, k, w):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
        for _ in range(w):
            flush.fill_(1)
            fn()
        torch.cuda.synchronize()
        for i in range(k):
            flush.fill_(i & 0xff)
            ev[i][0].record(stream)
            fn()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
        return [a.elapsed_time(b) for a, b in ev]

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ms = timed(step, args.steps, args.warmup)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_step = statistics.mean(ms)
    t_total = sum(ms)
    if world > 1:
        tt = torch.tensor([t_total], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_total = float(tt.item())
    value = world * U * args.steps / (t_total * 1e-3) / 1e9
    ms_per_step = t_total / args.steps

    # per-kernel times (Bit: Huffman decode and LZ77 launched separately, same stream, same events)
    T = gomp.token_bytes(c) if info.mode == 1 else 0   # Bit token buffer: 4 B per record + 1 B per literal
    if info.mode == 1:
        kd = statistics.mean(timed(lambda: gomp.decompress_into(info, d_src, out, ws, args.strategy, stream,
                                                                phase="decode"), 10, 3))
        kl = statistics.mean(timed(lambda: gomp.decompress_into(info, d_src, out, ws, args.strategy, stream,
                                                                phase="lz77"), 10, 3))
        # algorithmic bytes per launch: decode reads the compressed file and writes the tokens;
        # LZ77 reads the tokens and writes the output
        kern = {f"huff_{gomp.huff_variant(info)}_kernel": (kd, C + T),
                "lz77_batch_kernel" if args.strategy in ("auto", "de") and info.de else "lz77_kernel": (kl, T + U)}
    else:
        kern = {"lz77_batch_kernel (Byte, fused)" if args.strategy in ("auto", "de") and info.de else
                "lz77_kernel (Byte, fused)": (t_step, C + U)}
    dom = max(kern, key=lambda k: kern[k][0])
    P, peak_src = peaks()
    kd_ms, kbytes = kern[dom]
    achieved = kbytes / (kd_ms * 1e-3) / 1e9
    traffic = ncu_traffic(dom.split(" ")[0], args.config)
    roofline = {"bound": "hbm", "achieved": round(achieved, 2), "peak": P, "unit": "GB/s",
                "frac": round(achieved / P, 4), "traffic": traffic["bytes"] if traffic else None,
                "kernel": dom, "kernel_ms": round(kd_ms, 4), "algorithmic_bytes_per_launch": kbytes,
                "traffic_source": traffic["source"] if traffic else None, "peak_source": peak_src,
                "issue": traffic.get("issue") if traffic else None,
                "kernels_ms": {k: round(v[0], 4) for k, v in kern.items()},
                "step": {"algorithmic_bytes": U + C, "achieved": round((U + C) / (t_step * 1e-3) / 1e9, 2),
                         "frac": round((U + C) / (t_step * 1e-3) / 1e9 / P, 4)}}

    e2e = None
    if not args.no_e2e:
        h_src = c.pin_memory()
        h_dst = torch.empty(U, dtype=torch.uint8, pin_memory=True)
        d_src2 = torch.empty(C, dtype=torch.uint8, device=dev)
        bufs = (d_src2, out, ws)

        def e2e_step():
            gomp.lib().gomp_decompress_host(
                gomp.ctypes.byref(info), h_src.data_ptr(), C, h_dst.data_ptr(), U, d_src2.data_ptr(), out.data_ptr(),
                ws.data_ptr(), ws.numel(), gomp.STRATEGIES[args.strategy], gomp.ctypes.c_void_p(stream.cuda_stream))

        me = timed(e2e_step, max(3, min(args.steps, 10)), 2)
        assert np.array_equal(h_dst.numpy(), x)
        te = statistics.mean(me)
        if world > 1:
            tt = torch.tensor([te], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = float(tt.item())
        e2e = {"value": round(world * U / (te * 1e-3) / 1e9, 3), "unit": "GB/s", "h2d_bytes_per_step": C,
               "d2h_bytes_per_step": U, "api": "gomp_decompress_host (pinned host buffers)"}
        del bufs

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, nbytes, dt = oracle_rate(c.numpy(), info.block_size, info.n_blocks, args.cpu_budget, U)
        cpu = {"value": round(v, 4), "unit": "GB/s", "cores": 1, "kind": "oracle",
               "sample": f"{nbytes} B ({nbytes // info.block_size} blocks) of the same file in {dt:.1f} s, "
                         f"single thread, oracle.decompress_blocks"}

    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
                "config": {"workload": workload, "uncompressed_bytes_per_gpu": U, "compressed_bytes_per_gpu": C,
                           "ratio": round(U / C, 4), "strategy": args.strategy, "l2": "flushed (512 MiB write) between steps",
                           "parallelism": f"blocks sharded over {world} GPU(s), no collective",
                           "compress_s": round(t_compress, 2)},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches_per_step * args.steps, "clocks": clk.summary(), "parity": ok}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
