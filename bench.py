#!/usr/bin/env python
"""bench.py — Gompresso decompression throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2|C4|...] [--impl ours|reference]

A step = one decompression of the rank's shard through gomp_decompress (every hot-path step of SURVEY.md
§8(a): tables, sub-block scans, LUT build, Huffman decode, LZ77 with DE/MRR). Default workload = BASELINE.json
configs[1] (C2): 256 MiB Wikipedia-shaped synthetic text, Gompresso/Bit, 256 KiB blocks, 16 sub-blocks per
block, DE. Multi-GPU (torchrun, one rank per GPU): the corpus is the C2 file's blocks tiled
`tiles` times (blocks are independent and the window is 8 KiB, so tiling keeps every block's
statistics); gomp_plan_shards splits the tiled file into contiguous block ranges and every rank decodes only
the shard file of its range (rebased tables, O(shard) device memory). Default tiles = N (weak scaling, 256 MiB
per GPU); C4 = 64 tiles = 16 GiB split over the N GPUs (strong scaling). The only collectives are outside the
data path: the barrier, the gather of per-rank {bytes, error word, time} and the max over ranks.

Timing: CUDA events on the launching stream around each step; the L2 (126 MB) is flushed by writing a 512 MiB
buffer between steps (outside the events). ms_per_step = median step time (max over ranks); value = the
uncompressed bytes of all ranks / that time (GB/s, 1e9).
e2e = the same through gomp_decompress_host with pinned host buffers (H2D + kernels + D2H inside the events).
roofline: algorithmic bytes = compressed C (read) + uncompressed U (written) per step, over
the median step time, against the measured HBM copy bandwidth in MEASURED_PEAKS.json; traffic = ncu DRAM bytes
(read + write) of one whole step from the committed capture of the same sources (profiles/ncu_traffic.json).
cpu_baseline: the oracle (oracle/, test infrastructure) on a bounded sample on rank 0 — one thread, and all host
cores pulling blocks from a shared queue (the paper's CPU methodology); --impl reference times the
oracle on all host cores as the reference arm.
"""
import argparse
import hashlib
import json
import os
import platform
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (generator, n_bytes, seed, compression kwargs, workload string, tiles (None = one per rank))
    "C1": ("text", 1 << 20, 1, dict(mode="byte", de=True, block_size=65536),
           "C1: 1 MiB English-like text, Gompresso/Byte, 64 KiB blocks, DE", None),
    "C2": ("wiki", 256 << 20, 2, dict(mode="bit", de=True, block_size=262144, sub_blocks_per_block=16),
           "C2: 256 MiB Wikipedia-shaped text, Gompresso/Bit, 256 KiB blocks, 16 sub-blocks/block, DE", None),
    "C4": ("wiki", 256 << 20, 2, dict(mode="bit", de=True, block_size=262144, sub_blocks_per_block=16),
           "C4: 16 GiB Wikipedia-shaped corpus (the C2 file's blocks tiled 64x), Gompresso/Bit, 256 KiB blocks, "
           "16 sub-blocks/block, DE, blocks sharded across the GPUs", 64),
    "C2-g128": ("wiki", 256 << 20, 2, dict(mode="bit", de=True, block_size=262144, sub_blocks_per_block=16,
                                         de_group=128),
                "256 MiB Wikipedia-shaped text, Gompresso/Bit, 256 KiB blocks, 16 sub-blocks/block, DE over "
                "128-sequence groups (SURVEY 8(f) f3)", None),
    "C2-byte": ("wiki", 256 << 20, 2, dict(mode="byte", de=True, block_size=262144),
                "256 MiB Wikipedia-shaped text, Gompresso/Byte, 256 KiB blocks, DE", None),
    "C2-S16": ("wiki", 256 << 20, 2, dict(mode="bit", de=True, block_size=262144, sub_block_seqs=16),
               "256 MiB Wikipedia-shaped text, Gompresso/Bit, 256 KiB blocks, 16-sequence sub-blocks (P:556), DE",
               None),
    "C3-mrr": ("nested8", 256 << 20, 3, dict(mode="byte", de=False, block_size=262144),
               "C3: 256 MiB nesting-depth-8 data, Gompresso/Byte, MRR", None),
    "C3-de": ("nested8", 256 << 20, 3, dict(mode="byte", de=True, block_size=262144),
              "C3: 256 MiB nesting-depth-8 data, Gompresso/Byte, DE", None),
    "C5": ("matrix", 256 << 20, 5, dict(mode="bit", de=True, block_size=262144, sub_blocks_per_block=16),
           "256 MiB MatrixMarket-shaped numeric text, Gompresso/Bit, 256 KiB blocks, 16 sub-blocks/block, DE", None),
}
METRIC = "decompression GB/s (uncompressed bytes) at 1/2/4/8 B200; % of HBM roofline"


def gen(kind, n, seed):
    import datagen
    if kind.startswith("nested"):
        return datagen.nested(n, int(kind[6:]), seed=seed)
    return datagen.GENERATORS[kind](n, seed=seed)


def source_sha():
    """Hash of the product sources (csrc + include/gomp.h): ties a committed ncu capture to the build it measured."""
    h = hashlib.sha256()
    csrc = os.path.join(ROOT, "paper_1606_00519_b200", "csrc")
    files = sorted(os.path.join(csrc, f) for f in os.listdir(csrc) if f.endswith((".cu", ".cpp", ".hpp", ".cuh")))
    for f in files + [os.path.join(ROOT, "include", "gomp.h")]:
        with open(f, "rb") as fh:
            h.update(os.path.basename(f).encode() + b"\0" + fh.read())
    return h.hexdigest()[:16]


def ncu_traffic(config):
    """DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) of one whole step from the committed ncu --set full
    capture (profiles/ncu_traffic.json, written by tools/ncu_traffic.py), with per-kernel rows and issue
    utilisation; `same_build` says whether the capture measured these sources. None when absent."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as fh:
            t = json.load(fh)
        e = t[config]
        kern = e["kernels"]
        step = sum(int(k["dram_read"] + k["dram_write"]) for k in kern.values())
        return {"bytes": step, "kernels": kern, "source": e["source"], "src_sha": e["src_sha"],
                "same_build": e["src_sha"] == source_sha()}
    except (OSError, KeyError, ValueError, TypeError):
        return None


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


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


def oracle_run(c_np, block_size, n_blocks, total, seconds, threads):
    """The oracle as it stands (single-threaded C; ctypes releases the GIL) on `threads` host threads pulling
    4-block units of the file from a shared queue for ~`seconds`; returns (GB/s, bytes)."""
    import oracle
    lock = threading.Lock()
    nxt = [0]
    done = [0]
    t_end = time.perf_counter() + seconds

    def worker():
        while time.perf_counter() < t_end:
            with lock:
                b = nxt[0]
                nxt[0] = (b + 4) % n_blocks if b + 4 < n_blocks else 0
            nb = min(4, n_blocks - b)
            oracle.decompress_blocks(c_np, b, b + nb, block_size)
            with lock:
                done[0] += min((b + nb) * block_size, total) - b * block_size
    t0 = time.perf_counter()
    ts = [threading.Thread(target=worker) for _ in range(threads)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    dt = time.perf_counter() - t0
    return done[0] / dt / 1e9, done[0], dt


def cpu_baseline(c_np, block_size, n_blocks, total, budget):
    """Median of 3 runs each of the 1-thread and the all-cores oracle legs within ~budget seconds."""
    cores = os.cpu_count() or 1
    legs = {}
    for name, thr in (("1_thread", 1), ("all_cores", cores)):
        runs = [oracle_run(c_np, block_size, n_blocks, total, budget / 6, thr) for _ in range(3)]
        legs[name] = {"value": round(statistics.median(r[0] for r in runs), 4), "threads": thr,
                      "bytes": int(sum(r[1] for r in runs)), "seconds": round(sum(r[2] for r in runs), 2)}
    a = legs["all_cores"]
    return {"value": a["value"], "unit": "GB/s", "cores": cores, "kind": "oracle",
            "sample": f"blocks of the same file from a shared queue (4-block units), median of 3 runs of "
                      f"~{budget / 6:.1f} s per leg ({a['bytes']} B on {cores} threads, "
                      f"{legs['1_thread']['bytes']} B on 1 thread), oracle.decompress_blocks",
            "cpu_model": cpu_model(), "nproc": cores, "legs": legs}


def tiled_tables(c, tiles):
    """Header + block table of the virtual file holding `tiles` copies of c's blocks in order (C4: the C2 file
    tiled; needs whole blocks only). Enough for gomp_plan_shards (it reads the header and block table)."""
    import numpy as np
    import paper_1606_00519_b200 as gomp
    info = gomp.get_info(c)
    nb, ns = info.n_blocks, info.n_sub_total
    assert info.uncompressed_len == nb * info.block_size, "tiling needs whole blocks"
    pay = info.file_len - 16 - info.payload_base
    base = (64 + 32 * nb * tiles + 8 * ns * tiles + 15) & ~15
    hdr = c[:64].copy()
    hv = hdr.view(np.uint32)
    hv[5] = nb * tiles
    hdr[24:32] = np.frombuffer(np.uint64(nb * tiles * info.block_size).tobytes(), np.uint8)
    hdr[32:40] = np.frombuffer(np.uint64(base + pay * tiles + 16).tobytes(), np.uint8)
    hv[10] = ns * tiles
    hdr[48:56] = np.frombuffer(np.uint64(base).tobytes(), np.uint8)
    bt = np.tile(c[64:64 + 32 * nb].view(np.uint32).reshape(nb, 8), (tiles, 1)).copy()
    t = np.repeat(np.arange(tiles, dtype=np.uint64), nb)
    off = (bt[:, 0].astype(np.uint64) | (bt[:, 1].astype(np.uint64) << np.uint64(32))) - np.uint64(info.payload_base)
    off = off + np.uint64(base) + t * np.uint64(pay)
    bt[:, 0] = (off & np.uint64(0xffffffff)).astype(np.uint32)
    bt[:, 1] = (off >> np.uint64(32)).astype(np.uint32)
    bt[:, 5] = bt[:, 5] + (t * np.uint64(ns)).astype(np.uint32)
    return np.concatenate([hdr, bt.view(np.uint8).reshape(-1)])


def tiled_shard(c, b0, b1):
    """Standalone shard file of blocks [b0, b1) of the tiled virtual file (block b = c's block b mod n_blocks):
    what gomp_shard_file writes for that range of the (never materialised) tiled file: rebased block entries,
    the shard's sub-table entries and payloads in block order."""
    import numpy as np
    import paper_1606_00519_b200 as gomp
    info = gomp.get_info(c)
    nb = info.n_blocks
    bt = c[64:64 + 32 * nb].view(np.uint32).reshape(nb, 8)
    st = c[64 + 32 * nb: 64 + 32 * nb + 8 * info.n_sub_total]
    off = bt[:, 0].astype(np.int64) | (bt[:, 1].astype(np.int64) << 32)
    plen, sub_first, n_sub = bt[:, 2].astype(np.int64), bt[:, 5].astype(np.int64), bt[:, 7].astype(np.int64)
    runs = []
    for t in range(b0 // nb, (b1 - 1) // nb + 1 if b1 > b0 else b0 // nb):
        j0, j1 = max(b0 - t * nb, 0), min(b1 - t * nb, nb)
        if j1 > j0:
            runs.append((j0, j1))
    n = b1 - b0
    ent = np.concatenate([bt[j0:j1] for j0, j1 in runs]).copy() if runs else np.zeros((0, 8), np.uint32)
    nsub = int(sum(int(n_sub[j0:j1].sum()) for j0, j1 in runs))
    base = (64 + 32 * n + 8 * nsub + 15) & ~15
    pays = [c[off[j0]: off[j1 - 1] + plen[j1 - 1]] for j0, j1 in runs]
    subs = [st[8 * sub_first[j0]: 8 * (sub_first[j1 - 1] + n_sub[j1 - 1])] for j0, j1 in runs]
    pl = ent[:, 2].astype(np.int64)
    new_off = base + np.concatenate([[0], np.cumsum(pl)[:-1]]) if n else np.zeros(0, np.int64)
    ns_e = ent[:, 7].astype(np.int64)
    new_sf = np.concatenate([[0], np.cumsum(ns_e)[:-1]]) if n else np.zeros(0, np.int64)
    ent[:, 0] = (new_off & 0xffffffff).astype(np.uint32)
    ent[:, 1] = (new_off >> 32).astype(np.uint32)
    if info.mode == 1:
        ent[:, 5] = new_sf.astype(np.uint32)
    flen = base + int(pl.sum()) + 16
    hdr = c[:64].copy()
    hv = hdr.view(np.uint32)
    hv[5] = n
    hdr[24:32] = np.frombuffer(np.uint64(n * info.block_size).tobytes(), np.uint8)
    hdr[32:40] = np.frombuffer(np.uint64(flen).tobytes(), np.uint8)
    hv[10] = nsub
    if info.mode == 1 and n:
        hv[11] = int((4 * ent[:, 3].astype(np.int64) + ent[:, 4]).max())
    hdr[48:56] = np.frombuffer(np.uint64(base).tobytes(), np.uint8)
    out = np.zeros(flen, np.uint8)
    out[:64] = hdr
    out[64:64 + 32 * n] = ent.view(np.uint8).reshape(-1)
    at = 64 + 32 * n
    for sb in subs:
        out[at:at + len(sb)] = sb
        at += len(sb)
    at = base
    for pb in pays:
        out[at:at + len(pb)] = pb
        at += len(pb)
    return out


def run_reference(args, cfg):
    """Reference arm: the oracle as it stands on all host cores (blocks from a shared queue; no GPU work)."""
    import numpy as np
    import paper_1606_00519_b200 as gomp
    kind, n, seed, ckw, workload, _ = CONFIGS[cfg]
    x = gen(kind, n, seed)
    c = gomp.compress(x, **ckw).numpy()
    info = gomp.get_info(c)
    import oracle
    cores = os.cpu_count() or 1
    y = oracle.decompress_blocks(c, 0, 1, info.block_size)           # parity of the arm on its first unit
    assert np.array_equal(y, x[:len(y)])
    per_step = max(0.5, min(3.0, 60.0 / max(args.steps + args.warmup, 1)))
    vals, nbytes = [], []
    for s in range(args.warmup + args.steps):
        v, nb, dt = oracle_run(c, info.block_size, info.n_blocks, info.uncompressed_len, per_step, cores)
        if s >= args.warmup:
            vals.append(v)
            nbytes.append(nb)
    val = statistics.median(vals)
    step_bytes = int(statistics.median(nbytes))
    sample = (f"~{per_step:.1f} s of 4-block units of the {cfg} file per step from a shared queue on {cores} host "
              f"threads ({cpu_model()}), oracle.decompress_blocks; median over steps")
    line = {"metric": METRIC, "impl": "reference", "value": round(val, 4), "unit": "GB/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * per_step, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": workload, "bytes_per_step": step_bytes, "l2": "n/a (CPU)"},
            "cpu_baseline": {"value": round(val, 4), "unit": "GB/s", "cores": cores, "kind": "oracle",
                             "sample": sample, "cpu_model": cpu_model(), "nproc": cores},
            "e2e": {"value": round(val, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2", choices=sorted(CONFIGS))
    ap.add_argument("--tiles", type=int, default=0, help="copies of the config's blocks (0: config default / N)")
    ap.add_argument("--strategy", default="auto")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=12.0, help="seconds of oracle work for cpu_baseline")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    args.steps = max(args.steps, 5)        # median of >= 5 timed steps

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

    kind, n, seed, ckw, workload, cfg_tiles = CONFIGS[args.config]
    tiles = args.tiles or cfg_tiles or world
    x = gen(kind, n, seed)
    t0 = time.time()
    c_full = gomp.compress(x, **ckw).numpy()
    t_compress = time.time() - t0
    base_info = gomp.get_info(c_full)
    # the corpus: `tiles` copies of the file's blocks; this rank's contiguous range from gomp_plan_shards
    if tiles == 1 and world == 1:
        b0, b1 = 0, base_info.n_blocks
        c = c_full
    else:
        first = gomp.plan_shards(tiled_tables(c_full, tiles), world)
        b0, b1 = first[rank], first[rank + 1]
        c = tiled_shard(c_full, b0, b1)
    info = gomp.get_info(c)
    U, C = info.uncompressed_len, info.file_len
    nb_file = base_info.n_blocks
    d_src = torch.from_numpy(c).to(dev)
    out = torch.empty(max(U, 1), dtype=torch.uint8, device=dev)
    ws = torch.empty(gomp.workspace_size(info), dtype=torch.uint8, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    launches_per_step = 1 if info.mode == 0 else 2
    x_d = torch.from_numpy(x).to(dev)

    def step():
        gomp.decompress_into(info, d_src, out, ws, args.strategy, stream)

    def parity():
        """rank output == the tiled input: block b of the shard is input block (b0 + b) mod nb_file"""
        bs = info.block_size
        for t in range(b0 // nb_file, (b1 - 1) // nb_file + 1 if b1 > b0 else 0):
            j0, j1 = max(b0 - t * nb_file, 0), min(b1 - t * nb_file, nb_file)
            o = (t * nb_file + j0 - b0) * bs
            hi = min(j1 * bs, len(x))
            if not torch.equal(out[o:o + hi - j0 * bs], x_d[j0 * bs:hi]):
                return False
        return True

    # correctness of the timed configuration (parity in every timed run)
    step()
    e = gomp.read_error(ws, stream)
    if e.status:
        raise SystemExit(f"device error {gomp.STATUS.get(e.status)} block {e.block}")
    ok = parity()
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

    def gather_max(v):
        if world == 1:
            return v, [v]
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        g = [torch.zeros(1, dtype=torch.float64, device=dev) for _ in range(world)]
        dist.all_gather(g, t)
        vals = [float(z.item()) for z in g]
        return max(vals), vals

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ms = timed(step, args.steps, args.warmup)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_med = statistics.median(ms)
    ms_per_step, per_rank_ms = gather_max(t_med)
    # gather per-rank {uncompressed bytes, compressed bytes, error word} (setup/report only, not the data path)
    e = gomp.read_error(ws, stream)
    rec = torch.tensor([U, C, e.status, int(ok)], dtype=torch.int64, device=dev)
    if world > 1:
        g = [torch.zeros(4, dtype=torch.int64, device=dev) for _ in range(world)]
        dist.all_gather(g, rec)
        recs = [z.tolist() for z in g]
    else:
        recs = [rec.tolist()]
    U_all = sum(r[0] for r in recs)
    C_all = sum(r[1] for r in recs)
    all_ok = all(r[2] == 0 and r[3] == 1 for r in recs)
    value = U_all / (ms_per_step * 1e-3) / 1e9

    # roofline: algorithmic bytes C + U per step over the median step time, per GPU (rank 0)
    P, peak_src = peaks()
    achieved = (U + C) / (t_med * 1e-3) / 1e9
    kern = {}
    T = gomp.token_bytes(c) if info.mode == 1 else 0   # Bit token stream: 4 B per record + 1 B per literal
    if info.mode == 1:
        kd = statistics.median(timed(lambda: gomp.decompress_into(info, d_src, out, ws, args.strategy, stream,
                                                                  phase="decode"), 10, 3))
        kl = statistics.median(timed(lambda: gomp.decompress_into(info, d_src, out, ws, args.strategy, stream,
                                                                  phase="lz77"), 10, 3))
        lzname = "lz77_batch_kernel" if args.strategy in ("auto", "de") and info.de else "lz77_kernel"
        kern = {f"huff_{gomp.huff_variant(info)}_kernel": {"ms": round(kd, 4), "share": round(kd / (kd + kl), 3),
                                                           "algorithmic_bytes": C, "implementation_bytes": T},
                lzname: {"ms": round(kl, 4), "share": round(kl / (kd + kl), 3), "algorithmic_bytes": U,
                         "implementation_bytes": T}}
    else:
        kern = {("lz77_batch_kernel" if args.strategy in ("auto", "de") and info.de else "lz77_kernel"):
                {"ms": round(t_med, 4), "share": 1.0, "algorithmic_bytes": C + U, "implementation_bytes": 0}}
    tr = ncu_traffic(args.config) if tiles == 1 and world == 1 else None
    roofline = {"bound": "hbm", "achieved": round(achieved, 2), "peak": P, "unit": "GB/s",
                "frac": round(achieved / P, 4), "traffic": tr["bytes"] if tr and tr["same_build"] else None,
                "kernel": "whole step (" + " + ".join(kern) + ")", "algorithmic_bytes_per_step": U + C,
                "step_ms": round(t_med, 4), "peak_source": peak_src,
                "traffic_source": (tr["source"] + (" (same sources)" if tr["same_build"] else
                                                   f" (capture of sources {tr['src_sha']}, not these "
                                                   f"{source_sha()}: not reported)")) if tr else None,
                "kernels": kern,
                "note": "T (token stream, written by decode and read by LZ77) is implementation traffic"}
    if tr:
        roofline["ncu_kernels"] = tr["kernels"]

    e2e = None
    if not args.no_e2e:
        try:
            h_src = torch.from_numpy(c).pin_memory()
            h_dst = torch.empty(max(U, 1), dtype=torch.uint8, pin_memory=True)
            d_src2 = torch.empty(C, dtype=torch.uint8, device=dev)

            def e2e_step():
                gomp.lib().gomp_decompress_host(
                    gomp.ctypes.byref(info), h_src.data_ptr(), C, h_dst.data_ptr(), U, d_src2.data_ptr(),
                    out.data_ptr(), ws.data_ptr(), ws.numel(), gomp.STRATEGIES[args.strategy],
                    gomp.ctypes.c_void_p(stream.cuda_stream))

            me = timed(e2e_step, max(5, min(args.steps, 10)), 2)
            if gomp.read_error(ws, stream).status or not parity():
                raise SystemExit("e2e output differs from the input")
            if tiles == 1 and world == 1:
                assert np.array_equal(h_dst.numpy()[:U], x)
            te, _ = gather_max(statistics.median(me))
            e2e = {"value": round(U_all / (te * 1e-3) / 1e9, 3), "unit": "GB/s", "h2d_bytes_per_step": C,
                   "d2h_bytes_per_step": U, "api": "gomp_decompress_host (pinned host buffers)",
                   "ms_per_step": round(te, 4)}
            del d_src2, h_src, h_dst
        except RuntimeError as ex:      # e.g. pinned host memory for a 16 GiB shard not available
            e2e = {"value": None, "unit": "GB/s", "h2d_bytes_per_step": C, "d2h_bytes_per_step": U,
                   "error": str(ex)[:200]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(c_full, base_info.block_size, base_info.n_blocks, base_info.uncompressed_len,
                           args.cpu_budget)

    if rank == 0:
        strong = cfg_tiles is not None and not args.tiles
        line = {"metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
                "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
                "config": {"workload": workload, "uncompressed_bytes": U_all, "compressed_bytes": C_all,
                           "uncompressed_bytes_per_gpu": U, "compressed_bytes_per_gpu": C,
                           "ratio": round(U_all / C_all, 4), "strategy": args.strategy, "tiles": tiles,
                           "blocks": [b0, b1], "l2": "flushed (512 MiB write) between steps",
                           "timing": "median of the timed steps, max over ranks",
                           "parallelism": f"blocks sharded over {world} GPU(s) by gomp_plan_shards, no collective "
                                          f"in the data path", "compress_s": round(t_compress, 2),
                           "per_rank_ms": [round(v, 4) for v in per_rank_ms]},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches_per_step * args.steps, "clocks": clk.summary(), "parity": all_ok}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
