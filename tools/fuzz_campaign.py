"""Dev helper: a long GPU-vs-oracle fuzz campaign over corrupted files (complements the fixed-seed fuzz tests).

For `seconds` of wall time: draw a data kind, a format configuration (Byte / Bit, DE or not, block size, sub-block
shape, code-length limit, DE group) and a corruption (bit flips in the payloads, the block table or the sub-block
table), decode the corrupted file with the oracle and on the GPU (launcher's choice, and every decoder / LZ77
strategy that applies), and require the GPU to fail iff the oracle fails, with identical output when both accept.
Prints one JSON line of counts; exits non-zero on the first disagreement (after printing it).

With --clean: no corruption, inputs up to 64 blocks of up to 1 MiB (full grids of every kernel variant), every
output compared with the oracle's. With --clean --host: the same files through the end-to-end path
(gomp_decompress_host: pinned host file -> chunked H2D / kernels / D2H pipeline -> host output).

usage: python tools/fuzz_campaign.py [seconds] [seed] [--clean [--host]]
"""
import json
import struct
import sys
import time

sys.path.insert(0, '.')
import numpy as np
import torch

import datagen
import oracle
import paper_1606_00519_b200 as gomp

FORMAT_ERRORS = ("CORRUPT_STREAM", "MALFORMED_BACKREF", "HEADER_INCONSISTENT")
clean = "--clean" in sys.argv
host = "--host" in sys.argv
argv = [v for v in sys.argv if v not in ("--clean", "--host")]
seconds = float(argv[1]) if len(argv) > 1 else 300.0
rng = np.random.default_rng(int(argv[2]) if len(argv) > 2 else 0)
KINDS = ["wiki", "text", "matrix", "random", "zeros", "nested2", "nested8"]


def data(kind, n, seed):
    if kind == "zeros":
        return datagen.zeros(n)
    if kind.startswith("nested"):
        return datagen.nested(n, int(kind[6:]), seed=seed)
    return datagen.GENERATORS[kind](n, seed=seed)


def gpu(f, strategy, huff):
    try:
        if host:
            return "ok", gomp.decompress_host(torch.as_tensor(f).pin_memory(), strategy=strategy).numpy().copy()
        y = gomp.decompress(torch.as_tensor(f).cuda(), strategy=strategy, huff=huff)
        return "ok", y.cpu().numpy()
    except gomp.GompError as e:
        return e.name, None


counts = {"files": 0, "decodes": 0, "oracle_ok": 0, "oracle_err": 0}
t0 = time.time()
while time.time() - t0 < seconds:
    kind = KINDS[int(rng.integers(len(KINDS)))]
    mode = "bit" if rng.random() < 0.6 else "byte"
    de = bool(rng.random() < 0.7) and kind != "nested2"
    bs = int(rng.choice([4096, 16384, 65536, 262144] + ([1 << 20] if clean else [])))
    n = int(rng.integers(1, 65 if clean else 8)) * bs - int(rng.integers(0, bs))
    if clean:
        n = min(n, 48 << 20)
    kw = dict(mode=mode, de=de, block_size=bs)
    if mode == "bit":
        if rng.random() < 0.5:
            kw.update(sub_block_seqs=0, sub_blocks_per_block=int(rng.choice([1, 2, 4, 8, 16, 32])))
        else:
            kw.update(sub_block_seqs=int(rng.choice([16, 64, 200])))
        kw["cwl"] = int(rng.choice([10, 10, 11, 13, 15]))
    if de and rng.random() < 0.2:
        kw["de_group"] = int(rng.choice([64, 128]))
    x = data(kind, max(n, 1), int(rng.integers(1 << 30)))
    c = gomp.compress(x, **kw).numpy()
    info = gomp.get_info(c)
    off = struct.unpack_from("<Q", c.tobytes(), 64)[0]
    sub_lo = 64 + 32 * info.n_blocks
    regions = [(off, len(c) - 16), (off, min(len(c) - 16, off + 4096)), (64, sub_lo)]
    if info.n_sub_total:
        regions.append((sub_lo, sub_lo + 8 * info.n_sub_total))
    lo, hi = regions[int(rng.integers(len(regions)))]
    if hi <= lo:
        continue
    f = c.copy()
    for _ in range(0 if clean else int(rng.integers(1, 4))):
        p = int(rng.integers(lo, hi))
        f[p] ^= np.uint8(1 << int(rng.integers(0, 8)))
    try:
        ref, o_st = oracle.decompress(f), "ok"
    except oracle.OracleError as e:
        ref, o_st = None, e.name
    counts["files"] += 1
    counts["oracle_ok" if o_st == "ok" else "oracle_err"] += 1
    runs = [("auto", None)]
    runs += [("mrr", None)] if de else [("sc", None)]
    if host:
        pass
    elif mode == "bit":
        runs += [("auto", "thread"), ("auto", "warp")]
    else:
        runs += [("de", None)]
    for strategy, huff in runs:
        g_st, y = gpu(f, strategy, huff)
        counts["decodes"] += 1
        bad = None
        if clean and g_st != "ok":
            bad = f"clean file rejected: {g_st}"
        elif (o_st == "ok") != (g_st == "ok"):
            bad = f"verdicts differ: oracle {o_st}, gpu {g_st}"
        elif g_st == "ok" and not np.array_equal(y, ref):
            bad = "both accept, outputs differ"
        elif g_st != "ok" and g_st not in FORMAT_ERRORS:
            bad = f"gpu status {g_st} is not a format error"
        if bad:
            print(json.dumps({"disagreement": bad, "kind": kind, "params": kw, "n": n, "region": [lo, hi],
                              "strategy": strategy, "huff": huff}), flush=True)
            sys.exit(1)
counts["seconds"] = round(time.time() - t0, 1)
print(json.dumps({"fuzz_campaign": ("clean files through gomp_decompress_host: output == oracle output" if host else
                                   "clean files: GPU output == oracle output" if clean else
                                   "GPU fails iff the oracle fails, identical output otherwise"), **counts}))
