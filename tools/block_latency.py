"""Dev helper: device time of decode / lz77 for the first n blocks of C2 (per-block lifetime vs load)."""
import sys, statistics
sys.path.insert(0, '.')
import torch, bench, paper_1606_00519_b200 as gomp
kind, n, seed, ckw = bench.CONFIGS["C2"][:4]
x = bench.gen(kind, n, seed)
c = gomp.compress(x, **ckw)
info = gomp.get_info(c)
d = c.cuda(); out = torch.empty(info.uncompressed_len, dtype=torch.uint8, device="cuda")
ws = torch.empty(gomp.workspace_size(info), dtype=torch.uint8, device="cuda")
for nb in (1, 2, 8, 32, 148, 296, 592, 1024):
    r = {}
    for ph in ("decode", "lz77", None):
        gomp.decompress_into(info, d, out, ws, phase="decode", n_blocks=nb)
        ts = []
        for _ in range(8):
            if ph == "lz77":
                gomp.decompress_into(info, d, out, ws, phase="decode", n_blocks=nb)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); gomp.decompress_into(info, d, out, ws, phase=ph, n_blocks=nb); b.record(); torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        r[ph or "all"] = round(statistics.median(ts[2:]), 4)
    print(nb, r, flush=True)
