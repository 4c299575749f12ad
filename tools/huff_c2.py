"""Dev helper: C2 decode time with the warp (speculative) and thread (paper) decoders, forced."""
import sys, statistics
sys.path.insert(0, '.')
import torch, bench, paper_1606_00519_b200 as gomp
kind, n, seed, ckw = bench.CONFIGS["C2"][:4]
x = bench.gen(kind, n, seed)
c = gomp.compress(x, **ckw)
info = gomp.get_info(c)
d = c.cuda(); out = torch.empty(info.uncompressed_len, dtype=torch.uint8, device="cuda")
ws = torch.empty(gomp.workspace_size(info), dtype=torch.uint8, device="cuda")
xd = torch.from_numpy(x).cuda()
for huff in ("warp", "thread"):
    gomp.decompress_into(info, d, out, ws, huff=huff)
    ok = gomp.read_error(ws).status == 0 and torch.equal(out, xd)
    r = {}
    for nb in (148, 1024):
        ts = []
        for _ in range(8):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); gomp.decompress_into(info, d, out, ws, phase="decode", n_blocks=nb, huff=huff); b.record(); torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        r[nb] = round(statistics.median(ts[2:]), 4)
    print(huff, ok, r, flush=True)
