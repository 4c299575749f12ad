"""Dev helper: the thread decoder forced on the first n blocks of C2, libgompresso.so vs exp/*.so."""
import sys, statistics, glob
sys.path.insert(0, '.')
import torch, bench, paper_1606_00519_b200 as gomp
kind, n, seed, ckw = bench.CONFIGS["C2"][:4]
x = bench.gen(kind, n, seed)
c = gomp.compress(x, **ckw)
for path in [gomp.LIB_PATH] + sorted(glob.glob("exp/*.so")):
    gomp.LIB_PATH, gomp._lib = path, None
    info = gomp.get_info(c)
    d = c.cuda(); out = torch.empty(info.uncompressed_len, dtype=torch.uint8, device="cuda")
    ws = torch.empty(gomp.workspace_size(info), dtype=torch.uint8, device="cuda")
    r = {}
    for nb in (148, 1024):
        ts = []
        for _ in range(6):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); gomp.decompress_into(info, d, out, ws, phase="decode", n_blocks=nb, huff="thread"); b.record(); torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        r[nb] = round(statistics.median(ts[2:]), 4)
    print(path.split('/')[-1], r, flush=True)
