"""Dev helper: whole C2 decompression (CUDA events, L2 flushed between steps, median of 15) for libgompresso.so and
every exp/*.so, with parity."""
import sys, statistics, glob
sys.path.insert(0, '.')
import torch, bench, paper_1606_00519_b200 as gomp
cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
kind, n, seed, ckw = bench.CONFIGS[cfg][:4]
x = bench.gen(kind, n, seed)
c = gomp.compress(x, **ckw)
xd = torch.from_numpy(x).cuda()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for path in [gomp.LIB_PATH] + sorted(glob.glob("exp/*.so")):
    gomp.LIB_PATH, gomp._lib = path, None
    info = gomp.get_info(c)
    d = c.cuda(); out = torch.empty(info.uncompressed_len, dtype=torch.uint8, device="cuda")
    ws = torch.empty(gomp.workspace_size(info), dtype=torch.uint8, device="cuda")
    gomp.decompress_into(info, d, out, ws)
    ok = gomp.read_error(ws).status == 0 and torch.equal(out, xd)
    ts = []
    for _ in range(15):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); gomp.decompress_into(info, d, out, ws); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = statistics.median(ts[3:])
    print(path.split('/')[-1], cfg, "ms", round(ms, 4), "GB/s", round(info.uncompressed_len / ms / 1e6, 1), "parity", ok, flush=True)
