"""Dev helper: C2 In/Out wall time through gomp_decompress_host for libgompresso.so and every exp/*.so, interleaved."""
import glob, statistics, sys, time
sys.path.insert(0, '.')
import torch, bench, paper_1606_00519_b200 as gomp
DEV = torch.device("cuda:0")
kind, n, seed, ckw = bench.CONFIGS["C2"][:4]
x = bench.gen(kind, n, seed)
c = gomp.compress(x, **ckw).pin_memory()
info = gomp.get_info(c)
bufs = (torch.empty(info.file_len, dtype=torch.uint8, device=DEV),
        torch.empty(info.uncompressed_len, dtype=torch.uint8, device=DEV),
        torch.empty(gomp.workspace_size(info), dtype=torch.uint8, device=DEV))
out_h = torch.empty(info.uncompressed_len, dtype=torch.uint8, pin_memory=True)
libs = [gomp.LIB_PATH] + sorted(glob.glob("exp/*.so"))
res = {l: [] for l in libs}
for rnd in range(6):
    for l in libs:
        gomp.LIB_PATH, gomp._lib = l, None
        for i in range(4):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            gomp.decompress_host(c, out_host=out_h, device=DEV, bufs=bufs, info=info)
            torch.cuda.synchronize()
            if i: res[l].append(time.perf_counter() - t0)
for l, ts in res.items():
    print(l.split('/')[-1], "median GB/s", round(n / statistics.median(ts) / 1e9, 2), "best", round(n / min(ts) / 1e9, 2))
