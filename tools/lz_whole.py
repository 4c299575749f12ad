"""Dev helper: whole-file device time of configs (default strategy and MRR) for libgompresso.so and exp/*.so."""
import sys, statistics, glob
sys.path.insert(0, '.')
import torch, bench, paper_1606_00519_b200 as gomp
cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["C1", "C2", "C2-byte", "C3-de", "C3-mrr", "C5"]
data = {}
for cfg in cfgs:
    kind, n, seed, ckw = bench.CONFIGS[cfg][:4]
    x = bench.gen(kind, n, seed)
    data[cfg] = (x, gomp.compress(x, **ckw))
for path in [gomp.LIB_PATH] + sorted(glob.glob("exp/*.so")):
    gomp.LIB_PATH, gomp._lib = path, None
    r = {}
    for cfg, (x, c) in data.items():
        info = gomp.get_info(c)
        d = c.cuda(); out = torch.empty(info.uncompressed_len, dtype=torch.uint8, device="cuda")
        ws = torch.empty(gomp.workspace_size(info), dtype=torch.uint8, device="cuda")
        xd = torch.from_numpy(x).cuda()
        gomp.decompress_into(info, d, out, ws)
        ok = gomp.read_error(ws).status == 0 and torch.equal(out, xd)
        ts = []
        for _ in range(12):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); gomp.decompress_into(info, d, out, ws); b.record(); torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        r[cfg] = (round(statistics.median(ts[2:]), 4), ok)
    print(path, r, flush=True)
