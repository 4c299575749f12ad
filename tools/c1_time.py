"""Dev helper: C1 kernel time (CUDA graph of 32 decompressions) for libgompresso.so and every exp/*.so."""
import sys, statistics, glob
sys.path.insert(0, '.')
import torch, datagen, paper_1606_00519_b200 as gomp
x = datagen.text(1 << 20, seed=1)
c = gomp.compress(x, mode="byte", de=True, block_size=65536)
xd = torch.from_numpy(x).cuda()
for path in [gomp.LIB_PATH] + sorted(glob.glob("exp/*.so")):
    gomp.LIB_PATH, gomp._lib = path, None
    info = gomp.get_info(c)
    d = c.cuda(); out = torch.empty(info.uncompressed_len, dtype=torch.uint8, device="cuda")
    ws = torch.empty(gomp.workspace_size(info), dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        gomp.decompress_into(info, d, out, ws, stream=s)
    torch.cuda.synchronize()
    ok = bool(torch.equal(out, xd))
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(32):
            gomp.decompress_into(info, d, out, ws, stream=s)
    g.replay(); torch.cuda.synchronize()
    ms = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); b.record(); torch.cuda.synchronize()
        ms.append(a.elapsed_time(b) / 32 * 1e3)
    print(path.split('/')[-1], "us", round(statistics.median(ms), 2), "parity", ok, flush=True)
