"""Dev helper: how much of the LZ77 kernel hides under the decode kernel when both run at once (C2).

Decodes copy A (decode phase only) on one stream while the LZ77 phase of copy B (tokens decoded beforehand)
runs on another, and compares that with the two phases back to back. Independent data, so no flags: an upper
bound on what a block-granular decode -> LZ77 overlap could gain."""
import sys, statistics
sys.path.insert(0, '.')
import torch, bench, paper_1606_00519_b200 as gomp
kind, n, seed, ckw = bench.CONFIGS["C2"][:4]
x = bench.gen(kind, n, seed)
c = gomp.compress(x, **ckw)
info = gomp.get_info(c)
d = c.cuda()
outs = [torch.empty(info.uncompressed_len, dtype=torch.uint8, device="cuda") for _ in range(2)]
wss = [torch.empty(gomp.workspace_size(info), dtype=torch.uint8, device="cuda") for _ in range(2)]
gomp.decompress_into(info, d, outs[1], wss[1], phase="decode")
torch.cuda.synchronize()
lo, hi = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else (0, -1)


def timed(fn, reps=15):
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return round(statistics.median(ts[3:]), 4)


def dec():
    gomp.decompress_into(info, d, outs[0], wss[0], phase="decode")


def lz():
    gomp.decompress_into(info, d, outs[1], wss[1], phase="lz77")


def both(prio_dec):
    s1 = torch.cuda.Stream(priority=-1 if prio_dec else 0)
    s2 = torch.cuda.Stream(priority=0)
    cur = torch.cuda.current_stream()

    def run():
        s1.wait_stream(cur); s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            gomp.decompress_into(info, d, outs[0], wss[0], phase="decode", stream=s1)
        with torch.cuda.stream(s2):
            gomp.decompress_into(info, d, outs[1], wss[1], phase="lz77", stream=s2)
        cur.wait_stream(s1); cur.wait_stream(s2)
    return run


full = lambda: gomp.decompress_into(info, d, outs[0], wss[0])
print({"full": timed(full), "decode": timed(dec), "lz77": timed(lz), "seq": timed(lambda: (dec(), lz())),
       "conc": timed(both(False)), "conc_prio_dec": timed(both(True))}, flush=True)
