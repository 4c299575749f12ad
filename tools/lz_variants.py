"""Dev helper: LZ77 kernel device time, flow (default) vs batch (GOMP_FLAG_LZ77_BATCH), on the first n blocks
of C2 (Bit tokens from one decode) and on whole C1 / C2-byte / C3-de files; checks every output."""
import statistics
import sys
sys.path.insert(0, '.')
import torch
import bench
import paper_1606_00519_b200 as gomp


def med(fn, k=10):
    ts = []
    for _ in range(k + 2):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return round(statistics.median(ts[2:]), 4)


for cfg in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["C2", "C1", "C2-byte", "C3-de", "C5"]):
    kind, n, seed, ckw = bench.CONFIGS[cfg][:4]
    x = bench.gen(kind, n, seed)
    c = gomp.compress(x, **ckw)
    info = gomp.get_info(c)
    d = c.cuda()
    xd = torch.from_numpy(x).cuda()
    out = torch.empty(info.uncompressed_len, dtype=torch.uint8, device="cuda")
    ws = torch.empty(gomp.workspace_size(info), dtype=torch.uint8, device="cuda")
    res = {}
    for lz in ("default",):
        out.zero_()
        gomp.decompress_into(info, d, out, ws, "de")
        e = gomp.read_error(ws)
        ok = e.status == 0 and torch.equal(out, xd)
        r = {"ok": ok}
        if info.mode == 1:
            for nb in (1, 8, 148, 1024):
                nb = min(nb, info.n_blocks)
                gomp.decompress_into(info, d, out, ws, "de", phase="decode", n_blocks=nb)
                r[f"lz_{nb}"] = med(lambda: gomp.decompress_into(info, d, out, ws, "de", phase="lz77", n_blocks=nb))
        r["all"] = med(lambda: gomp.decompress_into(info, d, out, ws, "de"))
        res[lz] = r
    print(cfg, res, flush=True)
