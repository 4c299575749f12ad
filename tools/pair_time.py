"""Dev helper: Bit decode time (CUDA events, median) and parity of the warp (K1b) and pair (K1c) decoders on C2
and a few C5-like shapes (256 MiB each)."""
import sys, statistics
sys.path.insert(0, '.')
import torch, bench, datagen, paper_1606_00519_b200 as gomp
shapes = [("wiki", 262144, 16), ("matrix", 262144, 16), ("wiki", 65536, 16), ("matrix", 1 << 20, 16),
          ("wiki", 262144, 8), ("wiki", 262144, 4)]
only = sys.argv[1:] and int(sys.argv[1])
for i, (kind, bs, k) in enumerate(shapes):
    if only and i >= only:
        break
    x = bench.gen(kind, 256 << 20, 2 if kind == "wiki" else 5)
    c = gomp.compress(x, mode="bit", de=True, block_size=bs, sub_blocks_per_block=k)
    info = gomp.get_info(c)
    d = c.cuda(); out = torch.empty(info.uncompressed_len, dtype=torch.uint8, device="cuda")
    ws = torch.empty(gomp.workspace_size(info), dtype=torch.uint8, device="cuda")
    xd = torch.from_numpy(x).cuda()
    r = {}
    for huff in ("warp", "pair"):
        out.zero_()
        gomp.decompress_into(info, d, out, ws, huff=huff)
        ok = gomp.read_error(ws).status == 0 and torch.equal(out, xd)
        ts = []
        for _ in range(9):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); gomp.decompress_into(info, d, out, ws, phase="decode", huff=huff); b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        r[huff] = (round(statistics.median(ts[2:]), 4), ok)
    print(kind, bs, k, "avg_bits", (info.file_len - info.payload_base) * 8 // info.n_sub_total, r, flush=True)
