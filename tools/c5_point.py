"""Dev helper: decode time of C5-shaped points (256 MiB matrix text) with the thread and warp decoders forced.
usage: c5_point.py block_size k|S<n> [...]"""
import sys, statistics
sys.path.insert(0, '.')
import torch, bench, paper_1606_00519_b200 as gomp
x = bench.gen("matrix", 256 << 20, 5)
xd = torch.from_numpy(x).cuda()
pts = [(int(sys.argv[i]), sys.argv[i + 1]) for i in range(1, len(sys.argv), 2)]
for bs, sub in pts:
    kw = dict(sub_block_seqs=int(sub[1:])) if sub[0] == "S" else dict(sub_blocks_per_block=int(sub), sub_block_seqs=0)
    c = gomp.compress(x, mode="bit", de=True, block_size=bs, **kw)
    info = gomp.get_info(c)
    d = c.cuda(); out = torch.empty(info.uncompressed_len, dtype=torch.uint8, device="cuda")
    ws = torch.empty(gomp.workspace_size(info), dtype=torch.uint8, device="cuda")
    r = {}
    for huff in ("thread", "warp"):
        gomp.decompress_into(info, d, out, ws, huff=huff)
        ok = gomp.read_error(ws).status == 0 and torch.equal(out, xd)
        ts = []
        for _ in range(8):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); gomp.decompress_into(info, d, out, ws, phase="decode", huff=huff); b.record(); torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        r[huff] = (round(statistics.median(ts[2:]), 4), ok)
    avg_bits = (info.file_len - info.payload_base) * 8 // max(info.n_sub_total, 1)
    print(bs, sub, "avg_bits", avg_bits, "auto:", gomp.huff_variant(info), r, flush=True)
