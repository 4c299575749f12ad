"""Dev helper: decode time of C5-shaped points (256 MiB matrix text, launcher's decoder) for libgompresso.so and
every exp/*.so, with parity. usage: c5_exp.py block_size k|S<n> [...]"""
import sys, statistics, glob
sys.path.insert(0, '.')
import torch, bench, paper_1606_00519_b200 as gomp
x = bench.gen("matrix", 256 << 20, 5)
xd = torch.from_numpy(x).cuda()
base = gomp.LIB_PATH
pts = [(int(sys.argv[i]), sys.argv[i + 1]) for i in range(1, len(sys.argv), 2)]
for bs, sub in pts:
    kw = dict(sub_block_seqs=int(sub[1:])) if sub[0] == "S" else dict(sub_blocks_per_block=int(sub), sub_block_seqs=0)
    c = gomp.compress(x, mode="bit", de=True, block_size=bs, **kw)
    for path in [base] + sorted(glob.glob("exp/*.so")):
        gomp.LIB_PATH, gomp._lib = path, None
        info = gomp.get_info(c)
        d = c.cuda(); out = torch.empty(info.uncompressed_len, dtype=torch.uint8, device="cuda")
        ws = torch.empty(gomp.workspace_size(info), dtype=torch.uint8, device="cuda")
        out.zero_()
        gomp.decompress_into(info, d, out, ws)
        ok = gomp.read_error(ws).status == 0 and torch.equal(out, xd)
        ts = []
        for _ in range(8):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); gomp.decompress_into(info, d, out, ws, phase="decode"); b.record(); torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        print(bs, sub, gomp.huff_variant(info), path.split('/')[-1], "decode ms", round(statistics.median(ts[2:]), 4), "parity", ok, flush=True)
