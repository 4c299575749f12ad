"""Dev helper: thread-per-sub-block decoder (K1a) device time for libgompresso.so and every exp/*.so on the
paper-default sub-blocks (S = 16 sequences) and on short fixed-count sub-blocks."""
import sys, statistics, glob
sys.path.insert(0, '.')
import torch, datagen, paper_1606_00519_b200 as gomp
cases = [("C3-D1 S16", datagen.nested(256 << 20, 1, seed=3), dict(sub_block_seqs=16)),
         ("C3-D8 S16", datagen.nested(256 << 20, 8, seed=3), dict(sub_block_seqs=16)),
         ("wiki S16", datagen.wiki(256 << 20, seed=2), dict(sub_block_seqs=16)),
         ("matrix 64k k64", datagen.matrix(64 << 20, seed=5), dict(block_size=65536, sub_blocks_per_block=64))]
files = []
for name, x, kw in cases:
    p = dict(mode="bit", de=True, block_size=262144); p.update(kw)
    files.append((name, gomp.compress(x, **p)))
for path in [gomp.LIB_PATH] + sorted(glob.glob("exp/*.so")):
    gomp.LIB_PATH, gomp._lib = path, None
    r = {}
    for name, c in files:
        info = gomp.get_info(c)
        d = c.cuda(); out = torch.empty(info.uncompressed_len, dtype=torch.uint8, device="cuda")
        ws = torch.empty(gomp.workspace_size(info), dtype=torch.uint8, device="cuda")
        ts = []
        for _ in range(8):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); gomp.decompress_into(info, d, out, ws, phase="decode", huff="thread"); b.record(); torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        r[name] = round(statistics.median(ts[2:]), 4)
    print(path.split('/')[-1], r, flush=True)
