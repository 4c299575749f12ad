"""Dev helper: thread-decoder configurations (C3 Bit S=16 at D=1/8/32, C2-S16, C5 S16) whole-file and decode-phase
device time for libgompresso.so and every exp/*.so."""
import sys, statistics, glob
sys.path.insert(0, '.')
import torch, datagen, bench, paper_1606_00519_b200 as gomp
files = {
    "C3-D1-bit": (datagen.nested(256 << 20, 1, seed=3), dict(mode="bit", de=True, block_size=262144, sub_block_seqs=16)),
    "C3-D8-bit": (datagen.nested(256 << 20, 8, seed=3), dict(mode="bit", de=True, block_size=262144, sub_block_seqs=16)),
    "C3-D16-bit": (datagen.nested(256 << 20, 16, seed=3), dict(mode="bit", de=True, block_size=262144, sub_block_seqs=16)),
    "C2-S16": (bench.gen("wiki", 256 << 20, 2), dict(mode="bit", de=True, block_size=262144, sub_block_seqs=16)),
    "C5-64k-S16": (datagen.matrix(256 << 20, seed=5), dict(mode="bit", de=True, block_size=65536, sub_block_seqs=16)),
}
comp = {k: (x, gomp.compress(x, **kw)) for k, (x, kw) in files.items()}
for path in [gomp.LIB_PATH] + sorted(glob.glob("exp/*.so")):
    gomp.LIB_PATH, gomp._lib = path, None
    r = {}
    for k, (x, c) in comp.items():
        info = gomp.get_info(c)
        d = c.cuda(); out = torch.empty(info.uncompressed_len, dtype=torch.uint8, device="cuda")
        ws = torch.empty(gomp.workspace_size(info), dtype=torch.uint8, device="cuda")
        gomp.decompress_into(info, d, out, ws)
        ok = gomp.read_error(ws).status == 0 and torch.equal(out, torch.from_numpy(x).cuda())
        res = []
        for ph in ("decode", None):
            ts = []
            for _ in range(8):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(); gomp.decompress_into(info, d, out, ws, phase=ph); b.record(); torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            res.append(round(statistics.median(ts[2:]), 4))
        r[k] = (res[0], res[1], ok)
    print(path.split('/')[-1], r, flush=True)
