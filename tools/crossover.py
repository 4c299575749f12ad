"""Dev helper: Bit decoder crossover on C5-shaped data (256 MiB matrix text, one tile of C5): decode-phase device ms
for the thread decoder and the speculative (warp) decoder forced, per block size x sub-blocks per block, for
libgompresso.so and every exp/*.so."""
import sys, statistics, glob
sys.path.insert(0, '.')
import torch, datagen, paper_1606_00519_b200 as gomp
x = datagen.matrix(256 << 20, seed=5)
xd = torch.from_numpy(x).cuda()
cases = {}
for bs in (65536, 262144, 1 << 20):
    for k in (4, 8, 16, 32, 64):
        cases[(bs // 1024, k)] = gomp.compress(x, mode="bit", de=True, block_size=bs, sub_blocks_per_block=k)
for path in [gomp.LIB_PATH] + sorted(glob.glob("exp/*.so")):
    gomp.LIB_PATH, gomp._lib = path, None
    for key, c in cases.items():
        info = gomp.get_info(c)
        d = c.cuda(); out = torch.empty(info.uncompressed_len, dtype=torch.uint8, device="cuda")
        ws = torch.empty(gomp.workspace_size(info), dtype=torch.uint8, device="cuda")
        bits = (info.file_len - info.payload_base) * 8 // info.n_sub_total
        r = {}
        for huff in ("thread", "warp"):
            ts = []
            for _ in range(7):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(); gomp.decompress_into(info, d, out, ws, phase="decode", huff=huff); b.record(); torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            r[huff] = round(statistics.median(ts[2:]), 3)
        gomp.decompress_into(info, d, out, ws, huff="warp")
        ok = gomp.read_error(ws).status == 0 and torch.equal(out, xd)
        print(path.split('/')[-1], key, "bits/sub", bits, "auto", gomp.huff_variant(info), r, "warp parity", ok, flush=True)
