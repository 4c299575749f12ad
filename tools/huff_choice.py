"""Dev helper: decode time of the thread vs warp Huffman decoders over block size x sub-blocks (matrix data)."""
import sys, statistics
sys.path.insert(0, '.')
import torch, datagen, paper_1606_00519_b200 as gomp
x = datagen.matrix(64 << 20, seed=5)
for bs in (65536, 131072, 262144, 524288):
    for k in (4, 8, 16, 32, 64, 128):
        c = gomp.compress(x, mode="bit", de=True, block_size=bs, sub_blocks_per_block=k)
        info = gomp.get_info(c)
        d = c.cuda(); out = torch.empty(info.uncompressed_len, dtype=torch.uint8, device="cuda")
        ws = torch.empty(gomp.workspace_size(info), dtype=torch.uint8, device="cuda")
        res = {}
        for h in ("thread", "warp"):
            for _ in range(2): gomp.decompress_into(info, d, out, ws, phase="decode", huff=h)
            ts = []
            for _ in range(5):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(); gomp.decompress_into(info, d, out, ws, phase="decode", huff=h); b.record(); torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            res[h] = statistics.median(ts)
        avg_bits = (info.file_len - info.payload_base) * 8 / info.n_sub_total
        print(f"bs {bs>>10}k k {k}: avg_sub {info.n_sub_total/info.n_blocks:.0f} avg_bits {avg_bits:.0f} "
              f"thread {res['thread']:.3f} warp {res['warp']:.3f} pick {gomp.huff_variant(info)}", flush=True)
