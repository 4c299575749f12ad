"""Dev helper: the thread-per-sub-block decoder (K1a) on 256 MiB nesting-depth-8 data, S = 16 (C3 Bit, DE)."""
import sys, statistics
sys.path.insert(0, '.')
import torch, datagen, paper_1606_00519_b200 as gomp
x = datagen.nested(256 << 20, 8, seed=3)
c = gomp.compress(x, mode="bit", de=True, block_size=262144, sub_block_seqs=16)
info = gomp.get_info(c)
d = c.cuda(); out = torch.empty(info.uncompressed_len, dtype=torch.uint8, device="cuda")
ws = torch.empty(gomp.workspace_size(info), dtype=torch.uint8, device="cuda")
for _ in range(3): gomp.decompress_into(info, d, out, ws, phase="decode")
ts = []
for _ in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); gomp.decompress_into(info, d, out, ws, phase="decode"); b.record(); torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
print("decode ms", statistics.median(ts), "n_sub", info.n_sub_total, "blocks", info.n_blocks)
