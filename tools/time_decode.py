"""Dev helper: time the Bit decode phase alone on the C2 workload (no correctness check)."""
import sys, statistics
sys.path.insert(0, '.')
import torch, datagen, paper_1606_00519_b200 as gomp
x = datagen.wiki(256 << 20, seed=2)
c = gomp.compress(x, mode="bit", de=True, block_size=262144, sub_blocks_per_block=16)
info = gomp.get_info(c)
d = c.cuda(); out = torch.empty(info.uncompressed_len, dtype=torch.uint8, device="cuda")
ws = torch.empty(gomp.workspace_size(info), dtype=torch.uint8, device="cuda")
for _ in range(3): gomp.decompress_into(info, d, out, ws, phase="decode")
ts = []
for _ in range(10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); gomp.decompress_into(info, d, out, ws, phase="decode"); b.record(); torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
print(sys.argv[1] if len(sys.argv) > 1 else "", "decode ms", statistics.mean(ts))
