"""Dev helper: time one phase ("decode" / "lz77" / "all") of the C2 workload (no correctness check)."""
import sys, statistics
sys.path.insert(0, '.')
import torch, datagen, paper_1606_00519_b200 as gomp
phase = sys.argv[1] if len(sys.argv) > 1 else "all"
x = datagen.wiki(256 << 20, seed=2)
grp = int(sys.argv[2]) if len(sys.argv) > 2 else 32
c = gomp.compress(x, mode="bit", de=True, block_size=262144, sub_blocks_per_block=16, de_group=grp)
info = gomp.get_info(c)
d = c.cuda(); out = torch.empty(info.uncompressed_len, dtype=torch.uint8, device="cuda")
ws = torch.empty(gomp.workspace_size(info), dtype=torch.uint8, device="cuda")
gomp.decompress_into(info, d, out, ws, phase="decode")
ph = None if phase == "all" else phase
for _ in range(3): gomp.decompress_into(info, d, out, ws, phase=ph)
ts = []
for _ in range(10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); gomp.decompress_into(info, d, out, ws, phase=ph); b.record(); torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
print(phase, "ms", statistics.mean(ts))
