"""Dev helper: the C1 data at 148 blocks of 64 KiB (one latency-variant LZ77 CTA per SM; ncu capture target)."""
import sys
sys.path.insert(0, '.')
import torch, datagen, paper_1606_00519_b200 as gomp
x = datagen.text(148 * 65536, seed=1)
c = gomp.compress(x, mode="byte", de=True, block_size=65536)
info = gomp.get_info(c)
d = c.cuda(); out = torch.empty(info.uncompressed_len, dtype=torch.uint8, device="cuda")
ws = torch.empty(gomp.workspace_size(info), dtype=torch.uint8, device="cuda")
for _ in range(4):
    gomp.decompress_into(info, d, out, ws)
torch.cuda.synchronize()
print("ok", bool(torch.equal(out, torch.from_numpy(x).cuda())))
