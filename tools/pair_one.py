"""Dev helper: C2 decode phase with the pair decoder forced (ncu capture target)."""
import sys
sys.path.insert(0, '.')
import torch, bench, paper_1606_00519_b200 as gomp
kind, n, seed, ckw = bench.CONFIGS["C2"][:4]
x = bench.gen(kind, n, seed)
c = gomp.compress(x, **ckw)
info = gomp.get_info(c)
d = c.cuda(); out = torch.empty(info.uncompressed_len, dtype=torch.uint8, device="cuda")
ws = torch.empty(gomp.workspace_size(info), dtype=torch.uint8, device="cuda")
huff = sys.argv[1] if len(sys.argv) > 1 else "pair"
for _ in range(3):
    gomp.decompress_into(info, d, out, ws, phase="decode", huff=huff)
torch.cuda.synchronize()
print("done")
