"""Dev helper: C2 decode phase (ncu capture target) with the library at argv[1] (default libgompresso.so)."""
import sys
sys.path.insert(0, '.')
import torch, bench, paper_1606_00519_b200 as gomp
if len(sys.argv) > 1:
    gomp.LIB_PATH = sys.argv[1]
kind, n, seed, ckw = bench.CONFIGS["C2"][:4]
x = bench.gen(kind, n, seed)
c = gomp.compress(x, **ckw)
info = gomp.get_info(c)
d = c.cuda(); out = torch.empty(info.uncompressed_len, dtype=torch.uint8, device="cuda")
ws = torch.empty(gomp.workspace_size(info), dtype=torch.uint8, device="cuda")
for _ in range(3):
    gomp.decompress_into(info, d, out, ws, phase="decode")
torch.cuda.synchronize()
print("done")
