"""Dev helper: the thread-per-sub-block decoder (paper scheme) forced on the first n blocks of C2 (for ncu)."""
import sys
sys.path.insert(0, '.')
import torch, bench, paper_1606_00519_b200 as gomp
kind, n, seed, ckw = bench.CONFIGS["C2"][:4]
x = bench.gen(kind, n, seed)
c = gomp.compress(x, **ckw)
info = gomp.get_info(c)
d = c.cuda(); out = torch.empty(info.uncompressed_len, dtype=torch.uint8, device="cuda")
ws = torch.empty(gomp.workspace_size(info), dtype=torch.uint8, device="cuda")
nb = int(sys.argv[1]) if len(sys.argv) > 1 else 148
gomp.decompress_into(info, d, out, ws, phase="decode", n_blocks=nb, huff="thread")
torch.cuda.synchronize()
