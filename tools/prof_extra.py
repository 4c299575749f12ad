"""Dev helper: one launch of each secondary kernel for ncu: the GPU compressor on 64 MiB of C2-shaped text, and
the MRR kernel on a 64 MiB nesting-depth-8 Byte file (non-DE)."""
import sys
sys.path.insert(0, '.')
import torch, datagen, paper_1606_00519_b200 as gomp
x = datagen.wiki(64 << 20, seed=2)
xd = torch.from_numpy(x).cuda()
c = gomp.compress_device(xd, mode="bit", de=True, block_size=262144, sub_blocks_per_block=16)
y = datagen.nested(64 << 20, 8, seed=3)
f = gomp.compress(y, mode="byte", de=False, block_size=262144)
out = gomp.decompress(f.cuda(), strategy="mrr")
torch.cuda.synchronize()
print("ok", bool(torch.equal(out.cpu(), torch.from_numpy(y))))
