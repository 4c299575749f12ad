"""Dev helper: one launch of each secondary kernel for ncu: the GPU compressor on 64 MiB of C2-shaped text, the
MRR kernel on a 64 MiB nesting-depth-8 Byte file (non-DE), the thread-per-sub-block decoder on a 256 MiB
nesting-depth-8 Bit file with S = 16 (C3), and the fused Byte DE path on the same data."""
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
print("mrr ok", bool(torch.equal(out.cpu(), torch.from_numpy(y))))
z = datagen.nested(256 << 20, 8, seed=3)
for kw in (dict(mode="bit", de=True, sub_block_seqs=16), dict(mode="byte", de=True)):
    f = gomp.compress(z, block_size=262144, **kw)
    out = gomp.decompress(f.cuda())
    torch.cuda.synchronize()
    print(kw["mode"], "ok", bool(torch.equal(out.cpu(), torch.from_numpy(z))))
