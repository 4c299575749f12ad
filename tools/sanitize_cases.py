"""Dev helper: one decompression per kernel configuration, for compute-sanitizer (memcheck / racecheck /
synccheck): Byte DE with the three LZ77 variants (4-warp batches with instruction-lean or load-first copies,
16-warp batches), Bit with the speculative decoder
(whole grid and split grid, one- and two-warp groups) and the thread decoder (with long sub-blocks handed to
one warp), MRR and SC on a non-DE file. Exits non-zero on a mismatch."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch, datagen, paper_1606_00519_b200 as gomp
cases = [
    ("byte DE 537 blocks", datagen.wiki(2_200_000, seed=21), dict(mode="byte", de=True, block_size=4096), "auto"),
    ("byte DE 19 blocks (16-warp batches)", datagen.wiki(300_000, seed=21), dict(mode="byte", de=True, block_size=16384), "auto"),
    ("byte DE 300 blocks (load-first copies)", datagen.wiki(300 * 4096, seed=21), dict(mode="byte", de=True, block_size=4096), "auto"),
    ("bit warp 600 blocks", datagen.wiki(600 * 16384, seed=2), dict(mode="bit", de=True, block_size=16384, sub_blocks_per_block=2), "auto"),
    ("bit warp split", datagen.wiki(20 * 262144, seed=2), dict(mode="bit", de=True, block_size=262144, sub_blocks_per_block=16), "auto"),
    ("bit thread S16", datagen.nested(2_000_000, 8, seed=3), dict(mode="bit", de=True, block_size=65536, sub_block_seqs=16), "auto"),
    ("bit thread S16, long sub-blocks to one warp", datagen.nested(1_500_000, 1, seed=3), dict(mode="bit", de=True, block_size=262144, sub_block_seqs=16), "auto"),
    ("bit warp G=1 (~12 kbit sub-blocks)", datagen.wiki(40 * 65536, seed=2), dict(mode="bit", de=True, block_size=65536, sub_blocks_per_block=16), "auto"),
    ("byte MRR", datagen.nested(1_000_000, 8, seed=3), dict(mode="byte", de=False, block_size=65536), "mrr"),
    ("byte SC", datagen.nested(500_000, 8, seed=3), dict(mode="byte", de=False, block_size=65536), "sc"),
]
bad = 0
for name, x, kw, strat in cases:
    c = gomp.compress(x, **kw)
    y = gomp.decompress(c.cuda(), strategy=strat).cpu().numpy()
    ok = np.array_equal(y, x)
    bad += not ok
    print(name, gomp.get_info(c).n_blocks, "blocks", "ok" if ok else "MISMATCH", flush=True)
sys.exit(1 if bad else 0)
