import sys; sys.path.insert(0,'.')
import numpy as np, torch, datagen, paper_1606_00519_b200 as gomp
x = datagen.wiki(200_000, seed=1)
c = gomp.compress(x, mode="byte", de=True, block_size=65536)
for s in ("de", "mrr"):
    try:
        y = gomp.decompress(c.cuda(), strategy=s)
        yy = y.cpu().numpy(); bad = np.flatnonzero(yy != x)
        print(s, "equal", np.array_equal(yy, x), bad[:10], len(bad))
    except Exception as e:
        print(s, e)
