"""Dev helper (exp/btrace.so, -DGOMP_BATCH_TRACE): per-phase cycles of the LZ77 batch loop, block 0, C2 tokens."""
import sys, ctypes; sys.path.insert(0, '.')
import numpy as np, torch, bench
import paper_1606_00519_b200 as gomp
gomp.LIB_PATH = "exp/btrace.so"; gomp._lib = None
kind, n, seed, ckw = bench.CONFIGS["C2"][:4]
x = bench.gen(kind, n, seed)
c = gomp.compress(x, **ckw)
info = gomp.get_info(c)
d = c.cuda(); out = torch.empty(info.uncompressed_len, dtype=torch.uint8, device="cuda")
ws = torch.empty(gomp.workspace_size(info), dtype=torch.uint8, device="cuda")
L = gomp.lib(); L.gomp_debug_trace.restype = ctypes.c_int; L.gomp_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_uint32]
buf = np.zeros(1 << 22, np.uint32)
names = ["cpwait->scan+checks", "->syncthreads", "->flush+offsets", "litcopy", "nonInb copy", "chain wait", "inb+arrive+zero"]
for nb in [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "1,1024").split(",")]:
    gomp.decompress_into(info, d, out, ws, phase="decode", n_blocks=nb)
    L.gomp_debug_trace(buf.ctypes.data, 0)
    gomp.decompress_into(info, d, out, ws, phase="lz77", n_blocks=nb)
    m = L.gomp_debug_trace(buf.ctypes.data, 1 << 22)
    t = buf[:m].reshape(-1, 8).astype(np.int64)
    for w in range(4):
        tw = t[(t[:, 0] & 255) == w]
        print(nb, "blocks, warp", w, "batches", len(tw), {nm: int(np.median(tw[:, q + 1])) for q, nm in enumerate(names)},
              "sum", int(np.median(tw[:, 1:].sum(1))))
