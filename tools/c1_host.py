"""Dev helper: where C1's single-launch latency goes (Python binding, C enqueue, kernel, synchronise)."""
import sys, time, statistics, ctypes
sys.path.insert(0, '.')
import torch, datagen, paper_1606_00519_b200 as gomp
x = datagen.text(1 << 20, seed=1)
c = gomp.compress(x, mode="byte", de=True, block_size=65536)
info = gomp.get_info(c)
d = c.cuda(); out = torch.empty(info.uncompressed_len, dtype=torch.uint8, device="cuda")
ws = torch.empty(gomp.workspace_size(info), dtype=torch.uint8, device="cuda")
L = gomp.lib()
args = (ctypes.byref(info), 0, info.n_blocks, d.data_ptr(), d.numel(), out.data_ptr(), out.numel(), ws.data_ptr(),
        ws.numel(), 0, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
def med(f, n=40):
    ts = []
    for i in range(n):
        torch.cuda.synchronize()
        t0 = time.perf_counter(); f(); t1 = time.perf_counter()
        ts.append((t1 - t0) * 1e6)
    return round(statistics.median(ts[5:]), 1)
r = {}
r["py_call_enqueue_only"] = med(lambda: gomp.decompress_into(info, d, out, ws))
r["py_call_plus_sync"] = med(lambda: (gomp.decompress_into(info, d, out, ws), torch.cuda.synchronize()))
r["c_call_enqueue_only"] = med(lambda: L.gomp_decompress_blocks(*args))
r["c_call_plus_sync"] = med(lambda: (L.gomp_decompress_blocks(*args), torch.cuda.synchronize()))
r["empty_sync"] = med(lambda: torch.cuda.synchronize())
ev = []
for _ in range(20):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); L.gomp_decompress_blocks(*args); b.record(); torch.cuda.synchronize()
    ev.append(a.elapsed_time(b) * 1e3)
r["events_us"] = round(statistics.median(ev[3:]), 1)
print(r)
