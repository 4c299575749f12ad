"""Dev helper: host link ceiling for the e2e path: H2D of the compressed C2 file and D2H of its output, alone and concurrently."""
import torch
C, U = 99225968, 268435456
hs, hd = torch.empty(C, dtype=torch.uint8, pin_memory=True), torch.empty(U, dtype=torch.uint8, pin_memory=True)
ds, dd = torch.empty(C, dtype=torch.uint8, device="cuda"), torch.empty(U, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(h2d, d2h):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    s1.wait_event(a); s2.wait_event(a)
    if h2d:
        with torch.cuda.stream(s1): ds.copy_(hs, non_blocking=True)
    if d2h:
        with torch.cuda.stream(s2): hd.copy_(dd, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b)
for _ in range(2): run(1, 1)
for name, h, d in (("h2d C", 1, 0), ("d2h U", 0, 1), ("both", 1, 1)):
    t = min(run(h, d) for _ in range(5))
    print(name, round(t, 3), "ms", "-> U/t", round(U / t / 1e6, 1), "GB/s")
