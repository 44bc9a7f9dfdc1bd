"""Pinned host<->device copy bandwidth, alone and concurrent (the e2e floor)."""
import torch

def t(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3

nb = 13434880
h = torch.empty(nb, dtype=torch.uint8).pin_memory()
h2 = torch.empty(nb, dtype=torch.uint8).pin_memory()
d = torch.empty(nb, dtype=torch.uint8, device="cuda")
d2 = torch.empty(nb, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
h2d = t(lambda: d.copy_(h, non_blocking=True))
d2h = t(lambda: h2.copy_(d2, non_blocking=True))

def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)
bo = t(both)
print(f"H2D {h2d:.1f} us = {nb/h2d/1e3:.1f} GB/s; D2H {d2h:.1f} us = {nb/d2h/1e3:.1f} GB/s; both {bo:.1f} us = {2*nb/bo/1e3:.1f} GB/s")
