"""Write-bandwidth probe: how fast can HBM absorb pure writes of V-sized buffers?"""
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

for mb in (51, 105, 256, 1024):
    n = mb * 2**20 // 4
    x = torch.empty(n, device="cuda")
    y = torch.empty(n, device="cuda")
    us = t(lambda: x.fill_(1.0))
    us2 = t(lambda: y.copy_(x))
    print(f"{mb} MiB: fill {us:.1f} us = {n*4/us/1e3:.0f} GB/s ; copy {us2:.1f} us = {2*n*4/us2/1e3:.0f} GB/s (r+w)")
