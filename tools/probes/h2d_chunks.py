"""H2D copy bandwidth vs chunking and concurrent streams (pinned host memory)."""
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
h = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
h.fill_(3)
d = torch.empty(nb, dtype=torch.uint8, device="cuda")
d2 = torch.empty(nb, dtype=torch.uint8, device="cuda")
h2 = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
streams = [torch.cuda.Stream() for _ in range(8)]

def chunked(nchunks, nstreams, d2h=False):
    cur = torch.cuda.current_stream()
    for s in streams[:nstreams]:
        s.wait_stream(cur)
    step = nb // nchunks
    for i in range(nchunks):
        s = streams[i % nstreams]
        with torch.cuda.stream(s):
            sl = slice(i * step, nb if i == nchunks - 1 else (i + 1) * step)
            d[sl].copy_(h[sl], non_blocking=True)
            if d2h:
                h2[sl].copy_(d2[sl], non_blocking=True)
    for s in streams[:nstreams]:
        cur.wait_stream(s)

for nc, ns in ((1, 1), (4, 1), (4, 2), (4, 4), (8, 4), (8, 8), (16, 8)):
    us = t(lambda: chunked(nc, ns))
    print(f"H2D {nc} chunks / {ns} streams: {us:.0f} us = {nb / us / 1e3:.1f} GB/s")
us = t(lambda: chunked(4, 4, True))
print(f"H2D+D2H 4 chunks / 4 streams: {us:.0f} us")
