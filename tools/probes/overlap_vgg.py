"""VGG-16 forward (batch 256) as `chunks` image chunks on `chunks` streams, issued layer
by layer round-robin so one chunk's HBM-bound transforms overlap another chunk's
FP32-bound contraction.  Times the multi-stream forward (CUDA graph) against the
one-stream forward and checks the final activations are bitwise equal."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_1803_10986_b200 as W  # noqa: E402
from paper_1803_10986_b200.stack import VGG16, ConvStack, he_normal_weights  # noqa: E402

N = int(os.environ.get("PROBE_N", "256"))
ts = W.build_transforms(3, 6, W.parse_points("0,-1,1,1/2,-1/2,2,-2,inf"))
cfg = W.ConvConfig("fp32", "huffman", "pairwise")
ws = he_normal_weights(VGG16, 3)
x = torch.rand(N, 3, 224, 224, device="cuda") * 2 - 1


def timed(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


full = ConvStack(ts, cfg, VGG16, N, 224)
full.set_weights(ws)
t1 = timed(lambda: full.forward(x))
ref = full.act[-1].clone()
print(f"one stream: {t1:.2f} ms", flush=True)
for chunks in (2, 4):
    n = N // chunks
    sts = [ConvStack(ts, cfg, VGG16, n, 224) for _ in range(chunks)]
    for st in sts:
        st.share_weights(full)
    streams = [torch.cuda.Stream() for _ in range(chunks)]

    def fwd():
        cur = torch.cuda.current_stream()
        acts = [x[i * n:(i + 1) * n] for i in range(chunks)]
        for s in streams:
            s.wait_stream(cur)
        for li in range(len(VGG16)):
            for i, (st, s) in enumerate(zip(sts, streams)):
                with torch.cuda.stream(s):
                    acts[i] = st.layer_forward(li, acts[i], stream=s.cuda_stream)
        for s in streams:
            cur.wait_stream(s)

    t = timed(fwd)
    out = torch.cat([st.act[-1] for st in sts])
    same = bool(torch.equal(out.view(torch.int32), ref.view(torch.int32)))
    print(f"{chunks} chunks x {n} images on {chunks} streams: {t:.2f} ms ({t1 / t:.3f}x), bitwise={same}", flush=True)
    del sts
