"""VGG-16 forward (batch 256) as image chunks whose contractions (K3, FP32-pipe bound) run on
HIGH-priority streams and whose transforms (K1+K2, K4+act, HBM bound) run on LOW-priority
streams, so the block scheduler places a pending contraction CTA before the other chunk's
transform blocks and the transforms fill the SM resources the contraction leaves free.
Times the CUDA-graph replay against the one-stream forward; checks bitwise equality."""
import ctypes
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import tuning_env  # noqa: E402,F401
import paper_1803_10986_b200 as W  # noqa: E402
from paper_1803_10986_b200 import _native  # noqa: E402
from paper_1803_10986_b200 import device as D  # noqa: E402
from paper_1803_10986_b200.stack import VGG16, ConvStack, he_normal_weights  # noqa: E402

N = int(os.environ.get("PROBE_N", "256"))
GRAPH = os.environ.get("PROBE_GRAPH", "1") == "1"
ts = W.build_transforms(3, 6, W.parse_points("0,-1,1,1/2,-1/2,2,-2,inf"))
cfg = W.ConvConfig("fp32", "huffman", "pairwise")
ws = he_normal_weights(VGG16, 3)
x = torch.rand(N, 3, 224, 224, device="cuda") * 2 - 1
lib = _native.lib()


def timed(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    if GRAPH:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        run = g.replay
    else:
        run = fn
    run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        run()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


full = ConvStack(ts, cfg, VGG16, N, 224)
full.set_weights(ws)
t1 = timed(lambda: full.forward(x))
ref = full.act[-1].clone()
print(f"one stream: {t1:.2f} ms", flush=True)
lo_p, hi_p = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else (0, -1)
print("priority range", lo_p, hi_p, flush=True)

for chunks, mode in ((2, "prio"), (2, "flat"), (4, "prio")):
    n = N // chunks
    sts = [ConvStack(ts, cfg, VGG16, n, 224) for _ in range(chunks)]
    for st in sts:
        st.share_weights(full)
    hi = [torch.cuda.Stream(priority=hi_p if mode == "prio" else 0) for _ in range(chunks)]
    lo = [torch.cuda.Stream(priority=lo_p if mode == "prio" else 0) for _ in range(chunks)]

    def layer(st, i, cur, s_lo, s_hi):
        op = st.ops[i]
        pool = st.shapes[i][4]
        sh = ctypes.byref(op.shape)
        U, V, M = st._uvm(op.layout)
        _native.check(lib.wino_transforms(op.plan.handle, sh, D.ptr(cur), D.ptr(st.weights[i]), ctypes.c_void_p(U),
                                          ctypes.c_void_p(V), s_lo.cuda_stream), "K1")
        s_hi.wait_stream(s_lo)
        _native.check(lib.wino_contract(op.plan.handle, sh, ctypes.c_void_p(U), ctypes.c_void_p(V),
                                        ctypes.c_void_p(M), s_hi.cuda_stream), "K3")
        s_lo.wait_stream(s_hi)
        _native.check(lib.wino_output_transform_act(op.plan.handle, sh, ctypes.c_void_p(M), D.ptr(st.act[i]),
                                                    1 if pool else 0, s_lo.cuda_stream), "K4")
        return st.act[i]

    def fwd():
        cur = torch.cuda.current_stream()
        acts = [x[i * n:(i + 1) * n] for i in range(chunks)]
        for s in lo + hi:
            s.wait_stream(cur)
        for li in range(len(VGG16)):
            for i in range(chunks):
                acts[i] = layer(sts[i], li, acts[i], lo[i], hi[i])
        for s in lo + hi:
            cur.wait_stream(s)

    t = timed(fwd)
    out = torch.cat([st.act[-1] for st in sts])
    same = bool(torch.equal(out.view(torch.int32), ref.view(torch.int32)))
    print(f"{mode}: {chunks} chunks x {n} images: {t:.2f} ms ({t1 / t:.3f}x), bitwise={same}", flush=True)
    del sts
