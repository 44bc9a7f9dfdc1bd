"""Fused exact K3 + K4 (wino_conv2d_fused, accumulators parked in TMEM) vs the unfused layer
(K2+K1, K3, K4) on one layer shape, L2 flushed between steps.  PROBE_SHAPE=N,C,K,H  PROBE_SUM"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1803_10986_b200 as W  # noqa: E402

N, C, K, H = (int(v) for v in os.environ.get("PROBE_SHAPE", "32,128,128,28").split(","))
cs = os.environ.get("PROBE_SUM", "linear")
ts = W.build_transforms(3, 2, W.parse_points("0,1,-1,inf"))
op = W.layer_op(ts, W.ConvConfig("fp32", "huffman", cs), N, C, H, H, K, 1)
torch.manual_seed(3)
x = torch.rand(N, C, H, H, device="cuda") * 2 - 1
w = torch.randn(K, C, 3, 3, device="cuda") * 0.05
y0 = torch.empty(op.out_shape, device="cuda")
y1 = torch.empty(op.out_shape, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def t(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    g.replay()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / reps * 1e3


a = t(lambda: op(x, w, out=y0))
b = t(lambda: op.call_fused(x, w, out=y1))
assert torch.equal(y0.view(torch.int32), y1.view(torch.int32))
tf = op.direct_flops / 1e6
print(f"N={N} C={C} K={K} H={H} {cs}: unfused {a:.1f} us ({tf / a:.1f} TFLOP/s)  fused {b:.1f} us ({tf / b:.1f} TFLOP/s)  "
      f"{a / b:.3f}x, bitwise equal", flush=True)
