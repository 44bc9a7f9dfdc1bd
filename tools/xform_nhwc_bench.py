"""K1 / K4 alone: NCHW gather kernels vs the NHWC-native kernels vs NHWC through device
permutes (the pre-round-2 path), on one layer shape.  PROBE_SHAPE=N,C,K,H  PROBE_M=6"""
import ctypes
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1803_10986_b200 as W  # noqa: E402
from paper_1803_10986_b200 import _native  # noqa: E402
from paper_1803_10986_b200 import device as D  # noqa: E402

N, C, K, H = (int(v) for v in os.environ.get("PROBE_SHAPE", "64,256,256,28").split(","))
m = int(os.environ.get("PROBE_M", "6"))
pts = {2: "0,1,-1,inf", 4: "0,1,-1,1/2,-1/2,inf", 6: "0,-1,1,1/2,-1/2,2,-2,inf"}[m]
ts = W.build_transforms(3, m, W.parse_points(pts))
cfg = W.ConvConfig("fp32", "huffman", os.environ.get("PROBE_SUM", "linear"))
op = W.layer_op(ts, cfg, N, C, H, H, K, 1)
op.prepare(_native.PREPARE_STAGES | _native.PREPARE_NHWC)
L = op.layout
lib = _native.lib()
torch.manual_seed(1)
x = torch.rand(N, C, H, H, device="cuda") * 2 - 1
w = torch.randn(K, C, 3, 3, device="cuda") * 0.05
xh = x.permute(0, 2, 3, 1).contiguous()
V = op.input_transform(x)
M = op.contract(op.filter_transform(w), V)
y = op.output_transform(M)
yh = torch.empty(N, L.Ho, L.Wo, K, device="cuda")
V2 = torch.empty_like(V)
sh = ctypes.byref(op.shape)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def t(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / reps * 1e3


s = D.stream_handle()
k1 = t(lambda: _native.check(lib.wino_input_transform(op.plan.handle, sh, D.ptr(x), D.ptr(V2), s)))
k1h = t(lambda: _native.check(lib.wino_input_transform_nhwc(op.plan.handle, sh, D.ptr(xh), D.ptr(V2), s)))
assert torch.equal(V.view(torch.int32), V2.view(torch.int32))
k1p = t(lambda: _native.check(lib.wino_input_transform(op.plan.handle, sh, D.ptr(xh.permute(0, 3, 1, 2).contiguous()),
                                                       D.ptr(V2), s)))
k4 = t(lambda: _native.check(lib.wino_output_transform(op.plan.handle, sh, D.ptr(M), D.ptr(y), s)))
k4h = t(lambda: _native.check(lib.wino_output_transform_nhwc(op.plan.handle, sh, D.ptr(M), D.ptr(yh), s)))
assert torch.equal(y.view(torch.int32), yh.permute(0, 3, 1, 2).contiguous().view(torch.int32))
y_tmp = torch.empty_like(y)


def k4_perm():
    _native.check(lib.wino_output_transform(op.plan.handle, sh, D.ptr(M), D.ptr(y_tmp), s))
    yh.copy_(y_tmp.permute(0, 2, 3, 1))


k4p = t(k4_perm)
yn = torch.empty_like(y)
full = t(lambda: op(x, w, out=yn))
fullh = t(lambda: op.call_nhwc(xh, w, out=yh))
assert torch.equal(yn.view(torch.int32), yh.permute(0, 3, 1, 2).contiguous().view(torch.int32))


def full_perm():
    op(xh.permute(0, 3, 1, 2).contiguous(), w, out=yn)
    yh.copy_(yn.permute(0, 2, 3, 1))


fullp = t(full_perm)
tf = op.direct_flops / 1e6
print(f"  whole layer (K2 K1 K3 K4): NCHW {full:.1f} us ({tf / full:.1f} TFLOP/s)  NHWC native {fullh:.1f} us "
      f"({tf / fullh:.1f} TFLOP/s)  NHWC via permutes {fullp:.1f} us ({tf / fullp:.1f} TFLOP/s)", flush=True)
b1 = x.numel() * 4 + L.v_bytes
b4 = L.m_bytes + y.numel() * 4
print(f"N={N} C={C} K={K} H={H} m={m}:  K1 NCHW {k1:.1f} us ({b1 / k1 / 1e6:.2f} TB/s)  NHWC native {k1h:.1f} us "
      f"({b1 / k1h / 1e6:.2f} TB/s)  NHWC via permute {k1p:.1f} us | K4 NCHW {k4:.1f} us ({b4 / k4 / 1e6:.2f} TB/s)  "
      f"NHWC native {k4h:.1f} us ({b4 / k4h / 1e6:.2f} TB/s)  NHWC via permute {k4p:.1f} us", flush=True)
