"""K1 alone, K2 alone and the combined K1 + K2 launch on the cfg4 / cfg2 / cfg3 shapes (50 launches back to back)."""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import tuning_env  # noqa: F401,E402
import ctypes  # noqa: E402
import paper_1803_10986_b200 as W  # noqa: E402
from paper_1803_10986_b200 import _native  # noqa: E402


def t(fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for name, (r, m, pts, N, C, K, H, pad, cs) in {
        "cfg4": (5, 4, "0,1,-1,1/2,-1/2,2,-2,inf", 32, 512, 512, 14, 2, "pairwise"),
        "cfg2": (3, 2, "0,1,-1,inf", 32, 128, 128, 28, 1, "linear"),
        "cfg3": (3, 6, "0,-1,1,1/2,-1/2,2,-2,inf", 64, 256, 256, 28, 1, "linear")}.items():
    ts = W.build_transforms(r, m, W.parse_points(pts))
    op = W.layer_op(ts, W.ConvConfig("fp32", "huffman", cs), N, C, H, H, K, pad)
    L = op.layout
    x = torch.rand((N, C, H, H), device="cuda") * 2 - 1
    w = torch.randn((K, C, r, r), device="cuda") * 0.05
    U = torch.empty(L.u_bytes, dtype=torch.uint8, device="cuda")
    V = torch.empty(L.v_bytes, dtype=torch.uint8, device="cuda")
    lib, sh, s = _native.lib(), ctypes.byref(op.shape), torch.cuda.current_stream().cuda_stream
    k1 = t(lambda: _native.check(lib.wino_input_transform(op.plan.handle, sh, _native.as_ptr(x), _native.as_ptr(V), s)))
    k2 = t(lambda: _native.check(lib.wino_filter_transform(op.plan.handle, sh, _native.as_ptr(w), _native.as_ptr(U), s)))
    k12 = t(lambda: _native.check(lib.wino_transforms(op.plan.handle, sh, _native.as_ptr(x), _native.as_ptr(w),
                                                      _native.as_ptr(U), _native.as_ptr(V), s)))
    b1 = 4 * N * C * H * H + 4 * L.P * C * L.T
    b2 = 4 * K * C * r * r + 4 * L.P * C * K
    print(f"{name}: K1 {k1:.1f} us ({b1 / k1 / 1e3:.0f} GB/s)  K2 {k2:.1f} us ({b2 / k2 / 1e3:.0f} GB/s)  "
          f"K1+K2 one launch {k12:.1f} us ({(b1 + b2) / k12 / 1e3:.0f} GB/s)")
