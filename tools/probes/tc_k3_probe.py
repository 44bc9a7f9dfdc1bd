"""K3t alone on the cfg2 / cfg3 shapes: mean of 50 back-to-back launches (A/B of the epilogue variants,
  WINO_TC_EPW=1|2|4 python tools/probes/tc_k3_probe.py)."""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import tuning_env  # noqa: F401,E402
import paper_1803_10986_b200 as W  # noqa: E402

for name, (m, pts, N, C, K, H) in {"cfg2": (2, "0,1,-1,inf", 32, 128, 128, 28),
                                   "cfg3": (6, "0,-1,1,1/2,-1/2,2,-2,inf", 64, 256, 256, 28)}.items():
    ts = W.build_transforms(3, m, W.parse_points(pts))
    op = W.layer_op(ts, W.ConvConfig(), N, C, H, H, K, 1, contraction="tc_bf16")
    x = torch.rand((N, C, H, H), device="cuda") * 2 - 1
    w = torch.randn((K, C, 3, 3), device="cuda") * 0.05
    U, V = op.filter_transform(w), op.input_transform(x)
    for _ in range(5):
        M = op.contract(U, V)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        M = op.contract(U, V)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 50 * 1e3
    print(f"{name} epw={os.environ.get('WINO_TC_EPW', 'auto')}: K3t {us:.2f} us  {op.contraction_flops / us / 1e6:.1f} TFLOP/s")
