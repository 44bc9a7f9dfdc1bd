"""Stage times of a cfg2 layer at small batch (the e2e pipeline's chunks), alone."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import os as _os, sys as _sys  # noqa: E401
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import tuning_env  # noqa: E402,F401  (WINO_* env -> libwino tuning keys)
import paper_1803_10986_b200 as W
from paper_1803_10986_b200 import pointsets

ts = W.build_transforms(3, 2, W.parse_points(pointsets.curated_text(4, 2)))
for N in (4, 8, 16, 32):
    op = W.layer_op(ts, W.ConvConfig(), N, 128, 28, 28, 128, 1)
    x = torch.randn(N, 128, 28, 28, device="cuda")
    w = torch.randn(128, 128, 3, 3, device="cuda") * 0.04
    for _ in range(3):
        U = op.filter_transform(w); V = op.input_transform(x); M = op.contract(U, V); y = op.output_transform(M)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    res = []
    for rep in range(10):
        ev[0].record(); U = op.filter_transform(w); ev[1].record(); V = op.input_transform(x); ev[2].record()
        M = op.contract(U, V); ev[3].record(); y = op.output_transform(M); ev[4].record()
        torch.cuda.synchronize()
        res.append([ev[i].elapsed_time(ev[i + 1]) * 1e3 for i in range(4)])
    r = np.median(np.array(res), axis=0)
    print(f"N={N}: filter {r[0]:.1f} input {r[1]:.1f} contract {r[2]:.1f} output {r[3]:.1f} us")
