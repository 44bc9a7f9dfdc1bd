"""HostPipeline end-to-end timing under different L2-flush preambles (cfg2)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import os as _os, sys as _sys  # noqa: E401
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import tuning_env  # noqa: E402,F401  (WINO_* env -> libwino tuning keys)
import paper_1803_10986_b200 as W
from paper_1803_10986_b200 import pointsets

N, C, H, K, pad = 32, 128, 28, 128, 1
ts = W.build_transforms(3, 2, W.parse_points(pointsets.curated_text(4, 2)))
cfg = W.ConvConfig()
rng = np.random.default_rng(0)
xh = torch.from_numpy(rng.random((N, C, H, H), dtype=np.float32) * 2 - 1).pin_memory()
wh = torch.from_numpy(rng.standard_normal((K, C, 3, 3), dtype=np.float32) * 0.04).pin_memory()
yh = torch.empty((N, K, H, H), dtype=torch.float32).pin_memory()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
clean = torch.ones(64 << 20, dtype=torch.float32, device="cuda")
for chunks, graph in ((4, False), (8, False), (4, True), (8, True), ([6, 5, 5, 4, 4, 3, 3, 2], True),
                      ([8, 7, 6, 5, 4, 2], True), (16, True)):
    pipe = W.HostPipeline(ts, cfg, N, C, H, H, K, pad, chunks=chunks, graph=graph)
    for _ in range(3):
        pipe(xh, wh, yh)
    torch.cuda.synchronize()
    for name, pre in (("none", lambda: None), ("zero", lambda: flush.zero_()),
                      ("zero+sum", lambda: (flush.zero_(), clean.sum()))):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts_ = []
        for _ in range(10):
            pre()
            e0.record()
            pipe(xh, wh, yh)
            e1.record()
            torch.cuda.synchronize()
            ts_.append(e0.elapsed_time(e1))
        print(f"chunks {chunks} graph {graph} flush {name:9s} e2e {np.mean(ts_)*1e3:.0f} us (min {np.min(ts_)*1e3:.0f})")
