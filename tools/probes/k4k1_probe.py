"""K4(i) + activation + K1(i+1) fused (wino_output_input_transform) vs the two kernels, VGG-16 layer pairs.
usage: [WINO_K4K1_KS=k] python tools/probes/k4k1_probe.py [N]"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
import tuning_env  # noqa: E402,F401
import paper_1803_10986_b200 as W
from paper_1803_10986_b200 import _native

N = int(sys.argv[1]) if len(sys.argv) > 1 else 256
ts = W.build_transforms(3, 6, W.parse_points("0,-1,1,1/2,-1/2,2,-2,inf"))
cfg = W.ConvConfig("fp32", "huffman", "pairwise")
lib = _native.lib()
s = torch.cuda.current_stream().cuda_stream
for (C, K, H, pool, K2) in [(64, 64, 224, 1, 128), (64, 128, 112, 0, 128), (128, 128, 112, 1, 256), (256, 256, 56, 0, 256),
                            (256, 256, 56, 1, 512), (512, 512, 28, 0, 512), (512, 512, 28, 1, 512), (512, 512, 14, 0, 512)]:
    op = W.layer_op(ts, cfg, N, C, H, H, K, 1)
    op.prepare(_native.PREPARE_ACT)
    Ho = op.layout.Ho
    H2 = Ho // 2 if pool else Ho
    nxt = W.layer_op(ts, cfg, N, K, H2, H2, K2, 1)
    nxt.prepare(_native.PREPARE_K4K1 | _native.PREPARE_STAGES)
    L, L2 = op.layout, nxt.layout
    M = torch.randn(L.m_bytes // 4, device="cuda")
    act = torch.empty((N, K, H2, H2), device="cuda")
    Va = torch.empty(L2.v_bytes // 4, device="cuda")
    Vb = torch.full((L2.v_bytes // 4,), 7.0, device="cuda")
    sh, sh2 = ctypes.byref(op.shape), ctypes.byref(nxt.shape)

    def unfused():
        _native.check(lib.wino_output_transform_act(op.plan.handle, sh, _native.as_ptr(M), _native.as_ptr(act), pool, s))
        _native.check(lib.wino_input_transform(nxt.plan.handle, sh2, _native.as_ptr(act), _native.as_ptr(Va), s))

    def fused():
        _native.check(lib.wino_output_input_transform(op.plan.handle, sh, _native.as_ptr(M), pool, sh2, _native.as_ptr(Vb), s))

    def timeit(f, reps=10):
        for _ in range(3):
            f()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
        e[0].record()
        for i in range(reps):
            f()
            e[i + 1].record()
        torch.cuda.synchronize()
        return float(np.median([e[i].elapsed_time(e[i + 1]) for i in range(reps)]))

    tu, tf = timeit(unfused), timeit(fused)
    same = torch.equal(Va.view(torch.int32), Vb.view(torch.int32))
    gb = (4 * L.P * K * L.T + 4 * L2.P * K * L2.T) / 1e9
    print(f"C={C} K={K} H={H} pool={pool}: K4act + K1 {tu:.3f} ms, fused {tf:.3f} ms ({tu / tf:.2f}x, "
          f"{gb / tf:.2f} TB/s), bitwise {same}", flush=True)
    del M, act, Va, Vb
    torch.cuda.empty_cache()
