"""VGG-16 layer 1 (N x 3 x 224 x 224 -> 64 filters, F(6x6,3x3), pairwise): K3 + K4act (M through HBM)
vs the fused small-C kernel (wino_contract_output_smallc).  Bitwise check + CUDA-event timing.
usage: [WINO_SC2_KG=k] python tools/probes/layer1_fused.py [N]"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1803_10986_b200 as W
from paper_1803_10986_b200 import _native

sys.path.insert(0, "tools")
import tuning_env  # noqa: E402,F401  (WINO_SC2_KG -> libwino tuning key)

N = int(sys.argv[1]) if len(sys.argv) > 1 else 256
P8 = "0,-1,1,1/2,-1/2,2,-2,inf"
ts = W.build_transforms(3, 6, W.parse_points(P8))
lib = _native.lib()
for (C, K, H, mode) in [(3, 64, 224, 1), (3, 64, 224, 2), (4, 64, 224, 1), (1, 32, 224, 1)]:
    op = W.layer_op(ts, W.ConvConfig("fp32", "huffman", "pairwise"), N, C, H, H, K, 1)
    op.prepare(_native.PREPARE_CONV | _native.PREPARE_ACT)
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.rand((N, C, H, H), device="cuda", generator=g) * 2 - 1
    w = torch.randn((K, C, 3, 3), device="cuda", generator=g) * 0.3
    U, V = op.filter_transform(w), op.input_transform(x)
    M = op.contract(U, V)
    s = torch.cuda.current_stream().cuda_stream
    Ho, Wo = op.layout.Ho, op.layout.Wo
    shp = (N, K, Ho // 2, Wo // 2) if mode == 2 else (N, K, Ho, Wo)
    want = torch.empty(shp, device="cuda")
    got = torch.full(shp, 7.0, device="cuda")
    sh = ctypes.byref(op.shape)

    def unfused():
        _native.check(lib.wino_contract(op.plan.handle, sh, _native.as_ptr(U), _native.as_ptr(V), _native.as_ptr(M), s))
        _native.check(lib.wino_output_transform_act(op.plan.handle, sh, _native.as_ptr(M), _native.as_ptr(want), mode - 1, s))

    def fused():
        _native.check(lib.wino_contract_output_smallc(op.plan.handle, sh, _native.as_ptr(U), _native.as_ptr(V),
                                                      _native.as_ptr(got), mode, s))

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
    same = torch.equal(got.view(torch.int32), want.view(torch.int32))
    L = op.layout
    print(f"C={C} K={K} H={H} N={N} mode={mode} tile {L.bm}x{L.bn}: K3+K4act {tu:.3f} ms, fused {tf:.3f} ms "
          f"({tu / tf:.2f}x), bitwise {same}", flush=True)
    del U, V, M, want, got, x
    torch.cuda.empty_cache()
