"""Contraction tile-config sweep on VGG-16 layer shapes (batch 256, F(6,3) P8, pairwise
exact): time of wino_contract per tuning "gemm" config, and M bit-equality with the
default config.   python tools/probes/contract_sweep.py "cfgA;cfgB;..." [layers]"""
import ctypes
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_1803_10986_b200 as W  # noqa: E402
from paper_1803_10986_b200 import _native  # noqa: E402
from paper_1803_10986_b200.stack import VGG16  # noqa: E402

cfgs = [c for c in sys.argv[1].split(";") if c] if len(sys.argv) > 1 else []
layers = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [2, 3, 6, 9, 12]
prec = os.environ.get("PROBE_PREC", "fp32")
cs = os.environ.get("PROBE_SUM", "pairwise")
N = int(os.environ.get("PROBE_N", "256"))
shapes, h = [], 224
for C, K, pool in VGG16:
    shapes.append((C, K, h))
    h = h // 2 if pool else h
lib = _native.lib()
s = torch.cuda.current_stream().cuda_stream
for li in layers:
    C, K, H = shapes[li - 1]
    x = torch.rand(N, C, H, H, device="cuda") * 2 - 1
    w = torch.randn(K, C, 3, 3, device="cuda") * 0.05
    ref = None
    for cfg in ["default"] + cfgs:
        _native.set_tuning("gemm", None if cfg == "default" else cfg)
        ts = W.build_transforms(3, 6, W.parse_points("0,-1,1,1/2,-1/2,2,-2,inf"))
        op = W.layer_op(ts, W.ConvConfig(prec, "huffman", cs), N, C, H, H, K, 1)
        L = op.layout
        U, V = op.filter_transform(w), op.input_transform(x)
        M = op.contract(U, V)
        sh = ctypes.byref(op.shape)
        for _ in range(2):
            _native.check(lib.wino_contract(op.plan.handle, sh, _native.as_ptr(U), _native.as_ptr(V),
                                            _native.as_ptr(M), s))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            _native.check(lib.wino_contract(op.plan.handle, sh, _native.as_ptr(U), _native.as_ptr(V),
                                            _native.as_ptr(M), s))
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        got = M[:, :K, :L.T].contiguous()
        same = True if ref is None else bool(torch.equal(got.view(torch.int32), ref.view(torch.int32)))
        if ref is None:
            ref = got.clone()
        print(f"layer {li} C{C} K{K} H{H} cfg={cfg} tile={L.bm}x{L.bn} ms={ms:.3f} "
              f"tflops={op.contraction_flops / (ms * 1e-3) / 1e12:.2f} bitwise={same}", flush=True)
        del U, V, M, got
    _native.set_tuning("gemm", None)
