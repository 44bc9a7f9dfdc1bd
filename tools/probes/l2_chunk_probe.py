"""L2 blocking of one VGG-16 layer: run the batch as chunks of n images (K1 -> K3 -> K4+act
per chunk, U transformed once) so that a chunk's V and M (P x C x tiles x 4 B each) stay in
the 126 MB L2 between the kernels instead of making the HBM round trip.  Prints ms per
256-image layer for each chunk size (CUDA-graph replay) and checks bitwise equality."""
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
from paper_1803_10986_b200.stack import VGG16  # noqa: E402

N = int(os.environ.get("PROBE_N", "256"))
layers = [int(v) for v in os.environ.get("PROBE_LAYERS", "2,4,6,9").split(",")]
sizes = [int(v) for v in os.environ.get("PROBE_CHUNKS", "256,16,8,4,2,1").split(",")]
ts = W.build_transforms(3, 6, W.parse_points("0,-1,1,1/2,-1/2,2,-2,inf"))
cfg = W.ConvConfig("fp32", "huffman", "pairwise")
MODE = os.environ.get("PROBE_MODE", "exact")  # tc_bf16 / tc_fp16: the HBM-bound tensor-core contraction
lib = _native.lib()
s = torch.cuda.current_stream().cuda_stream

for layer in layers:
    C, K, pool = VGG16[layer - 1]
    H = 224
    for (_, _, p_) in VGG16[:layer - 1]:
        H = H // 2 if p_ else H
    torch.manual_seed(layer)
    x = torch.rand(N, C, H, H, device="cuda")
    w = torch.randn(K, C, 3, 3, device="cuda") * (2.0 / (9 * C)) ** 0.5
    ref = None
    for n in sizes:
        if n > N:
            continue
        op = W.layer_op(ts, cfg, n, C, H, H, K, 1, MODE)
        if not op.tensor_core:
            op.prepare(_native.PREPARE_CONV | _native.PREPARE_ACT | _native.PREPARE_STAGES)
        L = op.layout
        U = op.filter_transform(w)
        V = torch.empty(L.v_bytes, dtype=torch.uint8, device="cuda")
        M = torch.empty(L.m_bytes, dtype=torch.uint8, device="cuda")
        Ho = L.Ho // 2 if pool else L.Ho
        act = torch.empty(N, K, Ho, Ho, device="cuda")
        sh = ctypes.byref(op.shape)

        def run():
            s = torch.cuda.current_stream().cuda_stream
            for a in range(0, N, n):
                _native.check(lib.wino_input_transform(op.plan.handle, sh, D.ptr(x[a:a + n]), D.ptr(V), s), "K1")
                _native.check(lib.wino_contract(op.plan.handle, sh, D.ptr(U), D.ptr(V), D.ptr(M), s), "K3")
                _native.check(lib.wino_output_transform_act(op.plan.handle, sh, D.ptr(M), D.ptr(act[a:a + n]),
                                                            1 if pool else 0, s), "K4")

        run()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            run()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        if ref is None:
            ref = act.clone()
        same = bool(torch.equal(act.view(torch.int32), ref.view(torch.int32)))
        print(f"layer {layer} (C={C} K={K} H={H}) chunk {n:3d}: {ms:7.3f} ms  V+M per chunk "
              f"{(L.v_bytes + L.m_bytes) / 1e6:7.1f} MB  tile {L.bm}x{L.bn}  bitwise={same}", flush=True)
        del g, V, M, U
