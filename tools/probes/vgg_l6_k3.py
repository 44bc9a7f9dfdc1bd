"""VGG-16 layer-6 contraction probe (C=K=256, 56², batch 256, F(6,3) pairwise exact):
wino_contract time under the current WINO_GEMM override."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, ".")
import os as _os, sys as _sys  # noqa: E401
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import tuning_env  # noqa: E402,F401  (WINO_* env -> libwino tuning keys)
import paper_1803_10986_b200 as W  # noqa: E402
from paper_1803_10986_b200 import _native  # noqa: E402

N, C, K, H = (int(v) for v in os.environ.get('PROBE_SHAPE', '256,256,256,56').split(','))
ts = W.build_transforms(3, 6, W.parse_points("0,-1,1,1/2,-1/2,2,-2,inf"))
op = W.layer_op(ts, W.ConvConfig("fp32", "huffman", "pairwise"), N, C, H, H, K, 1)
torch.manual_seed(7)
x = torch.rand(N, C, H, H, device="cuda") * 2 - 1
w = torch.randn(K, C, 3, 3, device="cuda") * 0.05
U, V = op.filter_transform(w), op.input_transform(x)
M = op.contract(U, V)
lib = _native.lib()
s = torch.cuda.current_stream().cuda_stream
sh = ctypes.byref(op.shape)
for _ in range(2):
    _native.check(lib.wino_contract(op.plan.handle, sh, _native.as_ptr(U), _native.as_ptr(V), _native.as_ptr(M), s))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    _native.check(lib.wino_contract(op.plan.handle, sh, _native.as_ptr(U), _native.as_ptr(V), _native.as_ptr(M), s))
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
L = op.layout
y = op.output_transform(M)
chk = int(y.view(torch.int32).to(torch.int64).sum().item())  # bitwise checksum: must not depend on the tile config
print(f"chk={chk:x} WINO_GEMM={os.environ.get('WINO_GEMM', 'default')} bm_bn={L.bm}x{L.bn} ms={ms:.3f} "
      f"tflops={op.contraction_flops / (ms * 1e-3) / 1e12:.2f}", flush=True)
