"""cfg2 contraction probe (F(2,3), N=32, C=K=128, 28², linear exact): wino_contract time
under the current WINO_GEMM override (PROBE_PREC / PROBE_SUM select the mode), x in L2-cold state not controlled (K3 alone)."""
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

N, C, K, H = 32, 128, 128, 28
ts = W.build_transforms(3, 2, W.parse_points("0,1,-1,inf"))
PREC, CS = os.environ.get("PROBE_PREC", "fp32"), os.environ.get("PROBE_SUM", "linear")
op = W.layer_op(ts, W.ConvConfig(PREC, "huffman", CS), N, C, H, H, K, 1)
x = torch.rand(N, C, H, H, device="cuda") * 2 - 1
w = torch.randn(K, C, 3, 3, device="cuda") * 0.2
U, V = op.filter_transform(w), op.input_transform(x)
M = op.contract(U, V)
lib = _native.lib()
s = torch.cuda.current_stream().cuda_stream
sh = ctypes.byref(op.shape)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ts_ = []
for i in range(23):
    flush.fill_(i)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _native.check(lib.wino_contract(op.plan.handle, sh, _native.as_ptr(U), _native.as_ptr(V), _native.as_ptr(M), s))
    e1.record()
    torch.cuda.synchronize()
    if i >= 3:
        ts_.append(e0.elapsed_time(e1))
ts_.sort()
L = op.layout
print(f"{PREC}/{CS} WINO_GEMM={os.environ.get('WINO_GEMM', 'default')} bm_bn={L.bm}x{L.bn} median_ms={ts_[len(ts_) // 2]:.4f} "
      f"min_ms={ts_[0]:.4f} tflops={op.contraction_flops / (ts_[len(ts_) // 2] * 1e-3) / 1e12:.1f}", flush=True)
