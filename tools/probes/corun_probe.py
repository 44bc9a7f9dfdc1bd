"""Do the contraction (K3) and a transform kernel (K1+K2 or K4+act) of ANOTHER image chunk
really run at the same time on one GPU?  VGG-16 layer `PROBE_LAYER` (default 9), N images
per chunk: times K3 alone, K1 / K4 alone, and K3 on stream A with K1+K4 of a second stack on
stream B, with per-kernel start/end events placed on a common timeline."""
import ctypes
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import tuning_env  # noqa: E402,F401  (WINO_* env -> libwino tuning keys)
import paper_1803_10986_b200 as W  # noqa: E402
from paper_1803_10986_b200 import _native  # noqa: E402
from paper_1803_10986_b200 import device as D  # noqa: E402
from paper_1803_10986_b200.stack import VGG16, ConvStack, he_normal_weights  # noqa: E402

N = int(os.environ.get("PROBE_N", "128"))
LI = int(os.environ.get("PROBE_LAYER", "9")) - 1
ts = W.build_transforms(3, 6, W.parse_points("0,-1,1,1/2,-1/2,2,-2,inf"))
cfg = W.ConvConfig("fp32", "huffman", "pairwise")
lib = _native.lib()
C, K, _ = VGG16[LI]
H = 224
for (_, _, pool) in VGG16[:LI]:
    H = H // 2 if pool else H
layers = [(C, K, False)]
ws = he_normal_weights(layers, 3)
sa = ConvStack(ts, cfg, layers, N, H)
sb = ConvStack(ts, cfg, layers, N, H)
sa.set_weights(ws)
sb.share_weights(sa)
xa = torch.rand(N, C, H, H, device="cuda")
xb = torch.rand(N, C, H, H, device="cuda")
A, B = torch.cuda.Stream(priority=-1), torch.cuda.Stream(priority=0)


def k1(st, x, s):
    op = st.ops[0]
    U, V, M = st._uvm(op.layout)
    _native.check(lib.wino_transforms(op.plan.handle, ctypes.byref(op.shape), D.ptr(x), D.ptr(st.weights[0]),
                                      ctypes.c_void_p(U), ctypes.c_void_p(V), s.cuda_stream), "K1")


def k3(st, s):
    op = st.ops[0]
    U, V, M = st._uvm(op.layout)
    _native.check(lib.wino_contract(op.plan.handle, ctypes.byref(op.shape), ctypes.c_void_p(U), ctypes.c_void_p(V),
                                    ctypes.c_void_p(M), s.cuda_stream), "K3")


def k4(st, s):
    op = st.ops[0]
    U, V, M = st._uvm(op.layout)
    _native.check(lib.wino_output_transform_act(op.plan.handle, ctypes.byref(op.shape), ctypes.c_void_p(M),
                                                D.ptr(st.act[0]), 0, s.cuda_stream), "K4")


def ev():
    return torch.cuda.Event(enable_timing=True)


def alone(fn, s, reps=5):
    with torch.cuda.stream(s):
        fn()
        torch.cuda.synchronize()
        e0, e1 = ev(), ev()
        e0.record(s)
        for _ in range(reps):
            fn()
        e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for st, x_ in ((sa, xa), (sb, xb)):
    k1(st, x_, A)
    k3(st, A)
    k4(st, A)
torch.cuda.synchronize()
t3 = alone(lambda: k3(sa, A), A)
t1 = alone(lambda: k1(sb, xb, B), B)
t4 = alone(lambda: k4(sb, B), B)
print(f"layer {LI + 1} N={N}: alone K3 {t3:.3f} ms, K1+K2 {t1:.3f} ms, K4+act {t4:.3f} ms", flush=True)

for order in ("k3_first", "xf_first"):
    base = ev()
    e = [ev() for _ in range(6)]
    torch.cuda.synchronize()
    cur = torch.cuda.current_stream()
    base.record(cur)
    A.wait_stream(cur)
    B.wait_stream(cur)

    def run_a():
        with torch.cuda.stream(A):
            e[0].record(A)
            k3(sa, A)
            e[1].record(A)

    def run_b():
        with torch.cuda.stream(B):
            e[2].record(B)
            k4(sb, B)
            e[3].record(B)
            k1(sb, xb, B)
            e[4].record(B)

    if order == "k3_first":
        run_a()
        run_b()
    else:
        run_b()
        run_a()
    cur.wait_stream(A)
    cur.wait_stream(B)
    e[5].record(cur)
    torch.cuda.synchronize()
    tl = [base.elapsed_time(x_) for x_ in e]
    print(f"{order}: K3 [{tl[0]:.3f}, {tl[1]:.3f}]  K4 [{tl[2]:.3f}, {tl[3]:.3f}]  K1 [{tl[3]:.3f}, {tl[4]:.3f}]  "
          f"all done {tl[5]:.3f} ms (serial sum {t3 + t1 + t4:.3f})", flush=True)
