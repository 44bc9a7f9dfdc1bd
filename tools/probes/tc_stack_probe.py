"""Per-layer stage times of the VGG-16 stack in a tensor-core mode (K1+K2 | K3t | K4+act).
  WINO_K1TC_STAGED=0 python tools/probes/tc_stack_probe.py [tc_bf16] [batch]   (A/B of the staged K1)"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import tuning_env  # noqa: F401,E402
import paper_1803_10986_b200 as W  # noqa: E402
from paper_1803_10986_b200.stack import VGG16, ConvStack, he_normal_weights  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "tc_bf16"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
ts = W.build_transforms(3, 6, W.parse_points("0,-1,1,1/2,-1/2,2,-2,inf"))
st = ConvStack(ts, W.ConvConfig("fp32", "huffman", "pairwise"), VGG16, n, 224, contraction=mode)
st.set_weights(he_normal_weights(VGG16, 3))
x = (torch.rand((n, 3, 224, 224), device="cuda") * 2 - 1)
for _ in range(2):
    st.forward(x)
torch.cuda.synchronize()
tot = np.zeros(3)
cur = x
for i in range(len(st.ops)):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    cur = st.layer_forward(i, cur, events=ev)
    torch.cuda.synchronize()
    t = np.array([ev[j].elapsed_time(ev[j + 1]) for j in range(3)])
    tot += t
    C, K, h, w, pool = st.shapes[i]
    print(f"layer {i + 1:2d} C={C:3d} K={K:3d} H={h:3d} pool={int(pool)}  K1+K2 {t[0]:7.3f}  K3 {t[1]:7.3f}  K4+act {t[2]:7.3f} ms")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    st.forward(x)
e1.record()
torch.cuda.synchronize()
print(f"{mode} batch {n} staged={os.environ.get('WINO_K1TC_STAGED', '1')}: K1+K2 {tot[0]:.3f}  K3 {tot[1]:.3f}  K4+act {tot[2]:.3f}  "
      f"forward {e0.elapsed_time(e1) / 5:.3f} ms  ({st.direct_flops / (e0.elapsed_time(e1) / 5 * 1e-3) / 1e12:.1f} TFLOP/s direct-eq)")
