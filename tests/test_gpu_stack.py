"""GPU parity of the conv stack (VGG-16 shape, BASELINE config 5) vs the oracle."""
import numpy as np
import pytest

import _golden as G
from oracle import wino_oracle as O

pytestmark = pytest.mark.gpu
W = pytest.importorskip("paper_1803_10986_b200")
torch = pytest.importorskip("torch")

P8 = "0,-1,1,1/2,-1/2,2,-2,inf"


def test_small_vgg_like_stack_bitwise():
    from paper_1803_10986_b200.stack import ConvStack, he_normal_weights
    layers = [(3, 16, False), (16, 16, True), (16, 32, False), (32, 32, True), (32, 40, False)]
    ts = W.build_transforms(3, 6, W.parse_points(P8))
    trip = O.Triple.from_points(3, 6, P8)
    N, H = 2, 30
    x = np.stack([O.synthetic((3, H, H), 5, i) for i in range(N)])
    ws = he_normal_weights(layers, 3, seed=11)
    st = ConvStack(ts, W.ConvConfig("fp32", "huffman", "pairwise"), layers, N, H)
    st.set_weights(ws)
    xt = torch.from_numpy(x).cuda()
    out = st.forward(xt).cpu().numpy()
    ref_outs, ref = O.stack_forward(trip, x, ws, layers)
    for i, y in enumerate(ref_outs):
        assert G.same_bits(st.conv_out[i].cpu().numpy(), y), i
    assert G.same_bits(out, ref)
    errs = st.layer_errors(xt)
    assert len(errs) == len(layers) and all(e["rel_l1"] < 1e-4 for e in errs)


def test_vgg16_geometry():
    from paper_1803_10986_b200.stack import VGG16, ConvStack
    ts = W.build_transforms(3, 6, W.parse_points(P8))
    st = ConvStack(ts, W.ConvConfig("fp32", "huffman", "pairwise"), VGG16, 1, 224)
    assert st.out_hw == (14, 14)
    assert abs(st.direct_flops * 256 - 7.86e12) / 7.86e12 < 0.01   # 7.86 TFLOP per batch-256
