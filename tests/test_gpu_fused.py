"""Fused exact K3 + K4 (wino_conv2d_fused: alpha^2 accumulators parked in tensor memory)
against the unfused layer path and the oracle, bit for bit."""
import numpy as np
import pytest

import _golden as G
from oracle import wino_oracle as O

pytestmark = pytest.mark.gpu
W = pytest.importorskip("paper_1803_10986_b200")
torch = pytest.importorskip("torch")

CASES = [
    # r, m, points, N, C, K, H, W, pad
    (3, 2, "0,1,-1,inf", 3, 33, 70, 15, 17, 1),        # odd sizes, K > one filter block, partial tiles
    (3, 2, "0,1,-1,inf", 4, 128, 128, 28, 28, 1),      # cfg2-like, several tile blocks
    (2, 3, "0,1,-1,inf", 2, 7, 9, 11, 11, 0),          # alpha = 4 with m = 3 (odd m: scalar stores)
    (2, 2, "0,1,inf", 2, 20, 5, 9, 10, 1),             # alpha = 3 (9 points)
    (3, 2, "0,1,-1,inf", 1, 1100, 3, 6, 6, 1),         # deep channel sums
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"r{c[0]}m{c[1]}C{c[4]}K{c[5]}")
@pytest.mark.parametrize("cs", ["linear", "pairwise"])
def test_fused_layer_vs_oracle_and_unfused(case, cs):
    r, m, pts, N, C, K, H, Wd, pad = case
    ts = W.build_transforms(r, m, W.parse_points(pts))
    trip = O.Triple.from_points(r, m, pts)
    x = O.synthetic((N, C, H, Wd), 21, 0)
    w = O.synthetic((K, C, r, r), 21, 1)
    cfg = W.ConvConfig("fp32", "huffman", cs)
    op = W.layer_op(ts, cfg, N, C, H, Wd, K, pad)
    assert op.fused_exact_supported
    xt, wt = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
    y = op.call_fused(xt, wt)
    want = O.layer_conv2d(trip, x, w, pad, "fp32", "huffman", cs)
    assert G.same_bits(y.cpu().numpy(), want)
    assert torch.equal(y.view(torch.int32), op(xt, wt).view(torch.int32))
    # activations: ReLU, and ReLU of the 2x2 max-pool for even m
    relu = O.relu_pool(want, False)
    assert G.same_bits(op.call_fused(xt, wt, mode=1).cpu().numpy(), relu)
    if m % 2 == 0:
        assert G.same_bits(op.call_fused(xt, wt, mode=2).cpu().numpy(), O.relu_pool(want, True))


def test_fused_is_refused_where_it_does_not_apply():
    import ctypes
    from paper_1803_10986_b200 import _native
    ts6 = W.build_transforms(3, 4, W.parse_points("0,1,-1,1/2,-1/2,inf"))     # alpha = 6: 36 points
    op = W.layer_op(ts6, W.ConvConfig(), 2, 8, 12, 12, 8, 1)
    assert not op.fused_exact_supported
    need = ctypes.c_size_t(0)
    rc = _native.lib().wino_fused_workspace(op.plan.handle, ctypes.byref(op.shape), ctypes.byref(need))
    assert rc != 0 and b"alpha^2 <= 16" in _native.lib().wino_last_error()
    ts = W.build_transforms(3, 2, W.parse_points("0,1,-1,inf"))
    assert not W.layer_op(ts, W.ConvConfig("mixed", "huffman", "linear"), 2, 8, 12, 12, 8, 1).fused_exact_supported
    assert not W.layer_op(ts, W.ConvConfig(), 2, 8, 12, 12, 8, 1, "tc_bf16").fused_exact_supported
    op2 = W.layer_op(ts, W.ConvConfig(), 2, 8, 12, 12, 8, 1)
    x = torch.zeros(2, 8, 12, 12, device="cuda")
    w = torch.zeros(8, 8, 3, 3, device="cuda")
    with pytest.raises(ValueError):
        op2.call_fused(x, w, mode=3)
