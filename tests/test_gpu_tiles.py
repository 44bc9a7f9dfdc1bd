"""Every contraction tile configuration a plan can pick (wino_host.cu cands: the
layout is chosen per layer shape) and the scalar (unpacked) form must give the
oracle's bits: the tile shape, stage depth and packed f32x2 arithmetic change
the schedule, never the per-output operation order.  The "gemm" tuning key
(wino_tuning_set) forces one config for plans created while it is set."""
import numpy as np
import pytest

from oracle import wino_oracle as O

pytestmark = pytest.mark.gpu
W = pytest.importorskip("paper_1803_10986_b200")

#            tm,tn,thm,thn,bk,stages,maxreg,ku,noprod,pack
LINEAR = ["8,8,16,8,16,4,0,16,0,1",    # 128 x 64 (default)
          "8,8,8,16,16,4,0,16,0,1",    # 64 x 128
          "4,8,16,8,16,4,0,16,0,1",    # 64 x 64
          "4,4,16,8,16,4,0,16,0,1",    # 64 x 32
          "8,8,16,8,8,4,0,8,0,1",      # 8-channel stages (C <= 8)
          "8,8,16,8,16,4,0,8,0,0"]     # scalar FMUL + FADD
PAIRWISE = ["4,4,16,16,64,2,168,8,0,1",  # default: 8 consumer warps, 64 x 64, 64-channel stages
            "4,4,16,16,32,3,168,8,0,1",  # 32-channel stages (C not a multiple of 64)
            "4,4,16,16,8,4,168,8,0,1",   # 8-channel stages
            "4,8,16,16,8,4,168,8,0,1",   # 8-channel stages, 64 x 128 (pairwise C <= 8 candidate)
            "4,4,8,16,32,4,168,8,0,1",   # 32 x 64
            "4,4,8,16,32,4,168,8,0,0"]   # scalar

CASES = [
    # r, m, points, N, C, K, H, W, pad
    (3, 2, "0,1,-1,inf", 3, 33, 70, 15, 17, 1),
    (3, 4, "0,1,-1,1/2,-1/2,inf", 2, 3, 24, 20, 20, 1),
    (3, 6, "0,-1,1,1/2,-1/2,2,-2,inf", 1, 70, 130, 29, 23, 1),
]


@pytest.mark.parametrize("cs,gemm", [("linear", g) for g in LINEAR] + [("pairwise", g) for g in PAIRWISE])
@pytest.mark.parametrize("prec", ["fp32", "mixed"])
def test_tile_config_bits(cs, gemm, prec, gemm_tuning):
    gemm_tuning(gemm)
    for r, m, pts, N, C, K, H, Wd, pad in CASES:
        ts = W.build_transforms(r, m, W.parse_points(pts))   # fresh plan cache
        trip = O.Triple.from_points(r, m, pts)
        x = O.synthetic((N, C, H, Wd), 5, 0)
        w = O.synthetic((K, C, r, r), 5, 1)
        y = W.conv2d_layer(ts, x, w, W.ConvConfig(prec, "huffman", cs), pad=pad)
        want = O.layer_conv2d(trip, x, w, pad, prec, "huffman", cs)
        assert y.dtype == want.dtype and y.tobytes() == want.tobytes(), (gemm, r, m, C, K)

