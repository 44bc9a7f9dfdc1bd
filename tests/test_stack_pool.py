"""The process-parallel oracle driver (oracle/stack_pool.py, the VGG CPU baseline and
the checker of the full-size VGG parity test) is bit-identical to the plain oracle."""
import numpy as np

from oracle import wino_oracle as O
from oracle.stack_pool import OraclePool

P8 = "0,-1,1,1/2,-1/2,2,-2,inf"


def test_pool_layers_equal_plain_oracle():
    trip = O.Triple.from_points(3, 6, P8)
    layers = [(3, 8, False), (8, 20, True), (20, 33, False)]
    ws = [O.synthetic((K, C, 3, 3), 4, 100 + i) for i, (C, K, _) in enumerate(layers)]
    x = O.synthetic((2, 3, 37, 29), 4, 0)          # partial edge tiles in both directions
    with OraclePool(trip, ws, x.size * 40, procs=3) as pool:
        outs, act = pool.stack_forward(x, layers)
    ref_outs, ref = O.stack_forward(trip, x, ws, layers)
    for a, b in zip(outs, ref_outs):
        assert a.tobytes() == b.tobytes()
    assert act.tobytes() == ref.tobytes()


def test_pool_linear_sum_and_single_process():
    trip = O.Triple.from_points(3, 4, "0,1,-1,1/2,-1/2,inf")
    w = O.synthetic((40, 5, 3, 3), 6, 1)
    x = O.synthetic((3, 5, 26, 21), 6, 0)
    want = O.layer_conv2d(trip, x, w, 1, "fp32", "huffman", "linear")
    for procs in (1, 4):
        with OraclePool(trip, [w], x.size * 2, procs=procs) as pool:
            got = pool.layer(0, x, pad=1, csum="linear")
        assert got.tobytes() == want.tobytes(), procs
