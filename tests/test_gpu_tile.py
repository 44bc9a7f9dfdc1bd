"""GPU parity of the tile-level drop-in API (conv_2d, hadamard_2d, output_2d,
channel_reduce, conv_1d, conv_direct, pairwise_sum, dot_with_order, trial
draws, measure_error) against the reference's own outputs, bit for bit."""

from fractions import Fraction

import numpy as np
import pytest

import _golden as G
from oracle import wino_oracle as O

pytestmark = pytest.mark.gpu

W = pytest.importorskip("paper_1803_10986_b200")
torch = pytest.importorskip("torch")

TILE = G.cases("tile_cases.json")
F23 = None


def _ts(name):
    d = G.transforms()[name]
    return W.build_transforms(d["r"], d["m"], W.parse_points(d["points"]))


@pytest.mark.parametrize("case", TILE["cases"], ids=lambda c: c["name"])
def test_tile_api_golden(case):
    arr = G.npz("tile.npz")
    ts = _ts(case["ts"])
    nm = case["name"]
    h, x = arr[nm + "/h"], arr[nm + "/x"]
    assert G.same_bits(W.conv_direct(h, x, 2, "fp64", "linear"), arr[nm + "/direct64"])
    for prec, order, cs in TILE["modes"]:
        cfg = W.ConvConfig(prec, order, cs)
        key = f"{nm}/{prec}-{order}-{cs}"
        z = W.hadamard_2d(ts, h, x, cfg)
        assert G.same_bits(z, arr[key + "/z"])
        assert G.same_bits(W.output_2d(ts, W.channel_reduce(z, 2, cs), cfg), arr[key + "/y"])
        assert G.same_bits(W.conv_2d(ts, h, x, cfg), arr[key + "/y"])
        assert G.same_bits(W.conv_1d(ts, arr[nm + "/h1"], arr[nm + "/x1"], cfg), arr[key + "/y1"])


def test_trial_draws_golden():
    arr = G.npz("philox.npz")
    for key in arr:
        if key.endswith("/h"):
            seed, t, dims, n, C = (int(v) for v in key.split("/")[:5])
            h, x = W.trial_inputs(seed, t, dims, 3, n, C)
            assert G.same_bits(h, arr[key]) and G.same_bits(x, arr[key[:-1] + "x"])


def test_pairwise_sum_golden():
    arr = G.npz("tile.npz")
    for L in range(1, 71):
        s = W.pairwise_sum(arr[f"pw/{L}/v"], "fp32")
        assert G.same_bits(np.asarray(s), arr[f"pw/{L}/s"])
    assert W.pairwise_sum([1.0, 2.0, 3.0, 4.0], "fp32") == 10.0
    with pytest.raises(ValueError):
        W.pairwise_sum([], "fp32")


def test_halving_tree_equals_counter_many_lengths():
    rng = np.random.default_rng(5)
    for C in list(range(1, 70)) + [127, 128, 129, 255, 256, 1000, 4096]:
        z = rng.uniform(-1, 1, (C, 3, 5)).astype(np.float32)
        got = W.channel_reduce(z[None], 2, "pairwise")[0]
        assert G.same_bits(got, O.reduce_channels(z, 0, "pairwise")), C
        got = W.channel_reduce(z[None], 2, "linear")[0]
        assert G.same_bits(got, O.reduce_channels(z, 0, "linear")), C


def test_dot_with_order_matches_tree_eval():
    rng = np.random.default_rng(42)
    for _ in range(20):
        row = [Fraction(int(rng.integers(-8, 9)), int(rng.integers(1, 5))) for _ in range(6)]
        tree = W.huffman_order(row)
        if tree is None:
            continue
        x = rng.uniform(-1, 1, (4, 6)).astype(np.float32)
        got = W.dot_with_order(tree, x, "fp32")
        otree = O.huffman_tree(row)
        want = O._eval(otree, lambda j: x[..., j], "fp32")
        assert G.same_bits(np.asarray(got), np.asarray(want))
    assert W.dot_with_order(None, np.ones(3), "fp32") == 0.0


def test_reference_engine_properties():
    """Ports of reference test_engine.py properties onto the GPU path."""
    f23 = W.build_modified(3, 2, W.parse_points("0,1,-1,inf"))
    # zero input -> zero output in every mode (test_engine.py:184-190, 257-260)
    for prec in ("fp32", "fp64", "mixed"):
        for order in ("linear", "huffman"):
            out = W.conv_1d(f23, np.zeros(3, np.float32), np.zeros(4, np.float32), W.ConvConfig(prec, order))
            assert np.all(out == 0.0)
    out = W.conv_2d(f23, np.zeros((2, 3, 3)), np.zeros((2, 4, 4)), W.ConvConfig("mixed", channel_sum="pairwise"))
    assert np.all(out == 0.0)
    # exact channel cancellation (test_engine.py:192-198)
    h1 = np.array([0.3, -0.7, 0.2], dtype=np.float32)
    x1 = np.array([0.1, 0.5, -0.4, 0.9], dtype=np.float32)
    out = W.conv_1d(f23, np.stack([h1, -h1]), np.stack([x1, x1]), W.ConvConfig(channel_sum="linear"))
    assert np.all(out == 0.0)
    # mixed returns float64 (test_engine.py:223-226)
    hb, xb = W.trial_inputs(52, 0, 1, 3, 4)
    assert W.conv_1d(f23, hb, xb, W.ConvConfig(precision="mixed")).dtype == np.float64
    assert W.conv_1d(f23, hb, xb, W.ConvConfig(precision="fp32")).dtype == np.float32
    # batched == scalar (test_engine.py:215-221)
    pairs = [W.trial_inputs(51, t, 2, 3, 4, 3) for t in range(10)]
    hb = np.stack([p[0] for p in pairs])
    xb = np.stack([p[1] for p in pairs])
    out = W.conv_2d(f23, hb, xb)
    for t in range(10):
        assert G.same_bits(out[t], W.conv_2d(f23, hb[t], xb[t]))
    # point-order invariance under Huffman (test_engine.py:206-213), 2D
    base = W.build_transforms(3, 3, W.parse_points("0,-1,1,1/2,inf"))
    pairs = [W.trial_inputs(50, t, 2, 3, 5, 2) for t in range(50)]
    hb = np.stack([p[0] for p in pairs])
    xb = np.stack([p[1] for p in pairs])
    out0 = W.conv_2d(base, hb, xb)
    for ptxt in ("-1,1,0,1/2,inf", "1/2,1,-1,0,inf", "1,1/2,0,-1,inf"):
        assert G.same_bits(out0, W.conv_2d(W.build_transforms(3, 3, W.parse_points(ptxt)), hb, xb))
    # shape validation (test_engine.py:200-204)
    with pytest.raises(ValueError):
        W.conv_1d(f23, np.zeros(4), np.zeros(4))
    with pytest.raises(ValueError):
        W.conv_1d(f23, np.zeros((2, 3)), np.zeros((3, 4)))
    with pytest.raises(ValueError):
        W.conv_direct(np.zeros(5), np.zeros(3), 1)


ROWS = G.measure_rows()


@pytest.mark.parametrize("row", ROWS, ids=lambda r: f"{r['set']}-{r['precision']}-{r['dot_order']}-{r['channel_sum']}-C{r['channels']}")
def test_measure_error_golden_repr(row):
    """the reference's measure_error numbers, repr for repr."""
    if row["set"] == "direct":
        spec = W.DirectSpec(3, 1)
    elif row["set"].startswith("cur1d"):
        spec = W.curated_transform(int(row["set"].split("_n")[1]), 1, "fp32")
    else:
        spec = _ts(row["set"])
    rep = W.measure_error(spec, row["dims"], W.ConvConfig(row["precision"], row["dot_order"], row["channel_sum"]),
                          row["trials"], row["seed"], row["channels"])
    assert repr(rep.total_l1_mean) == row["total_l1_mean"]
    assert repr(rep.per_point_l1_mean) == row["per_point_l1_mean"]


def test_measure_per_trial_golden():
    arr = G.npz("measure_per_trial.npz")
    for key, want in arr.items():
        setname, prec, cs, C = key.split("/")
        rep = W.measure_error(_ts(setname), 2, W.ConvConfig(prec, "huffman", cs), 200, 0, int(C))
        assert G.same_bits(rep.per_trial, want), key
