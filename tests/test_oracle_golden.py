"""Pin the CPU oracle (oracle/wino_oracle.py) against golden vectors produced by
the reference toolkit itself (tests/golden/make_golden.py), and -- when the
reference is mounted -- directly against it on fresh inputs."""

import sys
from fractions import Fraction

import numpy as np
import pytest

from _golden import REFERENCE_SRC, reference_available
from oracle import wino_oracle as O
import _golden as G

SPECS = sorted(G.transforms())


def trip_for(name):
    d = G.transforms()[name]
    return O.Triple.from_points(d["r"], d["m"], d["points"])


@pytest.mark.parametrize("name", SPECS)
def test_matrices_rounding_and_trees(name):
    d = G.transforms()[name]
    t = trip_for(name)
    assert [("inf" if p is None else str(p)) for p in t.points] == d["ordered_points"]
    for mat in ("A_T", "G", "B_T"):
        assert t.mats[mat] == [[Fraction(v) for v in row] for row in d[mat]]
        for fmt in ("fp32", "fp64"):
            got = np.array([[O.round_fraction(v, fmt) for v in row] for row in t.mats[mat]],
                           dtype=np.float32 if fmt == "fp32" else np.float64)
            bits = [format(int(v), "x") for v in got.view(np.uint32 if fmt == "fp32" else np.uint64).ravel()]
            assert bits == d[f"{mat}_{fmt}_bits"], (mat, fmt)
        for order in ("huffman", "linear"):
            want = [G.tree_from_json(x) for x in d[f"trees/{mat}/{order}"]]
            assert t.trees(mat, order) == want, (mat, order)


def test_round_fraction_edge_cases():
    # ties to even, subnormals, overflow threshold (reference exact.py:23-28, 61-91)
    assert O.round_fraction(Fraction(1, 3), "fp32") == np.float32(1 / 3)
    assert O.round_fraction(Fraction(2**24 + 1), "fp32") == np.float32(2**24)
    assert O.round_fraction(Fraction(2**24 + 3), "fp32") == np.float32(2**24 + 4)
    tiny = Fraction(1, 2**149)
    assert O.round_fraction(tiny, "fp32") == np.float32(2.0**-149)
    assert O.round_fraction(tiny / 2, "fp32") == np.float32(0.0)          # tie -> even (0)
    assert O.round_fraction(tiny * 3 / 2, "fp32") == np.float32(2.0**-148)  # tie -> even
    with pytest.raises(OverflowError):
        O.round_fraction(Fraction(2**128 - 2**103), "fp32")
    assert O.round_fraction(Fraction(2**128 - 2**104), "fp32") == np.float32(3.4028234663852886e38)


LAYER = G.cases("layer_cases.json")


@pytest.mark.parametrize("case", LAYER["cases"], ids=lambda c: c["name"])
def test_layer_composition_bitwise(case):
    arr = G.npz("layer.npz")
    t = trip_for(case["ts"])
    x, w = arr[case["name"] + "/x"], arr[case["name"] + "/w"]
    y64 = O.layer_direct_fp64(x, w, case["pad"])
    assert G.same_bits(y64, arr[case["name"] + "/y64"])
    for prec, order, cs in LAYER["modes"]:
        y = O.layer_conv2d(t, x, w, case["pad"], prec, order, cs, tile_chunk=7)
        assert G.same_bits(y, arr[f"{case['name']}/{prec}-{order}-{cs}/y"]), (prec, order, cs)


TILE = G.cases("tile_cases.json")


@pytest.mark.parametrize("case", TILE["cases"], ids=lambda c: c["name"])
def test_tile_level_bitwise(case):
    arr = G.npz("tile.npz")
    t = trip_for(case["ts"])
    nm = case["name"]
    h, x = arr[nm + "/h"], arr[nm + "/x"]
    # the Philox draws themselves
    for tr in range(case["trials"]):
        hh, xx = O.trial_draw(case["seed"], tr, 2, t.r, t.n, case["C"])
        assert G.same_bits(hh, h[tr]) and G.same_bits(xx, x[tr])
    assert G.same_bits(O.reduce_channels(O.direct_products(h, x, 2, "fp64"), -3, "linear"),
                       arr[nm + "/direct64"])
    for prec, order, cs in TILE["modes"]:
        key = f"{nm}/{prec}-{order}-{cs}"
        z = O.hadamard2d(t, h, x, prec, order)
        assert G.same_bits(z, arr[key + "/z"])
        assert G.same_bits(O.tile_conv2d(t, h, x, prec, order, cs), arr[key + "/y"])
        assert G.same_bits(O.tile_conv1d(t, arr[nm + "/h1"], arr[nm + "/x1"], prec, order, cs),
                           arr[key + "/y1"])


def test_halving_sum_lengths_1_to_70():
    arr = G.npz("tile.npz")
    for L in range(1, 71):
        v = arr[f"pw/{L}/v"]
        assert G.same_bits(np.asarray(O.sum_halving(v)), arr[f"pw/{L}/s"])


def test_philox_golden():
    arr = G.npz("philox.npz")
    for key in arr:
        if not key.endswith("/h"):
            continue
        seed, t, dims, n, C = (int(v) for v in key.split("/")[:5])
        h, x = O.trial_draw(seed, t, dims, 3, n, C)
        assert G.same_bits(h, arr[key]) and G.same_bits(x, arr[key[:-1] + "x"])


def _rows(maxc):
    return [r for r in G.measure_rows() if r["channels"] <= maxc]


@pytest.mark.parametrize("row", _rows(64), ids=lambda r: f"{r['set']}-{r['precision']}-{r['dot_order']}-{r['channel_sum']}-C{r['channels']}")
def test_measure_error_golden(row):
    """SURVEY.md 8(c) golden table, reproduced bit for bit (repr equality)."""
    if row["set"] == "direct":
        per, tot, pp = O.measure_error(None, row["dims"], row["precision"], row["dot_order"],
                                       row["channel_sum"], row["trials"], row["seed"],
                                       row["channels"], direct=True)
    else:
        n = int(row["set"].split("_n")[1])
        t = O.Triple.from_points(3, n - 2, _curated(row["set"]))
        per, tot, pp = O.measure_error(t, row["dims"], row["precision"], row["dot_order"],
                                       row["channel_sum"], row["trials"], row["seed"], row["channels"])
    assert repr(tot) == row["total_l1_mean"]
    assert repr(pp) == row["per_point_l1_mean"]


def _curated(setname):
    if setname.startswith("cur1d"):
        n = int(setname.split("_n")[1])
        return {4: "0,-1,1", 6: "0,-1,1,1/2,-3"}[n] + ",inf"
    return G.transforms()[setname]["points"]


def test_measure_per_trial_and_chunking():
    arr = G.npz("measure_per_trial.npz")
    for key, want in arr.items():
        setname, prec, cs, C = key.split("/")
        n = int(setname.split("_n")[1])
        t = O.Triple.from_points(3, n - 2, G.transforms()[setname]["points"])
        per, _, _ = O.measure_error(t, 2, prec, "huffman", cs, 200, 0, int(C), chunk=37)
        assert G.same_bits(per, want), key


@pytest.mark.skipif(not reference_available(), reason="reference not mounted")
def test_oracle_vs_reference_fresh_inputs():
    sys.path.insert(0, REFERENCE_SRC)
    from toomcook import engine as E
    from toomcook.exact import parse_points
    from toomcook.transforms import build_transforms
    rng = np.random.default_rng(99)
    for r, m, pts in ((3, 3, "0,1,-1,1/2,inf"), (3, 5, "1/2,0,-1,2,-2,1,inf"), (2, 3, "0,1,-1,3"),
                      (5, 2, "0,-1,1,1/2,-2,inf")):
        ts = build_transforms(r, m, parse_points(pts))
        t = O.Triple.from_points(r, m, pts)
        h = rng.normal(size=(6, 5, r, r)).astype(np.float32)
        x = rng.normal(size=(6, 5, t.n, t.n)).astype(np.float32)
        for prec in ("fp32", "mixed", "fp64"):
            for order in ("huffman", "linear"):
                for cs in ("linear", "pairwise"):
                    want = E.conv_2d(ts, h, x, E.ConvConfig(prec, order, cs))
                    assert G.same_bits(O.tile_conv2d(t, h, x, prec, order, cs), want)
