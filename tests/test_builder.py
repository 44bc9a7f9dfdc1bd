"""Host-side builder of the product (exact matrices, rounding, evaluation
trees, lowered programs) against the reference's own values (golden
fixtures), plus ports of the reference's construction tests."""

import json
from fractions import Fraction as F

import numpy as np
import pytest

import _golden as G
import paper_1803_10986_b200 as W
from paper_1803_10986_b200 import pointsets, programs
from paper_1803_10986_b200.transforms import transform_set_from_json

SPECS = sorted(G.transforms())


def _tree_tuple(t):
    if t is None:
        return None
    if isinstance(t, W.EvalLeaf):
        return ("leaf", t.col, F(t.coeff))
    return ("add", _tree_tuple(t.left), _tree_tuple(t.right))


@pytest.mark.parametrize("name", SPECS)
def test_builder_matches_reference(name):
    d = G.transforms()[name]
    ts = W.build_transforms(d["r"], d["m"], W.parse_points(d["points"]))
    assert [str(p) for p in ts.points] == d["ordered_points"]
    assert ts.modified == d["modified"]
    for mat in ("A_T", "G", "B_T"):
        assert ts.matrix(mat) == tuple(tuple(F(v) for v in row) for row in d[mat])
        for fmt in ("fp32", "fp64"):
            arr = ts.matrix_fp(mat, fmt)
            bits = [format(int(v), "x") for v in arr.view(np.uint32 if fmt == "fp32" else np.uint64).ravel()]
            assert bits == d[f"{mat}_{fmt}_bits"]
        for order in ("huffman", "linear"):
            want = [G.tree_from_json(x) for x in d[f"trees/{mat}/{order}"]]
            assert [_tree_tuple(t) for t in W.row_trees(ts, mat, order)] == want


def test_curated_sets_match_golden():
    for n in range(4, 19):
        for fam in ("fp32", "mixed"):
            d = G.transforms()[f"cur2d_{fam}_n{n}"]
            assert pointsets.curated_text(n, 2, fam) == d["points"]


def test_f23_entries_and_structure():
    ts = W.build_modified(3, 2, W.parse_points("0,1,-1,inf"))
    g = ts.matrix("G")
    assert g[1] == (F(1, 2), F(1, 2), F(1, 2)) and g[2] == (F(1, 2), F(-1, 2), F(1, 2)) and g[3] == (0, 0, 1)
    assert ts.matrix("B_T")[3] == (0, -1, 0, 1)
    assert W.check_exactness(ts, 50, seed=12, dims=1) and W.check_exactness(ts, 10, seed=13, dims=2)
    with pytest.raises(ValueError):
        W.build_toom_cook(3, 2, W.parse_points("0,1,1,2"))
    with pytest.raises(ValueError):
        W.build_modified(3, 2, W.parse_points("0,1,-1,2"))
    with pytest.raises(ValueError):
        W.build_modified(3, 2, W.parse_points("0,1,inf,inf"))
    with pytest.raises(ValueError):
        W.ConvConfig(precision="fp16")


def test_to_nearest_float_contract():
    assert W.to_nearest_float(F(1, 3), "fp32") == np.float32(1 / 3)
    assert W.to_nearest_float(F(2**24 + 1), "fp32") == np.float32(2**24)
    with pytest.raises(OverflowError):
        W.to_nearest_float(F(2**128 - 2**103), "fp32")
    with pytest.raises(ValueError):
        W.to_nearest_float(F(1), "fp16")


def test_huffman_rules():
    t = W.huffman_order([1, 1, 2, 4])
    depths = {}

    def walk(n, d):
        if isinstance(n, W.EvalLeaf):
            depths[n.col] = d
        else:
            walk(n.left, d + 1)
            walk(n.right, d + 1)
    walk(t, 0)
    assert depths == {0: 3, 1: 3, 2: 2, 3: 1}
    assert W.huffman_order([0, 5, 0]) == W.EvalLeaf(1, F(5))
    assert W.huffman_order([0, 0]) is None
    a = W.build_toom_cook(3, 2, W.parse_points("0,1,-1,2"))
    b = W.build_toom_cook(3, 2, W.parse_points("2,1,-1,0"))
    ta, tb = W.row_trees(a, "B_T", "huffman"), W.row_trees(b, "B_T", "huffman")
    assert ta[0] == tb[3] and ta[3] == tb[0] and ta[1] == tb[1]


def test_lowered_programs_follow_trees():
    ts = W.curated_transform(8, 2)
    for order in ("huffman", "linear"):
        starts, ops, ncols = programs.lower(ts, "B_T", order, "fp32")
        assert ncols == 8 and len(starts) == 9
        for i in range(8):
            seg = ops[starts[i]:starts[i + 1]]
            leaves = [o for o in seg if o[0] == programs.OP_LEAF]
            adds = [o for o in seg if o[0] == programs.OP_ADD]
            nz = sum(1 for v in ts.matrix("B_T")[i] if v != 0)
            assert len(leaves) == nz and len(adds) == max(nz - 1, 0)
            for _, col, c in leaves:
                assert np.float32(c) == W.to_nearest_float(ts.matrix("B_T")[i][col], "fp32")


def test_json_roundtrip(tmp_path):
    ts = W.build_modified(3, 2, W.parse_points("0,1,-1,inf"))
    p = tmp_path / "t.json"
    ts.write_json(p)
    d = json.loads(p.read_text())
    assert list(d) == ["n_h", "n_o", "n", "modified", "points", "A_T", "G", "B_T", "A_T_fp64", "G_fp64", "B_T_fp64"]
    assert d["G"][1] == ["1/2", "1/2", "1/2"]
    back = W.read_transform_json(p)
    assert back.matrix("B_T") == ts.matrix("B_T")
    d["points"] = ["0", "1"]
    with pytest.raises(ValueError):
        transform_set_from_json(d)


def test_pairwise_counter_equals_halving_tree_symbolically():
    """The binary-counter order used on the GPU builds the same summation tree
    as the reference's halving reduction (engine.py:259-267) for C = 1..4096,
    and appending (-0) padding channels leaves it unchanged."""
    def halving(items):
        cur = list(items)
        while len(cur) > 1:
            nxt = [("+", cur[i], cur[i + 1]) for i in range(0, len(cur) - 1, 2)]
            if len(cur) % 2:
                nxt.append(cur[-1])
            cur = nxt
        return cur[0]

    def counter(items):
        slots = {}
        for c, z in enumerate(items):
            j, cy = 0, z
            while (c >> j) & 1:
                cy = ("+", slots.pop(j), cy)
                j += 1
            slots[j] = cy
        acc = None
        for j in sorted(slots):
            acc = slots[j] if acc is None else ("+", slots[j], acc)
        return acc

    def strip(t):  # x + (-0) == x
        if isinstance(t, tuple):
            a, b = strip(t[1]), strip(t[2])
            if a == "z":
                return b
            if b == "z":
                return a
            return ("+", a, b)
        return t

    for C in list(range(1, 300)) + [1000, 4095, 4096]:
        items = list(range(C))
        assert halving(items) == counter(items), C
        pad = -(-C // 16) * 16
        assert strip(counter(items + ["z"] * (pad - C))) == halving(items), C
