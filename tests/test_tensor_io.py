"""Tensor files + the convolve adapter (reference cli.py:57-98, 162-176).  The file
round trips and error behaviour run on CPU; the convolution runs on the GPU and
is checked against the oracle's tile-level composition."""
import json

import numpy as np
import pytest

import paper_1803_10986_b200 as W
from oracle import wino_oracle as O


@pytest.mark.parametrize("fmt", ["json", "csv"])
@pytest.mark.parametrize("shape,dims", [((3, 4, 4), 2), ((2, 6), 1), ((5, 5), 2)])
def test_tensor_roundtrip(tmp_path, fmt, shape, dims):
    arr = np.random.default_rng(1).standard_normal(shape)
    p = str(tmp_path / f"t.{fmt}")
    W.save_tensor(p, arr, dims, fmt)
    back, d = W.load_tensor(p)
    want = arr if arr.ndim > dims else arr[np.newaxis]
    assert d == dims and back.shape == want.shape and np.array_equal(back, want)


def test_tensor_errors(tmp_path):
    p = tmp_path / "bad.json"
    p.write_text(json.dumps({"dims": 2, "shape": [1, 3, 3], "data": [[[1, 2], [3, 4]]]}))
    with pytest.raises(ValueError):
        W.load_tensor(str(p))
    q = tmp_path / "bad.csv"
    q.write_text("1,2,3\n")
    with pytest.raises(ValueError):
        W.load_tensor(str(q))
    q.write_text("shape,2,3\n1,2,3\n")
    with pytest.raises(ValueError):
        W.load_tensor(str(q))
    h, x = tmp_path / "h.csv", tmp_path / "x.csv"
    W.save_tensor(str(h), np.ones((1, 3)), 1, "csv")
    W.save_tensor(str(x), np.ones((1, 4, 4)), 2, "csv")
    with pytest.raises(ValueError):
        W.convolve(str(h), str(x), matrix_path=None)


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", [("fp32", "huffman", "linear"), ("mixed", "huffman", "pairwise")])
def test_convolve_matches_oracle(tmp_path, cfg):
    pts = "0,1,-1,1/2,-1/2,inf"
    ts = W.build_transforms(3, 4, W.parse_points(pts))
    m = tmp_path / "t.json"
    ts.write_json(str(m))
    rng = np.random.default_rng(5)
    h = rng.uniform(-1, 1, (7, 3, 3))
    x = rng.uniform(-1, 1, (7, 6, 6))
    hp, xp, out = tmp_path / "h.json", tmp_path / "x.csv", tmp_path / "y.json"
    W.save_tensor(str(hp), h, 2, "json")
    W.save_tensor(str(xp), x, 2, "csv")
    from paper_1803_10986_b200.tensor_io import main
    assert main(["convolve", "--matrix", str(m), "--kernel", str(hp), "--input", str(xp), "--precision", cfg[0],
                 "--dot-order", cfg[1], "--channel-sum", cfg[2], "--format", "json", "--out", str(out)]) == 0
    y, dims = W.load_tensor(str(out))
    trip = O.Triple.from_points(3, 4, pts)
    want = O.tile_conv2d(trip, h.astype(np.float32), x.astype(np.float32), *cfg)
    assert dims == 2 and np.array_equal(y[0], np.asarray(want, dtype=np.float64))
    yd, _ = W.convolve(str(hp), str(xp), W.ConvConfig(), direct=True)
    assert np.allclose(yd, want, atol=1e-5)
