"""The alternative transform kernels (selected by libwino tuning keys, read once
per process -- wino_tuning_set) must produce the same bits as the default kernels:

  k1=tile          K1 parks V in smem and writes 16-byte rows (input_body) --
                   also the fallback for grids beyond 65535 tile chunks
  k4=staged        K4 stages M in smem (flat for m <= 2, banded otherwise)
  k1tc=4x8         TC K1 with 4 tiles x 8 channels per warp also for P <= 16
  cpt / kpt        gather K1 / K4 threads looping over several channels / filters

Each variant runs in a subprocess; its outputs are compared bitwise with the
default kernels' outputs computed here (exact mode also with the oracle)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_1803_10986_b200 as W
from oracle import wino_oracle as O

pytestmark = pytest.mark.gpu

CASES = [
    # r, m, points, N, C, K, H, W, pad
    (3, 2, "0,1,-1,inf", 3, 33, 70, 15, 17, 1),
    (3, 4, "0,1,-1,1/2,-1/2,inf", 2, 20, 24, 20, 20, 1),
    (3, 6, "0,-1,1,1/2,-1/2,2,-2,inf", 1, 17, 19, 29, 23, 1),
]
MODES = ["exact", "tc_bf16"]

_CHILD = r"""
import json, sys
import numpy as np
import paper_1803_10986_b200 as W
from oracle import wino_oracle as O
cases, modes, out = json.loads(sys.argv[1]), json.loads(sys.argv[2]), sys.argv[3]
for k, v in json.loads(sys.argv[4]).items():
    W._native.set_tuning(k, v)
res = {}
for i, (r, m, pts, N, C, K, H, Wd, pad) in enumerate(cases):
    ts = W.build_transforms(r, m, W.parse_points(pts))
    x = O.synthetic((N, C, H, Wd), 7, 0)
    w = O.synthetic((K, C, r, r), 7, 99)
    for mode in modes:
        res[f"{i}/{mode}"] = W.conv2d_layer(ts, x, w, W.ConvConfig(), pad=pad, contraction=mode)
np.savez(out, **res)
"""


def _run_variant(tuning, tmp_path):
    out = str(tmp_path / "variant.npz")
    env = dict(os.environ)
    here = os.path.dirname(os.path.abspath(__file__))
    env["PYTHONPATH"] = os.pathsep.join([os.path.dirname(here), env.get("PYTHONPATH", "")])
    subprocess.run([sys.executable, "-c", _CHILD, json.dumps(CASES), json.dumps(MODES), out, json.dumps(tuning)],
                   check=True, env=env, timeout=600)
    return np.load(out)


@pytest.mark.parametrize("env", [{"k1": "tile"}, {"k4": "staged"}, {"k1tc": "4x8"}, {"cpt": "4", "kpt": "8"}],
                         ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()))
def test_variant_bits(env, tmp_path):
    got = _run_variant(env, tmp_path)
    for i, (r, m, pts, N, C, K, H, Wd, pad) in enumerate(CASES):
        ts = W.build_transforms(r, m, W.parse_points(pts))
        x = O.synthetic((N, C, H, Wd), 7, 0)
        w = O.synthetic((K, C, r, r), 7, 99)
        for mode in MODES:
            want = W.conv2d_layer(ts, x, w, W.ConvConfig(), pad=pad, contraction=mode)
            assert np.array_equal(got[f"{i}/{mode}"].view(np.uint32), want.view(np.uint32)), (env, i, mode)
        trip = O.Triple.from_points(r, m, pts)
        oracle = O.layer_conv2d(trip, x, w, pad, "fp32", "huffman", "linear")
        assert np.array_equal(got[f"{i}/exact"].view(np.uint32), oracle.view(np.uint32)), (env, i)


def test_interpreted_tile_transforms_pass_the_tile_goldens():
    """tile_interp=1: the tile-level API through the program interpreter
    (used for alpha > 10) reproduces every tile golden of test_gpu_tile.py --
    z and y bits of hadamard_2d / output_2d / conv_2d / conv_1d, and the
    reference's measure_error values repr for repr."""
    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, WINO_TEST_TUNING="tile_interp=1")
    env["PYTHONPATH"] = os.pathsep.join([os.path.dirname(here), env.get("PYTHONPATH", "")])
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(here, "test_gpu_tile.py"), "-m", "gpu", "-q",
                        "-x", "-k", "golden"], env=env, cwd=os.path.dirname(here), capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stdout[-3000:]


@pytest.mark.parametrize("prec", ["fp32", "mixed"])
def test_bulk_staged_k1_equals_global_gather(prec):
    """K1 from bulk-copied image planes in shared memory (the default where the planes of a block
    fit) writes the V that the global-memory gather writes, bit for bit, padding included:
    several planes per block, partial edge tiles, padded channels and tiles, alpha = 4 and 8."""
    import torch
    import paper_1803_10986_b200 as W
    from paper_1803_10986_b200 import _native
    from oracle import wino_oracle as O
    try:
        for m, pts in ((6, "0,-1,1,1/2,-1/2,2,-2,inf"), (2, "0,1,-1,inf")):
            ts = W.build_transforms(3, m, W.parse_points(pts))
            for (N, C, H, Wd, K) in [(5, 6, 14, 14, 8), (3, 70, 28, 28, 16), (2, 9, 20, 24, 8), (17, 3, 8, 8, 4)]:
                op = W.layer_op(ts, W.ConvConfig(prec, "huffman", "pairwise"), N, C, H, Wd, K, 1)
                x = torch.from_numpy(O.synthetic((N, C, H, Wd), 33, C)).cuda()
                _native.set_tuning("k1", "gather")
                want = op.input_transform(x)
                _native.set_tuning("k1", None)
                got = op.input_transform(x)
                torch.cuda.synchronize()
                assert torch.equal(got.view(torch.int32), want.view(torch.int32)), (prec, m, N, C, H, Wd)
    finally:
        _native.set_tuning("k1", None)
