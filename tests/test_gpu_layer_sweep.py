"""GPU parity of the layer path over the BASELINE block-size sweeps (configs[2],
configs[3]): F(m, 3) for m = 5, 8, 9 (alpha 7, 10, 11) and F(m, 5) for m = 3, 5, 6
(alpha 7, 9, 10), with the curated ("good") and the canonical integer point sets,
across Huffman / linear transform order, fp32 / mixed precision and linear /
pairwise channel sums -- bit for bit against the oracle (the reference's
per-(filter, tile) arithmetic, engine.py:401-429 over the zero-padded image).
Plus one full-size image of configs[2] (m = 6) and configs[3] (m = 4)."""

import numpy as np
import pytest

import _golden as G
from oracle import wino_oracle as O

pytestmark = pytest.mark.gpu
W = pytest.importorskip("paper_1803_10986_b200")
torch = pytest.importorskip("torch")

from paper_1803_10986_b200.pointsets import canonical_text, curated_text  # noqa: E402

ALL4 = [("fp32", "huffman", "linear"), ("fp32", "linear", "pairwise"), ("mixed", "huffman", "pairwise"),
        ("mixed", "linear", "linear")]
TWO = [("fp32", "huffman", "pairwise"), ("mixed", "linear", "linear")]


def _points(r, m, family, prec):
    n = r + m - 1
    if family == "canonical":
        return canonical_text(n)
    return curated_text(n, 2, "mixed" if prec == "mixed" else "fp32")


# (r, m, point family, modes): every factor level appears at alpha 7 and 9; the
# alpha 10 / 11 plans (NVRTC-heavy straight-line transforms) get two modes
CASES = []
for r, m in ((3, 5), (5, 3), (5, 5)):
    CASES += [(r, m, "curated", md) for md in ALL4] + [(r, m, "canonical", md) for md in TWO]
for r, m in ((3, 8), (5, 6), (3, 9)):
    CASES += [(r, m, "curated", md) for md in TWO] + [(r, m, "canonical", TWO[0])]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"r{c[0]}m{c[1]}-{c[2]}-{'-'.join(c[3])}")
def test_sweep_layer_bitwise(case):
    r, m, family, mode = case
    pts = _points(r, m, family, mode[0])
    ts = W.build_transforms(r, m, W.parse_points(pts))
    trip = O.Triple.from_points(r, m, pts)
    pad = r // 2
    N, C, K = 2, 21, 70                      # odd C (padded stage), K spans two filter blocks
    H, Wd = 2 * m + 3, 3 * m - 1             # partial edge tiles in both directions
    x = O.synthetic((N, C, H, Wd), 31, r * 10 + m)
    w = O.synthetic((K, C, r, r), 31, 1000 + r * 10 + m)
    y = W.conv2d_layer(ts, x, w, W.ConvConfig(*mode), pad=pad)
    want = O.layer_conv2d(trip, x, w, pad, *mode)
    assert G.same_bits(y, want)


@pytest.mark.parametrize("cfgname", ["cfg3_m6", "cfg4_m4"])
def test_full_size_sweep_configs_sampled_image(cfgname):
    """configs[2] (F(6,3), N64 C=K=256 28^2, fp32 + mixed/pairwise) and configs[3]
    (F(4,5), N32 C=K=512 14^2, pad 2, pairwise, U[0,1] inputs) at full batch on the
    GPU (the tile picks of the real shape); the first and last image are checked
    bit for bit against the oracle."""
    if cfgname == "cfg3_m6":
        r, m, N, C, K, H, pad, dist = 3, 6, 64, 256, 256, 28, 1, "uniform"
        modes = [("fp32", "huffman", "linear"), ("mixed", "huffman", "pairwise")]
    else:
        r, m, N, C, K, H, pad, dist = 5, 4, 32, 512, 512, 14, 2, "uniform01"
        modes = [("fp32", "huffman", "pairwise")]
    x = np.stack([O.synthetic((C, H, H), 2024, i, dist) for i in range(N)])
    w = O.synthetic((K, C, r, r), 2024, 10_000_000, "normal") * np.float32(np.sqrt(2.0 / (r * r * C)))
    xt, wt = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
    for mode in modes:
        pts = curated_text(r + m - 1, 2, "mixed" if mode[0] == "mixed" else "fp32")
        ts = W.build_transforms(r, m, W.parse_points(pts))
        trip = O.Triple.from_points(r, m, pts)
        y = W.conv2d_layer(ts, xt, wt, W.ConvConfig(*mode), pad=pad).cpu().numpy()
        for i in (0, N - 1):
            want = O.layer_conv2d(trip, x[i:i + 1], w, pad, *mode)
            assert G.same_bits(y[i:i + 1], want), (mode, i)
