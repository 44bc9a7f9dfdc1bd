"""Out-of-bounds write guard (compute-sanitizer is unavailable on the GPU pool):
every stage kernel writes into a buffer embedded between two guard regions
filled with a sentinel; the guards must come back untouched, for the layer
shapes and contraction modes the plans pick between."""
import ctypes

import pytest

pytestmark = pytest.mark.gpu
W = pytest.importorskip("paper_1803_10986_b200")
torch = pytest.importorskip("torch")
from paper_1803_10986_b200 import _native  # noqa: E402

GUARD = 1 << 16  # 4-byte words per guard region
SENT = 0x7F7F7F7F


def _guarded(nbytes):
    words = (nbytes + 3) // 4
    buf = torch.full((2 * GUARD + words + 4,), SENT, dtype=torch.int32, device="cuda")
    return buf, buf[GUARD:GUARD + words]


def _intact(buf, nbytes):
    words = (nbytes + 3) // 4
    return bool((buf[:GUARD] == SENT).all() and (buf[GUARD + words:] == SENT).all())


CASES = [
    # r, m, points, N, C, K, H, pad, precision, channel_sum, contraction
    (3, 2, "0,1,-1,inf", 3, 33, 70, 15, 1, "fp32", "linear", "exact"),
    (3, 2, "0,1,-1,inf", 4, 128, 128, 28, 1, "fp32", "linear", "exact"),
    (3, 6, "0,-1,1,1/2,-1/2,2,-2,inf", 2, 3, 64, 30, 1, "fp32", "pairwise", "exact"),
    (3, 6, "0,-1,1,1/2,-1/2,2,-2,inf", 1, 70, 130, 29, 1, "mixed", "pairwise", "exact"),
    (5, 2, "0,-1,1,1/2,-2,inf", 2, 20, 12, 14, 2, "fp64", "linear", "exact"),
    (3, 4, "0,1,-1,1/2,-1/2,inf", 2, 20, 24, 20, 1, "fp32", "linear", "ffma"),
    (3, 4, "0,1,-1,1/2,-1/2,inf", 2, 20, 150, 20, 1, "fp32", "linear", "tc_bf16"),
    (3, 2, "0,1,-1,inf", 3, 24, 40, 13, 1, "fp32", "linear", "tcf_fp16"),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"m{c[1]}C{c[4]}K{c[5]}-{c[8]}-{c[9]}-{c[10]}")
def test_stage_kernels_stay_in_bounds(case):
    r, m, pts, N, C, K, H, pad, prec, cs, mode = case
    ts = W.build_transforms(r, m, W.parse_points(pts))
    op = W.layer_op(ts, W.ConvConfig(prec, "huffman", cs), N, C, H, H, K, pad, mode)
    L = op.layout
    lib = _native.lib()
    dt = torch.float64 if prec == "fp64" else torch.float32
    x = torch.rand((N, C, H, H), dtype=dt, device="cuda")
    w = torch.rand((K, C, r, r), dtype=dt, device="cuda")
    sh = ctypes.byref(op.shape)
    s = torch.cuda.current_stream().cuda_stream
    P = _native.as_ptr
    y_bytes = N * K * L.Ho * L.Wo * L.elem_bytes_y
    bU, U = _guarded(L.u_bytes)
    bV, V = _guarded(L.v_bytes)
    _native.check(lib.wino_transforms(op.plan.handle, sh, P(x), P(w), P(U), P(V), s))
    by, y = _guarded(y_bytes)
    if op.fused:
        _native.check(lib.wino_contract_output(op.plan.handle, sh, P(U), P(V), P(y), s))
        torch.cuda.synchronize()
        assert _intact(bU, L.u_bytes) and _intact(bV, L.v_bytes) and _intact(by, y_bytes)
        return
    bM, M = _guarded(L.m_bytes)
    _native.check(lib.wino_contract(op.plan.handle, sh, P(U), P(V), P(M), s))
    _native.check(lib.wino_output_transform(op.plan.handle, sh, P(M), P(y), s))
    torch.cuda.synchronize()
    assert _intact(bU, L.u_bytes), "K2 wrote outside U"
    assert _intact(bV, L.v_bytes), "K1 wrote outside V"
    assert _intact(bM, L.m_bytes), "K3 wrote outside M"
    assert _intact(by, y_bytes), "K4 wrote outside y"
