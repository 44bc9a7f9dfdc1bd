"""GPU parity of the layer-level hot path (K1-K4 through the C-ABI) against the
reference's own numbers (golden fixtures) and the CPU oracle, bit for bit."""

import numpy as np
import pytest

import _golden as G
from oracle import wino_oracle as O

pytestmark = pytest.mark.gpu

W = pytest.importorskip("paper_1803_10986_b200")
torch = pytest.importorskip("torch")


def _ts(name):
    d = G.transforms()[name]
    return W.build_transforms(d["r"], d["m"], W.parse_points(d["points"])), O.Triple.from_points(d["r"], d["m"], d["points"])


LAYER = G.cases("layer_cases.json")


@pytest.mark.parametrize("case", LAYER["cases"], ids=lambda c: c["name"])
def test_layer_golden_bitwise(case):
    arr = G.npz("layer.npz")
    ts, _ = _ts(case["ts"])
    x, w = arr[case["name"] + "/x"], arr[case["name"] + "/w"]
    for prec, order, cs in LAYER["modes"]:
        y = W.conv2d_layer(ts, x, w, W.ConvConfig(prec, order, cs), pad=case["pad"])
        want = arr[f"{case['name']}/{prec}-{order}-{cs}/y"]
        assert G.same_bits(y, want), (prec, order, cs, np.abs(y.astype(np.float64) - want).max())
    y64 = W.direct_layer_f64(x, w, case["pad"])
    assert G.same_bits(y64, arr[case["name"] + "/y64"])


RANDOM_CASES = [
    # r, m, points, N, C, K, H, W, pad
    (3, 2, "0,1,-1,inf", 3, 33, 70, 15, 17, 1),
    (3, 4, "0,1,-1,1/2,-1/2,inf", 2, 64, 64, 20, 20, 1),
    (3, 6, "0,-1,1,1/2,-1/2,2,-2,inf", 1, 40, 130, 29, 23, 1),
    (3, 7, "0,-1,1,1/2,-1/2,2,-2,-1/4,inf", 2, 9, 5, 16, 16, 0),
    (5, 2, "0,-1,1,1/2,-2,inf", 2, 20, 12, 14, 14, 2),
    (3, 3, "0,1,-1,2,-2", 1, 3, 64, 30, 30, 1),
    (2, 3, "0,1,-1,inf", 2, 7, 9, 11, 11, 0),
    (3, 2, "0,1,-1,inf", 1, 1100, 3, 6, 6, 1),   # deep channel sums: pairwise counter with 6 stage levels
    (3, 4, "0,1,-1,1/2,-1/2,inf", 1, 2049, 2, 4, 4, 1),  # C = 2^11 + 1: odd tail after 64 full stages
]


@pytest.mark.parametrize("case", RANDOM_CASES, ids=lambda c: f"r{c[0]}m{c[1]}C{c[4]}K{c[5]}")
@pytest.mark.parametrize("mode", [("fp32", "huffman", "linear"), ("fp32", "linear", "pairwise"),
                                  ("mixed", "huffman", "pairwise"), ("fp64", "linear", "linear"),
                                  ("fp64", "huffman", "pairwise")],
                         ids=lambda m: "-".join(m))
def test_layer_vs_oracle(case, mode):
    r, m, pts, N, C, K, H, Wd, pad = case
    ts = W.build_transforms(r, m, W.parse_points(pts))
    trip = O.Triple.from_points(r, m, pts)
    x = O.synthetic((N, C, H, Wd), 7, 0)
    w = O.synthetic((K, C, r, r), 7, 99)
    y = W.conv2d_layer(ts, x, w, W.ConvConfig(*mode), pad=pad)
    want = O.layer_conv2d(trip, x, w, pad, *mode)
    assert G.same_bits(y, want)


def test_stages_match_oracle_pieces():
    """U and V of the generated transforms equal the oracle's (G w G^T) and
    (B^T d B); padded channels hold +0 (U) and -0 (V)."""
    pts = "0,1,-1,1/2,-1/2,inf"
    ts = W.build_transforms(3, 4, W.parse_points(pts))
    trip = O.Triple.from_points(3, 4, pts)
    x = O.synthetic((2, 5, 9, 9), 3, 0)
    w = O.synthetic((3, 5, 3, 3), 3, 1)
    cfg = W.ConvConfig()
    op = W.layer_op(ts, cfg, 2, 5, 9, 9, 3, 1)
    L = op.layout
    U = op.unblock_u(op.filter_transform(torch.from_numpy(w).cuda())).cpu().numpy()
    V = op.unblock_v(op.input_transform(torch.from_numpy(x).cuda())).cpu().numpy()
    u_or = O.apply_2d(trip, "G", "huffman", "fp32", w)                     # [K, C, n, n]
    assert G.same_bits(U[:, :5, :3].reshape(6, 6, 5, 3).transpose(3, 2, 0, 1).copy(), u_or)
    assert np.all(U[:, 5:, :] == 0) and not np.any(np.signbit(U[:, 5:, :]))
    tiles = O.gather_tiles(x, 3, 4, 1)                                    # [T, C, n, n]
    v_or = O.apply_2d(trip, "B_T", "huffman", "fp32", tiles)
    T = tiles.shape[0]
    assert G.same_bits(V[:, :5, :T].reshape(6, 6, 5, T).transpose(3, 2, 0, 1).copy(), v_or)
    assert np.all(np.signbit(V[:, 5:, :T]))
    assert L.Cp % 8 == 0 and L.Tp >= T


@pytest.mark.parametrize("cfgname", ["cfg1", "cfg2"])
def test_full_size_configs_bitwise(cfgname):
    """BASELINE configs 1 and 2 at full size, compared with the oracle bit for bit."""
    if cfgname == "cfg1":
        r, m, pts, N, C, K, H = 3, 4, "0,1,-1,1/2,-1/2,inf", 8, 64, 64, 56
        w = O.synthetic((K, C, r, r), 2024, 10_000_000)
    else:
        r, m, pts, N, C, K, H = 3, 2, "0,1,-1,inf", 32, 128, 128, 28
        w = (O.synthetic((K, C, r, r), 2024, 10_000_000, "normal") * np.float32(np.sqrt(2.0 / (9 * C))))
    x = np.stack([O.synthetic((C, H, H), 2024, i) for i in range(N)])
    ts = W.build_transforms(r, m, W.parse_points(pts))
    trip = O.Triple.from_points(r, m, pts)
    y = W.conv2d_layer(ts, x, w, W.ConvConfig(), pad=1)
    want = O.layer_conv2d(trip, x, w, 1)
    assert G.same_bits(y, want)
    # error statistics vs fp64 direct agree to far better than 2 significant digits
    y64 = W.direct_layer_f64(x, w, 1)
    y64o = O.layer_direct_fp64(x[:1], w, 1)
    assert G.same_bits(y64[:1], y64o)


def test_device_tensors_in_device_tensor_out():
    ts = W.build_transforms(3, 2, W.parse_points("0,1,-1,inf"))
    x = torch.randn(2, 4, 10, 10, device="cuda")
    w = torch.randn(3, 4, 3, 3, device="cuda")
    y = W.conv2d_layer(ts, x, w, pad=1)
    assert isinstance(y, torch.Tensor) and y.is_cuda and y.shape == (2, 3, 10, 10)
    ref = torch.nn.functional.conv2d(x.double(), w.double(), padding=1)
    assert torch.allclose(y.double(), ref, atol=1e-4)


def test_layer_validation_errors():
    ts = W.build_transforms(3, 2, W.parse_points("0,1,-1,inf"))
    with pytest.raises(ValueError):
        W.conv2d_layer(ts, np.zeros((1, 2, 5, 5), np.float32), np.zeros((1, 3, 3, 3), np.float32))
    with pytest.raises(ValueError):
        W.conv2d_layer(ts, np.zeros((1, 2, 5, 5), np.float32), np.zeros((1, 2, 5, 5), np.float32))
    with pytest.raises(ValueError):
        W.conv2d_layer(ts, np.zeros((1, 2, 2, 2), np.float32), np.zeros((1, 2, 3, 3), np.float32), pad=0)


def test_layer_with_4_byte_aligned_tensors():
    """x and y that are only 4-byte aligned (views one element into a buffer): the 8-byte paired
    loads / stores of K1 and K4 must fall back to scalar accesses, same bits."""
    ts = W.build_transforms(3, 6, W.parse_points("0,-1,1,1/2,-1/2,2,-2,inf"))
    cfg = W.ConvConfig("fp32", "huffman", "pairwise")
    N, C, K, H = 2, 5, 6, 16                      # even width: the paired paths apply when aligned
    x = torch.from_numpy(O.synthetic((N, C, H, H), 11, 0)).cuda()
    w = torch.from_numpy(O.synthetic((K, C, 3, 3), 11, 1)).cuda()
    op = W.layer_op(ts, cfg, N, C, H, H, K, 1)
    want = op(x, w)
    xb = torch.empty(x.numel() + 1, device="cuda")
    xo = xb[1:].view(x.shape)
    xo.copy_(x)
    yb = torch.empty(want.numel() + 1, device="cuda")
    yo = yb[1:].view(want.shape)
    assert xo.data_ptr() % 8 == 4 and yo.data_ptr() % 8 == 4
    got = op(xo, w, out=yo)
    assert torch.equal(got.view(torch.int32), want.view(torch.int32))
    from paper_1803_10986_b200.stack import ConvStack
    st = ConvStack(ts, cfg, [(C, K, False)], N, H)
    st.set_weights([w.cpu().numpy()])
    a_ref = st.forward(x).clone()
    ab = torch.empty(a_ref.numel() + 1, device="cuda")
    st.act[0] = ab[1:].view(a_ref.shape)
    assert st.act[0].data_ptr() % 8 == 4
    assert torch.equal(st.forward(x).view(torch.int32), a_ref.view(torch.int32))


NHWC_CASES = [
    # r, m, points, N, C, K, H, W, pad  (odd C / K around the 16-channel block, partial edge tiles, pad 0 / 2)
    (3, 4, "0,1,-1,1/2,-1/2,inf", 2, 9, 5, 14, 11, 1),
    (3, 2, "0,1,-1,inf", 3, 33, 70, 15, 17, 1),
    (3, 6, "0,-1,1,1/2,-1/2,2,-2,inf", 1, 40, 19, 29, 23, 1),
    (5, 2, "0,-1,1,1/2,-2,inf", 2, 20, 12, 14, 14, 2),
    (2, 3, "0,1,-1,inf", 2, 7, 9, 11, 11, 0),
]


@pytest.mark.parametrize("case", NHWC_CASES, ids=lambda c: f"r{c[0]}m{c[1]}C{c[4]}K{c[5]}")
@pytest.mark.parametrize("mode", [("fp32", "huffman", "linear"), ("fp32", "linear", "pairwise"),
                                  ("mixed", "huffman", "pairwise"), ("fp64", "huffman", "linear")],
                         ids=lambda m: "-".join(m))
def test_layer_nhwc_layout(case, mode):
    """layout='NHWC' (native NHWC gather / store kernels, wino_conv2d_nhwc) gives the
    oracle's NCHW results transposed, bit for bit."""
    r, m, pts, N, C, K, H, Wd, pad = case
    ts = W.build_transforms(r, m, W.parse_points(pts))
    trip = O.Triple.from_points(r, m, pts)
    x = O.synthetic((N, C, H, Wd), 4, 0)
    w = O.synthetic((K, C, r, r), 4, 1)
    want = O.layer_conv2d(trip, x, w, pad, *mode)
    y = W.conv2d_layer(ts, np.ascontiguousarray(x.transpose(0, 2, 3, 1)), w, W.ConvConfig(*mode), pad=pad,
                       layout="NHWC")
    assert y.shape == (N,) + want.shape[2:] + (K,)
    assert G.same_bits(np.ascontiguousarray(y.transpose(0, 3, 1, 2)), want)


def test_layer_nhwc_stages_and_errors():
    """The NHWC stage entry points produce the NCHW stages' V (same blocked layout, padding
    signs included) and y; bad layouts and tensor-core plans are rejected loudly."""
    import ctypes
    from paper_1803_10986_b200 import _native
    from paper_1803_10986_b200 import device as D
    pts = "0,1,-1,1/2,-1/2,inf"
    ts = W.build_transforms(3, 4, W.parse_points(pts))
    cfg = W.ConvConfig("fp32", "huffman", "pairwise")
    N, C, K, H, Wd = 2, 19, 21, 13, 10
    x = torch.from_numpy(O.synthetic((N, C, H, Wd), 9, 0)).cuda()
    w = torch.from_numpy(O.synthetic((K, C, 3, 3), 9, 1)).cuda()
    op = W.layer_op(ts, cfg, N, C, H, Wd, K, 1)
    V = op.input_transform(x)
    V2 = torch.empty_like(V)
    xh = x.permute(0, 2, 3, 1).contiguous()
    lib = _native.lib()
    _native.check(lib.wino_input_transform_nhwc(op.plan.handle, ctypes.byref(op.shape), D.ptr(xh), D.ptr(V2),
                                                D.stream_handle()), "input_transform_nhwc")
    assert torch.equal(V.view(torch.int32), V2.view(torch.int32))
    M = op.contract(op.filter_transform(w), V)
    y = op.output_transform(M)
    y2 = torch.empty((N, op.layout.Ho, op.layout.Wo, K), device="cuda")
    _native.check(lib.wino_output_transform_nhwc(op.plan.handle, ctypes.byref(op.shape), D.ptr(M), D.ptr(y2),
                                                 D.stream_handle()), "output_transform_nhwc")
    assert torch.equal(y.view(torch.int32), y2.permute(0, 3, 1, 2).contiguous().view(torch.int32))
    with pytest.raises(ValueError):
        W.conv2d_layer(ts, x.cpu().numpy(), w.cpu().numpy(), cfg, pad=1, layout="CHWN")
    tc = W.layer_op(ts, W.ConvConfig(), N, C, H, Wd, K, 1, "tc_bf16")
    rc = lib.wino_input_transform_nhwc(tc.plan.handle, ctypes.byref(tc.shape), D.ptr(xh), D.ptr(V2), D.stream_handle())
    assert rc != 0 and b"FP32-pipe" in lib.wino_last_error()
    # tensor-core modes still accept layout="NHWC" (device permute around the NCHW kernels)
    yt = W.conv2d_layer(ts, xh, w, W.ConvConfig(), pad=1, contraction="tc_fp16", layout="NHWC")
    yn = W.conv2d_layer(ts, x, w, W.ConvConfig(), pad=1, contraction="tc_fp16")
    assert torch.equal(yt.permute(0, 3, 1, 2).contiguous().view(torch.int32), yn.view(torch.int32))


@pytest.mark.parametrize("by", ["batch", "filters"])
def test_sharded_layer_assembles_to_the_full_layer(by):
    """Per-rank shards (by images or by output channels) computed one after the
    other on one GPU reassemble into the single-GPU result, bit for bit."""
    from paper_1803_10986_b200 import distributed as Dd
    ts = W.build_transforms(3, 2, W.parse_points("0,1,-1,inf"))
    x = O.synthetic((5, 12, 10, 10), 6, 0)
    w = O.synthetic((9, 12, 3, 3), 6, 1)
    full = W.conv2d_layer(ts, x, w, W.ConvConfig(), pad=1)
    out = np.zeros_like(full)
    for r in range(4):
        ni, ki = Dd.layer_shard(5, 9, r, 4, by)
        out[ni, ki] = W.conv2d_layer(ts, x[ni], w[ki], W.ConvConfig(), pad=1)
    assert G.same_bits(out, full)


def test_empty_batch_layer_and_tiles():
    """Empty inputs (N = 0 images, B = 0 tiles) give empty outputs of the right shape
    and dtype, like the reference's ufunc composition on empty arrays."""
    ts = W.build_transforms(3, 2, W.parse_points("0,1,-1,inf"))
    for prec in ("fp32", "mixed"):
        y = W.conv2d_layer(ts, np.zeros((0, 4, 9, 9), np.float32), O.synthetic((3, 4, 3, 3), 1, 1),
                           W.ConvConfig(prec), pad=1)
        assert y.shape == (0, 3, 9, 9) and y.dtype == (np.float32 if prec == "fp32" else np.float64)
    z = W.conv_2d(ts, np.zeros((0, 2, 3, 3), np.float32), np.zeros((0, 2, 4, 4), np.float32))
    assert z.shape == (0, 2, 2)


def test_unsupported_combinations_fail_loudly():
    """Unsupported plans / calls raise instead of silently falling back."""
    import ctypes
    from paper_1803_10986_b200 import _native
    ts8 = W.build_transforms(3, 6, W.parse_points("0,-1,1,1/2,-1/2,2,-2,inf"))
    with pytest.raises(RuntimeError):     # fused tcf needs alpha^2 <= 32
        W.conv2d_layer(ts8, O.synthetic((1, 4, 12, 12), 1, 0), O.synthetic((2, 4, 3, 3), 1, 1), pad=1,
                       contraction="tcf_bf16")
    ts3 = W.build_transforms(3, 3, W.parse_points("0,1,-1,2,-2"))
    op = W.layer_op(ts3, W.ConvConfig(), 1, 4, 12, 12, 2, 1)
    M = torch.zeros((op.layout.P, op.layout.Kp, op.layout.Tp), device="cuda")
    act = torch.zeros((1, 2, 6, 6), device="cuda")
    rc = _native.lib().wino_output_transform_act(op.plan.handle, ctypes.byref(op.shape), _native.as_ptr(M),
                                                 _native.as_ptr(act), 1, torch.cuda.current_stream().cuda_stream)
    assert rc != 0                        # 2x2 pooling needs an even m
    ts18 = W.curated_transform(18, 2, "fp32")
    with pytest.raises(RuntimeError):     # layer kernels are generated for alpha <= 16 only
        W.conv2d_layer(ts18, O.synthetic((1, 2, 20, 20), 1, 0), O.synthetic((2, 2, 3, 3), 1, 1), pad=1)
