"""Tensor-core contraction mode (tcgen05, BF16/FP16 operands, FP32 accumulate):
not bitwise by design -- checked against an fp64 GEMM of the 16-bit-rounded
operands (layout correctness) and against the fp64 direct convolution (error)."""
import numpy as np
import pytest

from oracle import wino_oracle as O

pytestmark = pytest.mark.gpu
W = pytest.importorskip("paper_1803_10986_b200")
torch = pytest.importorskip("torch")


@pytest.mark.parametrize("mode,dt", [("tc_bf16", torch.bfloat16), ("tc_fp16", torch.float16)])
def test_tc_contraction_matches_rounded_gemm(mode, dt):
    ts = W.build_transforms(3, 4, W.parse_points("0,1,-1,1/2,-1/2,inf"))
    op = W.layer_op(ts, W.ConvConfig(), 3, 70, 20, 20, 150, 1, contraction=mode)
    L = op.layout
    Ud = torch.randn((L.P, L.Cp, L.Kp), device="cuda")
    Vd = torch.randn((L.P, L.Cp, L.Tp), device="cuda")
    U, V = op.block_u(Ud), op.block_v(Vd)
    assert torch.equal(op.unblock_u(U), Ud.to(dt)) and torch.equal(op.unblock_v(V), Vd.to(dt))
    M = op.contract(U, V)
    Uu = Ud.to(dt).double()
    Vu = Vd.to(dt).double()
    ref = torch.einsum("pck,pct->pkt", Uu, Vu)
    # M's padded filter rows (k >= K) are never read by K4 and are left unwritten
    err = (M.double() - ref)[:, :150].abs().max().item()
    scale = torch.einsum("pck,pct->pkt", Uu.abs(), Vu.abs()).max().item()
    assert err <= 1e-5 * scale, (err, scale)


@pytest.mark.parametrize("K", [64, 150, 7])
def test_tc_contraction_leaves_padded_filter_rows_unwritten(K):
    """K3t stores exactly the rows k < K of every point's [Kp][Tp] slab: poisoned padding rows stay
    poisoned (K = 64 pads to 128: half of the tile's store traffic), every real row is written,
    including the partially live lane quarter when K % 32 != 0."""
    import ctypes
    from paper_1803_10986_b200 import _native
    ts = W.build_transforms(3, 4, W.parse_points("0,1,-1,1/2,-1/2,inf"))
    op = W.layer_op(ts, W.ConvConfig(), 2, 40, 20, 20, K, 1, contraction="tc_fp16")
    L = op.layout
    Ud = torch.randn((L.P, L.Cp, L.Kp), device="cuda")
    Vd = torch.randn((L.P, L.Cp, L.Tp), device="cuda")
    U, V = op.block_u(Ud), op.block_v(Vd)
    poison = torch.full((L.P, L.Kp, L.Tp), float("nan"), device="cuda")
    M = poison.clone()
    _native.check(_native.lib().wino_contract(op.plan.handle, ctypes.byref(op.shape), _native.as_ptr(U),
                                              _native.as_ptr(V), _native.as_ptr(M),
                                              torch.cuda.current_stream().cuda_stream), "contract")
    torch.cuda.synchronize()
    assert not torch.isnan(M[:, :K]).any()
    assert torch.isnan(M[:, K:]).all() or L.Kp == K
    ref = torch.einsum("pck,pct->pkt", Ud.half().double(), Vd.half().double())[:, :K]
    scale = torch.einsum("pck,pct->pkt", Ud.half().double().abs(), Vd.half().double().abs()).max().item()
    assert (M[:, :K].double() - ref).abs().max().item() <= 1e-5 * scale


@pytest.mark.parametrize("mode", ["tc_bf16", "tc_fp16"])
def test_tc_transforms_write_rounded_operands(mode):
    """The tc transforms store exactly round16(fp32 exact transform) in the UMMA layout."""
    pts = "0,1,-1,1/2,-1/2,inf"
    ts = W.build_transforms(3, 4, W.parse_points(pts))
    x = torch.from_numpy(O.synthetic((2, 13, 11, 11), 4, 0)).cuda()
    w = torch.from_numpy(O.synthetic((9, 13, 3, 3), 4, 1)).cuda()
    ex = W.layer_op(ts, W.ConvConfig(), 2, 13, 11, 11, 9, 1)
    tc = W.layer_op(ts, W.ConvConfig(), 2, 13, 11, 11, 9, 1, contraction=mode)
    dt = torch.bfloat16 if mode == "tc_bf16" else torch.float16
    Le, Lt = ex.layout, tc.layout
    ue = ex.unblock_u(ex.filter_transform(w))[:, :13, :9]
    ut = tc.unblock_u(tc.filter_transform(w))[:, :13, :9]
    assert torch.equal(ut, ue.to(dt))
    ve = ex.unblock_v(ex.input_transform(x))[:, :13, :Le.T]
    vt = tc.unblock_v(tc.input_transform(x))[:, :13, :Lt.T]
    assert torch.equal(vt, ve.to(dt))


@pytest.mark.parametrize("mode", ["tc_bf16", "tc_fp16"])
@pytest.mark.parametrize("m,pts,geom,prec", [(6, "0,-1,1,1/2,-1/2,2,-2,inf", (3, 13, 37, 41, 9), "fp32"),
                                             (6, "0,-1,1,1/2,-1/2,2,-2,inf", (3, 13, 37, 41, 9), "mixed"),
                                             (6, "0,-1,1,1/2,-1/2,2,-2,inf", (2, 20, 64, 34, 5), "fp32"),
                                             (4, "0,1,-1,1/2,-1/2,inf", (2, 9, 40, 40, 7), "fp32"),
                                             (6, "0,-1,1,1/2,-1/2,2,-2,inf", (5, 11, 14, 14, 9), "fp32")],
                         ids=["a8_37x41", "a8_37x41_mixed", "a8_64x34", "a6_40x40", "a8_14x14_old_map"])
def test_tc_staged_input_transform_writes_rounded_operands(mode, m, pts, geom, prec):
    """K1 of the tc modes at 16 < alpha^2 <= 96: images above 32 x 32 take the warp-per-channel kernel that
    parks its 16-bit results in shared memory (wino_input_tcs / wino_transforms_tcs), smaller ones the
    4-tiles x 8-channels map; both store exactly round16(exact fp32 transform), through the standalone K1
    and through the K1 + K2 launch, with zeros in the padded channels and tiles."""
    import ctypes
    from paper_1803_10986_b200 import _native
    N, C, H, Wd, K = geom
    ts = W.build_transforms(3, m, W.parse_points(pts))
    x = torch.from_numpy(O.synthetic((N, C, H, Wd), 6, 0)).cuda()
    w = torch.from_numpy(O.synthetic((K, C, 3, 3), 6, 1)).cuda()
    ex = W.layer_op(ts, W.ConvConfig(prec), N, C, H, Wd, K, 1)
    tc = W.layer_op(ts, W.ConvConfig(prec), N, C, H, Wd, K, 1, contraction=mode)
    dt = torch.bfloat16 if mode == "tc_bf16" else torch.float16
    Le, Lt = ex.layout, tc.layout
    ve = ex.unblock_v(ex.input_transform(x))[:, :C, :Le.T].to(dt)
    vt = tc.unblock_v(tc.input_transform(x))
    assert torch.equal(vt[:, :C, :Lt.T], ve)
    assert not vt[:, C:, :].any() and not vt[:, :, Lt.T:].any()
    # the combined K1 + K2 launch
    U = torch.full((Lt.P * Lt.Cp * Lt.Kp,), 0x7fff, dtype=torch.int16, device="cuda")
    V = torch.full((Lt.P * Lt.Cp * Lt.Tp,), 0x7fff, dtype=torch.int16, device="cuda")
    _native.check(_native.lib().wino_transforms(tc.plan.handle, ctypes.byref(tc.shape), _native.as_ptr(x),
                                                _native.as_ptr(w), _native.as_ptr(U), _native.as_ptr(V),
                                                torch.cuda.current_stream().cuda_stream), "transforms")
    torch.cuda.synchronize()
    v2 = tc.unblock_v(V.view(dt))
    assert torch.equal(v2[:, :C, :Lt.T], ve) and not v2[:, C:, :].any() and not v2[:, :, Lt.T:].any()
    ue = ex.unblock_u(ex.filter_transform(w))[:, :C, :K].to(dt)
    assert torch.equal(tc.unblock_u(U.view(dt))[:, :C, :K], ue)


@pytest.mark.parametrize("mode", ["tc_bf16", "tc_fp16"])
def test_tc_layer_error_vs_fp64(mode):
    pts = "0,-1,1,1/2,-1/2,2,-2,inf"
    ts = W.build_transforms(3, 6, W.parse_points(pts))
    x = O.synthetic((4, 64, 28, 28), 3, 0)
    w = O.synthetic((96, 64, 3, 3), 3, 1) * np.float32(0.06)
    y = W.conv2d_layer(ts, x, w, W.ConvConfig(), pad=1, contraction=mode)
    y64 = O.layer_direct_fp64(x, w, 1)
    rel = np.abs(y.astype(np.float64) - y64).sum() / np.abs(y64).sum()
    # measured on B200: BF16 3.9e-2, FP16 ~3e-3 (F(6,3) transforms amplify the 16-bit operand rounding)
    assert rel < (6e-2 if mode == "tc_bf16" else 6e-3), rel
    yx = W.conv2d_layer(ts, x, w, W.ConvConfig(), pad=1)
    rel_exact = np.abs(yx.astype(np.float64) - y64).sum() / np.abs(y64).sum()
    assert rel_exact < rel


@pytest.mark.parametrize("mode,dt", [("tcf_bf16", torch.bfloat16), ("tcf_fp16", torch.float16)])
def test_tcf_alpha5_with_the_staged_input_transform(mode, dt):
    """alpha = 5 (P = 25) on an image above 32 x 32: the fused tensor-core plan's K1 is the staged
    warp-per-channel kernel writing the fused operand layout ([t/128][c/16][p]...): V == round16(exact V),
    and the fused layer agrees with the unfused tc mode (same operands) to accumulation accuracy."""
    ts = W.build_transforms(3, 3, W.parse_points("0,1,-1,2,inf"))
    N, C, H, Wd, K = 2, 19, 41, 50, 24
    x = torch.from_numpy(O.synthetic((N, C, H, Wd), 8, 0)).cuda()
    w = torch.from_numpy(O.synthetic((K, C, 3, 3), 8, 1)).cuda()
    ex = W.layer_op(ts, W.ConvConfig(), N, C, H, Wd, K, 1)
    op = W.layer_op(ts, W.ConvConfig(), N, C, H, Wd, K, 1, contraction=mode)
    assert op.layout.P == 25
    ve = ex.unblock_v(ex.input_transform(x))[:, :C, :ex.layout.T].to(dt)
    vt = op.unblock_v(op.input_transform(x))
    assert torch.equal(vt[:, :C, :op.layout.T], ve)
    assert not vt[:, C:, :].any() and not vt[:, :, op.layout.T:].any()
    y = W.conv2d_layer(ts, x, w, W.ConvConfig(), pad=1, contraction=mode)
    y3 = W.conv2d_layer(ts, x, w, W.ConvConfig(), pad=1, contraction=mode.replace("tcf", "tc"))
    yx = W.conv2d_layer(ts, x, w, W.ConvConfig(), pad=1)
    scale = yx.abs().max().item()
    assert (y.double() - y3.double()).abs().max().item() <= 1e-4 * scale
    assert (y.double() - yx.double()).abs().max().item() <= (0.1 if "bf16" in mode else 0.02) * scale


@pytest.mark.parametrize("mode,dt", [("tcf_bf16", torch.bfloat16), ("tcf_fp16", torch.float16)])
@pytest.mark.parametrize("geom", [(3, 70, 20, 20, 150, 1), (2, 16, 9, 11, 16, 0), (1, 33, 28, 28, 40, 1)],
                         ids=lambda g: "N{}C{}H{}W{}K{}".format(*g[:5]))
def test_tcf_fused_matches_rounded_gemm_then_output(mode, dt, geom):
    """Fused K3t+K4 (all alpha^2 accumulators in TMEM, output transform in the
    epilogue) == fp64 GEMM of the 16-bit operands followed by the fp64 output
    transform, to fp32 accumulation accuracy; and == the unfused tc mode's result
    within the same bound."""
    N, C, H, Wd, K, pad = geom
    pts = "0,1,-1,inf"
    ts = W.build_transforms(3, 2, W.parse_points(pts))
    op = W.layer_op(ts, W.ConvConfig(), N, C, H, Wd, K, pad, contraction=mode)
    L = op.layout
    x = torch.from_numpy(O.synthetic((N, C, H, Wd), 5, 0)).cuda()
    w = torch.from_numpy(O.synthetic((K, C, 3, 3), 5, 1)).cuda()
    U, V = op.filter_transform(w), op.input_transform(x)
    y = op.contract_output(U, V)
    torch.cuda.synchronize()
    Uu = op.unblock_u(U).double()
    Vu = op.unblock_v(V).double()
    M = torch.einsum("pck,pct->pkt", Uu, Vu)[:, :K, :L.T]  # [P][K][T]
    n = 4
    AT = torch.tensor(np.array(ts.matrix_fp("A_T", "fp64"), dtype=np.float64)).cuda()
    Mt = M.reshape(n, n, K, L.T).permute(2, 3, 0, 1)  # [K][T][n][n]
    Yt = AT @ Mt @ AT.T  # [K][T][2][2]
    Yt = Yt.reshape(K, N, L.th, L.tw, 2, 2).permute(1, 0, 2, 4, 3, 5).reshape(N, K, L.th * 2, L.tw * 2)
    ref = Yt[:, :, :L.Ho, :L.Wo]
    scale = torch.einsum("pck,pct->pkt", Uu.abs(), Vu.abs()).max().item() * 4
    err = (y.double() - ref).abs().max().item()
    assert err <= 2e-5 * scale, (err, scale)
    # whole-layer API (wino_conv2d) gives the same bits as the stage calls
    y2 = W.conv2d_layer(ts, x, w, W.ConvConfig(), pad=pad, contraction=mode)
    assert torch.equal(y2, y)
    # and agrees with the unfused tensor-core mode to accumulation accuracy
    y3 = W.conv2d_layer(ts, x, w, W.ConvConfig(), pad=pad, contraction=mode.replace("tcf", "tc"))
    assert (y3.double() - y.double()).abs().max().item() <= 2e-5 * scale
