"""GPU parity of the conv stack (VGG-16 shape, BASELINE config 5) vs the oracle."""
import numpy as np
import pytest

import _golden as G
from oracle import wino_oracle as O

pytestmark = pytest.mark.gpu
W = pytest.importorskip("paper_1803_10986_b200")
torch = pytest.importorskip("torch")

P8 = "0,-1,1,1/2,-1/2,2,-2,inf"


def test_small_vgg_like_stack_bitwise():
    from paper_1803_10986_b200.stack import ConvStack, he_normal_weights
    layers = [(3, 16, False), (16, 16, True), (16, 32, False), (32, 32, True), (32, 40, False)]
    ts = W.build_transforms(3, 6, W.parse_points(P8))
    trip = O.Triple.from_points(3, 6, P8)
    N, H = 2, 30
    x = np.stack([O.synthetic((3, H, H), 5, i) for i in range(N)])
    ws = he_normal_weights(layers, 3, seed=11)
    st = ConvStack(ts, W.ConvConfig("fp32", "huffman", "pairwise"), layers, N, H)
    st.set_weights(ws)
    xt = torch.from_numpy(x).cuda()
    assert st.fused_act
    out = st.forward(xt).cpu().numpy()                       # K4 + ReLU / max-pool fused
    ref_outs, ref = O.stack_forward(trip, x, ws, layers)
    assert G.same_bits(out, ref)
    st.use_smallc(True)                                      # layer 1 (C = 3): K3 + K4 + act fused
    assert st.smallc[0] and not any(st.smallc[1:])
    assert G.same_bits(st.forward(xt).cpu().numpy(), ref)
    st.use_smallc(False)
    st.use_fuse_next(True)                                   # K4 + act + K1 of the next layer in one kernel
    assert any(st.fuse_next)
    assert G.same_bits(st.forward(xt).cpu().numpy(), ref)
    st.use_fuse_next(False)
    out2 = st.forward(xt, keep_conv_out=True).cpu().numpy()  # unfused: y stored, wino_relu_pool
    for i, y in enumerate(ref_outs):
        assert G.same_bits(st.conv_out[i].cpu().numpy(), y), i
    assert G.same_bits(out2, ref)
    errs = st.layer_errors(xt)
    assert len(errs) == len(layers) and all(e["rel_l1"] < 1e-4 for e in errs)


@pytest.mark.parametrize("m,pts", [(4, "0,1,-1,1/2,-1/2,inf"), (3, "0,1,-1,2,-2")])
def test_fused_activation_matches_relu_pool(m, pts):
    """wino_output_transform_act == wino_output_transform + wino_relu_pool, bitwise,
    including partial edge tiles (odd output sizes) and ReLU-only for odd m."""
    import ctypes
    from paper_1803_10986_b200 import _native
    ts = W.build_transforms(3, m, W.parse_points(pts))
    lib = _native.lib()
    for (N, C, K, H, Wd) in [(2, 5, 7, 17, 23), (1, 16, 33, 30, 30)]:
        op = W.layer_op(ts, W.ConvConfig(), N, C, H, Wd, K, 1)
        x = torch.from_numpy(O.synthetic((N, C, H, Wd), 9, 0)).cuda()
        w = torch.from_numpy(O.synthetic((K, C, 3, 3), 9, 1)).cuda()
        U, V = op.filter_transform(w), op.input_transform(x)
        M = op.contract(U, V)
        y = op.output_transform(M)
        s = torch.cuda.current_stream().cuda_stream
        Ho, Wo = op.layout.Ho, op.layout.Wo
        for pool in ((0, 1) if m % 2 == 0 else (0,)):
            shp = (N, K, Ho // 2, Wo // 2) if pool else (N, K, Ho, Wo)
            want = torch.empty(shp, device="cuda")
            _native.check(lib.wino_relu_pool(0, N * K, Ho, Wo, pool, _native.as_ptr(y), _native.as_ptr(want), s))
            got = torch.full(shp, 7.0, device="cuda")
            _native.check(lib.wino_output_transform_act(op.plan.handle, ctypes.byref(op.shape), _native.as_ptr(M),
                                                        _native.as_ptr(got), pool, s))
            torch.cuda.synchronize()
            assert torch.equal(got.view(torch.int32), want.view(torch.int32)), (N, C, K, H, Wd, pool)


@pytest.mark.parametrize("mode", ["tc_bf16", "tc_fp16"])
def test_tensor_core_stack_fuses_activation(mode):
    """tc_* modes keep an fp32 M, so a stack runs K4 + ReLU (+ pool) as one kernel there too:
    same bits as the unfused forward (wino_conv2d then wino_relu_pool) of the same mode,
    on edge tiles and pooled / un-pooled layers."""
    from paper_1803_10986_b200.stack import ConvStack, he_normal_weights
    ts = W.build_transforms(3, 6, W.parse_points(P8))
    layers = [(3, 16, False), (16, 24, True), (24, 40, False), (40, 40, True)]
    st = ConvStack(ts, W.ConvConfig("fp32", "huffman", "pairwise"), layers, 3, 36, 44, contraction=mode)
    # the C = 3 layer has no contraction worth a tensor core: it runs the exact (fused small-C) path
    assert st.fused_act and not st.ops[0].tensor_core and all(op.tensor_core for op in st.ops[1:])
    assert st.kernels_per_forward in (2 + 3 * (len(layers) - 1), 3 * len(layers))
    st.set_weights(he_normal_weights(layers, 3))
    x = torch.from_numpy(O.synthetic((3, 3, 36, 44), 5, 0)).cuda()
    fused = st.forward(x).clone()
    acts = [a.clone() for a in st.act]
    plain = st.forward(x, keep_conv_out=True)
    torch.cuda.synchronize()
    for i, a in enumerate(acts):
        assert torch.equal(a.view(torch.int32), st.act[i].view(torch.int32)), i
    assert torch.equal(fused.view(torch.int32), plain.view(torch.int32))
    # and it is a convolution: final activation close to the exact path's
    ex = ConvStack(ts, W.ConvConfig("fp32", "huffman", "pairwise"), layers, 3, 36, 44)
    ex.set_weights(he_normal_weights(layers, 3))
    ref = ex.forward(x)
    rel = float((fused - ref).abs().sum() / ref.abs().sum())
    assert rel < (0.2 if mode == "tc_bf16" else 0.03), rel


def test_vgg16_geometry():
    from paper_1803_10986_b200.stack import VGG16, ConvStack
    ts = W.build_transforms(3, 6, W.parse_points(P8))
    st = ConvStack(ts, W.ConvConfig("fp32", "huffman", "pairwise"), VGG16, 1, 224)
    assert st.out_hw == (14, 14)
    assert abs(st.direct_flops * 256 - 7.86e12) / 7.86e12 < 0.01   # 7.86 TFLOP per batch-256


def test_vgg16_full_size_batch256_bitwise():
    """BASELINE config 5 at its real shape (batch 256, 224x224x3, the default tile
    picks of every layer): images 0 and 255 of the batch, every layer's
    pre-activation output and the final activation, bit for bit against the oracle
    (reference per-(filter, tile) arithmetic, run over host processes)."""
    import os
    from oracle.stack_pool import OraclePool
    from paper_1803_10986_b200.stack import VGG16, ConvStack, he_normal_weights
    ts = W.build_transforms(3, 6, W.parse_points(P8))
    trip = O.Triple.from_points(3, 6, P8)
    N = 256
    x = np.stack([O.synthetic((3, 224, 224), 2024, i) for i in range(N)])
    ws = he_normal_weights(VGG16, 3)
    st = ConvStack(ts, W.ConvConfig("fp32", "huffman", "pairwise"), VGG16, N, 224)
    st.set_weights(ws)
    xt = torch.from_numpy(x).cuda()
    fused = st.forward(xt).cpu().numpy()[[0, N - 1]]
    st.forward(xt, keep_conv_out=True)
    got = [st.conv_out[i][[0, N - 1]].cpu().numpy() for i in range(len(VGG16))]
    sample = x[[0, N - 1]]
    with OraclePool(trip, ws, 2 * 64 * 226 * 226, procs=min(16, len(os.sched_getaffinity(0)))) as pool:
        outs, act = pool.stack_forward(sample, VGG16)
    for i, (g, want) in enumerate(zip(got, outs)):
        assert G.same_bits(g, want), f"layer {i + 1}"
    assert G.same_bits(fused, act)


@pytest.mark.parametrize("cs", ["linear", "pairwise"])
def test_smallc_fused_kernel_matches_unfused(cs):
    """wino_contract_output_smallc (K3 + K4 + activation in one kernel for C <= 8) is
    bitwise equal to wino_contract + wino_output_transform[_act] for every C <= 8,
    modes y / ReLU / ReLU + max-pool, partial edge tiles, K not a multiple of 4."""
    import ctypes
    from paper_1803_10986_b200 import _native
    lib = _native.lib()
    s = torch.cuda.current_stream().cuda_stream
    for m, pts in ((6, P8), (4, "0,1,-1,1/2,-1/2,inf"), (3, "0,1,-1,2,-2")):
        ts = W.build_transforms(3, m, W.parse_points(pts))
        # odd output width (scalar stores), then an even one (the C <= 4 kernel's warp-cooperative row
        # stores: partial edge tiles, warps spanning tile rows and images, two U blocks for K = 70)
        for C, (N, K, H, Wd) in [(C, (2, 7 + C, 17 + C, 23)) for C in range(1, 9)] + \
                                [(C, (5, 70 if C == 2 else 9 + C, 20, 26)) for C in range(1, 5)]:
            op = W.layer_op(ts, W.ConvConfig("fp32", "huffman", cs), N, C, H, Wd, K, 1)
            assert lib.wino_smallc_supported(op.plan.handle, ctypes.byref(op.shape))
            x = torch.from_numpy(O.synthetic((N, C, H, Wd), 12, C)).cuda()
            w = torch.from_numpy(O.synthetic((K, C, 3, 3), 12, 100 + C)).cuda()
            U, V = op.filter_transform(w), op.input_transform(x)
            M = op.contract(U, V)
            Ho, Wo = op.layout.Ho, op.layout.Wo
            for mode in ((0, 1, 2) if m % 2 == 0 else (0, 1)):
                if mode == 0:
                    want = op.output_transform(M)
                else:
                    shp = (N, K, Ho // 2, Wo // 2) if mode == 2 else (N, K, Ho, Wo)
                    want = torch.empty(shp, device="cuda")
                    _native.check(lib.wino_output_transform_act(op.plan.handle, ctypes.byref(op.shape),
                                                                _native.as_ptr(M), _native.as_ptr(want), mode - 1, s))
                got = torch.full_like(want, 7.0)
                _native.check(lib.wino_contract_output_smallc(op.plan.handle, ctypes.byref(op.shape),
                                                              _native.as_ptr(U), _native.as_ptr(V),
                                                              _native.as_ptr(got), mode, s))
                torch.cuda.synchronize()
                assert torch.equal(got.view(torch.int32), want.view(torch.int32)), (m, C, K, H, Wd, cs, mode)


@pytest.mark.parametrize("chunks", [1, 3, [1, 3, 1], [32, 192, 32], [4, 4, 4, 4, 4, 4, 4]],
                         ids=lambda c: "chunks=" + str(c).replace(" ", ""))
def test_stack_pipeline_host_buffers_bitwise(chunks):
    """StackPipeline (pinned host images in, final activation out, copies overlapped over image
    chunks of equal or explicit sizes) equals the one-shot device forward, bit for bit."""
    from paper_1803_10986_b200.stack import ConvStack, StackPipeline, he_normal_weights
    layers = [(3, 8, True), (8, 12, False), (12, 9, True)]
    ts = W.build_transforms(3, 6, W.parse_points(P8))
    cfg = W.ConvConfig("fp32", "huffman", "pairwise")
    N, H = 5, 26
    x = np.stack([O.synthetic((3, H, H), 8, i) for i in range(N)])
    ws = he_normal_weights(layers, 3, seed=5)
    st = ConvStack(ts, cfg, layers, N, H)
    st.set_weights(ws)
    want = st.forward(torch.from_numpy(x).cuda()).cpu()
    pipe = StackPipeline(ts, cfg, layers, N, H, chunks=chunks)
    assert pipe.bounds[0][0] == 0 and pipe.bounds[-1][1] == N
    assert all(b > a for a, b in pipe.bounds) and all(p[1] == q[0] for p, q in zip(pipe.bounds, pipe.bounds[1:]))
    pipe.set_weights(ws)
    xh = torch.from_numpy(x).pin_memory()
    yh = torch.empty(pipe.out_shape, dtype=torch.float32).pin_memory()
    for _ in range(2):  # the second call reuses every buffer and event
        pipe(xh, yh)
        torch.cuda.synchronize()
        assert torch.equal(yh.view(torch.int32), want.view(torch.int32))


@pytest.mark.parametrize("cs", ["linear", "pairwise"])
def test_fused_output_input_transform_matches_k4_then_k1(cs):
    """wino_output_input_transform (K4 of a layer + ReLU / max-pool + K1 of the next layer in one
    kernel, the activation only in shared memory) writes the V that wino_output_transform_act
    followed by wino_input_transform writes, bit for bit: partial edge tiles, odd sizes after
    pooling, several planes per block, planes spanning several thread rounds, tile padding."""
    import ctypes
    from paper_1803_10986_b200 import _native
    lib = _native.lib()
    s = torch.cuda.current_stream().cuda_stream
    for m, pts in ((6, P8), (4, "0,1,-1,1/2,-1/2,inf"), (3, "0,1,-1,2,-2")):
        ts = W.build_transforms(3, m, W.parse_points(pts))
        for (N, C, K, H, Wd, K2) in [(3, 5, 16, 20, 26, 9), (7, 8, 64, 14, 14, 16), (2, 3, 32, 70, 52, 8)]:
            for pool in ((0, 1) if m % 2 == 0 else (0,)):
                cfg = W.ConvConfig("fp32", "huffman", cs)
                op = W.layer_op(ts, cfg, N, C, H, Wd, K, 1)
                Ho, Wo = op.layout.Ho, op.layout.Wo
                H2, W2 = (Ho // 2, Wo // 2) if pool else (Ho, Wo)
                nxt = W.layer_op(ts, cfg, N, K, H2, W2, K2, 1)
                if not lib.wino_output_input_supported(op.plan.handle, ctypes.byref(op.shape), pool,
                                                       ctypes.byref(nxt.shape)):
                    assert nxt.layout.Cp != K, (m, N, C, K, H, Wd, pool)   # only padded channels may refuse
                    continue
                nxt.prepare(_native.PREPARE_K4K1)
                x = torch.from_numpy(O.synthetic((N, C, H, Wd), 21, 0)).cuda()
                w = torch.from_numpy(O.synthetic((K, C, 3, 3), 21, 1)).cuda()
                M = op.contract(op.filter_transform(w), op.input_transform(x))
                act = torch.empty((N, K, H2, W2), device="cuda")
                _native.check(lib.wino_output_transform_act(op.plan.handle, ctypes.byref(op.shape), _native.as_ptr(M),
                                                            _native.as_ptr(act), pool, s))
                want = nxt.input_transform(act)
                got = torch.full_like(want, 7.0)
                _native.check(lib.wino_output_input_transform(op.plan.handle, ctypes.byref(op.shape), _native.as_ptr(M),
                                                              pool, ctypes.byref(nxt.shape), _native.as_ptr(got), s))
                torch.cuda.synchronize()
                assert torch.equal(got.view(torch.int32), want.view(torch.int32)), (m, cs, N, C, K, H, Wd, pool)


def test_transforms_smallc_leaves_padding_unwritten_and_unread():
    """wino_transforms_smallc writes only the C real channel rows of V (the rest stays as it was)
    and wino_contract_output_smallc never reads the others: poisoned padding, same bits."""
    import ctypes
    from paper_1803_10986_b200 import _native
    lib = _native.lib()
    s = torch.cuda.current_stream().cuda_stream
    ts = W.build_transforms(3, 6, W.parse_points(P8))
    N, C, K, H, Wd = 3, 3, 24, 32, 40
    op = W.layer_op(ts, W.ConvConfig("fp32", "huffman", "pairwise"), N, C, H, Wd, K, 1)
    assert lib.wino_smallc_supported(op.plan.handle, ctypes.byref(op.shape)) == 2
    op.prepare(_native.PREPARE_CONV | _native.PREPARE_ACT)
    x = torch.from_numpy(O.synthetic((N, C, H, Wd), 5, 0)).cuda()
    w = torch.from_numpy(O.synthetic((K, C, 3, 3), 5, 1)).cuda()
    L = op.layout
    U, V = op.filter_transform(w), op.input_transform(x)
    want = torch.empty((N, K, L.Ho, L.Wo), device="cuda")
    _native.check(lib.wino_output_transform_act(op.plan.handle, ctypes.byref(op.shape), _native.as_ptr(op.contract(U, V)),
                                                _native.as_ptr(want), 0, s))
    U2 = torch.full_like(U, float("nan"))
    V2 = torch.full_like(V, float("nan"))
    _native.check(lib.wino_transforms_smallc(op.plan.handle, ctypes.byref(op.shape), _native.as_ptr(x), _native.as_ptr(w),
                                             _native.as_ptr(U2), _native.as_ptr(V2), s))
    torch.cuda.synchronize()
    Vv, V2v = V.view(L.P, -1, L.Cp, L.bn), V2.view(L.P, -1, L.Cp, L.bn)
    assert torch.equal(V2v[:, :, :C].view(torch.int32), Vv[:, :, :C].view(torch.int32))   # real rows: same bits
    assert torch.isnan(V2v[:, :, C:]).all()                                             # padding: untouched
    got = torch.full_like(want, 7.0)
    _native.check(lib.wino_contract_output_smallc(op.plan.handle, ctypes.byref(op.shape), _native.as_ptr(U2),
                                                  _native.as_ptr(V2), _native.as_ptr(got), 1, s))
    torch.cuda.synchronize()
    assert torch.equal(got.view(torch.int32), want.view(torch.int32))
