"""Kernels of different layers/chunks running concurrently on several streams
must not disturb each other.  Regression test for a cross-proxy hazard in the
contraction pipeline: consumer warps read a stage with generic-proxy loads and
release it through an mbarrier; the producer's refill is an async-proxy bulk
copy, which needs a fence.proxy.async after the acquire -- without it the
refill overtook the reads whenever a load/store-heavy kernel (K1/K4 of another
chunk) shared the SMs, corrupting whole tiles of M (10 of 10 runs here)."""
import ctypes

import numpy as np
import pytest

from oracle import wino_oracle as O

pytestmark = pytest.mark.gpu
W = pytest.importorskip("paper_1803_10986_b200")
torch = pytest.importorskip("torch")
from paper_1803_10986_b200 import _native  # noqa: E402


def _three_stream_step(ts, cfg, x, w, K, pad, S):
    lib = _native.lib()
    N, C, H, _ = x.shape
    r = w.shape[-1]
    full = W.layer_op(ts, cfg, N, C, H, H, K, pad)
    bounds = [(i * N // S, (i + 1) * N // S) for i in range(S)]
    ops = [W.layer_op(ts, cfg, b - a, C, H, H, K, pad) for a, b in bounds]
    Us = [torch.empty((o.layout.P, o.layout.Cp, o.layout.Kp), device="cuda") for o in ops]
    Vs = [torch.empty((o.layout.P, o.layout.Cp, o.layout.Tp), device="cuda") for o in ops]
    Ms = [torch.empty((o.layout.P, o.layout.Kp, o.layout.Tp), device="cuda") for o in ops]
    y = torch.empty(full.out_shape, device="cuda")
    ss = [torch.cuda.Stream() for _ in range(3)]
    cur = torch.cuda.current_stream()
    for s in ss:
        s.wait_stream(cur)
    evs = []
    P = _native.as_ptr
    for i, (o, (a, b)) in enumerate(zip(ops, bounds)):
        sh = ctypes.byref(o.shape)
        _native.check(lib.wino_filter_transform(o.plan.handle, sh, P(w), P(Us[i]), ss[0].cuda_stream))
        _native.check(lib.wino_input_transform(o.plan.handle, sh, P(x[a:b]), P(Vs[i]), ss[0].cuda_stream))
        e = torch.cuda.Event()
        e.record(ss[0])
        ss[1].wait_event(e)
        _native.check(lib.wino_contract(o.plan.handle, sh, P(Us[i]), P(Vs[i]), P(Ms[i]), ss[1].cuda_stream))
        e2 = torch.cuda.Event()
        e2.record(ss[1])
        ss[2].wait_event(e2)
        _native.check(lib.wino_output_transform(o.plan.handle, sh, P(Ms[i]), P(y[a:b]), ss[2].cuda_stream))
        evs += [e, e2]
    for s in ss:
        cur.wait_stream(s)
    torch.cuda.synchronize()
    return y


@pytest.mark.parametrize("case", [(3, 6, "0,-1,1,1/2,-1/2,2,-2,inf", 64, 256, 256, 28, 1, "linear"),
                                  (3, 6, "0,-1,1,1/2,-1/2,2,-2,inf", 64, 256, 256, 28, 1, "pairwise"),
                                  (3, 2, "0,1,-1,inf", 32, 128, 128, 28, 1, "linear")],
                         ids=lambda c: f"m{c[1]}-{c[8]}")
def test_concurrent_chunks_bitwise(case):
    r, m, pts, N, C, K, H, pad, cs = case
    ts = W.build_transforms(r, m, W.parse_points(pts))
    cfg = W.ConvConfig("fp32", "huffman", cs)
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.rand((N, C, H, H), device="cuda", generator=g) * 2 - 1
    w = torch.randn((K, C, r, r), device="cuda", generator=g) * 0.05
    want = W.layer_op(ts, cfg, N, C, H, H, K, pad)(x, w)
    for S in (2, 4, 2, 4, 2):
        y = _three_stream_step(ts, cfg, x, w, K, pad, S)
        assert torch.equal(y, want), S


def test_pipeline_chunks_with_different_blockings():
    """HostPipeline chunks whose sizes pick different contraction tiles each get a
    U blocked for their own layout."""
    ts = W.build_transforms(3, 2, W.parse_points("0,1,-1,inf"))
    N, C, H, K = 12, 128, 28, 128
    full = W.layer_op(ts, W.ConvConfig(), 8, C, H, H, K, 1).layout
    part = W.layer_op(ts, W.ConvConfig(), 4, C, H, H, K, 1).layout
    assert (full.bm, full.bn) != (part.bm, part.bn)  # the premise of the test
    x = O.synthetic((N, C, H, H), 2, 0)
    w = O.synthetic((K, C, 3, 3), 2, 1)
    want = W.conv2d_layer(ts, x, w, W.ConvConfig(), pad=1)
    xh, wh = torch.from_numpy(x).pin_memory(), torch.from_numpy(w).pin_memory()
    yh = torch.empty(want.shape, dtype=torch.float32).pin_memory()
    pipe = W.HostPipeline(ts, W.ConvConfig(), N, C, H, H, K, 1, chunks=[8, 4], graph=False)
    pipe(xh, wh, yh)
    torch.cuda.synchronize()
    assert np.array_equal(yh.numpy().view(np.uint32), want.view(np.uint32))


def test_contract_rejects_a_u_blocked_for_another_shape():
    """A U transformed for one batch size must not be contracted under a shape whose
    contraction tile (hence U blocking) differs: wino_contract fails loudly."""
    import ctypes
    from paper_1803_10986_b200 import _native
    from paper_1803_10986_b200 import device as D
    ts = W.build_transforms(3, 2, W.parse_points("0,1,-1,inf"))
    C, H, K = 128, 28, 128
    big = W.layer_op(ts, W.ConvConfig(), 8, C, H, H, K, 1)
    small = W.layer_op(ts, W.ConvConfig(), 4, C, H, H, K, 1)
    assert (big.layout.bm, big.layout.Cp, big.layout.Kp) != (small.layout.bm, small.layout.Cp, small.layout.Kp)
    w = torch.from_numpy(O.synthetic((K, C, 3, 3), 2, 1)).cuda()
    x = torch.from_numpy(O.synthetic((4, C, H, H), 2, 0)).cuda()
    U = big.filter_transform(w)            # blocked for the 8-image shape
    V = small.input_transform(x)
    M = torch.empty((small.layout.P, small.layout.Kp, small.layout.Tp), device="cuda")
    lib = _native.lib()
    rc = lib.wino_contract(small.plan.handle, ctypes.byref(small.shape), D.ptr(U), D.ptr(V), D.ptr(M),
                           D.stream_handle())
    assert rc != 0 and b"blocking" in lib.wino_last_error()
    # transformed again for the shape it is used with: accepted, and the layer is right
    _native.check(lib.wino_filter_transform(small.plan.handle, ctypes.byref(small.shape), D.ptr(w), D.ptr(U),
                                            D.stream_handle()))
    _native.check(lib.wino_contract(small.plan.handle, ctypes.byref(small.shape), D.ptr(U), D.ptr(V), D.ptr(M),
                                    D.stream_handle()))
    y = small.output_transform(M)
    want = W.conv2d_layer(ts, x, w, W.ConvConfig(), pad=1)
    assert torch.equal(y.view(torch.int32), want.view(torch.int32))
