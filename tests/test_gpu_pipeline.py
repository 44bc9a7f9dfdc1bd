"""HostPipeline (the end-to-end host-buffer API used for bench.py's e2e leg):
chunked H2D | K1-K3-K4 | D2H on three streams, optionally captured into a CUDA
graph -- must give the same bits as the one-shot device path."""
import numpy as np
import pytest

from oracle import wino_oracle as O

pytestmark = pytest.mark.gpu
W = pytest.importorskip("paper_1803_10986_b200")
torch = pytest.importorskip("torch")


@pytest.mark.parametrize("mode", ["exact", "tcf_bf16"])
@pytest.mark.parametrize("chunks,graph", [(1, False), (3, False), (4, True), ([3, 2, 1, 1], True)],
                         ids=lambda v: str(v))
def test_pipeline_bits(mode, chunks, graph):
    N, C, H, K, pad = 7, 24, 13, 20, 1
    ts = W.build_transforms(3, 2, W.parse_points("0,1,-1,inf"))
    x = O.synthetic((N, C, H, H), 11, 0)
    w = O.synthetic((K, C, 3, 3), 11, 1)
    want = W.conv2d_layer(ts, x, w, W.ConvConfig(), pad=pad, contraction=mode)
    xh = torch.from_numpy(x).pin_memory()
    wh = torch.from_numpy(w).pin_memory()
    yh = torch.empty(want.shape, dtype=torch.float32).pin_memory()
    pipe = W.HostPipeline(ts, W.ConvConfig(), N, C, H, H, K, pad, chunks=chunks, contraction=mode, graph=graph)
    for _ in range(3):  # eager, capture, replay
        yh.zero_()
        pipe(xh, wh, yh)
        torch.cuda.synchronize()
        assert np.array_equal(yh.numpy().view(np.uint32), want.view(np.uint32))
    # a replay reads the host buffer's current contents
    xh.mul_(-1)
    pipe(xh, wh, yh)
    torch.cuda.synchronize()
    want2 = W.conv2d_layer(ts, -x, w, W.ConvConfig(), pad=pad, contraction=mode)
    assert np.array_equal(yh.numpy().view(np.uint32), want2.view(np.uint32))


def test_pipeline_rejects_bad_chunks():
    ts = W.build_transforms(3, 2, W.parse_points("0,1,-1,inf"))
    with pytest.raises(ValueError):
        W.HostPipeline(ts, W.ConvConfig(), 4, 3, 8, 8, 2, 1, chunks=[2, 1])
