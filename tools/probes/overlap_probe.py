"""Device-resident step with the HBM-bound transforms overlapped with the
FP32-bound contraction: the batch is split into image chunks; K1 of chunk i+1
(stream 1) and K4 of chunk i-1 (stream 3) run while K3 of chunk i (stream 2)
occupies the FP32 pipes.  Compares against the sequential 4-kernel step, both
CUDA-graph captured, L2 flushed between steps.

  python tools/probes/overlap_probe.py [--config cfg2] [--chunks 1,2,4]
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import os as _os, sys as _sys  # noqa: E401
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import tuning_env  # noqa: E402,F401  (WINO_* env -> libwino tuning keys)
import paper_1803_10986_b200 as W  # noqa: E402
from paper_1803_10986_b200 import _native  # noqa: E402

CFG = {"cfg2": (3, 2, "0,1,-1,inf", 32, 128, 128, 28, 1, "linear"),
       "cfg3_m6": (3, 6, "0,-1,1,1/2,-1/2,2,-2,inf", 64, 256, 256, 28, 1, "linear"),
       "cfg4_m4": (5, 4, "0,-1,1,1/2,-1/2,2,-2,inf", 32, 512, 512, 14, 2, "pairwise")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--chunks", default="1,2,4")
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    r, m, pts, N, C, K, H, pad, cs = CFG[a.config]
    ts = W.build_transforms(r, m, W.parse_points(pts))
    cfg = W.ConvConfig("fp32", "huffman", cs)
    lib = _native.lib()
    x = torch.rand((N, C, H, H), device="cuda") * 2 - 1
    w = torch.randn((K, C, r, r), device="cuda") * 0.05
    full = W.layer_op(ts, cfg, N, C, H, H, K, pad)
    y_ref = torch.empty(full.out_shape, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    clean = torch.ones(64 << 20, dtype=torch.float32, device="cuda")
    flops = 2 * N * K * C * full.layout.Ho * full.layout.Wo * r * r
    for S in [int(v) for v in a.chunks.split(",")]:
        bounds = [(i * N // S, (i + 1) * N // S) for i in range(S)]
        ops = [W.layer_op(ts, cfg, b - e0, C, H, H, K, pad) for e0, b in bounds]
        U = torch.empty((full.layout.P, full.layout.Cp, full.layout.Kp), device="cuda")
        Vs = [torch.empty((o.layout.P, o.layout.Cp, o.layout.Tp), device="cuda") for o in ops]
        Ms = [torch.empty((o.layout.P, o.layout.Kp, o.layout.Tp), device="cuda") for o in ops]
        y = torch.empty(full.out_shape, device="cuda")
        s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
        e1 = [torch.cuda.Event() for _ in ops]
        e3 = [torch.cuda.Event() for _ in ops]

        def step():
            cur = torch.cuda.current_stream()
            for s in (s1, s2, s3):
                s.wait_stream(cur)
            _native.check(lib.wino_filter_transform(full.plan.handle, ctypes.byref(full.shape), _native.as_ptr(w),
                                                    _native.as_ptr(U), s1.cuda_stream))
            for i, (o, (b0, b1)) in enumerate(zip(ops, bounds)):
                sh = ctypes.byref(o.shape)
                _native.check(lib.wino_input_transform(o.plan.handle, sh, _native.as_ptr(x[b0:b1]),
                                                       _native.as_ptr(Vs[i]), s1.cuda_stream))
                e1[i].record(s1)
                s2.wait_event(e1[i])
                _native.check(lib.wino_contract(o.plan.handle, sh, _native.as_ptr(U), _native.as_ptr(Vs[i]),
                                                _native.as_ptr(Ms[i]), s2.cuda_stream))
                e3[i].record(s2)
                s3.wait_event(e3[i])
                _native.check(lib.wino_output_transform(o.plan.handle, sh, _native.as_ptr(Ms[i]),
                                                        _native.as_ptr(y[b0:b1]), s3.cuda_stream))
            for s in (s1, s2, s3):
                cur.wait_stream(s)

        step()
        torch.cuda.synchronize()
        if S == 1:
            y_ref.copy_(y)
        same = bool(torch.equal(y, y_ref))
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            step()
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        ts_ = []
        for _ in range(a.reps):
            flush.zero_()
            clean.sum()
            e0, e9 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e9.record()
            torch.cuda.synchronize()
            ts_.append(e0.elapsed_time(e9))
        ts_.sort()
        ms = ts_[len(ts_) // 2]
        print(f"{a.config} chunks={S}: {ms * 1e3:.1f} us/step (median)  {flops / ms / 1e9:.1f} TFLOP/s  "
              f"bitwise_equal_to_1chunk={same}", flush=True)


if __name__ == "__main__":
    main()
