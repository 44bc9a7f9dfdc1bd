"""Transform-kernel (K1+K2, K4) micro-benchmark: times the generated transforms
of a real point set against the same kernels generated from trivial one-leaf
programs (memory traffic only) to separate arithmetic from memory cost.

  python tools/xform_bench.py --shape 64,256,28,256 --m 6
"""
import argparse
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import os as _os, sys as _sys  # noqa: E401
_sys.path.insert(0, _os.path.dirname(_os.path.abspath(__file__)))
import tuning_env  # noqa: E402,F401  (WINO_* env -> libwino tuning keys)
import paper_1803_10986_b200 as W  # noqa: E402
from paper_1803_10986_b200 import _native, pointsets  # noqa: E402


def trivial(rows, cols):
    starts, ops = [0], []
    for i in range(rows):
        ops.append((0, i % cols, 1.0))
        starts.append(len(ops))
    return (np.array(starts, dtype=np.int32), ops, cols)


def time_it(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="64,256,28,256")
    ap.add_argument("--m", type=int, default=6)
    ap.add_argument("--contraction", default="exact")
    a = ap.parse_args()
    N, C, H, K = (int(v) for v in a.shape.split(","))
    r, m = 3, a.m
    n = r + m - 1
    ts = W.build_transforms(r, m, W.parse_points(pointsets.curated_text(n, 2)))
    cfg = W.ConvConfig()
    real = W.engine.get_plan(ts, cfg, a.contraction)
    triv = _native.Plan(r, m, "fp32", "linear", a.contraction, trivial(n, r), trivial(n, n), trivial(m, n))
    L = real.layout(N, C, H, H, K, 1)
    g = torch.Generator(device="cuda").manual_seed(7)
    x = torch.randn(N, C, H, H, device="cuda", generator=g)
    w = torch.randn(K, C, r, r, device="cuda", generator=g)
    U = torch.empty(L.u_bytes // 4 + 64, device="cuda")
    V = torch.empty(L.v_bytes // 4 + 64, device="cuda")
    M = torch.randn(L.m_bytes // 4 + 64, device="cuda")
    y = torch.empty(N, K, L.Ho, L.Wo, device="cuda")
    shp = _native.LayerShape(N, C, H, H, K, 1)
    lib = _native.lib()
    s = torch.cuda.current_stream().cuda_stream
    P = _native.as_ptr
    res = {"shape": [N, C, H, K], "m": m}
    for name, plan in (("real", real), ("trivial", triv)):
        res[name + "_transforms_us"] = time_it(lambda: _native.check(lib.wino_transforms(
            plan.handle, ctypes.byref(shp), P(x), P(w), P(U), P(V), s)))
        res[name + "_input_us"] = time_it(lambda: _native.check(lib.wino_input_transform(
            plan.handle, ctypes.byref(shp), P(x), P(V), s)))
        res[name + "_output_us"] = time_it(lambda: _native.check(lib.wino_output_transform(
            plan.handle, ctypes.byref(shp), P(M), P(y), s)))
    import zlib
    _native.check(lib.wino_input_transform(real.handle, ctypes.byref(shp), P(x), P(V), s))
    torch.cuda.synchronize()
    res["V_crc32"] = zlib.crc32(V[: L.v_bytes // 4].cpu().numpy().tobytes())  # same bits across K1 variants
    k1 = 4 * N * C * H * H + L.elem_bytes_uv * L.P * L.T * C
    k4 = 4 * L.P * L.T * K + 4 * N * K * L.Ho * L.Wo
    for name in ("real", "trivial"):
        res[name + "_input_gbs"] = k1 / res[name + "_input_us"] / 1e3
        res[name + "_output_gbs"] = k4 / res[name + "_output_us"] / 1e3
    print(json.dumps(res))


if __name__ == "__main__":
    main()
