"""Per-chunk event timeline of HostPipeline (eager, cfg2): H2D end, compute end, D2H end."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import ctypes
import numpy as np
import torch
import os as _os, sys as _sys  # noqa: E401
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import tuning_env  # noqa: E402,F401  (WINO_* env -> libwino tuning keys)
import paper_1803_10986_b200 as W
from paper_1803_10986_b200 import pointsets, _native
from paper_1803_10986_b200 import device as D

N, C, H, K, pad = 32, 128, 28, 128, 1
ts = W.build_transforms(3, 2, W.parse_points(pointsets.curated_text(4, 2)))
cfg = W.ConvConfig()
rng = np.random.default_rng(0)
xh = torch.from_numpy(rng.random((N, C, H, H), dtype=np.float32) * 2 - 1).pin_memory()
wh = torch.from_numpy(rng.standard_normal((K, C, 3, 3), dtype=np.float32) * 0.04).pin_memory()
yh = torch.empty((N, K, H, H), dtype=torch.float32).pin_memory()
def run_once(pipe, lib, nb, ev, e0):
    cur = torch.cuda.current_stream()
    e0.record(cur)
    for s in (pipe.s_h2d, pipe.s_cmp, pipe.s_d2h):
        s.wait_stream(cur)
    with torch.cuda.stream(pipe.s_h2d):
        pipe.w_dev.copy_(wh, non_blocking=True)
        for i, ((a, b), (e_in, _)) in enumerate(zip(pipe.bounds, pipe.ev)):
            pipe.x_dev[a:b].copy_(xh[a:b], non_blocking=True)
            e_in.record(pipe.s_h2d)
            ev["h"][i].record(pipe.s_h2d)
    with torch.cuda.stream(pipe.s_cmp):
        sc = pipe.s_cmp.cuda_stream
        pipe.s_cmp.wait_event(pipe.ev[0][0])
        _native.check(lib.wino_filter_transform(pipe.full.plan.handle, ctypes.byref(pipe.full.shape),
                                                D.ptr(pipe.w_dev), D.ptr(pipe.U), sc))
        for i, (op, ws, (a, b), (e_in, e_out)) in enumerate(zip(pipe.ops, pipe.ws, pipe.bounds, pipe.ev)):
            pipe.s_cmp.wait_event(e_in)
            ev["c0"][i].record(pipe.s_cmp)
            V = ws
            M = ws[(op.layout.v_bytes + 255) // 256 * 64:]
            sh = ctypes.byref(op.shape)
            _native.check(lib.wino_input_transform(op.plan.handle, sh, D.ptr(pipe.x_dev[a:b]), D.ptr(V), sc))
            _native.check(lib.wino_contract(op.plan.handle, sh, D.ptr(pipe.U), D.ptr(V), D.ptr(M), sc))
            _native.check(lib.wino_output_transform(op.plan.handle, sh, D.ptr(M), D.ptr(pipe.y_dev[a:b]), sc))
            e_out.record(pipe.s_cmp)
            ev["c"][i].record(pipe.s_cmp)
    with torch.cuda.stream(pipe.s_d2h):
        for i, ((a, b), (_, e_out)) in enumerate(zip(pipe.bounds, pipe.ev)):
            pipe.s_d2h.wait_event(e_out)
            yh[a:b].copy_(pipe.y_dev[a:b], non_blocking=True)
            ev["d"][i].record(pipe.s_d2h)
    cur.wait_stream(pipe.s_d2h)


for chunks in (4, 8, [8, 7, 6, 5, 4, 2]):
    pipe = W.HostPipeline(ts, cfg, N, C, H, H, K, pad, chunks=chunks, graph=False)
    lib = _native.lib()
    nb = len(pipe.bounds)
    ev = {k: [torch.cuda.Event(enable_timing=True) for _ in range(nb)] for k in ("h", "c0", "c", "d")}
    e0 = torch.cuda.Event(enable_timing=True)
    run_once(pipe, lib, nb, ev, e0)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        run_once(pipe, lib, nb, ev, e0)
    for rep in range(4):
        g.replay()
        torch.cuda.synchronize()
    print(f"graph, chunks {chunks}:")
    for i in range(nb):
        f = lambda k: e0.elapsed_time(ev[k][i]) * 1e3
        print(f"  {i}: h2d end {f('h'):6.0f}  cmp start {f('c0'):6.0f} end {f('c'):6.0f}  d2h end {f('d'):6.0f}")
for chunks in ():
    pipe = W.HostPipeline(ts, cfg, N, C, H, H, K, pad, chunks=chunks, graph=False)
    lib = _native.lib()
    nb = len(pipe.bounds)
    for rep in range(4):
        ev = {k: [torch.cuda.Event(enable_timing=True) for _ in range(nb)] for k in ("h", "c0", "c", "d")}
        e0 = torch.cuda.Event(enable_timing=True)
        cur = torch.cuda.current_stream()
        torch.cuda.synchronize()
        e0.record(cur)
        for s in (pipe.s_h2d, pipe.s_cmp, pipe.s_d2h):
            s.wait_stream(cur)
        with torch.cuda.stream(pipe.s_h2d):
            pipe.w_dev.copy_(wh, non_blocking=True)
            for i, ((a, b), (e_in, _)) in enumerate(zip(pipe.bounds, pipe.ev)):
                pipe.x_dev[a:b].copy_(xh[a:b], non_blocking=True)
                e_in.record(pipe.s_h2d)
                ev["h"][i].record(pipe.s_h2d)
        with torch.cuda.stream(pipe.s_cmp):
            sc = pipe.s_cmp.cuda_stream
            pipe.s_cmp.wait_event(pipe.ev[0][0])
            _native.check(lib.wino_filter_transform(pipe.full.plan.handle, ctypes.byref(pipe.full.shape),
                                                    D.ptr(pipe.w_dev), D.ptr(pipe.U), sc))
            for i, (op, ws, (a, b), (e_in, e_out)) in enumerate(zip(pipe.ops, pipe.ws, pipe.bounds, pipe.ev)):
                pipe.s_cmp.wait_event(e_in)
                ev["c0"][i].record(pipe.s_cmp)
                V = ws
                M = ws[(op.layout.v_bytes + 255) // 256 * 64:]
                sh = ctypes.byref(op.shape)
                _native.check(lib.wino_input_transform(op.plan.handle, sh, D.ptr(pipe.x_dev[a:b]), D.ptr(V), sc))
                _native.check(lib.wino_contract(op.plan.handle, sh, D.ptr(pipe.U), D.ptr(V), D.ptr(M), sc))
                _native.check(lib.wino_output_transform(op.plan.handle, sh, D.ptr(M), D.ptr(pipe.y_dev[a:b]), sc))
                e_out.record(pipe.s_cmp)
                ev["c"][i].record(pipe.s_cmp)
        with torch.cuda.stream(pipe.s_d2h):
            for i, ((a, b), (_, e_out)) in enumerate(zip(pipe.bounds, pipe.ev)):
                pipe.s_d2h.wait_event(e_out)
                yh[a:b].copy_(pipe.y_dev[a:b], non_blocking=True)
                ev["d"][i].record(pipe.s_d2h)
        cur.wait_stream(pipe.s_d2h)
        torch.cuda.synchronize()
        if rep == 3:
            print(f"chunks {chunks}:")
            for i in range(nb):
                f = lambda k: e0.elapsed_time(ev[k][i]) * 1e3
                print(f"  {i}: h2d end {f('h'):6.0f}  cmp start {f('c0'):6.0f} end {f('c'):6.0f}  d2h end {f('d'):6.0f}")
