"""Layer-level Winograd convolution on the B200 -- the north-star hot path.

The reference has no layer API; its arithmetic is reached by
calling ``conv_2d(ts, w[k], X[tile], cfg)`` for every (output channel, tile)
of the zero-padded image.  ``conv2d_layer`` computes exactly
those numbers in four device stages:

  K2 filter transform    U[p][c][k] = (G w[k,c] G^T)[p]
  K1 input transform     V[p][c][t] = (B^T d[t,c] B)[p]   (gather + zero pad fused)
  K3 contraction         M[p][k][t] = sum_c U[p][c][k] V[p][c][t]   (linear | pairwise order)
  K4 output transform    y[n,k,tile] = A^T M[.][k][t] A   (crop + NCHW write-back)
"""

from __future__ import annotations

import ctypes
import threading

import numpy as np

from . import _native
from . import device as D
from .engine import ConvConfig, _input_dtype, _output_dtype, get_plan
from .transforms import TransformSet

_ws_lock = threading.Lock()
_workspaces: dict = {}


def _workspace(nbytes: int, stream: int):
    """Grow-only scratch for U, V and M, one per (device, stream): calls on different
    streams (or threads using different streams) never share it.  The buffer is
    allocated while its stream is current, so when it grows the caching allocator
    recycles the old block only after the work queued on that stream."""
    torch = D.torch
    dev = torch.cuda.current_device()
    key = (dev, stream)
    with _ws_lock:
        buf = _workspaces.get(key)
        if buf is None or buf.numel() < nbytes:
            _workspaces.pop(key, None)
            s = torch.cuda.ExternalStream(stream) if stream != torch.cuda.current_stream().cuda_stream else None
            with torch.cuda.stream(s) if s is not None else _nullcontext():
                buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=f"cuda:{dev}")
            _workspaces[key] = buf
        return buf


class _nullcontext:
    def __enter__(self):
        return None

    def __exit__(self, *a):
        return False


class LayerOp:
    """One layer geometry bound to a compiled plan (reusable across calls)."""

    def __init__(self, ts: TransformSet, cfg: ConvConfig, N, C, H, W, K, pad, contraction="exact"):
        if pad < 0:
            raise ValueError("pad must be >= 0")
        self.ts, self.cfg, self.contraction = ts, cfg, contraction
        self.plan = get_plan(ts, cfg, contraction)
        self.shape = _native.LayerShape(N, C, H, W, K, pad)
        self.layout = self.plan.layout(N, C, H, W, K, pad)
        self.N, self.C, self.H, self.W, self.K, self.pad = N, C, H, W, K, pad
        self.out_shape = (N, K, self.layout.Ho, self.layout.Wo)
        self.in_dtype = _input_dtype(cfg)
        self.out_dtype = _output_dtype(cfg)
        self.prepare(_native.PREPARE_CONV)

    def prepare(self, flags):
        """Compile (concurrently, cached on disk) the generated kernels this layer launches."""
        _native.check(_native.lib().wino_plan_prepare(self.plan.handle, ctypes.byref(self.shape), flags),
                      "plan_prepare")

    @property
    def direct_flops(self) -> int:
        """Direct-convolution-equivalent FLOPs, 2 N K C Ho Wo r^2."""
        r = self.ts.n_h
        return 2 * self.N * self.K * self.C * self.layout.Ho * self.layout.Wo * r * r

    @property
    def contraction_flops(self) -> int:
        L = self.layout
        return 2 * L.P * L.T * self.C * self.K

    def __call__(self, x, w, out=None, workspace=None, stream=None):
        """x, w: contiguous CUDA tensors of the plan's input dtype."""
        L = self.layout
        if out is None:
            out = D.empty(self.out_shape, self.out_dtype)
        s = D.stream_handle() if stream is None else stream
        ws = workspace if workspace is not None else _workspace(L.workspace_bytes, s)
        _native.check(_native.lib().wino_conv2d(self.plan.handle, ctypes.byref(self.shape), D.ptr(x), D.ptr(w),
                                                D.ptr(out), D.ptr(ws), ws.numel(), s), "conv2d")
        return out

    def call_nhwc(self, x, w, out=None, workspace=None, stream=None):
        """x (N, H, W, C), w (K, C, r, r) contiguous CUDA tensors -> y (N, Ho, Wo, K): the
        NHWC-native gather / store kernels (wino_conv2d_nhwc), no permuted copies."""
        L = self.layout
        N, K, Ho, Wo = self.out_shape
        if not getattr(self, "_nhwc_ready", False):
            self.prepare(_native.PREPARE_NHWC)  # compile the four kernels concurrently
            self._nhwc_ready = True
        if out is None:
            out = D.empty((N, Ho, Wo, K), self.out_dtype)
        s = D.stream_handle() if stream is None else stream
        ws = workspace if workspace is not None else _workspace(L.workspace_bytes, s)
        _native.check(_native.lib().wino_conv2d_nhwc(self.plan.handle, ctypes.byref(self.shape), D.ptr(x), D.ptr(w),
                                                     D.ptr(out), D.ptr(ws), ws.numel(), s), "conv2d_nhwc")
        return out

    @property
    def fused_exact_supported(self) -> bool:
        """alpha^2 <= 16, fp32, FP32-pipe contraction: K3 + K4 can run as one exact kernel."""
        return bool(_native.lib().wino_fused_supported(self.plan.handle, ctypes.byref(self.shape)))

    def call_fused(self, x, w, mode=0, out=None, stream=None):
        """K2 + K1, then the contraction and the output transform (+ ReLU / ReLU + 2x2 max-pool
        for mode 1 / 2) in ONE exact kernel: the alpha^2 accumulators of every (filter, tile)
        pair are parked in tensor memory, M never goes to HBM (wino_conv2d_fused).  Same bits
        as __call__ (followed by relu / max-pool)."""
        lib = _native.lib()
        need = ctypes.c_size_t(0)
        _native.check(lib.wino_fused_workspace(self.plan.handle, ctypes.byref(self.shape), ctypes.byref(need)),
                      "fused_workspace")
        N, K, Ho, Wo = self.out_shape
        if out is None:
            out = D.empty((N, K, Ho // 2, Wo // 2) if mode == 2 else self.out_shape, self.out_dtype)
        s = D.stream_handle() if stream is None else stream
        ws = _workspace(need.value, s)
        _native.check(lib.wino_conv2d_fused(self.plan.handle, ctypes.byref(self.shape), D.ptr(x), D.ptr(w), D.ptr(out),
                                            mode, D.ptr(ws), ws.numel(), s), "conv2d_fused")
        return out

    # -- individual stages (tests, profiling) --------------------------------
    @property
    def tensor_core(self) -> bool:
        return self.contraction.startswith(("tc_", "tcf_"))

    @property
    def fused(self) -> bool:
        """tcf_* modes: contraction + output transform in one kernel (no M)."""
        return self.contraction.startswith("tcf_")

    def _uv_dtype(self):
        if self.contraction in ("tc_bf16", "tcf_bf16"):
            return D.torch.bfloat16
        if self.contraction in ("tc_fp16", "tcf_fp16"):
            return D.torch.float16
        return D.torch.float64 if self.cfg.precision == "fp64" else D.torch.float32

    def _m_dtype(self):
        return D.torch.float32 if self.tensor_core else self._uv_dtype()

    def filter_transform(self, w):
        L = self.layout
        U = D.torch.empty((L.P, L.Cp, L.Kp), dtype=self._uv_dtype(), device="cuda")
        _native.check(_native.lib().wino_filter_transform(self.plan.handle, ctypes.byref(self.shape), D.ptr(w),
                                                          D.ptr(U), D.stream_handle()), "filter_transform")
        return U

    def input_transform(self, x):
        L = self.layout
        V = D.torch.empty((L.P, L.Cp, L.Tp), dtype=self._uv_dtype(), device="cuda")
        _native.check(_native.lib().wino_input_transform(self.plan.handle, ctypes.byref(self.shape), D.ptr(x),
                                                         D.ptr(V), D.stream_handle()), "input_transform")
        return V

    # Tensor-core modes keep U/V as 16-bit UMMA operands:
    #   X16[p][row/128][c/32][(c/8)%4][(row%128)/8][row%8][c%8]
    # Fused modes (tcf_*): every 16-channel stage of a (row block, all P) is contiguous:
    #   X16[row/B][c/16][p][(c/8)%2][(row%B)/8][row%8][c%8],  B = 128 (V) or NK (U)
    def _tc_unpack(self, X, R, B=128):
        L = self.layout
        if self.fused:
            return X.reshape(R // B, L.Cp // 16, L.P, 2, B // 8, 8, 8).permute(2, 1, 3, 6, 0, 4, 5).reshape(
                L.P, L.Cp, R)
        return X.reshape(L.P, R // 128, L.Cp // 32, 4, 16, 8, 8).permute(0, 2, 3, 6, 1, 4, 5).reshape(L.P, L.Cp, R)

    def _tc_pack(self, X, R, B=128):
        L = self.layout
        if self.fused:
            return X.reshape(L.P, L.Cp // 16, 2, 8, R // B, B // 8, 8).permute(4, 1, 0, 2, 5, 6, 3).contiguous()
        return X.reshape(L.P, L.Cp // 32, 4, 8, R // 128, 16, 8).permute(0, 4, 1, 2, 5, 6, 3).contiguous()

    def unblock_u(self, U):
        """device layout of U -> dense U[P][Cp][Kp]"""
        L = self.layout
        if self.tensor_core:
            return self._tc_unpack(U, L.Kp, L.bm if self.fused else 128)
        return U.reshape(L.P, L.Kp // L.bm, L.Cp, L.bm).permute(0, 2, 1, 3).reshape(L.P, L.Cp, L.Kp)

    def unblock_v(self, V):
        """device layout of V -> dense V[P][Cp][Tp]"""
        L = self.layout
        if self.tensor_core:
            return self._tc_unpack(V, L.Tp)
        return V.reshape(L.P, L.Tp // L.bn, L.Cp, L.bn).permute(0, 2, 1, 3).reshape(L.P, L.Cp, L.Tp)

    def block_u(self, U):
        """dense U[P][Cp][Kp] -> device layout"""
        L = self.layout
        if self.tensor_core:
            return self._tc_pack(U.to(self._uv_dtype()), L.Kp, L.bm if self.fused else 128)
        return U.reshape(L.P, L.Cp, L.Kp // L.bm, L.bm).permute(0, 2, 1, 3).contiguous()

    def block_v(self, V):
        """dense V[P][Cp][Tp] -> device layout"""
        L = self.layout
        if self.tensor_core:
            return self._tc_pack(V.to(self._uv_dtype()), L.Tp)
        return V.reshape(L.P, L.Cp, L.Tp // L.bn, L.bn).permute(0, 2, 1, 3).contiguous()

    def contract(self, U, V):
        L = self.layout
        M = D.torch.empty((L.P, L.Kp, L.Tp), dtype=self._m_dtype(), device="cuda")
        _native.check(_native.lib().wino_contract(self.plan.handle, ctypes.byref(self.shape), D.ptr(U), D.ptr(V),
                                                  D.ptr(M), D.stream_handle()), "contract")
        return M

    def contract_output(self, U, V, out=None):
        """fused modes: y = A^T (sum_c U_p V_p) A straight from the TMEM accumulators"""
        if out is None:
            out = D.empty(self.out_shape, self.out_dtype)
        _native.check(_native.lib().wino_contract_output(self.plan.handle, ctypes.byref(self.shape), D.ptr(U),
                                                         D.ptr(V), D.ptr(out), D.stream_handle()), "contract_output")
        return out

    def output_transform(self, M, out=None):
        if out is None:
            out = D.empty(self.out_shape, self.out_dtype)
        _native.check(_native.lib().wino_output_transform(self.plan.handle, ctypes.byref(self.shape), D.ptr(M),
                                                          D.ptr(out), D.stream_handle()), "output_transform")
        return out


class HostPipeline:
    """Host-buffer convolution with the copies overlapped: the batch is split
    into image chunks; chunk i's H2D copy, chunk i-1's K1-K3-K4 and chunk i-2's
    D2H run concurrently on three streams (PCIe is full duplex).  The filter
    transform K2 runs once per call (U does not depend on the images).

    x_host / y_host must be pinned CPU tensors (N, C, H, W) / (N, K, Ho, Wo).

    `chunks` is a count (equal chunks) or a list of image counts (e.g. decreasing
    sizes shorten the compute + D2H tail after the last H2D).  With `graph=True`
    the second call with the same host buffers captures the whole multi-stream
    pipeline (copies, kernels, cross-stream events) into a CUDA graph and later
    calls replay it -- one launch instead of ~5 per chunk from Python."""

    def __init__(self, ts: TransformSet, cfg: ConvConfig, N, C, H, W, K, pad, chunks=4, contraction="exact",
                 graph=True):
        self.full = layer_op(ts, cfg, N, C, H, W, K, pad, contraction)
        if isinstance(chunks, int):
            chunks = max(1, min(chunks, N))
            self.bounds = [(i * N // chunks, (i + 1) * N // chunks) for i in range(chunks)]
        else:
            sizes = [int(c) for c in chunks]
            if sum(sizes) != N or min(sizes) < 1:
                raise ValueError("chunk sizes must be >= 1 and sum to N")
            edges = np.cumsum([0] + sizes)
            self.bounds = [(int(a), int(b)) for a, b in zip(edges[:-1], edges[1:])]
        self.graph = graph
        self._graphs, self._seen = {}, set()
        self.ops = [layer_op(ts, cfg, b - a, C, H, W, K, pad, contraction) for a, b in self.bounds]
        # U is blocked by the contraction tile the layout picks (wino_host.cu pick());
        # chunks of a different size may pick another blocking: one U per blocking
        self.u_key = [(op.layout.bm, op.layout.Kp, op.layout.Cp) for op in self.ops]
        self.U = {}
        for key, op in zip(self.u_key, self.ops):
            if key not in self.U:
                L = op.layout
                self.U[key] = (op, D.torch.empty((L.P, L.Cp, L.Kp), dtype=op._uv_dtype(), device="cuda"))
        self.ws = [D.torch.empty((op.layout.v_bytes + op.layout.m_bytes + 512) // 4, dtype=D.torch.float32,
                                 device="cuda") for op in self.ops]
        self.x_dev = D.torch.empty((N, C, H, W), dtype=D._DT[self.full.in_dtype], device="cuda")
        self.w_dev = D.torch.empty((K, C, ts.n_h, ts.n_h), dtype=D._DT[self.full.in_dtype], device="cuda")
        self.y_dev = D.empty(self.full.out_shape, self.full.out_dtype)
        self.s_h2d, self.s_cmp, self.s_d2h = D.torch.cuda.Stream(), D.torch.cuda.Stream(), D.torch.cuda.Stream()
        self.ev = [(D.torch.cuda.Event(), D.torch.cuda.Event()) for _ in self.bounds]

    def __call__(self, x_host, w_host, y_host):
        if not self.graph:
            return self._run(x_host, w_host, y_host)
        torch = D.torch
        key = (x_host.data_ptr(), w_host.data_ptr(), y_host.data_ptr())
        g = self._graphs.get(key)
        if g is None and key in self._seen:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self._run(x_host, w_host, y_host)
            self._graphs[key] = g
        if g is None:
            self._seen.add(key)
            return self._run(x_host, w_host, y_host)
        g.replay()
        return y_host

    def _run(self, x_host, w_host, y_host):
        torch = D.torch
        lib = _native.lib()
        cur = torch.cuda.current_stream()
        for s in (self.s_h2d, self.s_cmp, self.s_d2h):
            s.wait_stream(cur)
        with torch.cuda.stream(self.s_h2d):
            self.w_dev.copy_(w_host, non_blocking=True)
            for (a, b), (e_in, _) in zip(self.bounds, self.ev):
                self.x_dev[a:b].copy_(x_host[a:b], non_blocking=True)
                e_in.record(self.s_h2d)
        with torch.cuda.stream(self.s_cmp):
            sc = self.s_cmp.cuda_stream
            self.s_cmp.wait_event(self.ev[0][0])
            for uop, U in self.U.values():
                _native.check(lib.wino_filter_transform(uop.plan.handle, ctypes.byref(uop.shape),
                                                        D.ptr(self.w_dev), D.ptr(U), sc), "filter_transform")
            for op, key, ws, (a, b), (e_in, e_out) in zip(self.ops, self.u_key, self.ws, self.bounds, self.ev):
                U = self.U[key][1]
                self.s_cmp.wait_event(e_in)
                V = ws
                M = ws[(op.layout.v_bytes + 255) // 256 * 64:]
                xs, ys = self.x_dev[a:b], self.y_dev[a:b]
                sh = ctypes.byref(op.shape)
                _native.check(lib.wino_input_transform(op.plan.handle, sh, D.ptr(xs), D.ptr(V), sc), "input")
                if op.fused:
                    _native.check(lib.wino_contract_output(op.plan.handle, sh, D.ptr(U), D.ptr(V), D.ptr(ys), sc),
                                  "contract_output")
                else:
                    _native.check(lib.wino_contract(op.plan.handle, sh, D.ptr(U), D.ptr(V), D.ptr(M), sc),
                                  "contract")
                    _native.check(lib.wino_output_transform(op.plan.handle, sh, D.ptr(M), D.ptr(ys), sc),
                                  "output")
                e_out.record(self.s_cmp)
        with torch.cuda.stream(self.s_d2h):
            for (a, b), (_, e_out) in zip(self.bounds, self.ev):
                self.s_d2h.wait_event(e_out)
                y_host[a:b].copy_(self.y_dev[a:b], non_blocking=True)
        cur.wait_stream(self.s_d2h)
        return y_host


_ops_lock = threading.Lock()


def layer_op(ts, cfg, N, C, H, W, K, pad, contraction="exact") -> LayerOp:
    key = ("layer_op", cfg, contraction, N, C, H, W, K, pad)
    with _ops_lock:
        op = ts._programs.get(key)
        if op is None:
            op = LayerOp(ts, cfg, N, C, H, W, K, pad, contraction)
            ts._programs[key] = op
    return op


def conv2d_layer(ts: TransformSet, x, w, cfg: ConvConfig = ConvConfig(), pad: int = 0,
                 contraction: str = "exact", layout: str = "NCHW", fused: bool = False):
    """Winograd F(m x m, r x r) convolution layer (stride 1, zero padding `pad`).

    x (N, C, H, W), w (K, C, r, r) -> y (N, K, Ho, Wo): numpy in -> numpy out
    (host<->device copies included), CUDA tensors in -> CUDA tensor out.
    Output dtype f32 in fp32 mode, f64 in mixed / fp64 mode (reference engine.py:378-387).
    layout="NHWC": x (N, H, W, C) -> y (N, Ho, Wo, K) through NHWC-native K1 / K4 kernels
    (wino_conv2d_nhwc; same values as the NCHW path, bit for bit).  Tensor-core
    contraction modes have no NHWC kernels: there the activations are permuted on the
    device around the NCHW kernels.
    fused=True (NCHW, fp32, alpha^2 <= 16, FP32-pipe contraction): the contraction and the
    output transform run as one exact kernel with the accumulators parked in tensor memory
    (wino_conv2d_fused) -- same bits, no M in HBM; faster than the unfused path on large
    transform-heavy layers (C <= 128, thousands of 64 x 64 blocks), slower on small ones."""
    if layout not in ("NCHW", "NHWC"):
        raise ValueError("layout must be 'NCHW' or 'NHWC'")
    if layout == "NHWC":
        xs, wsh = tuple(D.shape_of(x)), tuple(D.shape_of(w))
        if len(xs) != 4 or len(wsh) != 4:
            raise ValueError("x must be (N, H, W, C) and w (K, C, r, r)")
        N, H, W, C = xs
        K, C2, r1, r2 = wsh
        if C2 != C:
            raise ValueError("x and w disagree on the channel count")
        if r1 != ts.n_h or r2 != ts.n_h:
            raise ValueError(f"filter must be {ts.n_h}x{ts.n_h} for this transform set")
        if contraction.startswith(("tc_", "tcf_")):
            dt = np.float64 if cfg.precision == "fp64" else np.float32
            xt, hx = D.to_device(x, dt)
            wt, hw = D.to_device(w, dt)
            y = conv2d_layer(ts, xt.permute(0, 3, 1, 2).contiguous(), wt, cfg, pad, contraction)
            return D.finish(y.permute(0, 2, 3, 1).contiguous(), hx or hw)
        op = layer_op(ts, cfg, N, C, H, W, K, pad, contraction)
        xt, hx = D.to_device(x, op.in_dtype)
        wt, hw = D.to_device(w, op.in_dtype)
        return D.finish(op.call_nhwc(xt, wt), hx or hw)
    xs, wsh = tuple(D.shape_of(x)), tuple(D.shape_of(w))
    if len(xs) != 4 or len(wsh) != 4:
        raise ValueError("x must be (N, C, H, W) and w (K, C, r, r)")
    N, C, H, W = xs
    K, C2, r1, r2 = wsh
    if C2 != C:
        raise ValueError("x and w disagree on the channel count")
    if r1 != ts.n_h or r2 != ts.n_h:
        raise ValueError(f"filter must be {ts.n_h}x{ts.n_h} for this transform set")
    op = layer_op(ts, cfg, N, C, H, W, K, pad, contraction)
    xt, hx = D.to_device(x, op.in_dtype)
    wt, hw = D.to_device(w, op.in_dtype)
    if fused:
        if not op.fused_exact_supported:
            raise ValueError("fused=True needs an fp32 plan, an FP32-pipe contraction and alpha^2 <= 16")
        return D.finish(op.call_fused(xt, wt), hx or hw)
    return D.finish(op(xt, wt), hx or hw)


def direct_layer_f64(x, w, pad: int):
    """fp64 direct correlation of a layer on the device (the error oracle):
    per output, per channel the r*r taps in row-major order, channels left to
    right -- reference direct_products + channel_reduce("linear")."""
    xt, hx = D.to_device(x, np.float32)
    wt, hw = D.to_device(w, np.float32)
    N, C, H, W = xt.shape
    K, _, r, _ = wt.shape
    Ho, Wo = H + 2 * pad - r + 1, W + 2 * pad - r + 1
    y = D.empty((N, K, Ho, Wo), np.float64)
    s = _native.LayerShape(N, C, H, W, K, pad)
    _native.check(_native.lib().wino_direct_layer_f64(ctypes.byref(s), r, D.ptr(xt), D.ptr(wt), D.ptr(y),
                                                      D.stream_handle()), "direct_layer_f64")
    return D.finish(y, hx or hw)


def layer_error_stats(y, y64):
    """Per-image (sum|y - y64|, sum|y64|, count, max|y - y64|) on the device -> (N, 4) f64."""
    yt = y if isinstance(y, D.torch.Tensor) else D.to_device(y, np.asarray(y).dtype.type)[0]
    rt = y64 if isinstance(y64, D.torch.Tensor) else D.to_device(y64, np.float64)[0]
    N = yt.shape[0]
    per = int(yt.numel() // max(N, 1))
    stats = D.empty((N, 4), np.float64)
    _native.check(_native.lib().wino_layer_error_stats(N, per, 0 if yt.dtype == D.torch.float32 else 1,
                                                       D.ptr(yt), D.ptr(rt), D.ptr(stats), D.stream_handle()),
                  "layer_error_stats")
    return stats
