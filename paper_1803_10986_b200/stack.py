"""Winograd conv stacks (BASELINE.json config 5: the VGG-16 conv stack).

Thirteen 3x3 / pad-1 convolution layers, every one through the Winograd layer
path (K2 K1 K3 K4), each followed by ReLU and, after layers 2, 4, 7 and 10, a
2x2 max-pool (both in one libwino kernel).  Per-layer *isolated* error: every
layer's Winograd output is compared with the fp64 direct convolution of the
same fp32 input activation (SURVEY.md 7.2 "fp64 oracle at VGG scale").

Each layer's arithmetic is the reference's per-(filter, tile) ``conv_2d``
(engine.py:426-429 over the zero-padded image); the activation
between layers is the oracle's ``relu_pool``.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from . import device as D
from .engine import ConvConfig
from .layer import layer_op

# (C, K, pool after) of the 13 VGG-16 conv layers
VGG16 = [(3, 64, False), (64, 64, True), (64, 128, False), (128, 128, True), (128, 256, False),
         (256, 256, False), (256, 256, True), (256, 512, False), (512, 512, False), (512, 512, True),
         (512, 512, False), (512, 512, False), (512, 512, False)]


def he_normal_weights(layers, r, seed=2024):
    """He-normal filters N(0, 2/(r^2 C)) keyed Philox(seed, 10_000_000 + layer)."""
    out = []
    for i, (C, K, _) in enumerate(layers):
        g = np.random.Generator(np.random.Philox(key=np.array([seed, 10_000_000 + i], dtype=np.uint64)))
        w = g.standard_normal((K, C, r, r), dtype=np.float32) * np.float32(np.sqrt(2.0 / (r * r * C)))
        out.append(np.ascontiguousarray(w.astype(np.float32)))
    return out


class ConvStack:
    """A stack of same-transform Winograd conv layers with ReLU / max-pool."""

    def __init__(self, ts, cfg: ConvConfig, layers, N, H, W=None, pad=1, contraction="exact"):
        if cfg.precision != "fp32":
            raise ValueError("ConvStack chains fp32 activations: use precision='fp32'")
        W = H if W is None else W
        self.ts, self.cfg, self.layers, self.N, self.pad = ts, cfg, list(layers), N, pad
        self.H, self.W = H, W
        self.ops, self.shapes = [], []
        h, w = H, W
        self.contraction = contraction
        for C, K, pool in self.layers:
            # tc_* stacks: a layer with C <= 4 (VGG-16 layer 1) has no contraction worth a tensor core --
            # its 32-channel padded MMA only writes M -- so it runs the exact fp32 path (fused K3 + K4 +
            # activation where supported); tcf_* plans keep one mode throughout (no M anywhere)
            mode = "exact" if contraction.startswith("tc_") and C <= 4 else contraction
            op = layer_op(ts, cfg, N, C, h, w, K, pad, mode)
            if not op.tensor_core:
                op.prepare(_native.PREPARE_CONV | _native.PREPARE_ACT)
            self.ops.append(op)
            self.shapes.append((C, K, h, w, pool))
            h, w = op.layout.Ho, op.layout.Wo
            if pool:
                h, w = h // 2, w // 2
        self.out_hw = (h, w)
        # small-C layers (VGG-16 layer 1, C = 3) run K3 + K4 + activation in one kernel (M -- 6 GB
        # at batch 256 -- never stored, wino_contract_output_smallc) where the fast variant applies
        # (wino_smallc_supported == 2: 1.43 vs 2.73 ms at VGG layer 1)
        self._fuse_on = False
        self.use_smallc(True, fast_only=True)
        ws = max(op.layout.workspace_bytes for op in self.ops)
        self.workspace = D.torch.empty(ws, dtype=D.torch.uint8, device="cuda")
        # K4 of layer i + activation + K1 of layer i + 1 can run as one kernel (the activation between
        # them never goes to HBM, wino_output_input_transform; layer i + 1's V is written while layer
        # i's M is read, so layers then alternate between two workspaces).  Off by default: bitwise
        # equal, but at VGG-16 batch 256 only the 28 x 28 and 14 x 14 un-pooled pairs gain (1.03-1.07x);
        # the large planes lose (0.65-0.94x: one 128-thread block walks a whole plane in two
        # serial phases) and the forward is 67.3 vs 65.6 ms (profiles/r2_smallc2.md)
        self._workspace2 = None
        self.use_fuse_next(False)
        self._conv_out = None  # pre-activation outputs, allocated on first keep_conv_out forward
        self.act = []
        for op, (C, K, h, w, pool) in zip(self.ops, self.shapes):
            Ho, Wo = op.layout.Ho, op.layout.Wo
            self.act.append(D.empty((N, K, Ho // 2, Wo // 2) if pool else (N, K, Ho, Wo), np.float32))
        self.weights = None

    def use_smallc(self, on: bool = True, fast_only: bool = False):
        """Route qualifying small-C layers through the fused K3 + K4 + activation kernel
        (fast_only: only where libwino reports the faster-than-unfused variant)."""
        lib = _native.lib()
        sup = [0 if op.tensor_core else lib.wino_smallc_supported(op.plan.handle, ctypes.byref(op.shape))
               for op in self.ops]
        self._smallc_fast = [v == 2 for v in sup]
        self.smallc = [on and self.fused_act and v >= (2 if fast_only else 1) for v in sup]
        if hasattr(self, "fuse_next"):
            self.use_fuse_next(self._fuse_on)
        return self

    def use_fuse_next(self, on: bool = True):
        """Fuse K4 + activation of layer i with K1 of layer i + 1 where supported."""
        lib = _native.lib()
        self._fuse_on = on
        self.fuse_next = []
        for i, op in enumerate(self.ops):
            ok = on and self.fused_act and i + 1 < len(self.ops) and not self.smallc[i] and bool(
                lib.wino_output_input_supported(op.plan.handle, ctypes.byref(op.shape), 1 if self.shapes[i][4] else 0,
                                                ctypes.byref(self.ops[i + 1].shape)))
            self.fuse_next.append(ok)
        for i, ok in enumerate(self.fuse_next):
            if ok:
                self.ops[i + 1].prepare(_native.PREPARE_K4K1)
        if any(self.fuse_next) and self._workspace2 is None:
            self._workspace2 = D.torch.empty(self.workspace.numel(), dtype=D.torch.uint8, device="cuda")
        return self

    @property
    def conv_out(self):
        if self._conv_out is None:
            self._conv_out = [D.empty(op.out_shape, np.float32) for op in self.ops]
        return self._conv_out

    @property
    def out_shape(self):
        return tuple(self.act[-1].shape)

    def set_weights(self, weights):
        self.weights = [D.to_device(w, np.float32)[0] for w in weights]

    def share_weights(self, other: "ConvStack"):
        """Use another stack's device weights (same layers, e.g. a different batch size)."""
        self.weights = other.weights

    @property
    def direct_flops(self) -> int:
        return sum(op.direct_flops for op in self.ops)

    @property
    def contraction_flops(self) -> int:
        return sum(op.contraction_flops for op in self.ops)

    @property
    def fused_act(self) -> bool:
        """K4 writes the activation directly (ReLU / 2x2 max-pool fused, y not stored)."""
        pools = any(pool for _, _, pool in self.layers)
        # tc_* modes keep an fp32 M, so the same fused K4 applies; tcf_* modes have no M at all
        return not self.contraction.startswith("tcf_") and (self.ts.n_o % 2 == 0 or not pools)

    @property
    def kernels_per_forward(self) -> int:
        if not self.fused_act:
            return 4 * len(self.ops)
        return sum(2 if sc else 3 for sc in self.smallc)

    def _uvm(self, L, i=0):
        al = lambda v: (v + 255) // 256 * 256
        ws = self._workspace2 if (i & 1) and self._workspace2 is not None else self.workspace
        U = ws.data_ptr()
        V = U + al(L.u_bytes)
        return U, V, V + al(L.v_bytes)

    def layer_forward(self, i, cur, stream=None, events=None, after_kernel=None):
        """Layer i on activation `cur` (fused path): K1+K2, K3, K4+ReLU(+pool) -> self.act[i].
        Where fuse_next[i - 1] holds, layer i's V was already written by the previous layer's
        K4+K1 kernel (only K2 runs here and `cur` is not read); where fuse_next[i] holds, the
        last kernel is K4 + activation + K1 of layer i + 1 and the return value is None (the
        activation only ever exists in shared memory).
        events: optional 4 CUDA events recorded before K1+K2, before K3, before K4, after K4.
        after_kernel: optional callable issued after each of the three kernels (profiling)."""
        hook = after_kernel if after_kernel is not None else (lambda: None)
        lib = _native.lib()
        s = D.stream_handle() if stream is None else stream
        op = self.ops[i]
        pool = self.shapes[i][4]
        sh = ctypes.byref(op.shape)
        U, V, M = self._uvm(op.layout, i)
        if events is not None:
            events[0].record()
        if i > 0 and self.fuse_next[i - 1]:
            _native.check(lib.wino_filter_transform(op.plan.handle, sh, D.ptr(self.weights[i]), ctypes.c_void_p(U), s),
                          f"layer {i + 1} K2")
        else:
            # a layer that goes through the fast small-C kernel needs only the C real channel rows of V
            k12 = lib.wino_transforms_smallc if self.smallc[i] and self._smallc_fast[i] else lib.wino_transforms
            _native.check(k12(op.plan.handle, sh, D.ptr(cur), D.ptr(self.weights[i]),
                              ctypes.c_void_p(U), ctypes.c_void_p(V), s), f"layer {i + 1} K1/K2")
        hook()
        if events is not None:
            events[1].record()
        if self.smallc[i]:  # K3 + K4 + ReLU (+ pool) in one launch
            _native.check(lib.wino_contract_output_smallc(op.plan.handle, sh, ctypes.c_void_p(U), ctypes.c_void_p(V),
                                                          D.ptr(self.act[i]), 2 if pool else 1, s),
                          f"layer {i + 1} K3+K4+act")
            hook()
            if events is not None:
                events[2].record()
                events[3].record()
            return self.act[i]
        _native.check(lib.wino_contract(op.plan.handle, sh, ctypes.c_void_p(U), ctypes.c_void_p(V),
                                        ctypes.c_void_p(M), s), f"layer {i + 1} K3")
        hook()
        if events is not None:
            events[2].record()
        if self.fuse_next[i]:  # K4 + ReLU (+ pool) + K1 of the next layer: writes the next layer's V
            nxt = self.ops[i + 1]
            _, V2, _ = self._uvm(nxt.layout, i + 1)
            _native.check(lib.wino_output_input_transform(op.plan.handle, sh, ctypes.c_void_p(M), 1 if pool else 0,
                                                          ctypes.byref(nxt.shape), ctypes.c_void_p(V2), s),
                          f"layer {i + 1} K4+act+K1")
            hook()
            if events is not None:
                events[3].record()
            return None
        _native.check(lib.wino_output_transform_act(op.plan.handle, sh, ctypes.c_void_p(M),
                                                    D.ptr(self.act[i]), 1 if pool else 0, s),
                      f"layer {i + 1} K4+act")
        hook()
        if events is not None:
            events[3].record()
        return self.act[i]

    def forward(self, x, keep_conv_out=False, stream=None, before_last=None):
        """x: CUDA f32 tensor (N, C0, H, W) -> activation after the last layer.

        Per layer: K2+K1 (one launch), K3, then K4 with ReLU (+ max-pool) fused
        (wino_output_transform_act) -- bitwise the same activations as K4 followed
        by wino_relu_pool.  keep_conv_out=True takes the unfused path and keeps
        every layer's pre-activation output in self.conv_out (layer_errors).
        before_last: called just before the last layer is issued (pipelines insert
        a wait for the read-back of the previous chunk's final activation there)."""
        lib = _native.lib()
        s = D.stream_handle() if stream is None else stream
        cur = x
        for i, op in enumerate(self.ops):
            C, K, h, w, pool = self.shapes[i]
            if before_last is not None and i == len(self.ops) - 1:
                before_last()
            if keep_conv_out or not self.fused_act:
                y = self.conv_out[i]
                _native.check(lib.wino_conv2d(op.plan.handle, ctypes.byref(op.shape), D.ptr(cur),
                                              D.ptr(self.weights[i]), D.ptr(y), D.ptr(self.workspace),
                                              self.workspace.numel(), s), f"layer {i + 1}")
                _native.check(lib.wino_relu_pool(0, op.N * K, op.layout.Ho, op.layout.Wo, 1 if pool else 0,
                                                 D.ptr(y), D.ptr(self.act[i]), s), "relu_pool")
                cur = self.act[i]
            else:
                cur = self.layer_forward(i, cur, s)
        return cur

    def layer_errors(self, x, images=None):
        """Per-layer isolated error over the first `images` images: (layer, rel_l1,
        per_point_l1, max_abs) vs fp64 direct conv of the same fp32 input
        activation (runs one unfused forward to keep the pre-activation outputs)."""
        from .layer import direct_layer_f64, layer_error_stats
        self.forward(x, keep_conv_out=True)
        n = self.N if images is None else min(images, self.N)
        res = []
        inp = x
        for i, op in enumerate(self.ops):
            y64 = direct_layer_f64(inp[:n].contiguous(), self.weights[i], self.pad)
            st = layer_error_stats(self.conv_out[i][:n].contiguous(), y64).cpu().numpy()
            res.append({"layer": i + 1, "C": self.shapes[i][0], "K": self.shapes[i][1], "H": self.shapes[i][2],
                        "rel_l1": float(st[:, 0].sum() / st[:, 1].sum()),
                        "per_point_l1": float(st[:, 0].sum() / st[:, 2].sum()), "max_abs": float(st[:, 3].max())})
            inp = self.act[i]
        return res


class StackPipeline:
    """Host-buffer forward of a conv stack with the PCIe copies hidden: the batch is
    split into image chunks; chunk i+1's H2D copy and chunk i-1's D2H copy of the
    final activation run on their own streams while chunk i's 13 layers run on the
    compute stream (the copy engines and the SMs overlap).

    x_host (N, C0, H, W) and out_host (N, K_last, h, w) must be pinned f32 CPU
    tensors.  Weights stay resident on the device (set_weights once)."""

    def __init__(self, ts, cfg: ConvConfig, layers, N, H, W=None, chunks=4, pad=1, contraction="exact"):
        if isinstance(chunks, (list, tuple)):
            # explicit image counts (scaled to N if they do not add up): a small first chunk starts
            # the compute stream early, a small last chunk shortens the exposed D2H tail
            sizes_ = [max(1, int(round(c * N / sum(chunks)))) for c in chunks]
            sizes_[-1] = N - sum(sizes_[:-1])
            if min(sizes_) < 1:  # batch too small for this split: equal chunks
                k = max(1, min(len(chunks), N))
                sizes_ = [(i + 1) * N // k - i * N // k for i in range(k)]
            edges = np.cumsum([0] + sizes_)
            self.bounds = [(int(a), int(b)) for a, b in zip(edges[:-1], edges[1:])]
        else:
            chunks = max(1, min(int(chunks), N))
            self.bounds = [(i * N // chunks, (i + 1) * N // chunks) for i in range(chunks)]
        sizes = sorted({b - a for a, b in self.bounds})
        self.stacks = {n: ConvStack(ts, cfg, layers, n, H, W, pad, contraction) for n in sizes}
        first = self.stacks[sizes[0]]
        self.N, self.layers = N, list(layers)
        self.in_shape = (N, layers[0][0], H, H if W is None else W)
        self.out_shape = (N,) + first.out_shape[1:]
        self.x_dev = D.empty(self.in_shape, np.float32)
        self.s_h2d, self.s_cmp, self.s_d2h = D.torch.cuda.Stream(), D.torch.cuda.Stream(), D.torch.cuda.Stream()
        self.ev_in = [D.torch.cuda.Event() for _ in self.bounds]
        self.ev_out = [D.torch.cuda.Event() for _ in self.bounds]
        self.ev_d2h = [D.torch.cuda.Event() for _ in self.bounds]

    def set_weights(self, weights):
        stacks = list(self.stacks.values())
        stacks[0].set_weights(weights)
        for st in stacks[1:]:
            st.share_weights(stacks[0])

    @property
    def direct_flops(self) -> int:
        return sum(self.stacks[b - a].direct_flops for a, b in self.bounds)

    @property
    def kernels_per_forward(self) -> int:
        return sum(self.stacks[b - a].kernels_per_forward for a, b in self.bounds)

    def __call__(self, x_host, out_host):
        torch = D.torch
        cur = torch.cuda.current_stream()
        for s in (self.s_h2d, self.s_cmp, self.s_d2h):
            s.wait_stream(cur)
        with torch.cuda.stream(self.s_h2d):
            for (a, b), ev in zip(self.bounds, self.ev_in):
                self.x_dev[a:b].copy_(x_host[a:b], non_blocking=True)
                ev.record(self.s_h2d)
        prev = {}  # stack size -> index of the last chunk whose final activation it holds
        for j, ((a, b), e_in, e_out) in enumerate(zip(self.bounds, self.ev_in, self.ev_out)):
            st = self.stacks[b - a]
            with torch.cuda.stream(self.s_cmp):
                self.s_cmp.wait_event(e_in)
                hook = None
                if (b - a) in prev:  # the final-activation buffer must have been read back
                    hook = (lambda ev: lambda: self.s_cmp.wait_event(ev))(self.ev_d2h[prev[b - a]])
                st.forward(self.x_dev[a:b], stream=self.s_cmp.cuda_stream, before_last=hook)
                e_out.record(self.s_cmp)
            with torch.cuda.stream(self.s_d2h):
                self.s_d2h.wait_event(e_out)
                out_host[a:b].copy_(st.act[-1], non_blocking=True)
                self.ev_d2h[j].record(self.s_d2h)
            prev[b - a] = j
        cur.wait_stream(self.s_d2h)
        cur.wait_stream(self.s_cmp)
        return out_host
