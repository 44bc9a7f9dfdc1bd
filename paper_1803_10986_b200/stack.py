"""Winograd conv stacks (BASELINE.json config 5: the VGG-16 conv stack).

Thirteen 3x3 / pad-1 convolution layers, every one through the Winograd layer
path (K2 K1 K3 K4), each followed by ReLU and, after layers 2, 4, 7 and 10, a
2x2 max-pool (both in one libwino kernel).  Per-layer *isolated* error: every
layer's Winograd output is compared with the fp64 direct convolution of the
same fp32 input activation (SURVEY.md 7.2 "fp64 oracle at VGG scale").
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
        self.ops, self.shapes = [], []
        h, w = H, W
        for C, K, pool in self.layers:
            op = layer_op(ts, cfg, N, C, h, w, K, pad, contraction)
            self.ops.append(op)
            self.shapes.append((C, K, h, w, pool))
            h, w = op.layout.Ho, op.layout.Wo
            if pool:
                h, w = h // 2, w // 2
        self.out_hw = (h, w)
        ws = max(op.layout.workspace_bytes for op in self.ops)
        self.workspace = D.torch.empty(ws, dtype=D.torch.uint8, device="cuda")
        self.conv_out = [D.empty(op.out_shape, np.float32) for op in self.ops]
        self.act = []
        for op, (C, K, h, w, pool) in zip(self.ops, self.shapes):
            Ho, Wo = op.layout.Ho, op.layout.Wo
            self.act.append(D.empty((N, K, Ho // 2, Wo // 2) if pool else (N, K, Ho, Wo), np.float32))
        self.weights = None

    def set_weights(self, weights):
        self.weights = [D.to_device(w, np.float32)[0] for w in weights]

    @property
    def direct_flops(self) -> int:
        return sum(op.direct_flops for op in self.ops)

    @property
    def fused_act(self) -> bool:
        """K4 writes the activation directly (ReLU / 2x2 max-pool fused, y not stored)."""
        pools = any(pool for _, _, pool in self.layers)
        return not self.ops[0].tensor_core and (self.ts.n_o % 2 == 0 or not pools)

    @property
    def kernels_per_forward(self) -> int:
        return (3 if self.fused_act else 4) * len(self.ops)

    def forward(self, x, keep_conv_out=False):
        """x: CUDA f32 tensor (N, C0, H, W) -> activation after the last layer.

        Per layer: K2+K1 (one launch), K3, then K4 with ReLU (+ max-pool) fused
        (wino_output_transform_act) -- bitwise the same activations as K4 followed
        by wino_relu_pool.  keep_conv_out=True takes the unfused path and keeps
        every layer's pre-activation output in self.conv_out (layer_errors)."""
        lib = _native.lib()
        s = D.stream_handle()
        cur = x
        al = lambda v: (v + 255) // 256 * 256
        for i, op in enumerate(self.ops):
            C, K, h, w, pool = self.shapes[i]
            sh = ctypes.byref(op.shape)
            if keep_conv_out or not self.fused_act:
                y = self.conv_out[i]
                _native.check(lib.wino_conv2d(op.plan.handle, sh, D.ptr(cur), D.ptr(self.weights[i]), D.ptr(y),
                                              D.ptr(self.workspace), self.workspace.numel(), s), f"layer {i + 1}")
                _native.check(lib.wino_relu_pool(0, op.N * K, op.layout.Ho, op.layout.Wo, 1 if pool else 0,
                                                 D.ptr(y), D.ptr(self.act[i]), s), "relu_pool")
            else:
                L = op.layout
                U = self.workspace.data_ptr()
                V = U + al(L.u_bytes)
                M = V + al(L.v_bytes)
                _native.check(lib.wino_transforms(op.plan.handle, sh, D.ptr(cur), D.ptr(self.weights[i]),
                                                  ctypes.c_void_p(U), ctypes.c_void_p(V), s), f"layer {i + 1} K1/K2")
                _native.check(lib.wino_contract(op.plan.handle, sh, ctypes.c_void_p(U), ctypes.c_void_p(V),
                                                ctypes.c_void_p(M), s), f"layer {i + 1} K3")
                _native.check(lib.wino_output_transform_act(op.plan.handle, sh, ctypes.c_void_p(M),
                                                            D.ptr(self.act[i]), 1 if pool else 0, s),
                              f"layer {i + 1} K4+act")
            cur = self.act[i]
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
