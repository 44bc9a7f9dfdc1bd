"""Drop-in convolution API of the reference (toomcook.engine,
/root/reference/pkg/src/toomcook/engine.py), executed by libwino on the GPU.

Same names, argument meaning, dtypes and errors as the reference; the
arithmetic (every product and sum rounded exactly as the reference rounds it)
runs in generated sm_100a kernels.  Array-likes in -> numpy out (host round
trip); CUDA tensors in -> CUDA tensors out (device-resident).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from . import device as D
from .programs import (  # re-exported drop-in names
    EvalLeaf,
    EvalNode,
    coefficient_cast,
    compiled_programs,
    huffman_order,
    linear_order,
    lower,
    row_trees,
    tree_depth,
    tree_leaves,
)
from .transforms import TransformSet

PRECISION_MODES = ("fp32", "fp64", "mixed")
DOT_ORDERS = ("linear", "huffman")
CHANNEL_SUMS = ("linear", "pairwise")
CONTRACTIONS = ("exact", "ffma", "tc_bf16", "tc_fp16", "tcf_bf16", "tcf_fp16")

__all__ = [
    "ConvConfig", "EvalLeaf", "EvalNode", "huffman_order", "linear_order", "row_trees", "tree_depth",
    "tree_leaves", "compiled_programs", "dot_with_order", "pairwise_sum", "channel_reduce", "direct_products",
    "conv_direct", "hadamard_1d", "output_1d", "conv_1d", "hadamard_2d", "output_2d", "conv_2d", "get_plan",
]


@dataclass(frozen=True)
class ConvConfig:
    """Precision mode plus summation strategies (reference engine.py:27-55).

    mixed: fp64 transform arithmetic over the fp32-rounded constant tables,
    fp32 Hadamard product and channel sum (U, V narrowed round-to-nearest), fp64
    output transform returned in fp64."""

    precision: str = "fp32"
    dot_order: str = "huffman"
    channel_sum: str = "linear"

    def __post_init__(self):
        if self.precision not in PRECISION_MODES:
            raise ValueError(f"precision must be one of {PRECISION_MODES}")
        if self.dot_order not in DOT_ORDERS:
            raise ValueError(f"dot_order must be one of {DOT_ORDERS}")
        if self.channel_sum not in CHANNEL_SUMS:
            raise ValueError(f"channel_sum must be one of {CHANNEL_SUMS}")

    @property
    def transform_dtype(self):
        return np.float64 if self.precision in ("fp64", "mixed") else np.float32

    @property
    def working_dtype(self):
        return np.float64 if self.precision == "fp64" else np.float32


def _input_dtype(cfg: ConvConfig):
    """dtype the transforms read (reference _prepare_input, engine.py:356-360):
    fp32 and mixed read fp32 values (mixed widens them exactly), fp64 reads f64."""
    return np.float64 if cfg.precision == "fp64" else np.float32


def _output_dtype(cfg: ConvConfig):
    return np.float32 if cfg.precision == "fp32" else np.float64


def get_plan(ts: TransformSet, cfg: ConvConfig, contraction: str = "exact") -> _native.Plan:
    """Compiled native plan for (triple, precision, dot order, channel sum),
    cached on the TransformSet like the reference caches its programs."""
    if contraction not in CONTRACTIONS:
        raise ValueError(f"contraction must be one of {CONTRACTIONS}")
    key = ("native_plan", cfg.precision, cfg.dot_order, cfg.channel_sum, contraction)
    plan = ts._programs.get(key)
    if plan is None:
        low = [lower(ts, name, cfg.dot_order, cfg.precision) for name in ("G", "B_T", "A_T")]
        plan = _native.Plan(ts.n_h, ts.n_o, cfg.precision, cfg.channel_sum, contraction, *low)
        ts._programs[key] = plan
    return plan


# -- shape handling (reference engine.py:293-303) --------------------------------

def _channelled_shape(shape, dims: int, name: str, size: int | None = None) -> tuple:
    shape = tuple(shape)
    if len(shape) < dims:
        raise ValueError(f"{name} needs at least {dims} axes")
    if len(shape) == dims:
        shape = (1,) + shape
    if size is not None and shape[-1] != size:
        raise ValueError(f"{name} last axis is {shape[-1]}, expected {size}")
    if dims == 2 and shape[-1] != shape[-2]:
        raise ValueError(f"{name} must be square in its trailing axes")
    return shape


def _prod(t) -> int:
    p = 1
    for v in t:
        p *= int(v)
    return p


def _host_of(*arrays) -> bool:
    return any(not isinstance(a, D.torch.Tensor) or not a.is_cuda for a in arrays)


# -- channel reduction (reference engine.py:252-287, 336-338) -------------------

def _reduce(t, axis: int, strategy: str):
    """Device reduction of tensor t over `axis` (negative)."""
    shape = tuple(t.shape)
    ax = axis % len(shape)
    C = shape[ax]
    if C == 1:
        return t.reshape(shape[:ax] + shape[ax + 1:]).contiguous()
    if strategy not in CHANNEL_SUMS:
        raise ValueError(f"unknown channel_sum {strategy!r}")
    outer, inner = _prod(shape[:ax]), _prod(shape[ax + 1:])
    out = D.torch.empty(shape[:ax] + shape[ax + 1:], dtype=t.dtype, device=t.device)
    dt = 0 if t.dtype == D.torch.float32 else 1
    _native.check(_native.lib().wino_channel_reduce(dt, 1 if strategy == "pairwise" else 0, outer, C, inner,
                                                    D.ptr(t), D.ptr(out), D.stream_handle()), "channel_reduce")
    return out


def channel_reduce(z, dims: int, strategy: str):
    """Pointwise channel summation of (..., C, out...) data."""
    shape = D.shape_of(z)
    if len(shape) < dims + 1:
        raise ValueError("channel_reduce needs a channel axis")
    npdt = np.float32 if _dtype_is_f32(z) else np.float64
    t, host = D.to_device(z, npdt)
    return D.finish(_reduce(t, -(dims + 1), strategy), host)


def _dtype_is_f32(a) -> bool:
    if isinstance(a, D.torch.Tensor):
        return a.dtype == D.torch.float32
    return np.asarray(a).dtype == np.float32


def pairwise_sum(values, precision: str = "fp32"):
    """Balanced (halving-tree) summation of a nonempty 1-D list (engine.py:281-287)."""
    npdt = np.float32 if precision in ("fp32", "mixed") else np.float64
    shape = D.shape_of(values)
    if len(shape) != 1 or shape[0] == 0:
        raise ValueError("pairwise_sum expects a nonempty 1-D list")
    t, _ = D.to_device(values, npdt)
    out = D.torch.empty((), dtype=t.dtype, device=t.device)
    if shape[0] == 1:
        out.copy_(t[0])
    else:
        _native.check(_native.lib().wino_channel_reduce(0 if npdt is np.float32 else 1, 1, 1, shape[0], 1,
                                                        D.ptr(t), D.ptr(out), D.stream_handle()), "pairwise_sum")
    return npdt(out.item())


def dot_with_order(tree, vector, precision: str = "fp64"):
    """One dot product following the tree's summation order (engine.py:235-246),
    evaluated on the device; leading axes of `vector` are batched."""
    if precision not in ("fp32", "fp64"):
        raise ValueError(f"unknown precision: {precision!r}")
    npdt = np.float32 if precision == "fp32" else np.float64
    if tree is None:
        return npdt(0.0)
    cast = coefficient_cast(precision)
    from .programs import _postfix  # local: the flattening used for plans
    ops = []
    _postfix(tree, cast, ops)
    v, _ = D.to_device(vector, npdt)
    lead = tuple(v.shape[:-1])
    cols = v.shape[-1]
    opbuf = np.zeros(len(ops), dtype=[("kind", "<i4"), ("col", "<i4"), ("coeff", "<f8")])
    for i, (k, c, x) in enumerate(ops):
        opbuf[i] = (k, c, x)
    dops = D.torch.from_numpy(opbuf.view(np.uint8).copy()).cuda()
    out = D.torch.empty(lead, dtype=v.dtype, device=v.device)
    _native.check(_native.lib().wino_program_eval(0 if npdt is np.float32 else 1, D.ptr(dops), len(ops), cols,
                                                  _prod(lead), D.ptr(v), D.ptr(out), D.stream_handle()),
                  "dot_with_order")
    res = out.cpu().numpy()
    return npdt(res) if res.ndim == 0 else res


# -- direct convolution (reference engine.py:309-346) ---------------------------

def direct_products(h, x, dims: int = 1, precision: str = "fp64"):
    """Per-channel valid-region correlation, taps in kernel-index order; (..., C, out...)."""
    npdt = np.float64 if precision == "fp64" else np.float32
    hs = _channelled_shape(D.shape_of(h), dims, "kernel")
    xs = _channelled_shape(D.shape_of(x), dims, "input")
    if hs[:-dims] != xs[:-dims]:
        raise ValueError("kernel/input channel or batch shapes disagree")
    r, n = hs[-1], xs[-1]
    o = n - r + 1
    if o < 1:
        raise ValueError("input shorter than kernel")
    ht, host_h = D.to_device(h, npdt)
    xt, host_x = D.to_device(x, npdt)
    C = hs[-dims - 1]
    B = _prod(hs[:-dims - 1])
    out = D.empty(hs[:-dims] + (o,) * dims, npdt)
    dt = 0 if npdt is np.float32 else 1
    _native.check(_native.lib().wino_direct_products(dims, dt, dt, B, C, r, n, D.ptr(ht), D.ptr(xt), D.ptr(out),
                                                     D.stream_handle()), "direct_products")
    return D.finish(out, host_h or host_x)


def conv_direct(h, x, dims: int = 1, precision: str = "fp64", channel_sum: str = "linear"):
    """Valid-region correlation with channels summed pointwise."""
    p = direct_products(h, x, dims, precision)
    return channel_reduce(p, dims, channel_sum)


# -- Toom-Cook execution (reference engine.py:363-429) --------------------------

def _hadamard(ts, h, x, cfg, dims):
    hs = _channelled_shape(D.shape_of(h), dims, "kernel", ts.n_h)
    xs = _channelled_shape(D.shape_of(x), dims, "input", ts.n)
    if hs[:-dims] != xs[:-dims]:
        raise ValueError("kernel/input channel or batch shapes disagree")
    plan = get_plan(ts, cfg)
    ht, host_h = D.to_device(h, _input_dtype(cfg))
    xt, host_x = D.to_device(x, _input_dtype(cfg))
    C = hs[-dims - 1]
    B = _prod(hs[:-dims - 1])
    z = D.empty(hs[:-dims] + (ts.n,) * dims, cfg.working_dtype)
    fn = _native.lib().wino_tile_hadamard2d if dims == 2 else _native.lib().wino_tile_hadamard1d
    _native.check(fn(plan.handle, B, C, D.ptr(ht), D.ptr(xt), D.ptr(z), D.stream_handle()), "hadamard")
    return z, host_h or host_x


def _output(ts, y, cfg, dims):
    ys = tuple(D.shape_of(y))
    if len(ys) < dims or ys[-dims:] != (ts.n,) * dims:
        raise ValueError(f"output transform input must end in {(ts.n,) * dims}")
    plan = get_plan(ts, cfg)
    yt, host = D.to_device(y, cfg.working_dtype)
    B = _prod(ys[:-dims])
    out = D.empty(ys[:-dims] + (ts.n_o,) * dims, _output_dtype(cfg))
    fn = _native.lib().wino_tile_output2d if dims == 2 else _native.lib().wino_tile_output1d
    _native.check(fn(plan.handle, B, D.ptr(yt), D.ptr(out), D.stream_handle()), "output")
    return out, host


def hadamard_1d(ts: TransformSet, h, x, cfg: ConvConfig):
    z, host = _hadamard(ts, h, x, cfg, 1)
    return D.finish(z, host)


def output_1d(ts: TransformSet, y, cfg: ConvConfig):
    out, host = _output(ts, y, cfg, 1)
    return D.finish(out, host)


def conv_1d(ts: TransformSet, h, x, cfg: ConvConfig = ConvConfig()):
    """1D multi-channel convolution; kernel (..., C, n_h), input (..., C, n) -> (..., n_o)."""
    z, host = _hadamard(ts, h, x, cfg, 1)
    out, _ = _output(ts, _reduce(z, -2, cfg.channel_sum), cfg, 1)
    return D.finish(out, host)


def hadamard_2d(ts: TransformSet, h, x, cfg: ConvConfig):
    """G H_c G^T o B^T X_c B per channel: (..., C, n, n)."""
    z, host = _hadamard(ts, h, x, cfg, 2)
    return D.finish(z, host)


def output_2d(ts: TransformSet, y, cfg: ConvConfig):
    out, host = _output(ts, y, cfg, 2)
    return D.finish(out, host)


def conv_2d(ts: TransformSet, h, x, cfg: ConvConfig = ConvConfig()):
    """2D multi-channel convolution A^T (sum_c G H_c G^T o B^T X_c B) A."""
    z, host = _hadamard(ts, h, x, cfg, 2)
    out, _ = _output(ts, _reduce(z, -3, cfg.channel_sum), cfg, 2)
    return D.finish(out, host)
