"""ctypes binding of libwino.so (include/wino.h).

The compute path of this package is the native library and nothing else: if
libwino.so is missing or no CUDA device is present, every compute entry point
raises -- there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os
import threading
from ctypes import POINTER, c_char_p, c_double, c_int, c_int32, c_int64, c_size_t, c_uint64, c_void_p

import numpy as np

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libwino.so")

WINO_OK, WINO_EINVAL, WINO_EUNSUPPORTED, WINO_ECUDA, WINO_ECOMPILE = 0, -1, -2, -3, -4
PRECISION_CODE = {"fp32": 0, "fp64": 1, "mixed": 2}
SUM_CODE = {"linear": 0, "pairwise": 1}
CONTRACT_CODE = {"exact": 0, "ffma": 1, "tc_bf16": 2, "tc_fp16": 3, "tcf_bf16": 4, "tcf_fp16": 5}


class WinoOp(ctypes.Structure):
    _fields_ = [("kind", c_int32), ("col", c_int32), ("coeff", c_double)]


class WinoProg(ctypes.Structure):
    _fields_ = [("rows", c_int32), ("cols", c_int32), ("row_start", POINTER(c_int32)),
                ("ops", POINTER(WinoOp))]


class LayerShape(ctypes.Structure):
    _fields_ = [(k, c_int32) for k in ("N", "C", "H", "W", "K", "pad")]


class LayerLayout(ctypes.Structure):
    _fields_ = [("P", c_int32), ("th", c_int32), ("tw", c_int32), ("Ho", c_int32), ("Wo", c_int32),
                ("bm", c_int32), ("bn", c_int32), ("T", c_int64), ("Tp", c_int64), ("Cp", c_int64), ("Kp", c_int64),
                ("elem_bytes_uv", c_int32), ("elem_bytes_y", c_int32),
                ("u_bytes", c_size_t), ("v_bytes", c_size_t), ("m_bytes", c_size_t),
                ("workspace_bytes", c_size_t)]


PREPARE_CONV, PREPARE_ACT, PREPARE_STAGES, PREPARE_NHWC, PREPARE_K4K1 = 1, 2, 4, 8, 16  # wino_plan_prepare flags (include/wino.h)

# (name, restype, argtypes) of every exported symbol, in include/wino.h order
SIGNATURES = [
    ("wino_plan_create", c_int, [c_int, c_int, c_int, c_int, c_int, POINTER(WinoProg), POINTER(WinoProg),
                                 POINTER(WinoProg), POINTER(c_void_p)]),
    ("wino_plan_destroy", None, [c_void_p]),
    ("wino_plan_source", c_int, [c_void_p, c_int, c_char_p, c_size_t, POINTER(c_size_t)]),
    ("wino_plan_cubin", c_int, [c_void_p, c_int, c_int, c_void_p, c_size_t, POINTER(c_size_t)]),
    ("wino_plan_prepare", c_int, [c_void_p, POINTER(LayerShape), c_int]),
    ("wino_layer_layout_query", c_int, [c_void_p, POINTER(LayerShape), POINTER(LayerLayout)]),
    ("wino_filter_transform", c_int, [c_void_p, POINTER(LayerShape), c_void_p, c_void_p, c_void_p]),
    ("wino_input_transform", c_int, [c_void_p, POINTER(LayerShape), c_void_p, c_void_p, c_void_p]),
    ("wino_transforms", c_int, [c_void_p, POINTER(LayerShape), c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    ("wino_contract", c_int, [c_void_p, POINTER(LayerShape), c_void_p, c_void_p, c_void_p, c_void_p]),
    ("wino_output_transform", c_int, [c_void_p, POINTER(LayerShape), c_void_p, c_void_p, c_void_p]),
    ("wino_output_transform_act", c_int, [c_void_p, POINTER(LayerShape), c_void_p, c_void_p, c_int, c_void_p]),
    ("wino_transforms_smallc", c_int, [c_void_p, POINTER(LayerShape), c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    ("wino_output_input_supported", c_int, [c_void_p, POINTER(LayerShape), c_int, POINTER(LayerShape)]),
    ("wino_output_input_transform", c_int, [c_void_p, POINTER(LayerShape), c_void_p, c_int, POINTER(LayerShape),
                                            c_void_p, c_void_p]),
    ("wino_smallc_supported", c_int, [c_void_p, POINTER(LayerShape)]),
    ("wino_contract_output_smallc", c_int, [c_void_p, POINTER(LayerShape), c_void_p, c_void_p, c_void_p, c_int,
                                            c_void_p]),
    ("wino_contract_output", c_int, [c_void_p, POINTER(LayerShape), c_void_p, c_void_p, c_void_p, c_void_p]),
    ("wino_input_transform_nhwc", c_int, [c_void_p, POINTER(LayerShape), c_void_p, c_void_p, c_void_p]),
    ("wino_output_transform_nhwc", c_int, [c_void_p, POINTER(LayerShape), c_void_p, c_void_p, c_void_p]),
    ("wino_conv2d_nhwc", c_int, [c_void_p, POINTER(LayerShape), c_void_p, c_void_p, c_void_p, c_void_p, c_size_t,
                          c_void_p]),
    ("wino_fused_supported", c_int, [c_void_p, POINTER(LayerShape)]),
    ("wino_fused_workspace", c_int, [c_void_p, POINTER(LayerShape), POINTER(c_size_t)]),
    ("wino_conv2d_fused", c_int, [c_void_p, POINTER(LayerShape), c_void_p, c_void_p, c_void_p, c_int, c_void_p,
                           c_size_t, c_void_p]),
    ("wino_conv2d", c_int, [c_void_p, POINTER(LayerShape), c_void_p, c_void_p, c_void_p, c_void_p, c_size_t,
                            c_void_p]),
    ("wino_tile_hadamard2d", c_int, [c_void_p, c_int64, c_int, c_void_p, c_void_p, c_void_p, c_void_p]),
    ("wino_tile_output2d", c_int, [c_void_p, c_int64, c_void_p, c_void_p, c_void_p]),
    ("wino_tile_hadamard1d", c_int, [c_void_p, c_int64, c_int, c_void_p, c_void_p, c_void_p, c_void_p]),
    ("wino_tile_output1d", c_int, [c_void_p, c_int64, c_void_p, c_void_p, c_void_p]),
    ("wino_channel_reduce", c_int, [c_int, c_int, c_int64, c_int64, c_int64, c_void_p, c_void_p, c_void_p]),
    ("wino_direct_products", c_int, [c_int, c_int, c_int, c_int64, c_int, c_int, c_int, c_void_p, c_void_p,
                                     c_void_p, c_void_p]),
    ("wino_program_eval", c_int, [c_int, c_void_p, c_int, c_int, c_int64, c_void_p, c_void_p, c_void_p]),
    ("wino_relu_pool", c_int, [c_int, c_int64, c_int, c_int, c_int, c_void_p, c_void_p, c_void_p]),
    ("wino_direct_layer_f64", c_int, [POINTER(LayerShape), c_int, c_void_p, c_void_p, c_void_p, c_void_p]),
    ("wino_layer_error_stats", c_int, [c_int64, c_int64, c_int, c_void_p, c_void_p, c_void_p, c_void_p]),
    ("wino_trial_inputs", c_int, [c_uint64, c_int64, c_int64, c_int, c_int, c_int, c_int, c_void_p, c_void_p,
                                  c_void_p]),
    ("wino_trial_l1", c_int, [c_int64, c_int64, c_int, c_void_p, c_void_p, c_void_p, c_void_p]),
    ("wino_mean_f64", c_int, [c_int64, c_void_p, c_void_p, c_void_p]),
    ("wino_peak_probe", c_int, [c_int, c_int, c_int, c_void_p, c_void_p]),
    ("wino_launch_count", c_int64, []),
    ("wino_last_error", c_char_p, []),
    ("wino_tuning_set", c_int, [c_char_p, c_char_p]),
    ("wino_version", c_char_p, []),
]

_lib = None
_lock = threading.Lock()


def lib():
    """Load libwino.so (once).  Raises if it has not been built."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise RuntimeError(f"{LIB_PATH} is missing: build it with "
                                       "`python -c 'import __graft_entry__ as g; g.build()'`")
                L = ctypes.CDLL(LIB_PATH)
                for name, res, args in SIGNATURES:
                    fn = getattr(L, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = L
    return _lib


def check(rc: int, what: str = "") -> None:
    if rc == WINO_OK:
        return
    msg = lib().wino_last_error().decode(errors="replace")
    if rc == WINO_EINVAL:
        raise ValueError(f"{what}: {msg}" if what else msg)
    raise RuntimeError(f"libwino error {rc} in {what}: {msg}")


class ProgTable:
    """Owns the ctypes arrays of one lowered matrix (keeps them alive)."""

    def __init__(self, lowered):
        starts, ops, ncols = lowered
        self.starts = (c_int32 * len(starts))(*[int(v) for v in starts])
        self.ops = (WinoOp * max(1, len(ops)))(*[WinoOp(k, c, v) for (k, c, v) in ops])
        self.prog = WinoProg(len(starts) - 1, ncols, self.starts, self.ops)


class Plan:
    """A compiled libwino plan (transform triple + precision + summation)."""

    def __init__(self, r, m, precision, channel_sum, contraction, g_low, bt_low, at_low):
        self._tables = [ProgTable(g_low), ProgTable(bt_low), ProgTable(at_low)]
        handle = c_void_p()
        check(lib().wino_plan_create(r, m, PRECISION_CODE[precision], SUM_CODE[channel_sum],
                                     CONTRACT_CODE[contraction], ctypes.byref(self._tables[0].prog),
                                     ctypes.byref(self._tables[1].prog), ctypes.byref(self._tables[2].prog),
                                     ctypes.byref(handle)), "wino_plan_create")
        self.handle = handle
        self.r, self.m, self.n = r, m, r + m - 1
        self.precision, self.channel_sum, self.contraction = precision, channel_sum, contraction

    def __del__(self):
        try:
            if self.handle and _lib is not None:
                _lib.wino_plan_destroy(self.handle)
        except Exception:
            pass

    def source(self, which=0) -> str:
        n = c_size_t()
        check(lib().wino_plan_source(self.handle, which, None, 0, ctypes.byref(n)))
        buf = ctypes.create_string_buffer(n.value + 1)
        check(lib().wino_plan_source(self.handle, which, buf, n.value + 1, None))
        return buf.value.decode()

    def cubin(self, which=0, channels=64) -> bytes:
        n = c_size_t()
        check(lib().wino_plan_cubin(self.handle, which, channels, None, 0, ctypes.byref(n)), "plan_cubin")
        buf = ctypes.create_string_buffer(n.value)
        check(lib().wino_plan_cubin(self.handle, which, channels, buf, n.value, ctypes.byref(n)), "plan_cubin")
        return buf.raw[:n.value]

    def layout(self, N, C, H, W, K, pad) -> LayerLayout:
        s = LayerShape(N, C, H, W, K, pad)
        out = LayerLayout()
        check(lib().wino_layer_layout_query(self.handle, ctypes.byref(s), ctypes.byref(out)), "layout")
        return out


def set_tuning(key: str, value) -> None:
    """Tools / variant tests only: select an alternative kernel form or tile config
    (include/wino.h wino_tuning_set); value None clears the key."""
    check(lib().wino_tuning_set(key.encode(), None if value is None else str(value).encode()), "tuning_set")


def launch_count() -> int:
    return int(lib().wino_launch_count())


def as_ptr(t) -> int:
    return ctypes.c_void_p(t.data_ptr())


def f32_bits(a) -> np.ndarray:
    return np.ascontiguousarray(a).view(np.uint32)
