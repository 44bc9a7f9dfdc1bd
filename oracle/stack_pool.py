"""CPU ORACLE -- test infrastructure only, never the product path.

Process-parallel driver of ``wino_oracle.layer_conv2d`` for large layers (the
VGG-16 stack, BASELINE.json configs[4]).  Used by ``tests/`` as the checker and by
``bench.py``'s cpu_baseline / ``--impl reference`` legs as the CPU baseline.

Work split: every output tile of a layer depends only on its own zero-padded
alpha x alpha input window (reference engine.py:426-429 per
(filter, tile)), so a layer is cut into (image, band of tile rows, block of
filters) units and each unit runs the unmodified oracle arithmetic on its
window of the explicitly zero-padded input (pad=0).  The tiles a band sees are
exactly the tiles of the whole image (same origins at stride m), so the
assembled output is bit-identical to one ``layer_conv2d`` call -- checked by
``tests/test_stack_pool.py``.

The activation is published to the forked workers through one shared buffer;
filters are installed before the pool forks.
"""

from __future__ import annotations

import multiprocessing as mp
import os
from concurrent.futures import ProcessPoolExecutor

import numpy as np

from . import wino_oracle as O

_G: dict = {}


def _unit(args):
    """One (image, tile-row band, filter block) of layer `li`: y[1, kb, rows, Wo]."""
    li, shape, n, i0, i1, k0, k1, csum, order = args
    g = _G
    xp = np.frombuffer(g["buf"], dtype=np.float32, count=int(np.prod(shape))).reshape(shape)
    m, r = g["trip"].m, g["trip"].r
    rows = xp[n:n + 1, :, i0 * m:min(shape[2], i1 * m + r - 1)]
    return O.layer_conv2d(g["trip"], rows, g["weights"][li][k0:k1], 0, "fp32", order, csum)


class OraclePool:
    """fp32 oracle layers over `procs` forked worker processes (procs=1: in-process)."""

    def __init__(self, trip, weights, max_input_elems, procs=None):
        self.trip = trip
        self.weights = [np.ascontiguousarray(w, dtype=np.float32) for w in weights]
        self.procs = max(1, procs or len(os.sched_getaffinity(0)))
        self.buf = mp.RawArray("f", int(max_input_elems))
        _G.update(trip=trip, weights=self.weights, buf=self.buf)
        self.ex = None
        if self.procs > 1:
            self.ex = ProcessPoolExecutor(self.procs, mp_context=mp.get_context("fork"))

    def close(self):
        if self.ex is not None:
            self.ex.shutdown()
            self.ex = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def layer(self, li, x, pad=1, csum="pairwise", order="huffman"):
        """y = layer_conv2d(trip, x, weights[li], pad) (bit-identical), in parallel."""
        x = np.asarray(x, dtype=np.float32)
        if self.ex is None:
            return O.layer_conv2d(self.trip, x, self.weights[li], pad, "fp32", order, csum)
        N, C, H, W = x.shape
        K = self.weights[li].shape[0]
        r, m = self.trip.r, self.trip.m
        Ho, Wo, th, tw = O.layer_geometry(H, W, r, m, pad)
        shape = (N, C, H + 2 * pad, W + 2 * pad)
        if int(np.prod(shape)) > len(self.buf):
            raise ValueError("activation larger than the pool's shared buffer")
        xp = np.frombuffer(self.buf, dtype=np.float32, count=int(np.prod(shape))).reshape(shape)
        xp[...] = 0
        xp[:, :, pad:pad + H, pad:pad + W] = x
        # bands of tile rows per image; filter blocks when bands alone cannot fill the pool
        bands = max(1, min(th, -(-2 * self.procs // N)))
        kblocks = max(1, min(K // 16, -(-2 * self.procs // (N * bands))))
        units = []
        for n in range(N):
            for b in range(bands):
                i0, i1 = b * th // bands, (b + 1) * th // bands
                for q in range(kblocks):
                    k0, k1 = q * K // kblocks, (q + 1) * K // kblocks
                    if i1 > i0 and k1 > k0:
                        units.append((li, shape, n, i0, i1, k0, k1, csum, order))
        y = np.empty((N, K, Ho, Wo), dtype=np.float32)
        for u, part in zip(units, self.ex.map(_unit, units)):
            _, _, n, i0, i1, k0, k1, _, _ = u
            y[n, k0:k1, i0 * m:i0 * m + part.shape[2]] = part[0]
        return y

    def stack_forward(self, x, layers, pad=1, csum="pairwise", order="huffman", keep=True):
        """Oracle ConvStack forward (fp32): (conv outputs per layer | None, final activation)."""
        outs = [] if keep else None
        cur = np.asarray(x, dtype=np.float32)
        for li, (_, _, pool) in enumerate(layers):
            y = self.layer(li, cur, pad, csum, order)
            if keep:
                outs.append(y)
            cur = O.relu_pool(y, pool)
        return outs, cur
