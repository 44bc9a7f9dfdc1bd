"""CPU ORACLE -- test infrastructure only, never the product path.

A numpy restatement of the reference toolkit's Winograd / Toom-Cook arithmetic
(``/root/reference/pkg/src/toomcook``), used by ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s cpu_baseline / ``--impl reference`` leg as the checker and the
CPU baseline.  Nothing in ``paper_1803_10986_b200`` imports this module.

Parity pin: ``tests/test_oracle_golden.py`` checks every function below against
golden vectors produced by the reference itself (``tests/golden/make_golden.py``
imports the reference from /root/reference and writes the fixtures), and, when
/root/reference is mounted, directly against the reference on fresh inputs.

Semantics restated (reference file:line in each docstring):
  * exact-rational construction of (A^T, G, B^T) incl. the infinity point
  * per-row Huffman / left-to-right evaluation trees and their coefficient rounding
  * each product and each sum rounded individually (numpy elementwise ufuncs,
    never fused), 2D = left pass then right pass
  * channel summation: left-to-right, or the halving ("pairwise") tree
  * the fp64 direct-correlation reference and the per-trial L1 error metric
  * the layer-level composition (zero-padded overlapping alpha x alpha tiles at
    stride m, cropped output) of SURVEY.md section 3.4
"""

from __future__ import annotations

import math
from fractions import Fraction

import numpy as np

# ---------------------------------------------------------------------------
# exact scalars and points  (reference: exact.py:33-91, 175-232)
# ---------------------------------------------------------------------------

INF = None  # the infinity pseudo-point is represented by None


def parse_point_list(text):
    """"0,-1,1/2,inf" -> [Fraction|None, ...]   (reference exact.py:205-217)"""
    out = []
    for tok in text.split(","):
        tok = tok.strip().replace("−", "-")
        if not tok:
            continue
        if tok.lower() in ("inf", "infinity", "oo", "∞"):
            out.append(INF)
        elif "/" in tok:
            a, b = tok.split("/")
            out.append(Fraction(int(a), int(b)))
        else:
            out.append(Fraction(int(tok)))
    return out


def round_fraction(v, fmt):
    """Correctly rounded (ties-to-even) binary32/binary64 value of a rational.

    Reference: exact.py:61-91 (to_nearest_float).  Restated here by scaling the
    rational onto the target's integer significand grid."""
    v = Fraction(v)
    p, emin, emax = (24, -126, 127) if fmt == "fp32" else (53, -1022, 1023)
    limit = Fraction(2) ** (emax + 1) - Fraction(2) ** (emax - p)  # max + half ulp
    if abs(v) >= limit:
        raise OverflowError(f"{v} overflows {fmt}")
    if v == 0:
        return np.float32(0.0) if fmt == "fp32" else np.float64(0.0)
    neg = v < 0
    a = -v if neg else v
    e = a.numerator.bit_length() - a.denominator.bit_length()
    if Fraction(2) ** e > a:
        e -= 1
    e = max(e, emin)
    q = e - (p - 1)
    scaled = a / (Fraction(2) ** q)
    n = scaled.numerator // scaled.denominator
    rem = scaled - n
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and n % 2 == 1):
        n += 1
    val = math.ldexp(float(n), q) if n < (1 << 53) else float(Fraction(n) * Fraction(2) ** q)
    if neg:
        val = -val
    return np.float32(val) if fmt == "fp32" else np.float64(val)


# ---------------------------------------------------------------------------
# matrix construction  (reference: transforms.py:411-494)
# ---------------------------------------------------------------------------

def _poly_mul(a, b):
    out = [Fraction(0)] * (len(a) + len(b) - 1)
    for i, x in enumerate(a):
        for j, y in enumerate(b):
            out[i + j] += x * y
    return out


def _poly_from_roots(roots):
    poly = [Fraction(1)]
    for q in roots:
        poly = _poly_mul(poly, [-q, Fraction(1)])
    return poly


def build_triple(r, m, points):
    """Exact (A^T, G, B^T, ordered_points) for F(m, r).

    Finite points keep their order, the infinity point (if any) moves last.
    Toom-Cook (transforms.py:437-456) when all points are finite, otherwise the
    modified construction (transforms.py:459-486)."""
    n = r + m - 1
    if len(points) != n:
        raise ValueError("wrong number of points")
    finite = [p for p in points if p is not INF]
    n_inf = len(points) - len(finite)
    if n_inf > 1 or len(set(finite)) != len(finite):
        raise ValueError("points must be distinct with at most one infinity")
    ordered = finite + [INF] * n_inf
    nf = len(finite)
    # Lagrange scales N_i and cofactors M_i(a) = prod_{k != i} (a - p_k)
    scales, cof = [], []
    for i, pi in enumerate(finite):
        d = Fraction(1)
        for j, pj in enumerate(finite):
            if j != i:
                d *= pi - pj
        scales.append(1 / d)
        cof.append(_poly_from_roots([pj for j, pj in enumerate(finite) if j != i]))
    if n_inf == 0:
        at = [[p ** i for p in finite] for i in range(m)]
        g = [[finite[i] ** j * scales[i] for j in range(r)] for i in range(n)]
        bt = [c + [Fraction(0)] * (n - len(c)) for c in cof]
    else:
        at = [[q ** i for q in finite] + [Fraction(0)] for i in range(m)]
        at[m - 1][n - 1] = Fraction(1)
        g = [[finite[i] ** j * scales[i] for j in range(r)] for i in range(nf)]
        g.append([Fraction(0)] * (r - 1) + [Fraction(1)])
        bt = [c + [Fraction(0)] * (nf - len(c)) + [Fraction(0)] for c in cof]
        mp = _poly_from_roots(finite)
        bt.append(mp + [Fraction(0)] * (n - len(mp)))
    fr = lambda rows: [[Fraction(v) for v in row] for row in rows]
    return fr(at), fr(g), fr(bt), ordered


# ---------------------------------------------------------------------------
# evaluation trees  (reference: engine.py:76-108, 128-148, 157-188)
# tree := ("leaf", col, Fraction) | ("add", tree, tree) | None
# ---------------------------------------------------------------------------

def _point_key(p):
    return (1, Fraction(0)) if p is INF else (0, p)


def huffman_tree(row, keys=None):
    """Repeatedly merge the two lightest items; weight = |coefficient|.
    Ordering among equal weights: leaves first, then the leaf key (column or
    point key), then merge order (engine.py:76-95)."""
    items = []
    for j, c in enumerate(row):
        c = Fraction(c)
        if c != 0:
            items.append(((abs(c), 0, keys[j] if keys is not None else j), ("leaf", j, c)))
    if not items:
        return None
    made = 0
    while len(items) > 1:
        items.sort(key=lambda it: it[0])
        w = items[0][0][0] + items[1][0][0]
        merged = ((w, 1, made), ("add", items[0][1], items[1][1]))
        made += 1
        items = items[2:] + [merged]
    return items[0][1]


def linear_tree(row):
    """Left-deep chain over the nonzero coefficients (engine.py:98-108)."""
    t = None
    for j, c in enumerate(row):
        c = Fraction(c)
        if c == 0:
            continue
        leaf = ("leaf", j, c)
        t = leaf if t is None else ("add", t, leaf)
    return t


def matrix_trees(mat, name, order, points):
    if order == "linear":
        return [linear_tree(row) for row in mat]
    keys = [_point_key(p) for p in points] if name == "A_T" else None
    return [huffman_tree(row, keys) for row in mat]


def coeff_value(c, precision):
    """engine.py:163-171: fp32 table, fp64 table, or fp32 table widened."""
    if precision == "fp32":
        return round_fraction(c, "fp32")
    if precision == "fp64":
        return round_fraction(c, "fp64")
    return np.float64(round_fraction(c, "fp32"))


class Triple:
    """Transform triple plus per-(matrix, order, precision) trees.

    May be built from points (own restatement) or from golden data produced by
    the reference (``Triple.from_golden``)."""

    def __init__(self, r, m, points, at, g, bt):
        self.r, self.m, self.n = r, m, r + m - 1
        self.points = points
        self.mats = {"A_T": at, "G": g, "B_T": bt}
        self._trees = {}

    @classmethod
    def from_points(cls, r, m, text):
        at, g, bt, pts = build_triple(r, m, parse_point_list(text))
        return cls(r, m, pts, at, g, bt)

    def trees(self, name, order):
        key = (name, order)
        if key not in self._trees:
            self._trees[key] = matrix_trees(self.mats[name], name, order, self.points)
        return self._trees[key]


def _eval(tree, get, precision):
    """Evaluate one tree: leaf = one rounded product, node = one rounded sum
    (engine.py:191-208)."""
    if tree[0] == "leaf":
        return coeff_value(tree[2], precision) * get(tree[1])
    return _eval(tree[1], get, precision) + _eval(tree[2], get, precision)


def apply_rows(trip, name, order, precision, data, axis):
    """Apply matrix `name` along `axis` (-2: left pass, -1: right pass),
    one tree per output row (engine.py:211-232)."""
    data = np.asarray(data)
    outs = []
    for tree in trip.trees(name, order):
        get = (lambda j: data[..., j, :]) if axis == -2 else (lambda j: data[..., j])
        if tree is None:
            outs.append(np.zeros_like(get(0)))
        else:
            outs.append(_eval(tree, get, precision))
    return np.stack(outs, axis=axis)


def apply_2d(trip, name, order, precision, data):
    """(M D) M^T: left pass first, then right pass (engine.py:411-412, 423)."""
    return apply_rows(trip, name, order, precision,
                      apply_rows(trip, name, order, precision, data, -2), -1)


def apply_1d(trip, name, order, precision, data):
    return apply_rows(trip, name, order, precision, data, -1)


# ---------------------------------------------------------------------------
# channel sums  (reference: engine.py:252-287)
# ---------------------------------------------------------------------------

def sum_linear(stack):
    acc = stack[0]
    for c in range(1, stack.shape[0]):
        acc = acc + stack[c]
    return acc


def sum_halving(stack):
    """Pair neighbours level by level, an odd survivor rides to the end."""
    cur = stack
    while cur.shape[0] > 1:
        k = cur.shape[0]
        nxt = cur[0:k - 1:2] + cur[1:k:2]
        if k % 2 == 1:
            nxt = np.concatenate([nxt, cur[k - 1:k]], axis=0)
        cur = nxt
    return cur[0]


def reduce_channels(z, axis, strategy):
    s = np.moveaxis(np.asarray(z), axis, 0)
    if s.shape[0] == 1:
        return s[0]
    return sum_linear(s) if strategy == "linear" else sum_halving(s)


# ---------------------------------------------------------------------------
# tile-level convolution  (reference: engine.py:356-429)
# ---------------------------------------------------------------------------

def _widen(a, precision):
    a = np.asarray(a)
    if precision == "mixed":
        return a.astype(np.float32).astype(np.float64)
    return a.astype(np.float64 if precision == "fp64" else np.float32)


def hadamard2d(trip, h, x, precision, order):
    u = apply_2d(trip, "G", order, precision, _widen(h, precision))
    v = apply_2d(trip, "B_T", order, precision, _widen(x, precision))
    if precision == "mixed":
        u, v = u.astype(np.float32), v.astype(np.float32)
    return u * v


def output2d(trip, mred, precision, order):
    if precision == "mixed":
        mred = np.asarray(mred).astype(np.float64)
    return apply_2d(trip, "A_T", order, precision, mred)


def tile_conv2d(trip, h, x, precision="fp32", order="huffman", csum="linear"):
    """h (..., C, r, r), x (..., C, n, n) with equal leading shapes."""
    z = hadamard2d(trip, h, x, precision, order)
    return output2d(trip, reduce_channels(z, -3, csum), precision, order)


def hadamard1d(trip, h, x, precision, order):
    u = apply_1d(trip, "G", order, precision, _widen(h, precision))
    v = apply_1d(trip, "B_T", order, precision, _widen(x, precision))
    if precision == "mixed":
        u, v = u.astype(np.float32), v.astype(np.float32)
    return u * v


def tile_conv1d(trip, h, x, precision="fp32", order="huffman", csum="linear"):
    z = hadamard1d(trip, h, x, precision, order)
    red = reduce_channels(z, -2, csum)
    if precision == "mixed":
        red = red.astype(np.float64)
    return apply_1d(trip, "A_T", order, precision, red)


def direct_products(h, x, dims, precision="fp64"):
    """Per-channel valid correlation accumulated tap by tap in kernel-index
    order, products and sums rounded separately (engine.py:309-333)."""
    dt = np.float64 if precision == "fp64" else np.float32
    h = np.asarray(h).astype(dt)
    x = np.asarray(x).astype(dt)
    r = h.shape[-1]
    o = x.shape[-1] - r + 1
    acc = None
    if dims == 1:
        for a in range(r):
            t = h[..., a:a + 1] * x[..., a:a + o]
            acc = t if acc is None else acc + t
        return acc
    for a in range(r):
        for b in range(r):
            t = h[..., a:a + 1, b:b + 1] * x[..., a:a + o, b:b + o]
            acc = t if acc is None else acc + t
    return acc


# ---------------------------------------------------------------------------
# layer-level composition (bitwise equal to calling the
# reference's conv_2d per (output channel, tile))
# ---------------------------------------------------------------------------

def layer_geometry(H, W, r, m, pad):
    Ho, Wo = H + 2 * pad - r + 1, W + 2 * pad - r + 1
    th, tw = -(-Ho // m), -(-Wo // m)
    return Ho, Wo, th, tw


def gather_tiles(x, r, m, pad):
    """x [N,C,H,W] -> tiles [N*th*tw, C, n, n] of the zero-padded image."""
    N, C, H, W = x.shape
    n = r + m - 1
    Ho, Wo, th, tw = layer_geometry(H, W, r, m, pad)
    Hp, Wp = th * m + r - 1, tw * m + r - 1
    xp = np.zeros((N, C, Hp, Wp), dtype=x.dtype)
    hh, ww = min(H, Hp - pad), min(W, Wp - pad)
    xp[:, :, pad:pad + hh, pad:pad + ww] = x[:, :, :hh, :ww]
    tiles = np.empty((N, th, tw, C, n, n), dtype=x.dtype)
    for i in range(th):
        for j in range(tw):
            tiles[:, i, j] = xp[:, :, i * m:i * m + n, j * m:j * m + n]
    return tiles.reshape(N * th * tw, C, n, n)


def layer_conv2d(trip, x, w, pad, precision="fp32", order="huffman", csum="linear",
                 tile_chunk=None):
    """Winograd layer y[N,K,Ho,Wo] from x[N,C,H,W] (fp32) and w[K,C,r,r]."""
    x = np.asarray(x)
    w = np.asarray(w)
    N, C, H, W = x.shape
    K = w.shape[0]
    r, m = trip.r, trip.m
    Ho, Wo, th, tw = layer_geometry(H, W, r, m, pad)
    tiles = gather_tiles(x, r, m, pad)
    T = tiles.shape[0]
    if tile_chunk is None:
        tile_chunk = max(1, (4 << 20) // (K * C * trip.n * trip.n))
    u = apply_2d(trip, "G", order, precision, _widen(w, precision))
    if precision == "mixed":
        u = u.astype(np.float32)
    out_dt = np.float32 if precision == "fp32" else np.float64
    y_t = np.empty((K, T, m, m), dtype=out_dt)
    for s in range(0, T, tile_chunk):
        e = min(T, s + tile_chunk)
        v = apply_2d(trip, "B_T", order, precision, _widen(tiles[s:e], precision))
        if precision == "mixed":
            v = v.astype(np.float32)
        z = u[:, None] * v[None]                       # [K, t, C, n, n]
        red = reduce_channels(z, -3, csum)             # [K, t, n, n]
        y_t[:, s:e] = output2d(trip, red, precision, order)
    y = y_t.reshape(K, N, th, tw, m, m).transpose(1, 0, 2, 4, 3, 5)
    y = y.reshape(N, K, th * m, tw * m)[:, :, :Ho, :Wo]
    return np.ascontiguousarray(y)


def layer_direct_fp64(x, w, pad):
    """fp64 reference: per output, per channel the r*r taps in row-major
    order (products/sums rounded separately), then channels left to right --
    reference direct_products + channel_reduce("linear") (engine.py:309-346)
    applied to the zero-padded image."""
    x = np.asarray(x, dtype=np.float64)
    w = np.asarray(w, dtype=np.float64)
    N, C, H, W = x.shape
    K, _, r, _ = w.shape
    Ho, Wo = H + 2 * pad - r + 1, W + 2 * pad - r + 1
    xp = np.zeros((N, C, H + 2 * pad, W + 2 * pad))
    xp[:, :, pad:pad + H, pad:pad + W] = x
    y = np.empty((N, K, Ho, Wo))
    for k in range(K):
        acc = None
        for a in range(r):
            for b in range(r):
                t = w[k, None, :, a, b, None, None] * xp[:, :, a:a + Ho, b:b + Wo]
                acc = t if acc is None else acc + t
        y[:, k] = sum_linear(np.moveaxis(acc, 1, 0))
    return y


def layer_error_stats(y, y64):
    """Per-image fp64 partials (sum|err|, sum|ref|, count, max|err|)."""
    d = np.abs(np.asarray(y, dtype=np.float64) - y64)
    N = d.shape[0]
    return (d.reshape(N, -1).sum(axis=1), np.abs(y64).reshape(N, -1).sum(axis=1),
            np.full(N, d[0].size, dtype=np.int64), d.reshape(N, -1).max(axis=1))


# ---------------------------------------------------------------------------
# Monte-Carlo measurement  (reference: harness.py:97-183)
# ---------------------------------------------------------------------------

def trial_draw(seed, trial, dims, r, n, channels=1):
    """(h, x) of one trial: Philox keyed by (seed, trial), h drawn first, both
    uniform(-1, 1) as rng.random(float32)*2-1 (harness.py:97-107)."""
    gen = np.random.Generator(np.random.Philox(
        key=np.array([seed & 0xFFFFFFFFFFFFFFFF, trial], dtype=np.uint64)))
    h = gen.random((channels,) + (r,) * dims, dtype=np.float32) * np.float32(2) - np.float32(1)
    x = gen.random((channels,) + (n,) * dims, dtype=np.float32) * np.float32(2) - np.float32(1)
    return h, x


def measure_error(trip, dims, precision="fp32", order="huffman", csum="linear",
                  trials=5000, seed=0, channels=1, direct=False, chunk=None, t0=0):
    """Returns (per_trial L1 array, total_l1_mean, per_point_l1_mean)
    (harness.py:116-183).  `trip` may be None with direct=True (DirectSpec).
    t0 > 0: trials t0 .. t0+trials-1 (one rank's shard; draws keyed by trial index)."""
    r = 3 if trip is None else trip.r
    m = 1 if trip is None else trip.m
    n = r + m - 1
    n_out = m ** dims
    if chunk is None:
        chunk = max(1, min(trials, 2_000_000 // max(channels * n ** dims, 1)))
    per = np.empty(trials, dtype=np.float64)
    for s in range(0, trials, chunk):
        e = min(trials, s + chunk)
        pairs = [trial_draw(seed, t0 + t, dims, r, n, channels) for t in range(s, e)]
        hb = np.stack([p[0] for p in pairs])
        xb = np.stack([p[1] for p in pairs])
        ref = reduce_channels(direct_products(hb, xb, dims, "fp64"), -(dims + 1), "linear")
        if direct:
            prods = direct_products(hb, xb, dims, "fp64" if precision == "fp64" else "fp32")
            out = reduce_channels(prods, -(dims + 1), csum)
        elif dims == 2:
            out = tile_conv2d(trip, hb, xb, precision, order, csum)
        else:
            out = tile_conv1d(trip, hb, xb, precision, order, csum)
        diff = np.abs(out.astype(np.float64) - ref)
        per[s:e] = diff.reshape(e - s, -1).sum(axis=1)
    total = float(per.mean())
    return per, total, total / n_out


def synthetic(shape, seed, idx, dist="uniform"):
    """Seeded synthetic fp32 data keyed by (seed, idx)."""
    g = np.random.Generator(np.random.Philox(key=np.array([seed, idx], dtype=np.uint64)))
    if dist == "uniform":
        return g.random(shape, dtype=np.float32) * np.float32(2) - np.float32(1)
    if dist == "uniform01":
        return g.random(shape, dtype=np.float32)
    if dist == "normal":
        return g.standard_normal(shape, dtype=np.float32)
    raise ValueError(dist)


def relu_pool(y, pool):
    """ReLU then optional 2x2/stride-2 max-pool (between VGG conv layers)."""
    y = np.maximum(np.asarray(y), np.float32(0))
    if not pool:
        return y
    N, K, H, W = y.shape
    y = y[:, :, : H // 2 * 2, : W // 2 * 2].reshape(N, K, H // 2, 2, W // 2, 2)
    return y.max(axis=(3, 5))


def stack_forward(trip, x, weights, layers, pad=1, order="huffman", csum="pairwise"):
    """Oracle of paper_1803_10986_b200.stack.ConvStack (fp32): conv outputs per layer."""
    outs = []
    cur = x
    for w, (_, _, pool) in zip(weights, layers):
        y = layer_conv2d(trip, cur, w, pad, "fp32", order, csum)
        outs.append(y)
        cur = relu_pool(y, pool)
    return outs, cur
