"""Generate the golden fixtures in tests/golden/ FROM THE REFERENCE ITSELF.

Run in a container where /root/reference is mounted (it is not on the GPU box):

    python tests/golden/make_golden.py

Everything written here comes from calling the reference toolkit
(/root/reference/pkg/src/toomcook) on seeded inputs; the fixtures pin both the
CPU oracle (oracle/wino_oracle.py) and the product's host-side builder.

Layer-level fixtures use the chunked composition of reference internals from
SURVEY.md section 3.4 (gather zero-padded tiles, G / B^T programs, Hadamard,
channel_reduce, output_2d, scatter + crop); the script self-checks it against
per-(output channel, tile) calls of the reference's public conv_2d.
"""

from __future__ import annotations

import json
import os
import sys
from fractions import Fraction

import numpy as np

REF = os.environ.get("TOOMCOOK_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from toomcook import engine as E  # noqa: E402
from toomcook import harness as Hn  # noqa: E402
from toomcook import pointsets as PS  # noqa: E402
from toomcook.exact import parse_points  # noqa: E402
from toomcook.transforms import build_transforms  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def canonical_points(n):
    """'Canonical' comparison set for config 3 (not defined by the reference;
    recorded in DESIGN.md): integers first 0, 1, -1, 2, -2, ... then inf."""
    seq = ["0"]
    k = 1
    while len(seq) < n - 1:
        seq += [str(k), str(-k)]
        k += 1
    return ",".join(seq[:n - 1] + ["inf"])


def transform_specs():
    specs = []
    add = lambda name, r, m, pts: specs.append({"name": name, "r": r, "m": m, "points": pts})
    add("F23", 3, 2, "0,1,-1,inf")
    add("cfg1_F43", 3, 4, "0,1,-1,1/2,-1/2,inf")
    for fam in ("fp32", "mixed"):
        table = PS._FAMILIES[(fam, 2)]
        for n in sorted(table):
            add(f"cur2d_{fam}_n{n}", 3, n - 2, table[n] + ",inf")
    for n in range(4, 12):
        add(f"canon_n{n}", 3, n - 2, canonical_points(n))
    for m in range(2, 7):  # config 4: r = 5, alpha = m + 4, curated 2D fp32 set with n = alpha
        a = m + 4
        add(f"r5_m{m}", 5, m, PS._FP32_2D[a] + ",inf")
    add("tc_F23", 3, 2, "0,1,-1,2")
    add("tc_F43", 3, 4, "0,-1,1,1/2,-1/2,2")
    add("tc_r5", 5, 1, "0,1,-1,1/2,2")
    add("mod_r2", 2, 5, "0,-2/3,4,-1/4,3,inf")
    add("perm_F43", 3, 4, "1/2,inf,-1,0,-1/2,1")
    return specs


def tree_json(t):
    if t is None:
        return None
    if isinstance(t, E.EvalLeaf):
        return ["L", t.col, str(Fraction(t.coeff))]
    return ["+", tree_json(t.left), tree_json(t.right)]


def bits(arr):
    a = np.asarray(arr)
    return [format(int(v), "x") for v in a.view(np.uint32 if a.dtype == np.float32 else np.uint64).ravel()]


def dump_transforms(specs):
    out = []
    for s in specs:
        ts = build_transforms(s["r"], s["m"], parse_points(s["points"]))
        d = dict(s)
        d["ordered_points"] = [str(p) for p in ts.points]
        d["modified"] = ts.modified
        for name in ("A_T", "G", "B_T"):
            d[name] = [[str(v) for v in row] for row in ts.matrix(name)]
            d[name + "_fp32_bits"] = bits(ts.matrix_fp(name, "fp32"))
            d[name + "_fp64_bits"] = bits(ts.matrix_fp(name, "fp64"))
            for order in ("huffman", "linear"):
                d[f"trees/{name}/{order}"] = [tree_json(t) for t in E.row_trees(ts, name, order)]
        out.append(d)
    with open(os.path.join(OUT, "transforms.json"), "w") as fh:
        json.dump(out, fh, indent=0, separators=(",", ":"))
    print("transforms.json:", len(out), "sets")


# ----------------------------------------------------------------------------
# layer-level composition of reference internals
# ----------------------------------------------------------------------------

def ref_layer(ts, x, w, pad, cfg):
    r, m, n = ts.n_h, ts.n_o, ts.n
    N, C, H, W = x.shape
    K = w.shape[0]
    Ho, Wo = H + 2 * pad - r + 1, W + 2 * pad - r + 1
    th, tw = -(-Ho // m), -(-Wo // m)
    Hp, Wp = th * m + r - 1, tw * m + r - 1
    xp = np.zeros((N, C, Hp, Wp), dtype=x.dtype)
    xp[:, :, pad:pad + H, pad:pad + W] = x
    tiles = np.stack([xp[:, :, i * m:i * m + n, j * m:j * m + n]
                      for i in range(th) for j in range(tw)], axis=1)   # [N, th*tw, C, n, n]
    tiles = tiles.reshape(N * th * tw, C, n, n)
    label = cfg.precision
    g_p = E.compiled_programs(ts, "G", cfg.dot_order, label)
    b_p = E.compiled_programs(ts, "B_T", cfg.dot_order, label)
    u = E._apply_right(g_p, E._apply_left(g_p, E._prepare_input(w, cfg)))
    v = E._apply_right(b_p, E._apply_left(b_p, E._prepare_input(tiles, cfg)))
    if cfg.precision == "mixed":
        u, v = u.astype(np.float32), v.astype(np.float32)
    z = u[:, None] * v[None]
    y = E.output_2d(ts, E.channel_reduce(z, 2, cfg.channel_sum), cfg)   # [K, T, m, m]
    y = y.reshape(K, N, th, tw, m, m).transpose(1, 0, 2, 4, 3, 5).reshape(N, K, th * m, tw * m)
    return np.ascontiguousarray(y[:, :, :Ho, :Wo])


def ref_layer_per_tile(ts, x, w, pad, cfg):
    """Slow self-check: public conv_2d per (k, tile)."""
    r, m, n = ts.n_h, ts.n_o, ts.n
    N, C, H, W = x.shape
    K = w.shape[0]
    Ho, Wo = H + 2 * pad - r + 1, W + 2 * pad - r + 1
    th, tw = -(-Ho // m), -(-Wo // m)
    xp = np.zeros((N, C, th * m + r - 1, tw * m + r - 1), dtype=x.dtype)
    xp[:, :, pad:pad + H, pad:pad + W] = x
    dt = np.float32 if cfg.precision == "fp32" else np.float64
    y = np.zeros((N, K, th * m, tw * m), dtype=dt)
    for b in range(N):
        for k in range(K):
            for i in range(th):
                for j in range(tw):
                    y[b, k, i * m:(i + 1) * m, j * m:(j + 1) * m] = E.conv_2d(
                        ts, w[k], xp[b, :, i * m:i * m + n, j * m:j * m + n], cfg)
    return y[:, :, :Ho, :Wo]


def ref_direct_layer(x, w, pad):
    N, C, H, W = x.shape
    K = w.shape[0]
    xp = np.zeros((N, C, H + 2 * pad, W + 2 * pad))
    xp[:, :, pad:pad + H, pad:pad + W] = x
    out = []
    for b in range(N):
        out.append(np.stack([E.conv_direct(w[k].astype(np.float64), xp[b], 2, "fp64", "linear")
                             for k in range(K)]))
    return np.stack(out)


LAYER_CASES = [
    # name, transform spec name, N, C, K, H, pad
    ("L_f23", "F23", 2, 3, 4, 7, 1),
    ("L_cfg1", "cfg1_F43", 2, 5, 3, 10, 1),
    ("L_p8", "cur2d_fp32_n8", 1, 9, 2, 13, 1),
    ("L_r5", "r5_m4", 1, 4, 3, 11, 2),
    ("L_tc", "tc_F23", 1, 2, 2, 8, 0),
    ("L_n9c17", "cur2d_fp32_n9", 1, 17, 2, 9, 1),
    ("L_mix_n6", "cur2d_mixed_n6", 2, 11, 3, 9, 1),
    ("L_c1", "cfg1_F43", 3, 1, 1, 6, 1),
]

MODES = [
    ("fp32", "huffman", "linear"),
    ("fp32", "huffman", "pairwise"),
    ("fp32", "linear", "linear"),
    ("mixed", "huffman", "pairwise"),
    ("mixed", "linear", "linear"),
    ("fp64", "huffman", "pairwise"),
]


def dump_layers(specs):
    by = {s["name"]: s for s in specs}
    arrays = {}
    rng = np.random.default_rng(1803)
    for name, tsn, N, C, K, H, pad in LAYER_CASES:
        s = by[tsn]
        ts = build_transforms(s["r"], s["m"], parse_points(s["points"]))
        x = rng.uniform(-1, 1, (N, C, H, H)).astype(np.float32)
        w = rng.uniform(-1, 1, (K, C, s["r"], s["r"])).astype(np.float32)
        arrays[f"{name}/x"] = x
        arrays[f"{name}/w"] = w
        arrays[f"{name}/y64"] = ref_direct_layer(x, w, pad)
        for prec, order, cs in MODES:
            cfg = E.ConvConfig(prec, order, cs)
            y = ref_layer(ts, x, w, pad, cfg)
            arrays[f"{name}/{prec}-{order}-{cs}/y"] = y
        if name in ("L_f23", "L_cfg1"):
            for prec, order, cs in MODES[:4]:
                cfg = E.ConvConfig(prec, order, cs)
                slow = ref_layer_per_tile(ts, x, w, pad, cfg)
                fast = arrays[f"{name}/{prec}-{order}-{cs}/y"]
                assert np.array_equal(slow.view(np.uint8), fast.view(np.uint8)), (name, prec, order, cs)
    meta = [{"name": c[0], "ts": c[1], "N": c[2], "C": c[3], "K": c[4], "H": c[5], "pad": c[6]}
            for c in LAYER_CASES]
    np.savez_compressed(os.path.join(OUT, "layer.npz"), **arrays)
    with open(os.path.join(OUT, "layer_cases.json"), "w") as fh:
        json.dump({"cases": meta, "modes": MODES}, fh, indent=1)
    print("layer.npz:", len(arrays), "arrays")


TILE_CASES = [
    # name, spec, trials, channels, seed
    ("T_f23_c1", "F23", 32, 1, 5),
    ("T_cfg1_c4", "cfg1_F43", 24, 4, 6),
    ("T_p8_c13", "cur2d_fp32_n8", 16, 13, 7),
    ("T_n11_c2", "cur2d_fp32_n11", 8, 2, 8),
    ("T_r5_c3", "r5_m3", 8, 3, 9),
]


def dump_tiles(specs):
    by = {s["name"]: s for s in specs}
    arrays = {}
    for name, tsn, trials, C, seed in TILE_CASES:
        s = by[tsn]
        ts = build_transforms(s["r"], s["m"], parse_points(s["points"]))
        pairs = [Hn.trial_inputs(seed, t, 2, ts.n_h, ts.n, C) for t in range(trials)]
        hb = np.stack([p[0] for p in pairs])
        xb = np.stack([p[1] for p in pairs])
        arrays[f"{name}/h"] = hb
        arrays[f"{name}/x"] = xb
        for prec, order, cs in MODES:
            cfg = E.ConvConfig(prec, order, cs)
            z = E.hadamard_2d(ts, hb, xb, cfg)
            arrays[f"{name}/{prec}-{order}-{cs}/z"] = z
            red = E.channel_reduce(z, 2, cs)
            arrays[f"{name}/{prec}-{order}-{cs}/y"] = E.output_2d(ts, red, cfg)
            assert np.array_equal(arrays[f"{name}/{prec}-{order}-{cs}/y"], E.conv_2d(ts, hb, xb, cfg))
        arrays[f"{name}/direct64"] = E.conv_direct(hb, xb, 2, "fp64", "linear")
        # 1D pipeline on the first rows (same sets, 1D draws)
        p1 = [Hn.trial_inputs(seed, t, 1, ts.n_h, ts.n, C) for t in range(trials)]
        h1 = np.stack([p[0] for p in p1])
        x1 = np.stack([p[1] for p in p1])
        arrays[f"{name}/h1"] = h1
        arrays[f"{name}/x1"] = x1
        for prec, order, cs in MODES:
            cfg = E.ConvConfig(prec, order, cs)
            arrays[f"{name}/{prec}-{order}-{cs}/y1"] = E.conv_1d(ts, h1, x1, cfg)
    # pairwise_sum over lengths 1..70
    rng = np.random.default_rng(77)
    for L in range(1, 71):
        v = rng.uniform(0, 1, L).astype(np.float32)
        arrays[f"pw/{L}/v"] = v
        arrays[f"pw/{L}/s"] = np.asarray(E.pairwise_sum(v, "fp32"))
    meta = [{"name": c[0], "ts": c[1], "trials": c[2], "C": c[3], "seed": c[4]} for c in TILE_CASES]
    np.savez_compressed(os.path.join(OUT, "tile.npz"), **arrays)
    with open(os.path.join(OUT, "tile_cases.json"), "w") as fh:
        json.dump({"cases": meta, "modes": MODES}, fh, indent=1)
    print("tile.npz:", len(arrays), "arrays")


def dump_measure():
    """measure_error golden values and per-trial vectors."""
    rows = []
    per = {}
    for n in (4, 6, 8):
        ts = PS.curated_transform(n, 2, "fp32")
        for prec in ("fp32", "mixed"):
            for C, cs in ((1, "linear"), (32, "linear"), (32, "pairwise"), (64, "linear"), (64, "pairwise")):
                rep = Hn.measure_error(ts, 2, E.ConvConfig(prec, "huffman", cs), 5000, 0, C)
                rows.append({"set": f"cur2d_fp32_n{n}", "dims": 2, "precision": prec, "dot_order": "huffman",
                             "channel_sum": cs, "channels": C, "trials": 5000, "seed": 0,
                             "total_l1_mean": repr(rep.total_l1_mean),
                             "per_point_l1_mean": repr(rep.per_point_l1_mean)})
                if C <= 32:
                    per[f"cur2d_fp32_n{n}/{prec}/{cs}/{C}"] = rep.per_trial[:200].copy()
    rep = Hn.measure_error(PS.curated_transform(6, 2, "fp32"), 2, E.ConvConfig("fp32", "linear", "linear"), 5000, 0, 1)
    rows.append({"set": "cur2d_fp32_n6", "dims": 2, "precision": "fp32", "dot_order": "linear",
                 "channel_sum": "linear", "channels": 1, "trials": 5000, "seed": 0,
                 "total_l1_mean": repr(rep.total_l1_mean), "per_point_l1_mean": repr(rep.per_point_l1_mean)})
    for C, cs in ((1, "linear"), (32, "linear"), (64, "linear")):
        rep = Hn.measure_error(Hn.DirectSpec(3, 1), 2, E.ConvConfig("fp32", "huffman", cs), 5000, 0, C)
        rows.append({"set": "direct", "dims": 2, "precision": "fp32", "dot_order": "huffman",
                     "channel_sum": cs, "channels": C, "trials": 5000, "seed": 0,
                     "total_l1_mean": repr(rep.total_l1_mean), "per_point_l1_mean": repr(rep.per_point_l1_mean)})
    # 1D sample
    for n in (4, 6):
        ts = PS.curated_transform(n, 1, "fp32")
        rep = Hn.measure_error(ts, 1, E.ConvConfig("fp32", "huffman", "linear"), 2000, 3, 1)
        rows.append({"set": f"cur1d_fp32_n{n}", "dims": 1, "precision": "fp32", "dot_order": "huffman",
                     "channel_sum": "linear", "channels": 1, "trials": 2000, "seed": 3,
                     "total_l1_mean": repr(rep.total_l1_mean), "per_point_l1_mean": repr(rep.per_point_l1_mean)})
    with open(os.path.join(OUT, "measure.json"), "w") as fh:
        json.dump(rows, fh, indent=1)
    np.savez_compressed(os.path.join(OUT, "measure_per_trial.npz"), **per)
    # Philox draws
    ph = {}
    for seed, t, dims, n, C in ((0, 0, 2, 4, 1), (0, 4999, 2, 8, 64), (3, 17, 1, 6, 5), (2**40 + 7, 123, 2, 6, 3)):
        h, x = Hn.trial_inputs(seed, t, dims, 3, n, C)
        ph[f"{seed}/{t}/{dims}/{n}/{C}/h"] = h
        ph[f"{seed}/{t}/{dims}/{n}/{C}/x"] = x
    np.savez_compressed(os.path.join(OUT, "philox.npz"), **ph)
    print("measure.json:", len(rows), "rows")


if __name__ == "__main__":
    specs = transform_specs()
    dump_transforms(specs)
    dump_layers(specs)
    dump_tiles(specs)
    if "--no-measure" not in sys.argv:
        dump_measure()
