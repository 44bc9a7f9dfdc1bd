"""Fill libwino's on-disk cubin cache (paper_1803_10986_b200/kcache, travels with the
repo snapshot to the GPU box) for the bench workloads: NVRTC compiles on the CPU, so
the GPU run starts with every generated kernel already built.

  python tools/warm_kcache.py [vgg16 cfg sweep_cfg3 sweep_cfg4 ...]   (default: all)
"""
import os
import sys
from concurrent.futures import ProcessPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _layer(job):
    import paper_1803_10986_b200 as W
    from paper_1803_10986_b200 import _native
    r, m, pts, prec, order, cs, contraction, N, C, H, K, pad, flags = job
    ts = W.build_transforms(r, m, W.parse_points(pts))
    op = W.layer_op(ts, W.ConvConfig(prec, order, cs), N, C, H, H, K, pad, contraction)
    op.prepare(flags)
    return job[:3]


def jobs(which):
    import bench
    from paper_1803_10986_b200.stack import VGG16
    out = []
    if "vgg16" in which:
        for n in (256, 192, 128, 64, 32, 2):  # batch, e2e chunks (32, 192, 32), per-rank shards, the CPU slice
            h = 224
            for C, K, pool in VGG16:
                out.append((3, 6, bench.VGG_POINTS, "fp32", "huffman", "pairwise", "exact", n, C, h, K, 1, 3))
                h = h // 2 if pool else h
    if "cfg" in which:
        for name, c in bench.CONFIGS.items():
            r, m, pts, N, C, K, H, pad, _, _, prec, order, cs = c
            out.append((r, m, pts, prec, order, cs, "exact", N, C, H, K, pad, 1))
            for n in (N // 4, N - 3 * (N // 4)):
                out.append((r, m, pts, prec, order, cs, "exact", n, C, H, K, pad, 1))
    for sw in ("sweep_cfg3", "sweep_cfg4"):
        if sw in which:
            for v in bench.sweep_variants(sw):
                _, r, m, pts, N, C, K, H, pad, _, prec, order, cs = v
                out.append((r, m, pts, prec, order, cs, "exact", N, C, H, K, pad, 1))
    return out


if __name__ == "__main__":
    which = sys.argv[1:] or ["vgg16", "cfg", "sweep_cfg3", "sweep_cfg4"]
    js = jobs(which)
    with ProcessPoolExecutor(max(1, os.cpu_count() // 2)) as ex:
        for done in ex.map(_layer, js):
            pass
    print(f"warmed {len(js)} layer shapes")
