"""Golden values for the table sweep FROM THE REFERENCE:
runs the reference's own reproduce_table for Tables 2-8 with a shared cache and
records every measured per-point L1 mean in that cache, keyed like
paper_1803_10986_b200.sweep.key().  Needs /root/reference (not on the GPU box):

    python tests/golden/make_table_sweep.py [trials]      # default 5000, seed 0
"""
import json
import os
import sys
import time

REF = os.environ.get("TOOMCOOK_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

from toomcook import harness as Hn  # noqa: E402

from paper_1803_10986_b200 import sweep  # noqa: E402  (key format and the measurement list only)

OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    trials = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
    seed = 0
    cache = {}
    t0 = time.time()
    for which in ("2", "3", "4", "5", "6", "7", "8"):
        Hn.reproduce_table(which, trials=trials, seed=seed, cache=cache)
    secs = time.time() - t0
    values = {}
    for (n, family, dims, precision, order, cs, channels, tr, sd), rep in cache.items():
        assert (tr, sd, order) == (trials, seed, "huffman")
        values[sweep.key(family, dims, 0 if n == "direct" else n, channels, cs)] = repr(rep.per_point_l1_mean)
    want = {sweep.key(f, d, n, c, v) for f, d, n, c, vs in sweep.table_keys() for v in vs}
    assert set(values) == want, (sorted(set(values) ^ want))[:10]
    with open(os.path.join(OUT, f"table_sweep_{trials}.json"), "w") as fh:
        json.dump({"trials": trials, "seed": seed, "reference_cpu_seconds": round(secs, 1),
                   "source": "toomcook.harness.reproduce_table('2'..'8', shared cache)", "values": values},
                  fh, indent=1, sort_keys=True)
    print(len(values), "values in", round(secs, 1), "s")


if __name__ == "__main__":
    main()
