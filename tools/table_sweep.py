"""GPU table sweep: every measured cell of the reference's
Tables 2-8, timed on the GPU and checked repr-for-repr against the reference's
own values (tests/golden/table_sweep_<trials>.json, made by make_table_sweep.py).

  python tools/table_sweep.py [--trials 5000]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import os as _os, sys as _sys  # noqa: E401
_sys.path.insert(0, _os.path.dirname(_os.path.abspath(__file__)))
import tuning_env  # noqa: E402,F401  (WINO_* env -> libwino tuning keys)
from paper_1803_10986_b200 import sweep  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trials", type=int, default=5000)
    a = ap.parse_args()
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", f"table_sweep_{a.trials}.json")))
    sweep.table_measurements(trials=16, seed=0)  # plans compiled, context warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    got = sweep.table_measurements(trials=a.trials, seed=0)
    torch.cuda.synchronize()
    secs = time.perf_counter() - t0
    same = sum(repr(v) == gold["values"][k] for k, v in got.items())
    print(json.dumps({"trials": a.trials, "cells": len(got), "repr_identical": same, "gpu_seconds": round(secs, 2),
                      "reference_cpu_seconds": gold["reference_cpu_seconds"],
                      "speedup": round(gold["reference_cpu_seconds"] / secs, 1)}))


if __name__ == "__main__":
    main()
