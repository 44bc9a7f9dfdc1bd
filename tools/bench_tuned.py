"""tools/ only: run bench.py with WINO_<KEY> environment overrides applied through
libwino's tuning keys (tuning_env.py), for A/B runs of kernel variants:
  WINO_K4STAGE=0 python tools/bench_tuned.py --config cfg3_m6 --no-cpu"""
import os
import runpy
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import tuning_env  # noqa: E402,F401

sys.argv = [os.path.join(os.path.dirname(HERE), "bench.py")] + sys.argv[1:]
runpy.run_path(sys.argv[0], run_name="__main__")
