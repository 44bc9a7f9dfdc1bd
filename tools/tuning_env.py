"""tools/ only: map WINO_<KEY> environment variables onto libwino tuning keys
(include/wino.h wino_tuning_set) so the sweep scripts can select kernel variants
from the shell (e.g. WINO_GEMM=8,8,16,8,16,4,0,16,0,1 python tools/contract_bench.py).
The product package never reads these variables."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ("gemm", "dbuf", "k1", "k1order", "k4", "k1tc", "tile_interp", "cpt", "kpt", "tcf_nk", "tcf_dbg", "tc_epi", "k1rowwise", "k4rowwise", "sc2_kg", "k4k1_ks", "k1st_blocks", "k1_blocks", "k4_blocks", "k1tc_staged", "k1tc_blocks", "tc_epw", "k2coop")


def apply():
    if ROOT not in sys.path:
        sys.path.insert(0, ROOT)
    from paper_1803_10986_b200 import _native
    for k in KEYS:
        v = os.environ.get("WINO_" + k.upper())
        if v:
            _native.set_tuning(k, v)


apply()
