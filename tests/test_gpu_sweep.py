"""Table sweep: the GPU measurements behind the reference's
Tables 2-8 equal the reference's own reproduce_table values repr-for-repr
(golden: tests/golden/make_table_sweep.py)."""
import json
import os

import pytest

pytestmark = pytest.mark.gpu
sweep = pytest.importorskip("paper_1803_10986_b200.sweep")

HERE = os.path.dirname(os.path.abspath(__file__))


def test_table_sweep_matches_reference_500_trials():
    gold = json.load(open(os.path.join(HERE, "golden", "table_sweep_500.json")))
    got = sweep.table_measurements(trials=500, seed=0)
    assert set(got) == set(gold["values"])
    bad = {k: (repr(v), gold["values"][k]) for k, v in got.items() if repr(v) != gold["values"][k]}
    assert not bad, list(bad.items())[:5]
