"""The table-sweep measurement list covers exactly the cells the reference's
reproduce_table('2'..'8') measures (CPU; golden from the reference)."""
import json
import os

from paper_1803_10986_b200 import sweep

HERE = os.path.dirname(os.path.abspath(__file__))


def test_table_keys_match_reference_cache():
    gold = json.load(open(os.path.join(HERE, "golden", "table_sweep_500.json")))
    keys = {sweep.key(f, d, n, c, v) for f, d, n, c, vs in sweep.table_keys() for v in vs}
    assert keys == set(gold["values"]) and len(keys) == 176
