"""Helpers to read the golden fixtures written by tests/golden/make_golden.py."""
import json
import os
from fractions import Fraction
from functools import lru_cache

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
REFERENCE_SRC = "/root/reference/pkg/src"


def reference_available():
    return os.path.isdir(os.path.join(REFERENCE_SRC, "toomcook"))


@lru_cache(maxsize=None)
def transforms():
    with open(os.path.join(GOLDEN, "transforms.json")) as fh:
        return {d["name"]: d for d in json.load(fh)}


@lru_cache(maxsize=None)
def npz(name):
    return dict(np.load(os.path.join(GOLDEN, name)))


@lru_cache(maxsize=None)
def cases(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


@lru_cache(maxsize=None)
def measure_rows():
    with open(os.path.join(GOLDEN, "measure.json")) as fh:
        return json.load(fh)


def tree_from_json(t):
    """golden tree -> ('leaf', col, Fraction) | ('add', l, r) | None"""
    if t is None:
        return None
    if t[0] == "L":
        return ("leaf", t[1], Fraction(t[2]))
    return ("add", tree_from_json(t[1]), tree_from_json(t[2]))


def same_bits(a, b):
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    return a.dtype == b.dtype and a.shape == b.shape and a.tobytes() == b.tobytes()
