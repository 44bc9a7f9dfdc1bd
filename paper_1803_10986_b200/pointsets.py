"""Curated interpolation point sets (paper Tables 2/5; reference pointsets.py:20-107).

Each set is listed in its accretion order (the order the linear-evaluation
baseline follows); every set is completed by the infinity pseudo-point, so a
set of n points serves F(n-2, 3).  Also the config-3 "canonical" comparison
sets (integers first) used by this repo's benchmarks.
"""

from __future__ import annotations

from functools import lru_cache

from .exact import parse_points
from .transforms import build_transforms

KERNEL_SIZE = 3

_BASE4 = ("0", "-1", "1")
_BASE8 = _BASE4 + ("1/2", "-1/2", "2", "-2")
_BASE10 = _BASE8 + ("-1/4", "4")
_BASE14 = _BASE10 + ("1/4", "-3/4", "4/3", "-4")
_BASE12M = _BASE10 + ("3/4", "-4/3")
_BASE14M = _BASE12M + ("1/4", "-4")
_TAIL15 = ("-1", "1", "1/2", "-1/2", "2", "-2", "-1/4", "4")

# (family, dims) -> {n: finite points}
_SETS = {
    ("fp32", 1): {
        4: _BASE4, 5: _BASE4 + ("1/2",), 6: _BASE4 + ("1/2", "-3"),
        7: _BASE4 + ("1/2", "-1/2", "-3"), 8: _BASE8, 9: _BASE8 + ("-1/4",), 10: _BASE10,
        11: _BASE10 + ("1/4",), 12: _BASE10 + ("3/4", "-4/3"),
        13: _BASE10 + ("3/4", "-4/3", "1/4"), 14: _BASE14,
        15: _TAIL15 + ("1/4", "-3/4", "4/3", "-4", "2/3", "-3/2"),
        16: _BASE14 + ("2/3", "-3/2"), 17: _BASE14 + ("2/3", "-3/2", "-2/3"),
        18: _BASE14 + ("2/3", "-3/2", "-2/3", "3/2"),
    },
    ("fp32", 2): {
        4: _BASE4, 5: _BASE4 + ("1/2",), 6: _BASE4 + ("1/2", "-2"),
        7: _BASE4 + ("1/2", "-2", "-1/2"), 8: _BASE8, 9: _BASE8 + ("-1/4",), 10: _BASE10,
        11: _TAIL15 + ("3/4", "-4/3"), 12: _BASE10 + ("3/4", "-4/3"),
        13: _BASE10 + ("3/4", "-4/3", "1/4"), 14: _BASE14,
        15: _TAIL15 + ("1/4", "-3/4", "4/3", "-4", "3/4", "-4/3"),
        16: _BASE14 + ("3/4", "-4/3"), 17: _BASE14 + ("2/3", "-3/2", "3/2"),
        18: _BASE14 + ("2/3", "-3/2", "-2/3", "3/2"),
    },
    ("mixed", 1): {
        4: _BASE4, 5: _BASE4 + ("3",), 6: _BASE4 + ("3", "-1/2"),
        7: _BASE4 + ("3", "-1/2", "1/2"), 8: _BASE8, 9: _BASE8 + ("-1/4",), 10: _BASE10,
        11: _BASE10 + ("1/4",), 12: _BASE12M, 13: _BASE12M + ("1/4",), 14: _BASE14M,
        15: _TAIL15 + ("1/4", "-3/4", "4/3", "-4", "2/3", "-3/2"),
        16: _BASE14 + ("2/3", "-3/2"), 17: _BASE14 + ("2/3", "-3/2", "-2/3"),
        18: _BASE14 + ("2/3", "-3/2", "-2/3", "3/2"),
    },
    ("mixed", 2): {
        4: _BASE4, 5: _BASE4 + ("3",), 6: _BASE4 + ("3", "-1/2"),
        7: _BASE4 + ("3", "-1/2", "1/2"), 8: _BASE8, 9: _BASE8 + ("4",), 10: _BASE10,
        11: _TAIL15 + ("3/4", "-4/3"), 12: _BASE12M, 13: _BASE12M + ("-4",), 14: _BASE14M,
        15: _TAIL15 + ("3/4", "-4/3", "1/4", "-4", "-3/4", "4/3"),
        16: _BASE14M + ("-3/4", "4/3"), 17: _BASE14M + ("-3/4", "4/3", "3/2"),
        18: _BASE14M + ("2/3", "-3/2", "-2/3", "3/2"),
    },
}

SIZES = tuple(range(4, 19))


def curated_text(n: int, dims: int, family: str = "fp32") -> str:
    try:
        pts = _SETS[(family, dims)][n]
    except KeyError as exc:
        raise KeyError(f"no curated set for n={n}, dims={dims}, family={family!r}") from exc
    return ",".join(pts + ("inf",))


def curated_points(n: int, dims: int, family: str = "fp32") -> tuple:
    return parse_points(curated_text(n, dims, family))


@lru_cache(maxsize=None)
def curated_transform(n: int, dims: int, family: str = "fp32"):
    return build_transforms(KERNEL_SIZE, n - KERNEL_SIZE + 1, curated_points(n, dims, family))


def canonical_text(n: int) -> str:
    """Config-3 comparison set (the reference defines none): 0, 1, -1, 2, -2, ... + inf."""
    seq = ["0"]
    k = 1
    while len(seq) < n - 1:
        seq += [str(k), str(-k)]
        k += 1
    return ",".join(seq[:n - 1] + ["inf"])
